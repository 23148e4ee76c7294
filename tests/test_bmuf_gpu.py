"""BMUF on the GPU (include/bmuf.h) vs the oracle (Eqs. 1-4).

Simulated workers on one GPU use the oracle's rank-ordered double mean, so
every output is compared bit-exactly; so is world 1 (the mean of one model is
the model).  Multi-GPU (NCCL reduce-scatter sums in NCCL's order) is covered in
tests/test_multigpu.py with a derived error bound."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1904_10584_b200 as gtc  # noqa: E402

DEV = torch.device("cuda", 0)


def bits(t):
    return t.detach().cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("N", [1, 2, 3, 8])
@pytest.mark.parametrize("n", [1, 4097, 100_003])
def test_sim_workers_bit_exact(N, n):
    eta, zeta = 1 - 1 / max(N, 2), 1.0  # Eq. (5) with C = 1 ... ~ (C=N(1-eta)/zeta)
    ctx = gtc.bmuf_init(n)
    wg_h = synth.normal(n, 1, n)
    d_h = np.zeros(n, np.float32)
    wg, d = torch.from_numpy(wg_h.copy()).to(DEV), torch.zeros(n, device=DEV)
    for t in range(4):
        ws_h = [(wg_h + synth.normal(n, 10 + i, t) * np.float32(0.01)).astype(np.float32) for i in range(N)]
        ws = [torch.from_numpy(w.copy()).to(DEV) for w in ws_h]
        gtc.bmuf_sync_sim(ctx, [w.data_ptr() for w in ws], wg.data_ptr(), d.data_ptr(), eta, zeta,
                          torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        oracle.bmuf_step(ws_h, wg_h, d_h, eta, zeta)
        assert np.array_equal(bits(wg), wg_h.view(np.uint32)), t
        assert np.array_equal(bits(d), d_h.view(np.uint32)), t
        for i in range(N):
            assert np.array_equal(bits(ws[i]), ws_h[i].view(np.uint32)), (t, i)
    gtc.bmuf_destroy(ctx)


def test_world1_sync_bit_exact():
    n = 1_000_003
    b = gtc.BMUF(n, eta=0.5, zeta=1.0, w_init=torch.from_numpy(synth.normal(n, 3)).to(DEV))
    wg_h = synth.normal(n, 3)
    d_h = np.zeros(n, np.float32)
    w = b.local_buffer()
    for t in range(3):
        w_h = (wg_h + synth.normal(n, 4, t) * np.float32(0.1)).astype(np.float32)
        w[:n].copy_(torch.from_numpy(w_h))
        b.sync(w)
        torch.cuda.synchronize()
        ws = [w_h.copy()]
        oracle.bmuf_step(ws, wg_h, d_h, 0.5, 1.0)
        assert np.array_equal(bits(w[:n]), wg_h.view(np.uint32)), t
        assert np.array_equal(bits(b.wg[:n]), wg_h.view(np.uint32)), t
        assert np.array_equal(bits(b.delta[:n]), d_h.view(np.uint32)), t
    b.close()


def test_eq5_zeta():
    assert abs(gtc.bmuf_zeta(1, 8, 0.875) - 1.0) < 1e-12
    assert abs(gtc.bmuf_zeta(2, 64, 0.9) - 12.8) < 1e-9
