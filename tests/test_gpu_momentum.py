"""GPU parity of the SGD-momentum apply (GTC_ACCUM_MOMENTUM; SURVEY 8(f) #2,
DESIGN.md reading M1) against oracle_apply_momentum (pinned in
tests/test_momentum_oracle.py): weights, momentum buffer, residuals, messages
and counts bit-exact, through every kernel that applies -- the fused world-1
step (encode kernel), the counting decode (world 1 unfused, simulated
workers), on ragged sizes and at the LSTM-AM size."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1904_10584_b200 as gtc  # noqa: E402

DEV = torch.device("cuda", 0)
MODES = {"gt": oracle.CMP_GT, "ge": oracle.CMP_GE}
MU = 0.9


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def bits(t):
    return t.detach().cpu().numpy().view(np.uint32)


def inputs(n, tau, seed):
    g = [synth.normal(n, seed, t) * np.float32(0.7 * tau) for t in range(4)]
    r = synth.uniform(n, -tau, tau, seed + 1)
    w = synth.normal(n, seed + 2)
    b = synth.normal(n, seed + 3) * np.float32(0.01)  # a warm momentum buffer
    return g, r, w, b


@pytest.mark.parametrize("cmp", ["gt", "ge"])
@pytest.mark.parametrize("n", [1, 5, 4095, 4096, 4097, 3 * 4096 + 1234, 1_000_003])
@pytest.mark.parametrize("fused", [True, False])
def test_single_rank_momentum(n, cmp, fused):
    """world 1: gtc_step (momentum fused into the encode kernel) or encode ->
    exchange -> decode_apply (the counting decode's dense pass), 4 steps."""
    tau = 0.3
    gs, r_h, w_h, b_h = inputs(n, tau, 40 + n % 97)
    ctx = gtc.GTC(n, tau, cmp=cmp)
    rd, wd, bd = to_dev(r_h), to_dev(w_h), to_dev(b_h)
    ctx.bind_momentum(bd, MU)
    cnt = torch.empty(n, dtype=torch.int8, device=DEV)
    for t in range(4):
        gd = to_dev(gs[t])
        if fused:
            assert ctx.step(gd, rd, wd, -0.05, gtc.GTC_ACCUM_MOMENTUM) == gtc.GTC_OK
        else:
            ctx.encode(gd, rd)
            ctx.exchange()
            ctx.decode_apply(wd, -0.05, gtc.GTC_ACCUM_MOMENTUM, cnt if t % 2 else None)
        om, oc, _ = oracle.step([gs[t]], [r_h], w_h, tau, MODES[cmp], -0.05, oracle.ACCUM_MOMENTUM, buf=b_h, mu=MU)
        torch.cuda.synchronize()
        assert np.array_equal(ctx.message_tensor().cpu().numpy().view(np.uint32), om[0]), f"step {t}: message"
        if not fused and t % 2:
            assert np.array_equal(cnt.cpu().numpy().astype(np.int32), oc), f"step {t}: counts"
        assert np.array_equal(bits(rd), r_h.view(np.uint32)), f"step {t}: residual"
        assert np.array_equal(bits(bd), b_h.view(np.uint32)), f"step {t}: momentum buffer"
        assert np.array_equal(bits(wd), w_h.view(np.uint32)), f"step {t}: weights"
    assert ctx.check() == gtc.GTC_OK
    ctx.close()


@pytest.mark.parametrize("N", [2, 5])
def test_simulated_workers_momentum(N):
    """decode_apply_msgs over N simulated workers' messages (counts in [-N, N])."""
    n, tau = 300_007, 8.0
    ctxs = [gtc.GTC(n, tau, max_sim_msgs=N) for _ in range(N)]
    r_h = [synth.uniform(n, -tau, tau, synth.rank_seed(w)) for w in range(N)]
    w_h = synth.normal(n, 5)
    b_h = np.zeros(n, np.float32)
    rd = [to_dev(r) for r in r_h]
    wd, bd = to_dev(w_h), to_dev(b_h)
    ctxs[0].bind_momentum(bd, MU)
    cnt = torch.empty(n, dtype=torch.int8, device=DEV)
    for t in range(3):
        gs = [synth.correlated_gradient(n, 4.0, synth.BASE_SEED, t, w) for w in range(N)]
        for c, g, r in zip(ctxs, gs, rd):
            c.encode(to_dev(g), r)
        ctxs[0].decode_apply_msgs([c.message() for c in ctxs], wd, -0.5, gtc.GTC_ACCUM_MOMENTUM, counts_out=cnt)
        om, oc, _ = oracle.step(gs, r_h, w_h, tau, oracle.CMP_GT, -0.5, oracle.ACCUM_MOMENTUM, buf=b_h, mu=MU)
        torch.cuda.synchronize()
        assert np.array_equal(cnt.cpu().numpy().astype(np.int32), oc), f"step {t}: counts"
        assert np.abs(oc).max() >= 2  # correlated ranks: multi-quantum counts occur
        assert np.array_equal(bits(bd), b_h.view(np.uint32)), f"step {t}: momentum buffer"
        assert np.array_equal(bits(wd), w_h.view(np.uint32)), f"step {t}: weights"
    for c in ctxs:
        c.close()


def test_momentum_lstm_am_full_size():
    """The LSTM-AM size (n mod 4 = 3): 2 fused steps then 1 unfused, bit-exact."""
    n, tau = synth.LSTM_AM_PARAMS, 8.0
    sigma = synth.sigma_for_density(0.01, tau, synth.mean_abs_scale(n))
    gs = [synth.lstm_gradient(n, sigma, synth.BASE_SEED, t, 0) for t in range(3)]
    r_h = synth.uniform(n, -tau, tau, synth.rank_seed(0))
    w_h = synth.normal(n, synth.BASE_SEED, 0, 11) * np.float32(0.05)
    b_h = np.zeros(n, np.float32)
    ctx = gtc.GTC(n, tau)
    rd, wd, bd = to_dev(r_h), to_dev(w_h), to_dev(b_h)
    ctx.bind_momentum(bd, MU)
    for t in range(3):
        gd = to_dev(gs[t])
        if t < 2:
            ctx.step(gd, rd, wd, -1e-3, gtc.GTC_ACCUM_MOMENTUM)
        else:
            ctx.encode(gd, rd)
            ctx.exchange()
            ctx.decode_apply(wd, -1e-3, gtc.GTC_ACCUM_MOMENTUM)
        oracle.step([gs[t]], [r_h], w_h, tau, oracle.CMP_GT, -1e-3, oracle.ACCUM_MOMENTUM, buf=b_h, mu=MU)
    torch.cuda.synchronize()
    assert np.array_equal(bits(rd), r_h.view(np.uint32))
    assert np.array_equal(bits(bd), b_h.view(np.uint32))
    assert np.array_equal(bits(wd), w_h.view(np.uint32))
    ctx.close()


def test_momentum_errors():
    n = 10_000
    ctx = gtc.GTC(n, 8.0)
    w = torch.zeros(n, device=DEV)
    r = torch.zeros(n, device=DEV)
    with pytest.raises(gtc.GTCError) as e:  # no buffer bound
        ctx.step(None, r, w, -0.1, gtc.GTC_ACCUM_MOMENTUM)
    assert e.value.status == gtc.GTC_ESTATE
    big = torch.zeros(n + 1, device=DEV)
    with pytest.raises(gtc.GTCError) as e:
        gtc.gtc_bind_momentum(ctx.ctx, big[1:].data_ptr(), 0.9)
    assert e.value.status == gtc.GTC_EALIGN
    with pytest.raises(gtc.GTCError) as e:
        ctx.bind_momentum(torch.zeros(n, device=DEV), float("nan"))
    assert e.value.status == gtc.GTC_EINVAL
    with pytest.raises(gtc.GTCError) as e:
        ctx.step(None, r, w, -0.1, 3)
    assert e.value.status == gtc.GTC_EINVAL
    ctx.close()
