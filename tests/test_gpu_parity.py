"""GPU parity: the CUDA path (through the C ABI) vs. the CPU oracle.

Bar (BASELINE.json north_star): packed messages, word counts and integer
counts bit-exact; residuals bit-exact (same fp32 RNE adds); applied floats
within 1e-6 relative max-abs -- asserted bit-exact here because both sides pin
the same operation order (R8), with the 1e-6 check reported too.
"""
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


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def bits(t):
    return t.detach().cpu().numpy().view(np.uint32)


def assert_float_parity(got, exp, what):
    g, e = got.astype(np.float64), exp.astype(np.float64)
    scale = max(np.abs(e).max(initial=0.0), 1e-30)
    rel = np.abs(g - e).max(initial=0.0) / scale
    assert rel <= 1e-6, f"{what}: rel max-abs {rel}"
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32)), f"{what}: not bit-exact (rel {rel})"


class SimWorkers:
    """N simulated workers on one GPU: one context per worker for encode, the
    messages aggregated by decode_apply_msgs (no NCCL)."""

    def __init__(self, n, tau, N, cmp="gt"):
        self.ctx = [gtc.GTC(n, tau, cmp=cmp, max_sim_msgs=N) for _ in range(N)]

    def step(self, gd, rd, wd, alpha, mode, counts_out=None):
        for c, g, r in zip(self.ctx, gd, rd):
            c.encode(g, r)
        msgs = [c.message() for c in self.ctx]
        self.ctx[0].decode_apply_msgs(msgs, wd, alpha, mode, counts_out=counts_out)
        return [c.message_tensor().cpu().numpy().view(np.uint32) for c in self.ctx]

    def close(self):
        for c in self.ctx:
            c.close()


def run_parity(n, tau, N, steps, gen, cmp="gt", alpha=-0.5, mode=gtc.GTC_ACCUM_WEIGHTS, r0=None, seed=0):
    sim = SimWorkers(n, tau, N, cmp)
    r_host = [np.zeros(n, np.float32) if r0 is None else r0(w) for w in range(N)]
    w_host = synth.normal(n, 77 + seed)
    rd = [to_dev(r) for r in r_host]
    wd = to_dev(w_host)
    cnt = torch.empty(n, dtype=torch.int8, device=DEV)
    ks = []
    for t in range(steps):
        gs = [gen(t, w) for w in range(N)]
        gd = [to_dev(g) for g in gs]
        got_msgs = sim.step(gd, rd, wd, alpha, mode, cnt)
        om, oc, _ = oracle.step(gs, r_host, w_host, tau, MODES[cmp], alpha, mode)
        for w in range(N):
            assert np.array_equal(got_msgs[w], om[w]), f"step {t} worker {w}: message"
            assert np.array_equal(bits(rd[w]), r_host[w].view(np.uint32)), f"step {t} worker {w}: residual"
        assert np.array_equal(cnt.cpu().numpy().astype(np.int32), oc), f"step {t}: counts"
        assert_float_parity(wd.cpu().numpy(), w_host, f"step {t}: weights")
        ks.append([m.size for m in om])
    sim.close()
    return ks


# ------------------------------------------------------------------ config 1
@pytest.mark.parametrize("cmp", ["gt", "ge"])
def test_config1_dyadic_2workers_10steps(cmp):
    """C1(a): 1M params, 2 simulated workers, tau=8, 10 steps, dyadic gradients."""
    n, tau = 1_000_000, 8.0
    ks = run_parity(n, tau, 2, 10,
                    lambda t, w: synth.dyadic_gradient(n, 3.0, tau, synth.BASE_SEED, t, w), cmp)
    assert sum(sum(k) for k in ks) > 0


@pytest.mark.parametrize("cmp", ["gt", "ge"])
def test_config1_correlated_2workers_10steps(cmp):
    """C1(b): correlated ranks (counts of +-2 and cancellations), update mode."""
    n, tau = 1_000_000, 8.0
    run_parity(n, tau, 2, 10,
               lambda t, w: synth.correlated_gradient(n, 4.0, synth.BASE_SEED, t, w), cmp,
               alpha=1.0, mode=gtc.GTC_ACCUM_UPDATE,
               r0=lambda w: synth.uniform(n, -tau, tau, synth.rank_seed(w)))


# ------------------------------------------------------------------ N=1 API path
@pytest.mark.parametrize("cmp", ["gt", "ge"])
@pytest.mark.parametrize("n", [1, 3, 4, 5, 31, 4095, 4096, 4097, 3 * 4096 + 1234, 65536 * 3 + 7])
def test_single_rank_path_sizes(n, cmp):
    """encode -> exchange (no-op) -> decode_apply at world=1, ragged sizes
    (counts_out given: the tiled shared-memory count kernel)."""
    tau = 2.0
    g = synth.normal(n, 3, n) * np.float32(3.0)
    r_host = synth.uniform(n, -tau, tau, 4, n)
    r_host[::7] = 0.0
    g[::7] = np.float32(tau)  # exact ties
    w_host = synth.normal(n, 5, n)
    ctx = gtc.GTC(n, tau, cmp=cmp)
    rd, gd, wd = to_dev(r_host), to_dev(g), to_dev(w_host)
    cnt = torch.empty(n, dtype=torch.int8, device=DEV)
    ctx.encode(gd, rd)
    assert ctx.exchange() == gtc.GTC_OK
    ctx.decode_apply(wd, 0.25, gtc.GTC_ACCUM_WEIGHTS, cnt)
    torch.cuda.synchronize()
    om, oc, _ = oracle.step([g], [r_host], w_host, tau, MODES[cmp], 0.25, oracle.ACCUM_WEIGHTS)
    assert np.array_equal(ctx.message_tensor().cpu().numpy().view(np.uint32), om[0])
    assert ctx.last_counts() == [om[0].size]
    assert np.array_equal(bits(rd), r_host.view(np.uint32))
    assert np.array_equal(cnt.cpu().numpy().astype(np.int32), oc)
    assert_float_parity(wd.cpu().numpy(), w_host, "weights")
    assert ctx.check() == gtc.GTC_OK
    ctx.close()


@pytest.mark.parametrize("mode", [gtc.GTC_ACCUM_WEIGHTS, gtc.GTC_ACCUM_UPDATE])
@pytest.mark.parametrize("n", [1, 4097, 3 * 4096 + 1234, 2_000_003])
@pytest.mark.parametrize("use_step", [False, True])
def test_single_rank_word_parallel_apply(n, mode, use_step):
    """world=1 without counts_out: the word-parallel apply kernel (and gtc_step)."""
    tau = 0.1  # fl(c * tau) is inexact for general c, exact for c = +-1
    g = synth.normal(n, 21, n) * np.float32(0.3)
    r_host = synth.uniform(n, -tau, tau, 22, n)
    w_host = synth.normal(n, 23, n)
    ctx = gtc.GTC(n, tau)
    rd, gd, wd = to_dev(r_host), to_dev(g), to_dev(w_host)
    for t in range(3):
        if use_step:
            ctx.step(gd, rd, wd, -0.75, mode)
        else:
            ctx.encode(gd, rd)
            ctx.exchange()
            ctx.decode_apply(wd, -0.75, mode)
        oracle.step([g], [r_host], w_host, tau, oracle.CMP_GT, -0.75, mode)
    torch.cuda.synchronize()
    assert np.array_equal(bits(rd), r_host.view(np.uint32))
    assert_float_parity(wd.cpu().numpy(), w_host, "weights")
    ctx.close()


def test_sim_single_message_word_parallel():
    """decode_apply_msgs with one message and no counts_out."""
    n, tau = 300_007, 8.0
    v = synth.normal(n, 24) * np.float32(9.0)
    ctx = gtc.GTC(n, tau, max_sim_msgs=1)
    rd = to_dev(v)
    ctx.encode(None, rd)
    wd = torch.zeros(n, device=DEV)
    ctx.decode_apply_msgs([ctx.message()], wd, 2.0, gtc.GTC_ACCUM_WEIGHTS)
    words, _ = oracle.encode(None, v.copy(), tau)
    w_exp = np.zeros(n, np.float32)
    oracle.apply(oracle.decode_counts([words], n), w_exp, tau, 2.0, oracle.ACCUM_WEIGHTS)
    assert_float_parity(wd.cpu().numpy(), w_exp, "weights")
    ctx.close()


def test_empty_vector():
    ctx = gtc.GTC(0, 8.0)
    r = torch.zeros(0, device=DEV)
    ctx.encode(r, r)
    ctx.exchange()
    ctx.decode_apply(r)
    assert ctx.last_counts() == [0]
    ctx.close()


def test_grad_null_residual_holds_sum():
    n, tau = 50_000, 1.0
    v = synth.normal(n, 8) * np.float32(1.5)
    ctx = gtc.GTC(n, tau)
    rd = to_dev(v)
    ctx.encode(None, rd)
    torch.cuda.synchronize()
    r_host = v.copy()
    words, _ = oracle.encode(None, r_host, tau)
    assert np.array_equal(ctx.message_tensor().cpu().numpy().view(np.uint32), words)
    assert np.array_equal(bits(rd), r_host.view(np.uint32))
    ctx.close()


def test_all_emit_and_none_emit():
    n = 3 * 4096 + 77
    v = synth.normal(n, 9)
    for tau, expect_all in ((1e-30, True), (1e30, False)):
        ctx = gtc.GTC(n, tau)
        rd = to_dev(v)
        ctx.encode(None, rd)
        k = ctx.last_counts()[0]
        r_host = v.copy()
        words, _ = oracle.encode(None, r_host, tau)
        assert k == words.size == (np.count_nonzero(v) if expect_all else 0)
        assert np.array_equal(ctx.message_tensor().cpu().numpy().view(np.uint32), words)
        assert np.array_equal(bits(rd), r_host.view(np.uint32))
        ctx.close()


def test_nonfinite_flag_and_behaviour():
    n, tau = 10_000, 8.0
    v = synth.normal(n, 10)
    v[[3, 5000, 9999]] = [np.nan, np.inf, -np.inf]
    ctx = gtc.GTC(n, tau)
    rd = to_dev(v)
    ctx.encode(None, rd)
    assert ctx.exchange() == gtc.GTC_OK  # world 1: reported by check()
    r_host = v.copy()
    words, nf = oracle.encode(None, r_host, tau)
    assert nf
    assert np.array_equal(ctx.message_tensor().cpu().numpy().view(np.uint32), words)
    assert np.array_equal(bits(rd), r_host.view(np.uint32))
    assert ctx.check() == gtc.GTC_ENONFINITE
    assert ctx.check() == gtc.GTC_OK  # cleared once reported
    ctx.close()


def test_denormals_not_flushed():
    tiny = np.float32(1e-45)
    v = np.array([tiny, -tiny, 2 * tiny, 0, 0, 0, 0, 0], np.float32)
    g = np.array([tiny, 0, tiny, 0, 0, 0, 0, 0], np.float32)
    ctx = gtc.GTC(8, float(tiny))
    rd, gd = to_dev(v), to_dev(g)
    ctx.encode(gd, rd)
    r_host = v.copy()
    words, _ = oracle.encode(g, r_host, float(tiny))
    assert np.array_equal(ctx.message_tensor().cpu().numpy().view(np.uint32), words)
    assert np.array_equal(bits(rd), r_host.view(np.uint32))
    ctx.close()


def test_determinism_repeat():
    n, tau = 2_000_003, 8.0
    g = synth.lstm_gradient(n, synth.sigma_for_density(0.01, tau, synth.mean_abs_scale(n)), synth.BASE_SEED, 0)
    r0 = synth.uniform(n, -tau, tau, 1)
    outs = []
    for _ in range(2):
        ctx = gtc.GTC(n, tau)
        rd, gd = to_dev(r0), to_dev(g)
        ctx.encode(gd, rd)
        outs.append((ctx.message_tensor().cpu().numpy().copy(), bits(rd).copy()))
        ctx.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_repeated_calls_epochs():
    """Many encodes on one context (epoch-tagged look-back, ticket reset)."""
    n, tau = 300_001, 4.0
    ctx = gtc.GTC(n, tau)
    r_host = np.zeros(n, np.float32)
    rd = to_dev(r_host)
    for t in range(40):
        g = synth.normal(n, 12, t) * np.float32(1.3)
        ctx.encode(to_dev(g), rd)
        ctx.exchange()
        wd = torch.zeros(n, device=DEV)
        ctx.decode_apply(wd, 1.0, gtc.GTC_ACCUM_UPDATE)
        words, _ = oracle.encode(g, r_host, tau)
        if t % 8 == 0 or t == 39:
            assert np.array_equal(ctx.message_tensor().cpu().numpy().view(np.uint32), words), t
            assert np.array_equal(bits(rd), r_host.view(np.uint32)), t
    ctx.close()


# ------------------------------------------------------------------ errors
def test_error_paths():
    n = 10_000
    ctx = gtc.GTC(n, 8.0, max_sim_msgs=2)
    w = torch.zeros(n, device=DEV)
    with pytest.raises(gtc.GTCError) as e:
        ctx.decode_apply(w)
    assert e.value.status == gtc.GTC_ESTATE
    with pytest.raises(gtc.GTCError) as e:
        ctx.exchange()
    assert e.value.status == gtc.GTC_ESTATE
    big = torch.zeros(n + 1, device=DEV)
    with pytest.raises(gtc.GTCError) as e:
        ctx.encode(None, big[1:])
    assert e.value.status == gtc.GTC_EALIGN
    bad = torch.tensor([10, 4], dtype=torch.int32, device=DEV)  # descending
    with pytest.raises(gtc.GTCError) as e:
        ctx.decode_apply_msgs([bad], w)
    assert e.value.status == gtc.GTC_ECORRUPT
    oob = torch.tensor([2 * n], dtype=torch.int32, device=DEV)  # index n
    with pytest.raises(gtc.GTCError) as e:
        ctx.decode_apply_msgs([oob], w)
    assert e.value.status == gtc.GTC_ECORRUPT
    assert torch.count_nonzero(w).item() == 0  # nothing applied
    ctx.close()
    with pytest.raises(gtc.GTCError) as e:
        gtc.gtc_init(1 << 31, 8.0)
    assert e.value.status == gtc.GTC_EDIM
    with pytest.raises(gtc.GTCError):
        gtc.gtc_init(10, 0.0)


def test_capacity_bounds_only_the_contiguous_message():
    """The hot path's segmented message cannot overflow: the step applies in
    full; max_words_per_rank bounds only the contiguous wire format, which
    reports GTC_ECAPACITY when asked for."""
    n, tau = 100_000, 1.0
    ctx = gtc.GTC(n, tau, max_words_per_rank=100)
    v = synth.normal(n, 13) * np.float32(3.0)
    rd = to_dev(v)
    w = torch.zeros(n, device=DEV)
    ctx.encode(None, rd)
    ctx.exchange()
    ctx.decode_apply(w, 1.0, gtc.GTC_ACCUM_UPDATE)
    assert ctx.check() == gtc.GTC_OK
    r_host = v.copy()
    words, _ = oracle.encode(None, r_host, tau)
    w_exp = np.zeros(n, np.float32)
    oracle.apply(oracle.decode_counts([words], n), w_exp, tau, 1.0, oracle.ACCUM_UPDATE)
    assert_float_parity(w.cpu().numpy(), w_exp, "update")
    assert ctx.last_counts() == [words.size]
    with pytest.raises(gtc.GTCError) as e:
        ctx.message()
    assert e.value.status == gtc.GTC_ECAPACITY
    ctx.close()


# ------------------------------------------------------------------ config 2 / 4 (full LSTM-AM size)
def lstm_inputs(n, tau, rho, t, w, correlated=0.0):
    sigma = synth.sigma_for_density(rho, tau, synth.mean_abs_scale(n))
    return synth.lstm_gradient(n, sigma, synth.BASE_SEED, t, w, correlated)


@pytest.mark.parametrize("cmp", ["gt", "ge"])
def test_config2_lstm_am_full_size(cmp):
    """C2: n = 24,286,575 (PAPER.md:84-86 LSTM AM) at N=1, rho ~ 1%, 3 steps, full compare."""
    n, tau = synth.LSTM_AM_PARAMS, 8.0
    ks = run_parity(n, tau, 1, 3, lambda t, w: lstm_inputs(n, tau, 0.01, t, w), cmp,
                    r0=lambda w: synth.uniform(n, -tau, tau, synth.rank_seed(w)))
    rho = ks[0][0] / n
    assert 0.005 < rho < 0.02, rho


@pytest.mark.parametrize("rho", [1e-4, 1e-3, 1e-2, 1e-1])
def test_config4_density_sweep_8_workers(rho):
    """C4: LSTM-AM shape, tau=8, density 0.01%..10%, 8 simulated workers, full compare."""
    n, tau = synth.LSTM_AM_PARAMS, 8.0
    ks = run_parity(n, tau, 8, 1, lambda t, w: lstm_inputs(n, tau, rho, t, w, 0.5), "gt",
                    r0=lambda w: synth.uniform(n, -tau, tau, synth.rank_seed(w)))
    got = np.mean(ks[0]) / n
    assert rho / 2 < got < rho * 2, (rho, got)


# ------------------------------------------------------------------ config 5 (1e9 params, sampled)
def test_config5_1e9_params_sampled():
    """C5: n = 1e9 at N=1 in the bench's launch configuration; every word,
    residual, count and weight in sampled windows (tile edges, the ragged
    tail, random interior) is checked against the oracle on that window, plus
    whole-vector properties (k, ordering, support)."""
    n, tau = 1_000_000_000, 8.0
    free, _ = torch.cuda.mem_get_info()
    if free < 24 * 2**30:
        pytest.skip("needs ~24 GB free device memory")
    sigma = synth.sigma_for_density(0.01, tau)
    g = synth.normal(n, synth.rank_seed(0), 0) * np.float32(sigma)
    r0 = synth.uniform(n, -tau, tau, synth.rank_seed(0))
    ctx = gtc.GTC(n, tau, max_words_per_rank=n // 20)
    gd, rd = to_dev(g), to_dev(r0)
    wd = torch.zeros(n, device=DEV)
    cnt = torch.empty(n, dtype=torch.int8, device=DEV)
    ctx.encode(gd, rd)
    ctx.exchange()
    ctx.decode_apply(wd, -0.5, gtc.GTC_ACCUM_WEIGHTS, cnt)
    assert ctx.check() == gtc.GTC_OK
    del gd
    msg = ctx.message_tensor().cpu().numpy().view(np.uint32)
    idx = (msg >> 1).astype(np.int64)
    assert np.all(np.diff(idx) > 0) and idx[-1] < n
    rng = np.random.default_rng(0)
    T = gtc.GTC_TILE
    starts = [0, T - 100, 123_456 * T - 50, n - 4099, n - 1000] + list(rng.integers(0, n - 70_000, 12))
    for a in starts:
        b = min(n, a + 65_536)
        gw, rw = g[a:b].copy(), r0[a:b].copy()
        words, _ = oracle.encode(gw, rw, tau)
        exp_words = words + np.uint32(2 * a)  # global index a + i: word + 2a
        lo, hi = np.searchsorted(idx, a), np.searchsorted(idx, b)
        assert np.array_equal(msg[lo:hi], exp_words), a
        assert np.array_equal(bits(rd[a:b]), rw.view(np.uint32)), a
        c = oracle.decode_counts([words], b - a)
        assert np.array_equal(cnt[a:b].cpu().numpy().astype(np.int32), c), a
        w_exp = np.zeros(b - a, np.float32)
        oracle.apply(c, w_exp, tau, -0.5, oracle.ACCUM_WEIGHTS)
        assert np.array_equal(bits(wd[a:b]), w_exp.view(np.uint32)), a
    ctx.close()


# ------------------------------------------------------------------ bench launch configuration
def test_config2_fused_step_full_size():
    """The bench's N=1 step exactly: gtc_step (one fused kernel) on the LSTM-AM
    size, 3 steps over rotating gradients, residual + weights bit-exact."""
    n, tau = synth.LSTM_AM_PARAMS, 8.0
    sigma = synth.sigma_for_density(0.01, tau, synth.mean_abs_scale(n))
    gs = [synth.lstm_gradient(n, sigma, synth.BASE_SEED, t, 0) for t in range(3)]
    r_host = synth.uniform(n, -tau, tau, synth.rank_seed(0))
    w_host = synth.normal(n, synth.BASE_SEED, 0, 11) * np.float32(0.05)
    ctx = gtc.GTC(n, tau)
    gd = [to_dev(g) for g in gs]
    rd, wd = to_dev(r_host), to_dev(w_host)
    f = ctx.stepper(gd, rd, wd, -1e-3)
    for t in range(3):
        f(t)
        oracle.step([gs[t]], [r_host], w_host, tau, oracle.CMP_GT, -1e-3, oracle.ACCUM_WEIGHTS)
    torch.cuda.synchronize()
    assert np.array_equal(bits(rd), r_host.view(np.uint32))
    assert_float_parity(wd.cpu().numpy(), w_host, "weights")
    ctx.close()


def test_config5_fused_step_1e9_sampled():
    """n = 1e9 through gtc_step (the bench's launch configuration): residual and
    weights in sampled windows against the oracle on that window."""
    n, tau = 1_000_000_000, 8.0
    free, _ = torch.cuda.mem_get_info()
    if free < 24 * 2**30:
        pytest.skip("needs ~24 GB free device memory")
    sigma = synth.sigma_for_density(0.01, tau)
    g = synth.normal(n, synth.rank_seed(0), 0) * np.float32(sigma)
    r0 = synth.uniform(n, -tau, tau, synth.rank_seed(0))
    w0 = synth.normal(n, 5, 0) * np.float32(0.05)
    ctx = gtc.GTC(n, tau, max_words_per_rank=n // 20)
    gd, rd, wd = to_dev(g), to_dev(r0), to_dev(w0)
    ctx.step(gd, rd, wd, -0.5)
    assert ctx.check() == gtc.GTC_OK
    del gd
    rng = np.random.default_rng(1)
    T = gtc.GTC_TILE
    for a in [0, T - 100, n - 4099, n - 1000] + list(rng.integers(0, n - 70_000, 10)):
        b = min(n, a + 65_536)
        rw, ww = r0[a:b].copy(), w0[a:b].copy()
        oracle.step([g[a:b].copy()], [rw], ww, tau, oracle.CMP_GT, -0.5, oracle.ACCUM_WEIGHTS)
        assert np.array_equal(bits(rd[a:b]), rw.view(np.uint32)), a
        assert np.array_equal(bits(wd[a:b]), ww.view(np.uint32)), a
    ctx.close()


def test_serialized_message_matches_oracle_in_spec_layout():
    """A GPU message in SPEC.md:202's wire format (gtc_wire_pack over
    gtc_read_message): header and SPEC-layout words equal the oracle's
    message converted by hand (bit 31 = sign, bits 0..30 = index),
    and unpacking returns the canonical words."""
    import struct

    n, tau = 2 * gtc.GTC_TILE + 777, 8.0
    g = synth.correlated_gradient(n, 4.0, synth.BASE_SEED, 0, 0)
    r0 = synth.uniform(n, -tau, tau, synth.rank_seed(0))
    ctx = gtc.GTC(n, tau)
    ctx.encode(to_dev(g), to_dev(r0.copy()))
    blob = ctx.serialize_message()
    words, _ = oracle.encode(g, r0.copy(), tau, oracle.CMP_GT)
    assert blob[:4] == b"GTCU"
    assert struct.unpack_from("<QfI", blob, 4) == (n, tau, words.size)
    spec = np.frombuffer(blob, dtype="<u4", offset=20)
    assert np.array_equal(spec, ((words & 1) << 31) | (words >> 1))
    back, dim, t = gtc.gtc_wire_unpack(blob)
    assert np.array_equal(back, words) and dim == n and t == tau
    ctx.close()
