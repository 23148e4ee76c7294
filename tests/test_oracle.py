"""Pins for the CPU oracle (oracle/gtc_oracle.c) -- CPU only, no GPU.

Each test pins the oracle to something other than itself: a hand-worked vector
(tests/golden/*.json, cited), a closed form, an invariant the paper's rule
implies, a brute-force enumeration, or exact rational arithmetic.  The encode
rule is PAPER.md:222 (Sec. VI-A); readings R1..R10 are in DESIGN.md.
"""
from fractions import Fraction
import ctypes
import itertools
import math

import numpy as np
import pytest

import oracle
import synth

MODES = [oracle.CMP_GT, oracle.CMP_GE]
MODE_NAME = {oracle.CMP_GT: "GT", oracle.CMP_GE: "GE"}


def f32(x):
    return np.asarray(x, dtype=np.float32)


# ---------------------------------------------------------------- worked vectors
@pytest.mark.parametrize("mode", MODES)
def test_worked_vector_A(golden, mode):
    gv = golden("worked_vector_A.json")
    r = f32(gv["r0"]).copy()
    words, nf = oracle.encode(f32(gv["g"]), r, gv["tau"], mode)
    exp = gv[MODE_NAME[mode]]
    assert words.tolist() == exp["words"]
    assert r.tolist() == exp["r"]
    assert not nf


@pytest.mark.parametrize("mode", MODES)
def test_worked_vector_B_multistep(golden, mode):
    gv = golden("worked_vector_B.json")
    exp = gv[MODE_NAME[mode]]
    r = f32([0.0])
    emitted = []
    for t, gt in enumerate(gv["g"], start=1):
        words, _ = oracle.encode(f32([gt]), r, gv["tau"], mode)
        assert words.tolist() == exp["words_per_step"][t - 1]
        assert float(r[0]) == exp["r_after"][t - 1]
        if len(words):
            emitted.append(t)
    assert emitted == exp["emit_steps"]
    # conservation: sum g == r_T + tau * sum(signs)
    assert sum(gv["g"]) == float(r[0]) + gv["tau"] * len(emitted)


def test_worked_vector_C_decode_apply(golden):
    gv = golden("worked_vector_C.json")
    n, tau = gv["n"], gv["tau"]
    counts = oracle.decode_counts([np.array(m, np.uint32) for m in gv["messages"]], n)
    assert counts.tolist() == gv["counts"]
    u = np.zeros(n, np.float32)
    oracle.apply(counts, u, tau, 1.0, oracle.ACCUM_UPDATE)
    assert u.tolist() == gv["update"]
    w = np.full(n, gv["w0"], np.float32)
    oracle.apply(counts, w, tau, gv["alpha"], oracle.ACCUM_WEIGHTS)
    assert w.tolist() == gv["weights"]


def test_pack_layout_small_indices(golden):
    """Word layout R3 through the encoder: one selected element at index i."""
    for case in golden("pack_layout.json")["cases"]:
        i = case["index"]
        if i > 64:
            continue
        g = np.zeros(i + 1, np.float32)
        g[i] = -9.0 if case["negative"] else 9.0
        r = np.zeros_like(g)
        words, _ = oracle.encode(g, r, 8.0)
        assert words.tolist() == [case["word"]]
        # and decode maps it back to the same (index, sign)
        c = oracle.decode_counts([words], i + 1)
        assert c[i] == (-1 if case["negative"] else 1) and np.count_nonzero(c) == 1


# ---------------------------------------------------------------- library routine
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 31, 32, 33, 4095, 4097, 100_003])
def test_encode_matches_flatnonzero(mode, n):
    """Support set == np.flatnonzero(|v| > tau) (resp. >=); signs == v<0."""
    rng = np.random.default_rng(n + 17 * mode)
    r0 = rng.uniform(-8, 8, n).astype(np.float32)
    g = (rng.standard_normal(n) * 3).astype(np.float32)
    # plant exact ties
    if n > 4:
        r0[::5] = 0.0
        g[::5] = np.where(rng.random(g[::5].shape) < 0.5, 8.0, -8.0)
    v = (r0 + g).astype(np.float32)  # numpy float32 add is IEEE RNE
    r = r0.copy()
    words, _ = oracle.encode(g, r, 8.0, mode)
    sel = np.abs(v) > 8 if mode == oracle.CMP_GT else np.abs(v) >= 8
    idx = np.flatnonzero(sel)
    assert np.array_equal(words >> 1, idx.astype(np.uint32))
    assert np.array_equal((words & 1).astype(bool), v[idx] < 0)
    assert np.array_equal(r[~sel], v[~sel])


def test_counts_match_add_at():
    rng = np.random.default_rng(5)
    n, N = 50_000, 5
    msgs = []
    for _ in range(N):
        idx = np.sort(rng.choice(n, size=rng.integers(0, 5000), replace=False)).astype(np.uint32)
        neg = rng.random(idx.size) < 0.5
        msgs.append((idx << 1) | neg.astype(np.uint32))
    c = oracle.decode_counts(msgs, n)
    ref = np.zeros(n, np.int64)
    for m in msgs:
        np.add.at(ref, (m >> 1).astype(np.int64), np.where(m & 1, -1, 1))
    assert np.array_equal(c, ref)
    assert np.abs(c).max() <= N
    assert c.sum() == sum(int(np.sum(1 - 2 * (m & 1).astype(np.int64))) for m in msgs)


# ---------------------------------------------------------------- invariants
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("N", [1, 3])
def test_long_run_conservation_dyadic_exact(mode, N):
    """Sum_t g_t == r_T + tau * Sum_t s_t EXACTLY for 100 steps on dyadic input
    (every fp32 op is exact there), per worker."""
    n, tau, T = 20_000, 8.0, 100
    rs = [np.zeros(n, np.float32) for _ in range(N)]
    gsum = [np.zeros(n, np.float64) for _ in range(N)]
    ssum = [np.zeros(n, np.int64) for _ in range(N)]
    target = np.zeros(n, np.float32)
    ctot = np.zeros(n, np.int64)
    for t in range(T):
        gs = [synth.dyadic_gradient(n, 3.0, tau, synth.BASE_SEED, t, w) for w in range(N)]
        msgs, counts, _ = oracle.step(gs, rs, target, tau, mode, 1.0, oracle.ACCUM_UPDATE)
        ctot += counts
        for w in range(N):
            gsum[w] += gs[w]
            m = msgs[w]
            np.add.at(ssum[w], (m >> 1).astype(np.int64), np.where(m & 1, -1, 1))
    for w in range(N):
        assert np.array_equal(gsum[w], rs[w].astype(np.float64) + tau * ssum[w])
    # the applied update is the sum of all quanta sent by all workers
    assert np.array_equal(target.astype(np.float64), tau * ctot)
    assert np.array_equal(ctot, sum(ssum))


@pytest.mark.parametrize("tau", [0.125, 1.0, 8.0])
def test_per_step_reconstruction_exact_pow2_tau(tau):
    """r_new + s*tau == v bit-exactly when tau is a power of two (DESIGN R2/C4)."""
    n = 200_000
    rng = np.random.default_rng(1)
    r0 = rng.uniform(-tau, tau, n).astype(np.float32)
    g = (rng.standard_normal(n) * tau).astype(np.float32)
    v = (r0 + g).astype(np.float32)
    r = r0.copy()
    words, _ = oracle.encode(g, r, tau)
    s = np.zeros(n, np.float32)
    s[(words >> 1).astype(np.int64)] = np.where(words & 1, -tau, tau)
    assert np.array_equal((r + s).astype(np.float32), v)


def test_per_step_reconstruction_within_ulp_general_tau():
    n, tau = 200_000, 0.1
    rng = np.random.default_rng(2)
    r0 = rng.uniform(-tau, tau, n).astype(np.float32)
    g = (rng.standard_normal(n) * 3 * tau).astype(np.float32)
    v = (r0 + g).astype(np.float32)
    r = r0.copy()
    words, _ = oracle.encode(g, r, tau)
    s = np.zeros(n, np.float64)
    s[(words >> 1).astype(np.int64)] = np.where(words & 1, -1.0, 1.0) * np.float64(np.float32(tau))
    err = np.abs(r.astype(np.float64) + s - v.astype(np.float64))
    assert np.all(err <= np.spacing(np.abs(v)).astype(np.float64))


@pytest.mark.parametrize("mode", MODES)
def test_residual_bound_when_gradient_bounded(mode):
    """|g|inf <= tau each step => GE: |r| < tau, GT: |r| <= tau (DESIGN R2/C3)."""
    n, tau = 50_000, 1.0
    r = np.zeros(n, np.float32)
    for t in range(30):
        g = np.clip(synth.normal(n, 11, t) * 0.6, -tau, tau).astype(np.float32)
        oracle.encode(g, r, tau, mode)
        if mode == oracle.CMP_GE:
            assert np.abs(r).max() < tau
        else:
            assert np.abs(r).max() <= tau


def test_emits_at_most_one_quantum():
    """R2: |v| = 20 at tau=8 emits once; r keeps 12 (not 4)."""
    r = np.zeros(3, np.float32)
    words, _ = oracle.encode(f32([20, -100, 7]), r, 8.0)
    assert words.tolist() == [0, 3]
    assert r.tolist() == [12.0, -92.0, 7.0]


# ---------------------------------------------------------------- brute force
@pytest.mark.parametrize("mode", MODES)
def test_brute_force_tiny_grid(mode):
    """All v in {-2t,-1.5t,-t,-.5t,0,.5t,t,1.5t,2t}^(n*N) for N workers, n*N <= 6.

    Every combination is laid side by side in one long vector per worker (the
    rule is elementwise, so one oracle step evaluates all of them at once); the
    expected quanta are written out per element by plain Python."""
    tau = 8.0
    grid = np.array([x * tau for x in (-2, -1.5, -1, -0.5, 0, 0.5, 1, 1.5, 2)], np.float32)
    for n, N in [(1, 3), (2, 3), (3, 2), (6, 1)]:
        combos = np.array(list(itertools.product(range(9), repeat=n * N)), np.int64)
        vs = [grid[combos[:, w * n:(w + 1) * n]].reshape(-1).copy() for w in range(N)]
        rs = [v.copy() for v in vs]
        target = np.zeros(vs[0].size, np.float32)
        msgs, counts, _ = oracle.step(None, rs, target, tau, mode, 1.0, oracle.ACCUM_UPDATE)
        q_of = {}
        for x in grid.tolist():
            hit = abs(x) > tau if mode == oracle.CMP_GT else abs(x) >= tau
            q_of[x] = (tau if x > 0 else -tau) if hit else 0.0
        dense = np.zeros(vs[0].size, np.float64)
        for w in range(N):
            q = np.array([q_of[x] for x in vs[w].tolist()])
            dense += q
            assert np.array_equal(rs[w].astype(np.float64), vs[w].astype(np.float64) - q)
        assert np.array_equal(target.astype(np.float64), dense)
        assert np.array_equal(counts * tau, dense)


# ---------------------------------------------------------------- special cases
def test_zero_gradient_empty_message():
    r = np.array([1.0, -3.0, 0.0, 7.5], np.float32)
    r0 = r.copy()
    words, _ = oracle.encode(np.zeros(4, np.float32), r, 8.0)
    assert words.size == 0 and np.array_equal(r, r0)


def test_tau_below_min_is_sign_quantization():
    """tau below every nonzero |v| -> every nonzero coordinate is emitted."""
    rng = np.random.default_rng(3)
    v = rng.standard_normal(1000).astype(np.float32)
    v[::7] = 0
    r = v.copy()
    words, _ = oracle.encode(None, r, 1e-6)
    nz = np.flatnonzero(v)
    assert np.array_equal(words >> 1, nz.astype(np.uint32))
    assert np.array_equal((words & 1).astype(bool), v[nz] < 0)


def test_single_worker_counts_are_signs():
    rng = np.random.default_rng(4)
    g = (rng.standard_normal(10_000) * 8).astype(np.float32)
    r = np.zeros_like(g)
    target = np.zeros_like(g)
    msgs, counts, _ = oracle.step([g], [r], target, 8.0)
    m = msgs[0]
    exp = np.zeros(g.size, np.int32)
    exp[(m >> 1).astype(np.int64)] = np.where(m & 1, -1, 1)
    assert np.array_equal(counts, exp)


def test_nonfinite():
    """R9: NaN never emitted (|NaN| > tau is false), stays in r; +-Inf emitted."""
    r = np.zeros(4, np.float32)
    words, nf = oracle.encode(f32([np.nan, np.inf, -np.inf, 1.0]), r, 8.0)
    assert nf
    assert words.tolist() == [2, 5]
    assert np.isnan(r[0]) and r[1] == np.inf and r[2] == -np.inf and r[3] == 1.0
    r = np.zeros(2, np.float32)
    _, nf = oracle.encode(f32([1.0, 2.0]), r, 8.0)
    assert not nf


def test_denormals_preserved():
    tiny = np.float32(1e-45)  # smallest denormal
    r = f32([tiny, -tiny])
    words, _ = oracle.encode(f32([tiny, 0.0]), r, 1e-45)
    # |2*tiny| > tau=tiny -> emitted, residual = tiny (not flushed to 0)
    assert words.tolist() == [0]
    assert r[0] == tiny and r[1] == -tiny


# ---------------------------------------------------------------- apply arithmetic
def _round_f32(fr: Fraction) -> np.float32:
    """Correct round-to-nearest-even of an exact rational to binary32."""
    x = np.float32(float(fr))
    best = None
    for c in (np.nextafter(x, np.float32(-np.inf)), x, np.nextafter(x, np.float32(np.inf))):
        d = abs(Fraction(float(c)) - fr)
        key = (d, int(np.array(c, np.float32).view(np.uint32)) & 1)
        if best is None or key < best[0]:
            best = (key, c)
    return np.float32(best[1])


def test_apply_is_single_rounding_fma():
    """R8: W = fmaf(alpha, fl(c*tau), W): one rounding of the exact alpha*u + W."""
    rng = np.random.default_rng(6)
    n = 3000
    tau = np.float32(0.1)
    counts = rng.integers(-8, 9, n).astype(np.int32)
    w0 = rng.uniform(-1, 1, n).astype(np.float32)
    alpha = np.float32(-1.0 / 3.0)
    w = w0.copy()
    oracle.apply(counts, w, float(tau), float(alpha), oracle.ACCUM_WEIGHTS)
    differs_from_unfused = 0
    for i in range(n):
        c = int(counts[i])
        if c == 0:
            assert w[i] == w0[i]
            continue
        u = _round_f32(Fraction(c) * Fraction(float(tau)))
        exp = _round_f32(Fraction(float(alpha)) * Fraction(float(u)) + Fraction(float(w0[i])))
        assert w[i] == exp, i
        unfused = np.float32(np.float32(alpha * u) + w0[i])
        differs_from_unfused += int(unfused != exp)
    assert differs_from_unfused > 0  # the pin can tell fma from mul+add


def test_apply_update_mode_rounding():
    rng = np.random.default_rng(7)
    n = 2000
    tau = np.float32(7.3)
    counts = rng.integers(-8, 9, n).astype(np.int32)
    u0 = rng.uniform(-100, 100, n).astype(np.float32)
    u = u0.copy()
    oracle.apply(counts, u, float(tau), 1.0, oracle.ACCUM_UPDATE)
    for i in range(n):
        c = int(counts[i])
        if c == 0:
            assert u[i] == u0[i]
            continue
        q = _round_f32(Fraction(c) * Fraction(float(tau)))
        assert u[i] == _round_f32(Fraction(float(u0[i])) + Fraction(float(q)))


# ---------------------------------------------------------------- errors
def test_errors():
    L = oracle.lib()
    k = ctypes.c_int64()
    nf = ctypes.c_int()
    assert L.oracle_encode(1 << 31, 8.0, 0, None, None, None, ctypes.byref(k), ctypes.byref(nf)) == oracle.EDIM
    assert L.oracle_encode(-1, 8.0, 0, None, None, None, ctypes.byref(k), ctypes.byref(nf)) == oracle.EDIM
    for bad in (0.0, -1.0, float("nan"), float("inf")):
        with pytest.raises(oracle.OracleError):
            oracle.encode(None, np.zeros(3, np.float32), bad)
    with pytest.raises(oracle.OracleError):  # not strictly increasing
        oracle.decode_counts([np.array([4, 4], np.uint32)], 10)
    with pytest.raises(oracle.OracleError):  # descending
        oracle.decode_counts([np.array([8, 2], np.uint32)], 10)
    with pytest.raises(oracle.OracleError):  # index >= n
        oracle.decode_counts([np.array([20], np.uint32)], 10)


# ---------------------------------------------------------------- input recipe
def test_lstm_am_param_count():
    """5x768 LSTM, 192-dim input, 3,183 senones, 'about 24 M'."""
    assert synth.LSTM_AM_PARAMS == 24_286_575


def test_density_closed_form():
    """r0~U(-tau,tau), g~N(0,sigma): rho ~= sigma*sqrt(2/pi)/(2 tau) (statistical)."""
    n, tau = 1_000_000, 8.0
    for rho in (0.001, 0.01, 0.1):
        sigma = synth.sigma_for_density(rho, tau)
        r = synth.uniform(n, -tau, tau, 1)
        g = synth.normal(n, 2) * np.float32(sigma)
        words, _ = oracle.encode(g.astype(np.float32), r, tau)
        got = words.size / n
        assert abs(got - rho) / rho < 0.1, (rho, got)


@pytest.mark.parametrize("nb,corr", [(3, 0.0), (1, 0.0), (3, 0.5)])
def test_cycle_density_closed_form(nb, corr):
    """The bench's input recipe: nb LSTM-shaped gradients applied in rotation
    from synth.steady_residual; sigma_for_cycle_density's target density holds
    from the first cycle on and stays (oracle encode, statistical)."""
    n, tau, rho = 300_000, 8.0, 0.01
    sigma = synth.sigma_for_cycle_density(rho, tau, synth.mean_abs_scale(n), nb, corr)
    gs = [synth.lstm_gradient(n, sigma, synth.BASE_SEED, t, 1, corr) for t in range(nb)]
    r = synth.steady_residual(gs, tau, 5)
    dens = []
    for t in range(60):
        words, _ = oracle.encode(gs[t % nb], r, tau)
        dens.append(words.size / n)
    for a in (0, 30):
        got = float(np.mean(dens[a:a + 30]))
        assert abs(got - rho) / rho < 0.1, (a, got)


def test_determinism():
    g = synth.normal(100_000, 9) * np.float32(5)
    a, b = np.zeros(100_000, np.float32), np.zeros(100_000, np.float32)
    wa, _ = oracle.encode(g, a, 8.0)
    wb, _ = oracle.encode(g, b, 8.0)
    assert np.array_equal(wa, wb) and np.array_equal(a.view(np.uint32), b.view(np.uint32))
