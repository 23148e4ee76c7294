"""Pins of the oracle's SGD-momentum apply (oracle_apply_momentum; SURVEY
8(f) #2, reading M1) against things other than itself: SPEC's
worked sgd_step examples, a hand-worked dyadic run
(tests/golden/momentum_D.json), the reduction to ACCUM_WEIGHTS at mu = 0, and
the geometric closed form of a constant aggregate."""
from fractions import Fraction

import numpy as np
import pytest

import oracle

f32 = np.float32


def test_worked_vector_D(golden):
    gv = golden("momentum_D.json")
    w = np.array(gv["w0"], f32)
    buf = np.array(gv["buf0"], f32)
    for t, c in enumerate(gv["counts"]):
        oracle.apply_momentum(np.array(c, np.int32), w, buf, gv["tau"], gv["alpha"], gv["mu"])
        assert np.array_equal(buf, np.array(gv["buf"][t], f32)), f"buf at step {t}"
        assert np.array_equal(w, np.array(gv["weights"][t], f32)), f"weights at step {t}"


def test_spec_examples(golden):
    ex = golden("momentum_D.json")["spec_examples"]
    # one step, momentum 0
    w, buf = np.array([ex["p0"]], f32), np.zeros(1, f32)
    oracle.apply_momentum(np.array([ex["count"]], np.int32), w, buf, ex["tau"], -ex["lr"], 0.0)
    assert w[0] == f32(ex["one_step_mu0"])
    # g = 0 everywhere (and no momentum yet) -> unchanged, bitwise
    w0 = np.array([1.5, -0.0, 0.0, -3.25, 7e-39], f32)
    w, buf = w0.copy(), np.zeros(5, f32)
    oracle.apply_momentum(np.zeros(5, np.int32), w, buf, 0.5, -0.1, 0.9)
    assert np.array_equal(w.view(np.uint32), w0.view(np.uint32))
    assert not buf.any()
    # two steps, momentum 0.9, against the exact real recursion
    # (p = 1 - lr*g - lr*(mu*g + g) = 0.855): within 2 ulp of fp32
    w, buf = np.array([ex["p0"]], f32), np.zeros(1, f32)
    for _ in range(2):
        oracle.apply_momentum(np.array([ex["count"]], np.int32), w, buf, ex["tau"], -ex["lr"], ex["two_step_mu"])
    g, lr, mu = Fraction(1, 2), Fraction(1, 10), Fraction(9, 10)
    exact = 1 - lr * g - lr * (mu * g + g)
    assert float(exact) == ex["two_step_exact"]
    assert abs(float(w[0]) - float(exact)) <= 2 * float(np.spacing(f32(exact)))


def test_mu0_reduces_to_weights_mode():
    """mu = 0 and a zero buffer: the momentum apply is ACCUM_WEIGHTS on c != 0
    (oracle_apply, pinned by worked vector C) and the identity elsewhere."""
    rng = np.random.default_rng(7)
    n = 10_000
    c = rng.integers(-3, 4, n).astype(np.int32)
    w0 = (rng.standard_normal(n) * 3).astype(f32)
    w_m, buf = w0.copy(), np.zeros(n, f32)
    oracle.apply_momentum(c, w_m, buf, 0.37, -0.01, 0.0)
    w_a = w0.copy()
    oracle.apply(c, w_a, 0.37, -0.01, oracle.ACCUM_WEIGHTS)
    assert np.array_equal(w_m.view(np.uint32), w_a.view(np.uint32))
    assert np.array_equal(buf, (c.astype(f32) * f32(0.37)).astype(f32))


@pytest.mark.parametrize("cval", [1, -2, 3])
def test_constant_aggregate_closed_form(cval):
    """A constant count c for T steps from buf = 0, dyadic mu = 1/2:
    buf_T = u (1 - mu^T) / (1 - mu) and W_T = W_0 + alpha sum_t buf_t, exact."""
    tau, mu, alpha, T = 0.125, 0.5, -0.25, 12
    w, buf = np.array([2.0], f32), np.zeros(1, f32)
    u = Fraction(cval) * Fraction(tau)
    wsum = Fraction(2)
    for t in range(1, T + 1):
        oracle.apply_momentum(np.array([cval], np.int32), w, buf, tau, alpha, mu)
        b_t = u * (1 - Fraction(mu) ** t) / (1 - Fraction(mu))
        wsum += Fraction(alpha) * b_t
        assert Fraction(float(buf[0])) == b_t
        assert Fraction(float(w[0])) == wsum


def test_momentum_step_dispatch():
    """oracle.step in ACCUM_MOMENTUM mode is encode -> decode_counts ->
    apply_momentum; its messages and counts equal the WEIGHTS-mode step's."""
    rng = np.random.default_rng(3)
    n, tau = 5000, 1.0
    gs = [(rng.standard_normal(n) * 0.8).astype(f32) for _ in range(3)]
    r1 = [np.zeros(n, f32) for _ in range(3)]
    r2 = [np.zeros(n, f32) for _ in range(3)]
    w1, w2, buf = np.ones(n, f32), np.ones(n, f32), np.zeros(n, f32)
    m1, c1, _ = oracle.step(gs, r1, w1, tau, oracle.CMP_GT, -0.1, oracle.ACCUM_WEIGHTS)
    m2, c2, _ = oracle.step(gs, r2, w2, tau, oracle.CMP_GT, -0.1, oracle.ACCUM_MOMENTUM, buf=buf, mu=0.0)
    assert all(np.array_equal(a, b) for a, b in zip(m1, m2))
    assert np.array_equal(c1, c2)
    assert np.array_equal(w1.view(np.uint32), w2.view(np.uint32))  # mu = 0: the reduction above
