"""Pins for the BMUF oracle (Sec. VI-B, Eqs. 1-5) -- CPU only.

Each pin is something other than the oracle's own formula: the SPEC's worked
scalar run, reductions to plain model averaging and to the identity, a fixed
point, the Eq. (5) examples, and a multi-block run on dyadic values whose
closed form is evaluated exactly with Fractions."""
from fractions import Fraction

import numpy as np
import pytest

import oracle


def f32(x):
    return np.asarray(x, dtype=np.float32)


def test_worked_scalar_run():
    """Wg(0)=0, Delta(0)=0, eta=0.5, zeta=1, Wbar(1)=1 => G=1, Delta=1, Wg=1.5."""
    ws = [f32([1.0])]
    wg, d = f32([0.0]), f32([0.0])
    oracle.bmuf_step(ws, wg, d, 0.5, 1.0)
    assert wg.tolist() == [1.5] and d.tolist() == [1.0]
    assert ws[0].tolist() == [1.5]  # every worker restarts from Wg


@pytest.mark.parametrize("N", [1, 2, 3, 8])
def test_eta0_zeta1_is_model_averaging(N):
    """eta=0, zeta=1: Eqs. (2)-(4) collapse to Wg = Wbar, the plain model average (Eq. 1)."""
    rng = np.random.default_rng(N)
    n = 10_000
    ws = [rng.standard_normal(n).astype(np.float32) for _ in range(N)]
    # numpy's own mean of the float64 copies (a library routine), rounded once
    mean = np.mean(np.stack(ws).astype(np.float64), axis=0).astype(np.float32)
    wg = np.zeros(n, np.float32)       # Wg(t-1) = 0: G = Wbar and Wg = 0 + G exactly
    d = rng.standard_normal(n).astype(np.float32)  # eta = 0 forgets Delta(t-1)
    oracle.bmuf_step([w.copy() for w in ws], wg, d, 0.0, 1.0)
    assert np.array_equal(wg, mean) and np.array_equal(d, mean)


def test_identity_single_worker():
    """N=1, eta=0, zeta=1, Wg(t-1)=0: Wg = W exactly (SPEC.md:598 reduction)."""
    rng = np.random.default_rng(0)
    w = rng.standard_normal(5000).astype(np.float32)
    ws = [w.copy()]
    wg, d = np.zeros_like(w), np.zeros_like(w)
    oracle.bmuf_step(ws, wg, d, 0.0, 1.0)
    assert np.array_equal(wg, w) and np.array_equal(ws[0], w)


def test_fixed_point():
    """Wbar == Wg(t-1) and Delta(t-1) == 0: nothing moves."""
    rng = np.random.default_rng(1)
    wg = rng.standard_normal(3000).astype(np.float32)
    ws = [wg.copy(), wg.copy(), wg.copy()]
    wg0 = wg.copy()
    d = np.zeros_like(wg)
    oracle.bmuf_step(ws, wg, d, 0.9, 2.5)
    assert np.array_equal(wg, wg0) and not np.any(d)


@pytest.mark.parametrize("C,N,eta,zeta", [(1, 8, 0.875, 1.0), (1, 1, 0.0, 1.0), (2, 64, 0.9, 12.8)])
def test_eq5_zeta(C, N, eta, zeta):
    """Eq. (5) examples."""
    assert abs(oracle.bmuf_zeta(C, N, eta) - zeta) < 1e-9


def test_multi_block_dyadic_closed_form():
    """Workers always return c; eta = 1/2, zeta = 1; dyadic values keep every
    fp32 operation exact, so the oracle must equal the exact recurrence
    Delta_t = eta Delta_{t-1} + zeta (c - Wg_{t-1}), Wg_t = Wg_{t-1} + (1 + eta) Delta_t."""
    c = Fraction(3, 4)
    eta, zeta = Fraction(1, 2), Fraction(1)
    wg_e, d_e = Fraction(0), Fraction(0)
    wg, d = f32([0.0]), f32([0.0])
    for t in range(8):
        ws = [f32([float(c)]), f32([float(c)])]
        oracle.bmuf_step(ws, wg, d, float(eta), float(zeta))
        d_e = eta * d_e + zeta * (c - wg_e)
        wg_e = wg_e + (1 + eta) * d_e
        assert Fraction(float(d[0])) == d_e and Fraction(float(wg[0])) == wg_e, t
