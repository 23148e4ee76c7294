"""Seeded synthetic inputs for GTC: the ONLY module shared by the oracle side
(tests, bench cpu_baseline) and the CUDA side (tests, bench, smoke).

It holds none of the method's arithmetic -- no thresholding, no residual update,
no packing -- only the input recipe of DESIGN.md Sec. "Inputs": gradient vectors
shaped like the paper's LSTM acoustic model (Sec. II-B:
5 LSTM layers x 768 units on 64x3 stacked log-mel input, 3,183 senones) with
seeded numpy Philox streams.  Every value is float32 and produced on the host
(callers copy it to the GPU themselves), except ``cuda_normal``, which draws
the 1e9-parameter gradients on the GPU with torch's seeded Philox generator.
"""
from __future__ import annotations

import math

import numpy as np

BASE_SEED = 1904105840
_GOLDEN = 0x9E3779B97F4A7C15

# PAPER.md:84 "5 LSTM layers with 768 units", input 64-dim log-mel stacked x3
# (=192), "about 24 M parameters", output 3,183 senones.  One bias
# set per gate block (4 gates x 768 = 3072).  Sum = 24,286,575.
LSTM_HIDDEN = 768
LSTM_LAYERS = 5
LSTM_INPUT = 192
SENONES = 3183


def lstm_am_segments():
    """(name, numel) of every trainable tensor of the student LSTM AM, in order."""
    segs = []
    g4 = 4 * LSTM_HIDDEN
    for layer in range(LSTM_LAYERS):
        fan_in = LSTM_INPUT if layer == 0 else LSTM_HIDDEN
        segs.append((f"lstm{layer}.W_ih", g4 * fan_in))
        segs.append((f"lstm{layer}.W_hh", g4 * LSTM_HIDDEN))
        segs.append((f"lstm{layer}.b", g4))
    segs.append(("out.W", SENONES * LSTM_HIDDEN))
    segs.append(("out.b", SENONES))
    return segs


LSTM_AM_PARAMS = sum(s for _, s in lstm_am_segments())  # 24,286,575


def rank_seed(rank: int, base: int = BASE_SEED) -> int:
    """Per-rank seed: base XOR ((rank+1) * golden mod 2^63) (SPEC.md:341 idea)."""
    return base ^ (((rank + 1) * _GOLDEN) % (1 << 63))


def _rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([int(k) & ((1 << 63) - 1) for k in key])))


def normal(n: int, seed: int, step: int = 0, stream: int = 0) -> np.ndarray:
    """i.i.d. N(0,1) float32 of length n, from stream (seed, step, stream)."""
    return _rng(seed, step, stream).standard_normal(n, dtype=np.float32)


def uniform(n: int, lo: float, hi: float, seed: int, step: int = 0, stream: int = 7) -> np.ndarray:
    """U(lo, hi) float32 of length n."""
    u = _rng(seed, step, stream).random(n, dtype=np.float32)
    return (np.float32(lo) + u * np.float32(hi - lo)).astype(np.float32)


def segment_scales(seed: int = BASE_SEED, lo: float = 0.25, hi: float = 4.0):
    """Per-tensor gradient scale s_l, log-uniform in [lo, hi] (DESIGN.md inputs)."""
    segs = lstm_am_segments()
    u = _rng(seed, 0, 99).random(len(segs))
    return np.exp(np.log(lo) + u * (np.log(hi) - np.log(lo))).astype(np.float32)


def mean_abs_scale(n: int, seed: int = BASE_SEED) -> float:
    """Size-weighted mean of the per-segment scales over the first n params."""
    segs, scales = lstm_am_segments(), segment_scales(seed)
    tot, acc = 0, 0.0
    for (_, s), sc in zip(segs, scales):
        take = min(s, n - tot)
        if take <= 0:
            break
        acc += take * float(sc)
        tot += take
    if tot < n:  # padded variants repeat the last scale
        acc += (n - tot) * float(scales[-1])
    return acc / n


def lstm_gradient(n: int, sigma: float, seed: int, step: int, rank: int = 0,
                  correlated: float = 0.0) -> np.ndarray:
    """LSTM-AM-shaped gradient: segment l gets s_l * sigma * z.

    n may differ from LSTM_AM_PARAMS (the last segment's scale continues for
    padded sizes, earlier segments are cut for smaller sizes).  With
    ``correlated`` = c > 0 the unit noise is c*mu + z_r with mu shared across
    ranks (makes counts of +-2 and cancellations appear)."""
    z = normal(n, rank_seed(rank, seed), step, 0)
    if correlated:
        mu = normal(n, seed, step, 1)
        z = (np.float32(correlated) * mu + z).astype(np.float32)
    scales = segment_scales(seed)
    out = np.empty(n, dtype=np.float32)
    off = 0
    for (_, s), sc in zip(lstm_am_segments(), scales):
        if off >= n:
            break
        e = min(n, off + s)
        out[off:e] = z[off:e] * np.float32(sc * sigma)
        off = e
    if off < n:
        out[off:] = z[off:] * np.float32(scales[-1] * sigma)
    return out


def dyadic_gradient(n: int, sigma: float, clip: float, seed: int, step: int, rank: int = 0,
                    frac_bits: int = 10) -> np.ndarray:
    """round(sigma*z*2^b)/2^b clipped to [-clip, clip]: every value is a multiple
    of 2^-b, so sums of a few hundred of them stay exact in float32."""
    z = normal(n, rank_seed(rank, seed), step, 2).astype(np.float64)
    q = np.round(z * sigma * (1 << frac_bits)) / (1 << frac_bits)
    return np.clip(q, -clip, clip).astype(np.float32)


def correlated_gradient(n: int, scale: float, seed: int, step: int, rank: int = 0) -> np.ndarray:
    """scale * (0.5*mu + z_r), mu ~ N(0,1) shared by all ranks of (seed, step)."""
    mu = normal(n, seed, step, 3)
    z = normal(n, rank_seed(rank, seed), step, 4)
    return (np.float32(scale) * (np.float32(0.5) * mu + z)).astype(np.float32)


def sigma_for_density(rho: float, tau: float, mean_scale: float = 1.0) -> float:
    """Input calibration (not part of the method): with r0 ~ U(-tau, tau) and
    g ~ s*N(0, sigma), P(|r0+g| crosses tau) ~= E|g| / (2 tau)
    = sigma * mean_scale * sqrt(2/pi) / (2 tau).  Solve for sigma."""
    return rho * tau * math.sqrt(2.0 * math.pi) / mean_scale


def cuda_normal(n: int, seed: int, step: int, rank: int = 0, device="cuda"):
    """i.i.d. N(0,1) float32 of length n generated ON THE GPU (torch's Philox
    generator seeded with (rank_seed(rank, seed) + step) mod 2^63).  For the
    1e9-parameter config (BASELINE configs[4]) where a host generator would
    take longer than the run; the oracle side copies back the windows it
    checks.  Holds no arithmetic of the method."""
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed((rank_seed(rank, seed) + 1_000_003 * step) % (1 << 63))
    return torch.randn(n, generator=gen, dtype=torch.float32, device=device)


def sigma_for_cycle_density(rho: float, tau: float, mean_scale: float = 1.0, n_buffers: int = 1,
                            correlated: float = 0.0) -> float:
    """Input calibration of the benchmark (not part of the method).  The bench
    applies n_buffers fixed gradients in rotation, so every element drifts by
    d = sum_j g_j per cycle and, once the residual is stationary, sends |d|/tau
    quanta per cycle: rho = E|d| / (n_buffers * tau) = sigma_e * sqrt(2/pi) /
    (sqrt(n_buffers) * tau), with sigma_e = sigma * mean_scale * sqrt(1 + c^2)
    for lstm_gradient(..., correlated=c).  Solve for sigma."""
    return rho * tau * math.sqrt(n_buffers) / (mean_scale * math.sqrt(2.0 / math.pi) *
                                               math.sqrt(1.0 + correlated * correlated))


def steady_residual(grads, tau: float, seed: int) -> np.ndarray:
    """A stationary residual for gradients applied in rotation:
    r0 = sign(sum_j g_j) * U(0, tau) (an element drifting up sits in (0, tau]
    between quanta), so the measured density equals sigma_for_cycle_density's
    target from the first step instead of after ~500 steps."""
    d = grads[0] if len(grads) == 1 else np.sum(np.stack(grads), axis=0, dtype=np.float32)
    u = uniform(grads[0].size, 0.0, tau, seed)
    np.negative(u, out=u, where=d < 0)
    return u
