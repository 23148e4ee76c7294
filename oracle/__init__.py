"""CPU oracle for Gradient Threshold Compression (Sec. VI-A).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1904_10584_b200``) never imports it and
shares no code with it; ``liboracle.so`` is built from ``gtc_oracle.c`` alone.

This module is argument marshalling (numpy <-> ctypes) around ``liboracle.so``;
all arithmetic is in ``gtc_oracle.c``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gtc_oracle.c")
LIB_PATH = os.path.join(_HERE, "liboracle.so")

CMP_GT = 0
CMP_GE = 1
ACCUM_WEIGHTS = 0
ACCUM_UPDATE = 1
ACCUM_MOMENTUM = 2  # the same value as GTC_ACCUM_MOMENTUM; oracle.step's own dispatch

OK, EDIM, EINVAL, ECORRUPT = 0, 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with status {code}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain gcc, no CUDA)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "gtc_oracle.h"))
    ):
        cmd = ["gcc", "-std=c11", "-O2", "-fno-fast-math", "-ffp-contract=off",
               "-fPIC", "-shared", "-o", LIB_PATH, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        i64, f32, i32, vp = ctypes.c_int64, ctypes.c_float, ctypes.c_int, ctypes.c_void_p
        L.oracle_encode.argtypes = [i64, f32, i32, vp, vp, vp,
                                    ctypes.POINTER(i64), ctypes.POINTER(i32)]
        L.oracle_encode.restype = i32
        L.oracle_apply_momentum.argtypes = [i64, f32, vp, vp, vp, f32, f32]
        L.oracle_apply_momentum.restype = i32
        L.oracle_decode_counts.argtypes = [i64, i32, vp, vp, vp]
        L.oracle_decode_counts.restype = i32
        L.oracle_apply.argtypes = [i64, f32, vp, vp, f32, i32]
        L.oracle_apply.restype = i32
        L.oracle_step.argtypes = [i64, f32, i32, i32, vp, vp, vp, vp, vp, vp, f32, i32,
                                  ctypes.POINTER(i32)]
        L.oracle_step.restype = i32
        L.oracle_bmuf_step.argtypes = [i64, i32, vp, vp, vp, f32, f32, vp]
        L.oracle_bmuf_step.restype = i32
        L.oracle_bmuf_zeta.argtypes = [ctypes.c_double, i32, ctypes.c_double]
        L.oracle_bmuf_zeta.restype = ctypes.c_double
        _lib = L
    return _lib


def _f32(a, name):
    if not (isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags.c_contiguous):
        raise TypeError(f"{name} must be a C-contiguous float32 numpy array")
    return a


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def encode(g, r, tau: float, cmp_mode: int = CMP_GT):
    """Encode one worker (P:222 steps 1-4).  ``r`` is updated in place.

    Returns ``(words uint32[k], nonfinite bool)``.  ``g`` may be None (then
    ``r`` already holds r+g)."""
    _f32(r, "r")
    n = r.size
    if g is not None:
        _f32(g, "g")
        if g.size != n:
            raise ValueError("g and r differ in size")
    words = np.empty(max(n, 1), dtype=np.uint32)
    k = ctypes.c_int64(0)
    nf = ctypes.c_int(0)
    st = lib().oracle_encode(n, float(tau), cmp_mode, _ptr(g), _ptr(r), _ptr(words),
                             ctypes.byref(k), ctypes.byref(nf))
    if st != OK:
        raise OracleError(st, "encode")
    return words[: k.value].copy(), bool(nf.value)


def decode_counts(msgs, n: int):
    """Aggregate messages into int32 counts ("aggregated", reading R6)."""
    msgs = [np.ascontiguousarray(m, dtype=np.uint32) for m in msgs]
    counts = np.empty(max(n, 1), dtype=np.int32)
    ptrs = (ctypes.c_void_p * max(len(msgs), 1))(*[m.ctypes.data for m in msgs])
    ks = np.array([m.size for m in msgs] or [0], dtype=np.int64)
    st = lib().oracle_decode_counts(n, len(msgs), ctypes.cast(ptrs, ctypes.c_void_p),
                                    _ptr(ks), _ptr(counts))
    if st != OK:
        raise OracleError(st, "decode_counts")
    return counts[:n].copy()


def apply(counts, target, tau: float, alpha: float = 1.0, accum_mode: int = ACCUM_WEIGHTS):
    """Apply count*tau to ``target`` in place ("updated based on the aggregate", R8)."""
    counts = np.ascontiguousarray(counts, dtype=np.int32)
    _f32(target, "target")
    if counts.size != target.size:
        raise ValueError("counts and target differ in size")
    st = lib().oracle_apply(target.size, float(tau), _ptr(counts), _ptr(target),
                            float(alpha), accum_mode)
    if st != OK:
        raise OracleError(st, "apply")
    return target


def apply_momentum(counts, w, buf, tau: float, alpha: float, mu: float):
    """SGD-momentum apply of the aggregate (reading M1): for every i,
    buf = fl(fl(mu*buf) + fl(c*tau)); w = fmaf(alpha, buf, w).  In place."""
    counts = np.ascontiguousarray(counts, dtype=np.int32)
    _f32(w, "w")
    _f32(buf, "buf")
    if not (counts.size == w.size == buf.size):
        raise ValueError("counts, w and buf differ in size")
    st = lib().oracle_apply_momentum(w.size, float(tau), _ptr(counts), _ptr(w), _ptr(buf), float(alpha), float(mu))
    if st != OK:
        raise OracleError(st, "apply_momentum")
    return w


def step(gs, rs, target, tau: float, cmp_mode: int = CMP_GT, alpha: float = 1.0,
         accum_mode: int = ACCUM_WEIGHTS, buf=None, mu: float = 0.0):
    """One synchronous GTC step over len(rs) simulated workers.

    ``rs`` and ``target`` (and ``buf`` for ACCUM_MOMENTUM) are updated in
    place.  Returns ``(messages list[uint32 array], counts int32[n], nonfinite bool)``."""
    if accum_mode == ACCUM_MOMENTUM:
        # encode every worker, aggregate, then the momentum apply (all steps in liboracle)
        msgs, nfs = [], False
        for w, r in enumerate(rs):
            m, nf = encode(gs[w] if gs is not None else None, r, tau, cmp_mode)
            msgs.append(m)
            nfs |= nf
        counts = decode_counts(msgs, target.size)
        apply_momentum(counts, target, buf, tau, alpha, mu)
        return msgs, counts, nfs
    nw = len(rs)
    n = target.size
    for r in rs:
        _f32(r, "r")
    _f32(target, "target")
    if gs is not None:
        for g in gs:
            _f32(g, "g")
    words = [np.empty(max(n, 1), dtype=np.uint32) for _ in range(nw)]
    ks = np.zeros(nw, dtype=np.int64)
    counts = np.empty(max(n, 1), dtype=np.int32)
    VP = ctypes.c_void_p * nw
    gp = VP(*[g.ctypes.data for g in gs]) if gs is not None else None
    rp = VP(*[r.ctypes.data for r in rs])
    wp = VP(*[w.ctypes.data for w in words])
    nf = ctypes.c_int(0)
    st = lib().oracle_step(n, float(tau), cmp_mode, nw,
                           ctypes.cast(gp, ctypes.c_void_p) if gp is not None else None,
                           ctypes.cast(rp, ctypes.c_void_p), ctypes.cast(wp, ctypes.c_void_p),
                           _ptr(ks), _ptr(counts), _ptr(target), float(alpha), accum_mode,
                           ctypes.byref(nf))
    if st != OK:
        raise OracleError(st, "step")
    return [words[w][: ks[w]].copy() for w in range(nw)], counts[:n].copy(), bool(nf.value)


def bmuf_step(ws, wg, delta, eta: float, zeta: float):
    """One BMUF step (Eqs. 1-4).  ``wg`` and ``delta`` are
    updated in place; every worker model in ``ws`` is set to the new ``wg``."""
    nw = len(ws)
    for a in list(ws) + [wg, delta]:
        _f32(a, "bmuf array")
        if a.size != wg.size:
            raise ValueError("size mismatch")
    VP = ctypes.c_void_p * max(nw, 1)
    wp = VP(*[w.ctypes.data for w in ws])
    st = lib().oracle_bmuf_step(wg.size, nw, ctypes.cast(wp, ctypes.c_void_p), _ptr(wg), _ptr(delta),
                                float(eta), float(zeta), ctypes.cast(wp, ctypes.c_void_p))
    if st != OK:
        raise OracleError(st, "bmuf_step")
    return wg


def bmuf_zeta(C: float, N: int, eta: float) -> float:
    """Eq. (5): zeta = C * N * (1 - eta)."""
    return lib().oracle_bmuf_zeta(C, N, eta)
