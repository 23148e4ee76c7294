"""paper_1904_10584_b200 -- B200-native Gradient Threshold Compression (GTC).

The hot path of the distributed trainer of arXiv 1904.10584, PAPER.md:222
(Sec. VI-A): threshold-quantised gradient compression with residual
accumulation, the all-to-all exchange of the sparse updates, their
aggregation and the weight update.  All of it runs in libgtc.so
(hand-written sm_100a CUDA + NCCL, C ABI in include/gtc.h).  This module is a
thin ctypes binding with the same names as the C ABI (argument marshalling
only) plus ``GTC``, a convenience wrapper that lets PyTorch own the device
memory (workspace, tensors) and streams.

There is no CPU fallback: if libgtc.so is missing or no CUDA device is
present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GTC_LIB") or os.path.join(_PKG, "libgtc.so")  # GTC_LIB: experiment builds

GTC_OK = 0
GTC_EINVAL = 1
GTC_EDIM = 2
GTC_EALIGN = 3
GTC_ECUDA = 4
GTC_ENCCL = 5
GTC_ENONFINITE = 6
GTC_ECORRUPT = 7
GTC_ESTATE = 8
GTC_ECAPACITY = 9
GTC_EUNSUPPORTED = 10
GTC_EPEER = 11

GTC_CMP_GT = 0
GTC_CMP_GE = 1
GTC_EXCHANGE_P2P = 0
GTC_EXCHANGE_NCCL = 16
GTC_STEP_FUSED = 0
GTC_STEP_SPLIT = 32
GTC_LOOPBACK = 64
GTC_DECODE_SHARDED = 128
GTC_ACCUM_WEIGHTS = 0
GTC_ACCUM_UPDATE = 1
GTC_ACCUM_MOMENTUM = 2
GTC_MAX_MSGS = 64
GTC_TILE = 4096

# every entry point of include/gtc.h: name -> (restype, argtypes)
_vp, _i64, _i32, _u32, _f32, _sz = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                    ctypes.c_uint32, ctypes.c_float, ctypes.c_size_t)
_SIGS = {
    "gtc_get_unique_id": (_i32, [_vp]),
    "gtc_init": (_i32, [ctypes.POINTER(_vp), _i64, _f32, _i32, _i32, _vp, _i32, _u32]),
    "gtc_workspace_size": (_i32, [_vp, _i64, _i32, ctypes.POINTER(_sz)]),
    "gtc_bind_workspace": (_i32, [_vp, _vp, _sz, _i64, _i32]),
    "gtc_encode": (_i32, [_vp, _vp, _vp, _vp]),
    "gtc_exchange": (_i32, [_vp, _vp]),
    "gtc_decode_apply": (_i32, [_vp, _vp, _f32, _i32, _vp, _vp]),
    "gtc_step": (_i32, [_vp, _vp, _vp, _vp, _f32, _i32, _vp]),
    "gtc_bind_momentum": (_i32, [_vp, _vp, _f32]),
    "gtc_decode_apply_msgs": (_i32, [_vp, _vp, _vp, _i32, _vp, _f32, _i32, _vp, _vp]),
    "gtc_last_counts": (_i32, [_vp, _vp]),
    "gtc_local_count": (_i32, [_vp, ctypes.POINTER(_vp)]),
    "gtc_message": (_i32, [_vp, _i32, ctypes.POINTER(_vp), ctypes.POINTER(_i64)]),
    "gtc_read_message": (_i32, [_vp, _i32, _vp, _i64, ctypes.POINTER(_i64)]),
    "gtc_check": (_i32, [_vp, _vp]),
    "gtc_wire_pack": (_i32, [_vp, _i64, ctypes.c_uint64, _f32, _vp, _sz, ctypes.POINTER(_sz)]),
    "gtc_wire_unpack": (_i32, [_vp, _sz, _vp, _i64, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_uint64),
                               ctypes.POINTER(_f32)]),
    "gtc_connect_loopback": (_i32, [_vp, _i32]),
    "gtc_step_group": (_i32, [_vp, _i32, _vp, _vp, _vp, _f32, _i32, _u32, _vp]),
    "gtc_quiesce": (_i32, [_vp]),
    "gtc_exchange_mode": (_i32, [_vp]),
    "gtc_kernel_launches": (_i64, [_vp]),
    "gtc_debug_decode_trace": (_i32, [_vp, _i32]),
    "gtc_debug_step_trace": (_i32, [_vp, _i32]),
    "gtc_strerror": (ctypes.c_char_p, [_i32]),
    "gtc_last_error_detail": (ctypes.c_char_p, [_vp]),
    "gtc_destroy": (None, [_vp]),
    # include/bmuf.h
    "bmuf_init": (_i32, [ctypes.POINTER(_vp), _i64, _i32, _i32, _vp, _i32]),
    "bmuf_shard_len": (_i64, [_vp]),
    "bmuf_padded_len": (_i64, [_vp]),
    "bmuf_sync": (_i32, [_vp, _vp, _vp, _vp, _f32, _f32, _vp]),
    "bmuf_workspace_size": (_i32, [_vp, ctypes.POINTER(ctypes.c_size_t)]),
    "bmuf_bind_workspace": (_i32, [_vp, _vp, ctypes.c_size_t]),
    "bmuf_model": (_vp, [_vp]),
    "bmuf_check": (_i32, [_vp]),
    "bmuf_sync_sim": (_i32, [_vp, _vp, _i32, _vp, _vp, _f32, _f32, _vp]),
    "bmuf_zeta": (ctypes.c_double, [ctypes.c_double, _i32, ctypes.c_double]),
    "bmuf_quiesce": (_i32, [_vp]),
    "bmuf_destroy": (None, [_vp]),
}

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libgtc.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class GTCError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        msg = load_library().gtc_strerror(status).decode()
        super().__init__(f"{where}: {msg}" + (f" ({detail})" if detail else ""))
        self.status = status


def _chk(status: int, where: str, ctx=None, ok=(GTC_OK,)):
    if status not in ok:
        detail = load_library().gtc_last_error_detail(ctx).decode() if ctx else ""
        raise GTCError(status, where, detail)
    return status


# ----------------------------------------------------------------- C-ABI names
def gtc_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _chk(load_library().gtc_get_unique_id(buf), "gtc_get_unique_id")
    return buf.raw


def gtc_init(n_params: int, tau: float, rank: int = 0, world: int = 1, unique_id: bytes | None = None,
             cuda_device: int = 0, flags: int = GTC_CMP_GT):
    ctx = _vp()
    uid = ctypes.create_string_buffer(unique_id, 128) if unique_id is not None else None
    _chk(load_library().gtc_init(ctypes.byref(ctx), n_params, tau, rank, world, uid, cuda_device, flags),
         "gtc_init")
    return ctx


def gtc_workspace_size(ctx, max_words_per_rank: int = 0, max_sim_msgs: int = 0) -> int:
    out = _sz()
    _chk(load_library().gtc_workspace_size(ctx, max_words_per_rank, max_sim_msgs, ctypes.byref(out)),
         "gtc_workspace_size", ctx)
    return out.value


def gtc_bind_workspace(ctx, dev_ptr: int, nbytes: int, max_words_per_rank: int = 0, max_sim_msgs: int = 0):
    _chk(load_library().gtc_bind_workspace(ctx, dev_ptr, nbytes, max_words_per_rank, max_sim_msgs),
         "gtc_bind_workspace", ctx)


def gtc_encode(ctx, grad_ptr: int | None, residual_ptr: int, stream: int):
    _chk(load_library().gtc_encode(ctx, grad_ptr, residual_ptr, stream), "gtc_encode", ctx)


def gtc_exchange(ctx, stream: int) -> int:
    """Returns GTC_OK or GTC_ENONFINITE (exchange completed); raises otherwise."""
    return _chk(load_library().gtc_exchange(ctx, stream), "gtc_exchange", ctx, ok=(GTC_OK, GTC_ENONFINITE))


def gtc_decode_apply(ctx, target_ptr: int, alpha: float, mode: int, counts_out_ptr: int | None, stream: int):
    _chk(load_library().gtc_decode_apply(ctx, target_ptr, alpha, mode, counts_out_ptr, stream),
         "gtc_decode_apply", ctx)


def gtc_step(ctx, grad_ptr: int | None, residual_ptr: int, target_ptr: int, alpha: float, mode: int,
             stream: int) -> int:
    """encode + exchange + decode_apply; returns GTC_OK or GTC_ENONFINITE."""
    return _chk(load_library().gtc_step(ctx, grad_ptr, residual_ptr, target_ptr, alpha, mode, stream),
                "gtc_step", ctx, ok=(GTC_OK, GTC_ENONFINITE))


def gtc_bind_momentum(ctx, buf_ptr: int | None, mu: float):
    _chk(load_library().gtc_bind_momentum(ctx, buf_ptr, mu), "gtc_bind_momentum", ctx)


def gtc_decode_apply_msgs(ctx, msg_ptrs, counts, target_ptr: int, alpha: float, mode: int,
                          counts_out_ptr: int | None, stream: int):
    nm = len(msg_ptrs)
    P = (_vp * max(nm, 1))(*msg_ptrs)
    K = (_i64 * max(nm, 1))(*counts)
    _chk(load_library().gtc_decode_apply_msgs(ctx, P, K, nm, target_ptr, alpha, mode, counts_out_ptr, stream),
         "gtc_decode_apply_msgs", ctx)


def gtc_last_counts(ctx, world: int):
    buf = (_i64 * world)()
    _chk(load_library().gtc_last_counts(ctx, buf), "gtc_last_counts", ctx)
    return list(buf)


def gtc_local_count(ctx) -> int:
    p = _vp()
    _chk(load_library().gtc_local_count(ctx, ctypes.byref(p)), "gtc_local_count", ctx)
    return p.value


def gtc_message(ctx, rank: int):
    p, k = _vp(), _i64()
    _chk(load_library().gtc_message(ctx, rank, ctypes.byref(p), ctypes.byref(k)), "gtc_message", ctx)
    return p.value, k.value


def gtc_read_message(ctx, rank: int, max_words: int):
    """Host copy (numpy uint32) of a rank's message of the last step."""
    import numpy as np

    buf = np.empty(max(max_words, 1), dtype=np.uint32)
    k = _i64()
    _chk(load_library().gtc_read_message(ctx, rank, buf.ctypes.data_as(_vp), max_words, ctypes.byref(k)),
         "gtc_read_message", ctx)
    return buf[: k.value].copy()


def gtc_wire_pack(words, dim: int, tau: float) -> bytes:
    """SPEC.md:202 wire format ("GTCU", dim, tau, count, SPEC-layout words) of
    canonical words (index << 1 | neg, numpy uint32, ascending)."""
    import numpy as np

    w = np.ascontiguousarray(words, dtype=np.uint32)
    need = _sz()
    lib = load_library()
    lib.gtc_wire_pack(w.ctypes.data_as(_vp), w.size, dim, tau, None, 0, ctypes.byref(need))
    out = ctypes.create_string_buffer(max(need.value, 1))
    _chk(lib.gtc_wire_pack(w.ctypes.data_as(_vp), w.size, dim, tau, out, need.value, ctypes.byref(need)),
         "gtc_wire_pack")
    return out.raw[: need.value]


def gtc_wire_unpack(blob: bytes):
    """(canonical words numpy uint32, dim, tau) of a SPEC.md:202 serialized update."""
    import numpy as np

    n_max = max(0, (len(blob) - 20) // 4)
    words = np.empty(max(n_max, 1), dtype=np.uint32)
    k, dim, tau = _i64(), ctypes.c_uint64(), _f32()
    _chk(load_library().gtc_wire_unpack(blob, len(blob), words.ctypes.data_as(_vp), n_max, ctypes.byref(k),
                                        ctypes.byref(dim), ctypes.byref(tau)), "gtc_wire_unpack")
    return words[: k.value].copy(), dim.value, tau.value


def gtc_exchange_mode(ctx) -> int:
    return load_library().gtc_exchange_mode(ctx)


def gtc_check(ctx, stream: int) -> int:
    return load_library().gtc_check(ctx, stream)


def gtc_connect_loopback(ctxs):
    arr = (_vp * len(ctxs))(*[c.value if isinstance(c, _vp) else c for c in ctxs])
    _chk(load_library().gtc_connect_loopback(arr, len(ctxs)), "gtc_connect_loopback", ctxs[0])


def gtc_step_group(ctxs, grad_ptrs, residual_ptrs, target_ptrs, alpha: float, mode: int, debug_flags: int,
                   stream: int) -> int:
    w = len(ctxs)
    C = (_vp * w)(*[c.value if isinstance(c, _vp) else c for c in ctxs])
    G = (_vp * w)(*grad_ptrs) if grad_ptrs is not None else None
    R = (_vp * w)(*residual_ptrs)
    T = (_vp * w)(*target_ptrs)
    return _chk(load_library().gtc_step_group(C, w, G, R, T, alpha, mode, debug_flags, stream), "gtc_step_group",
                ctxs[0], ok=(GTC_OK, GTC_ENONFINITE))


def gtc_quiesce(ctx):
    _chk(load_library().gtc_quiesce(ctx), "gtc_quiesce", ctx)


def gtc_kernel_launches(ctx) -> int:
    return load_library().gtc_kernel_launches(ctx)


def gtc_debug_decode_trace(max_entries: int = 4096 * 6):
    """Debug: phase stamps (ns) of the last counting decode (GTC_DECODE_TRACE=1)."""
    import numpy as np

    buf = np.zeros(max_entries, dtype=np.uint64)
    _chk(load_library().gtc_debug_decode_trace(buf.ctypes.data_as(_vp), max_entries), "gtc_debug_decode_trace")
    return buf


def gtc_debug_step_trace(max_entries: int = 16384 * 6):
    """Debug: phase stamps (ns) + SM id per CTA of the last fused p2p step (GTC_DECODE_TRACE=1)."""
    import numpy as np

    buf = np.zeros(max_entries, dtype=np.uint64)
    _chk(load_library().gtc_debug_step_trace(buf.ctypes.data_as(_vp), max_entries), "gtc_debug_step_trace")
    return buf


def gtc_strerror(status: int) -> str:
    return load_library().gtc_strerror(status).decode()


def gtc_last_error_detail(ctx) -> str:
    return load_library().gtc_last_error_detail(ctx).decode()


def gtc_destroy(ctx):
    load_library().gtc_destroy(ctx)


# ----------------------------------------------------------------- torch glue
def broadcast_unique_id(rank: int, group=None) -> bytes:
    """Rank 0 creates the 128-byte NCCL id; every rank of ``group`` (an
    initialised torch.distributed group, any backend) receives the same bytes."""
    import torch.distributed as dist

    obj = [gtc_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    if not (isinstance(obj[0], bytes) and len(obj[0]) == 128):
        raise RuntimeError("NCCL unique id broadcast failed")
    return obj[0]


def _stream(stream, device):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def _ptr(t, name):
    import torch

    if t is None:
        return None
    if not (t.is_cuda and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous CUDA tensor")
    if t.dtype != torch.float32:
        raise TypeError(f"{name} must be float32")
    return t.data_ptr()


class GTC:
    """One rank's GTC context with torch-owned workspace.

    ``world > 1`` needs an initialised torch.distributed group (any backend)
    to broadcast the 128-byte NCCL id from rank 0; the exchange itself runs on
    libgtc's own NCCL communicator.  ``loopback=True``: one rank of an
    in-process group (no NCCL, no torch.distributed; see ``LoopbackGroup``).
    """

    def __init__(self, n_params: int, tau: float, rank: int = 0, world: int = 1, device=None,
                 cmp: str = "gt", max_words_per_rank: int = 0, max_sim_msgs: int = 0, group=None,
                 exchange: str = "p2p", fused_step: bool = True, loopback: bool = False, sharded: bool = False):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("GTC needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.n, self.tau, self.rank, self.world = int(n_params), float(tau), int(rank), int(world)
        self.cmp = {"gt": GTC_CMP_GT, "ge": GTC_CMP_GE}[cmp]
        flags = self.cmp | {"p2p": GTC_EXCHANGE_P2P, "nccl": GTC_EXCHANGE_NCCL}[exchange]
        flags |= GTC_STEP_FUSED if fused_step else GTC_STEP_SPLIT
        self.loopback = bool(loopback)
        if self.loopback:
            flags |= GTC_LOOPBACK
        if sharded:
            flags |= GTC_DECODE_SHARDED
        self.max_words = max_words_per_rank if max_words_per_rank > 0 else self.n
        uid = None
        if world > 1 and not self.loopback:
            uid = broadcast_unique_id(rank, group)
        with torch.cuda.device(self.device):
            self.ctx = gtc_init(self.n, self.tau, rank, world, uid, self.device.index, flags)
            nbytes = gtc_workspace_size(self.ctx, max_words_per_rank, max_sim_msgs)
            self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            gtc_bind_workspace(self.ctx, self.workspace.data_ptr(), nbytes, max_words_per_rank, max_sim_msgs)

    # --- optimizer state (GTC_ACCUM_MOMENTUM)
    def bind_momentum(self, buf, mu: float):
        """SGD-momentum state for mode GTC_ACCUM_MOMENTUM (float32[n] device
        tensor, zero at the start; ``None`` unbinds).  The tensor must outlive
        its use."""
        if buf is not None and buf.numel() != self.n:
            raise ValueError("momentum buffer length != n_params")
        self._mom = buf
        gtc_bind_momentum(self.ctx, _ptr(buf, "buf") if buf is not None else None, float(mu))

    # --- the three calls of a step
    def encode(self, grad, residual, stream=None):
        if residual.numel() != self.n or (grad is not None and grad.numel() != self.n):
            raise ValueError("grad/residual length != n_params")
        gtc_encode(self.ctx, _ptr(grad, "grad"), _ptr(residual, "residual"), _stream(stream, self.device))

    def exchange(self, stream=None) -> int:
        return gtc_exchange(self.ctx, _stream(stream, self.device))

    def decode_apply(self, target, alpha: float = 1.0, mode: int = GTC_ACCUM_WEIGHTS, counts_out=None,
                     stream=None):
        import torch

        if target.numel() != self.n:
            raise ValueError("target length != n_params")
        cptr = None
        if counts_out is not None:
            if counts_out.dtype != torch.int8 or counts_out.numel() != self.n or not counts_out.is_cuda:
                raise ValueError("counts_out must be int8[n] on the device")
            cptr = counts_out.data_ptr()
        gtc_decode_apply(self.ctx, _ptr(target, "target"), alpha, mode, cptr, _stream(stream, self.device))

    def step(self, grad, residual, target, alpha: float = 1.0, mode: int = GTC_ACCUM_WEIGHTS, stream=None) -> int:
        """encode -> exchange -> decode_apply in one C call."""
        for t, name in ((residual, "residual"), (target, "target")):
            if t.numel() != self.n:
                raise ValueError(f"{name} length != n_params")
        if grad is not None and grad.numel() != self.n:
            raise ValueError("grad length != n_params")
        return gtc_step(self.ctx, _ptr(grad, "grad"), _ptr(residual, "residual"), _ptr(target, "target"),
                        alpha, mode, _stream(stream, self.device))

    def stepper(self, grads, residual, target, alpha: float = 1.0, mode: int = GTC_ACCUM_WEIGHTS, stream=None):
        """A validated-once step closure for hot loops: ``f(i)`` runs one step
        on ``grads[i % len(grads)]`` with a single ctypes call."""
        for t in list(grads) + [residual, target]:
            _ptr(t, "tensor")
            if t.numel() != self.n:
                raise ValueError("tensor length != n_params")
        fn = load_library().gtc_step
        ctx, gp = self.ctx, [g.data_ptr() for g in grads]
        rp, tp, sp = residual.data_ptr(), target.data_ptr(), _stream(stream, self.device)
        ng, a, m = len(gp), float(alpha), int(mode)

        def f(i):
            st = fn(ctx, gp[i % ng], rp, tp, a, m, sp)
            if st != GTC_OK and st != GTC_ENONFINITE:
                _chk(st, "gtc_step", ctx)
            return st
        return f

    # --- simulated workers / tests
    def decode_apply_msgs(self, msgs, target, alpha: float = 1.0, mode: int = GTC_ACCUM_WEIGHTS,
                          counts_out=None, stream=None):
        """msgs: list of (device int32/uint32 tensor or raw ptr, k)."""
        ptrs, ks = [], []
        for m in msgs:
            if isinstance(m, tuple):
                ptrs.append(m[0] if isinstance(m[0], int) else m[0].data_ptr())
                ks.append(int(m[1]))
            else:
                ptrs.append(m.data_ptr())
                ks.append(m.numel())
        cptr = counts_out.data_ptr() if counts_out is not None else None
        gtc_decode_apply_msgs(self.ctx, ptrs, ks, _ptr(target, "target"), alpha, mode, cptr,
                              _stream(stream, self.device))

    def message(self, rank: int | None = None):
        """(device pointer, k) of a rank's message (local one when world == 1)."""
        return gtc_message(self.ctx, self.rank if rank is None else rank)

    def read_message(self, rank: int | None = None):
        """Host (numpy uint32) copy of a rank's message of the last step (any world)."""
        return gtc_read_message(self.ctx, self.rank if rank is None else rank, self.max_words)

    def serialize_message(self, rank: int | None = None) -> bytes:
        """A rank's message of the last step in SPEC.md:202's wire format."""
        return gtc_wire_pack(self.read_message(rank), self.n, self.tau)

    def exchange_mode(self) -> str:
        m = gtc_exchange_mode(self.ctx)
        return {0: "local", GTC_EXCHANGE_P2P: "p2p", GTC_EXCHANGE_NCCL: "nccl"}.get(m, "?") if self.world > 1 \
            else "local"

    def message_tensor(self, rank: int | None = None):
        """The message as an int32 view into this rank's workspace (bit pattern =
        uint32 words).  Only for messages that live in this workspace (world 1,
        or NCCL mode); use read_message() for peers' messages in p2p mode."""
        import torch

        ptr, k = self.message(rank)
        if not (self.workspace.data_ptr() <= ptr < self.workspace.data_ptr() + self.workspace.numel()):
            raise ValueError("message is not in this rank's workspace; use read_message()")
        off = ptr - self.workspace.data_ptr()
        return self.workspace[off: off + 4 * k].view(torch.int32)

    def local_count_tensor(self):
        import torch

        off = gtc_local_count(self.ctx) - self.workspace.data_ptr()
        return self.workspace[off: off + 8].view(torch.int64)

    def last_counts(self):
        return gtc_last_counts(self.ctx, self.world)

    def check(self, stream=None) -> int:
        return gtc_check(self.ctx, _stream(stream, self.device))

    def kernel_launches(self) -> int:
        return gtc_kernel_launches(self.ctx)

    def close(self):
        """Collective at world > 1 (every rank calls it): quiesce (device sync +
        NCCL barrier, so no peer still reads this workspace), then destroy."""
        if getattr(self, "ctx", None) is not None:
            try:
                if self.world > 1 and not self.loopback:
                    gtc_quiesce(self.ctx)
            finally:
                gtc_destroy(self.ctx)
                self.ctx = None

    def __del__(self):
        # never a collective here: ranks collect garbage at different times
        if getattr(self, "ctx", None) is not None:
            try:
                gtc_destroy(self.ctx)
            except Exception:
                pass
            self.ctx = None


class LoopbackGroup:
    """``world`` ranks of one data-parallel group inside ONE process
    (GTC_LOOPBACK contexts linked by gtc_connect_loopback): the real p2p
    kernels with every rank's workspace a plain device pointer.  For tests and
    single-process drivers; all ranks on ``device``.

    ``step`` runs the fused one-kernel step of every rank as ONE launch
    (gtc_step_group); ``split_step`` runs every rank's encode, then every
    rank's exchange, then every rank's decode_apply (the separate calls)."""

    def __init__(self, n_params: int, tau: float, world: int, device=None, cmp: str = "gt",
                 max_words_per_rank: int = 0, sharded: bool = False):
        import torch

        self.world = int(world)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.ranks = [GTC(n_params, tau, r, world, self.device, cmp=cmp, max_words_per_rank=max_words_per_rank,
                          loopback=True, sharded=sharded) for r in range(world)]
        gtc_connect_loopback([g.ctx for g in self.ranks])

    def step(self, grads, residuals, targets, alpha: float = 1.0, mode: int = GTC_ACCUM_WEIGHTS,
             debug_flags: int = 0, stream=None) -> int:
        gp = None if grads is None else [_ptr(g, "grad") for g in grads]
        return gtc_step_group([g.ctx for g in self.ranks], gp, [_ptr(r, "residual") for r in residuals],
                              [_ptr(t, "target") for t in targets], alpha, mode, debug_flags,
                              _stream(stream, self.device))

    def split_step(self, grads, residuals, targets, alpha: float = 1.0, mode: int = GTC_ACCUM_WEIGHTS,
                   counts_out=None, stream=None):
        """counts_out: None or a list of int8[n] device tensors, one per rank."""
        sts = []
        for r, g in enumerate(self.ranks):
            g.encode(None if grads is None else grads[r], residuals[r], stream)
        for g in self.ranks:
            sts.append(g.exchange(stream))
        for r, g in enumerate(self.ranks):
            g.decode_apply(targets[r], alpha, mode, None if counts_out is None else counts_out[r], stream)
        return sts

    def bind_momentum(self, bufs, mu: float):
        for g, b in zip(self.ranks, bufs):
            g.bind_momentum(b, mu)

    def check(self, stream=None):
        return [g.check(stream) for g in self.ranks]

    def close(self):
        for g in self.ranks:
            g.close()


# ----------------------------------------------------------------- BMUF (include/bmuf.h)
def bmuf_init(n: int, rank: int = 0, world: int = 1, unique_id: bytes | None = None, cuda_device: int = 0):
    ctx = _vp()
    uid = ctypes.create_string_buffer(unique_id, 128) if unique_id is not None else None
    _chk(load_library().bmuf_init(ctypes.byref(ctx), n, rank, world, uid, cuda_device), "bmuf_init")
    return ctx


def bmuf_shard_len(ctx) -> int:
    return load_library().bmuf_shard_len(ctx)


def bmuf_padded_len(ctx) -> int:
    return load_library().bmuf_padded_len(ctx)


def bmuf_sync(ctx, w_local_ptr: int, wg_shard_ptr: int, delta_shard_ptr: int, eta: float, zeta: float,
              stream: int):
    _chk(load_library().bmuf_sync(ctx, w_local_ptr, wg_shard_ptr, delta_shard_ptr, eta, zeta, stream), "bmuf_sync")


def bmuf_workspace_size(ctx) -> int:
    b = ctypes.c_size_t(0)
    _chk(load_library().bmuf_workspace_size(ctx, ctypes.byref(b)), "bmuf_workspace_size")
    return b.value


def bmuf_bind_workspace(ctx, ptr: int, nbytes: int):
    _chk(load_library().bmuf_bind_workspace(ctx, ptr, nbytes), "bmuf_bind_workspace")


def bmuf_model(ctx) -> int:
    return load_library().bmuf_model(ctx) or 0


def bmuf_check(ctx):
    _chk(load_library().bmuf_check(ctx), "bmuf_check")


def bmuf_sync_sim(ctx, w_ptrs, wg_ptr: int, delta_ptr: int, eta: float, zeta: float, stream: int):
    P = (_vp * max(len(w_ptrs), 1))(*w_ptrs)
    _chk(load_library().bmuf_sync_sim(ctx, P, len(w_ptrs), wg_ptr, delta_ptr, eta, zeta, stream), "bmuf_sync_sim")


def bmuf_zeta(C: float, N: int, eta: float) -> float:
    """Eq. (5): zeta = C * N * (1 - eta)."""
    return load_library().bmuf_zeta(C, N, eta)


def bmuf_quiesce(ctx):
    _chk(load_library().bmuf_quiesce(ctx), "bmuf_quiesce")


def bmuf_destroy(ctx):
    load_library().bmuf_destroy(ctx)


class BMUF:
    """One rank's BMUF-NBM synchroniser.  Holds this rank's
    shard of the global model Wg and of the block momentum Delta (torch-owned);
    ``sync(w_local)`` runs Eqs. (1)-(4) and leaves Wg(t) in ``w_local``.

    exchange="p2p" (default): the local model lives in an IPC-mapped workspace
    (``local_buffer()`` returns it) and a step is one kernel over NVLink,
    bit-exact with the oracle; "nccl": reduce-scatter + kernel + all-gather on
    any caller buffer of ``padded`` elements."""

    def __init__(self, n_params: int, eta: float, zeta: float, rank: int = 0, world: int = 1, device=None,
                 group=None, w_init=None, exchange: str = "p2p"):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("BMUF needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.n, self.rank, self.world = int(n_params), int(rank), int(world)
        self.eta, self.zeta = float(eta), float(zeta)
        uid = broadcast_unique_id(rank, group) if world > 1 else None
        with torch.cuda.device(self.device):
            self.ctx = bmuf_init(self.n, rank, world, uid, self.device.index)
        self.shard = bmuf_shard_len(self.ctx)
        self.padded = bmuf_padded_len(self.ctx)
        self.wg = torch.zeros(self.shard, dtype=torch.float32, device=self.device)
        self.delta = torch.zeros(self.shard, dtype=torch.float32, device=self.device)
        if exchange not in ("p2p", "nccl"):
            raise ValueError("exchange must be 'p2p' or 'nccl'")
        self.exchange = exchange
        self.workspace = None
        if exchange == "p2p":
            nbytes = bmuf_workspace_size(self.ctx)
            self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            with torch.cuda.device(self.device):
                bmuf_bind_workspace(self.ctx, self.workspace.data_ptr(), nbytes)
            off = bmuf_model(self.ctx) - self.workspace.data_ptr()
            self._model = self.workspace[off:off + 4 * self.padded].view(torch.float32)
            self._model.zero_()
        if w_init is not None:  # Wg(0): this rank's shard of the initial model
            lo = self.rank * self.shard
            hi = min(self.n, lo + self.shard)
            if hi > lo:
                self.wg[: hi - lo].copy_(w_init.reshape(-1)[lo:hi])

    def local_buffer(self):
        """The float[padded_len] local model buffer (p2p: the one in the
        workspace, zeroed at construction; nccl: a new zeroed tensor)."""
        import torch

        if self.workspace is not None:
            return self._model
        return torch.zeros(self.padded, dtype=torch.float32, device=self.device)

    def check(self):
        bmuf_check(self.ctx)

    def sync(self, w_local, stream=None):
        if w_local.numel() != self.padded:
            raise ValueError("w_local must have bmuf_padded_len elements")
        if self.workspace is not None and w_local.data_ptr() != self._model.data_ptr():
            raise ValueError("p2p BMUF: w_local must be local_buffer()")
        bmuf_sync(self.ctx, _ptr(w_local, "w_local"), _ptr(self.wg, "wg"), _ptr(self.delta, "delta"),
                  self.eta, self.zeta, _stream(stream, self.device))

    def close(self):
        """Collective at world > 1 (every rank calls it): quiesce, then destroy."""
        if getattr(self, "ctx", None) is not None:
            try:
                if self.world > 1:
                    bmuf_quiesce(self.ctx)
            finally:
                bmuf_destroy(self.ctx)
                self.ctx = None

    def __del__(self):
        # never a collective here: ranks collect garbage at different times
        if getattr(self, "ctx", None) is not None:
            try:
                bmuf_destroy(self.ctx)
            except Exception:
                pass
            self.ctx = None
