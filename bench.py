#!/usr/bin/env python
"""Benchmark of the GTC hot path: encode -> exchange -> decode_apply.

One "step" = one pass of the whole hot path over one synthetic gradient per
rank: residual accumulate + threshold + quantize + pack + compact (encode), the
NCCL all-gather of the messages (exchange, world > 1), integer aggregation +
sparse apply to the replicated weights (decode_apply).

Metric (BASELINE.json): params/sec of encode+exchange+apply per step, whole job
(= world * n_params / step time, weak scaling: every rank owns a full gradient).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gtc|reference]
                    [--workload lstm_am|lstm_am_30m|1e9] [--rho 0.01] [--cmp gt|ge]

N > 1 is launched by torchrun (RANK/LOCAL_RANK/WORLD_SIZE from the env).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "params/sec encode+exchange+apply per step"
UNIT = "params/s"
N_GRAD_BUFFERS = 3  # gradients rotate so each step reads a fresh 4n bytes

WORKLOADS = {
    # C2 (BASELINE configs[1]): the paper-shaped LSTM AM
    "lstm_am": dict(n=synth.LSTM_AM_PARAMS, desc="LSTM-AM gradient, 5x768 LSTM + 3183 senones (24,286,575 params)"),
    # north_star's "~30M params" variant
    "lstm_am_30m": dict(n=30_000_000, desc="LSTM-AM-shaped gradient padded to 30,000,000 params"),
    # C5: 1B params per rank
    "1e9": dict(n=1_000_000_000, desc="1e9-param synthetic gradient (HBM-bound regime)"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["gtc", "reference"], default="gtc")
    ap.add_argument("--algo", choices=["gtc", "bmuf"], default="gtc",
                    help="gtc: the GTC step (headline); bmuf: the paper's BMUF-NBM sync step (Eqs. 1-4)")
    ap.add_argument("--bmuf-eta", type=float, default=None, help="block momentum (default 1 - 1/N)")
    ap.add_argument("--bmuf-C", type=float, default=1.0, help="Eq. (5) constant C")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="lstm_am")
    ap.add_argument("--rho", type=float, default=0.01, help="target per-rank update density")
    ap.add_argument("--tau", type=float, default=8.0, help="gradient threshold (PAPER.md:249 uses 8)")
    ap.add_argument("--cmp", choices=["gt", "ge"], default="gt")
    ap.add_argument("--alpha", type=float, default=-1e-3, help="apply scale (e.g. -lr)")
    ap.add_argument("--exchange", choices=["p2p", "nccl"], default="p2p",
                    help="world > 1: NVLink peer reads fused into decode (p2p) or NCCL all-gather")
    ap.add_argument("--accum", choices=["weights", "momentum"], default="weights",
                    help="apply: sparse fmaf into the weights (headline) or the dense SGD-momentum update")
    ap.add_argument("--mu", type=float, default=0.9, help="SGD momentum for --accum momentum")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--split-step", action="store_true",
                    help="world > 1, p2p: gtc_step as encode + decode_apply kernels (GTC_STEP_SPLIT) "
                         "instead of the one fused kernel")
    ap.add_argument("--sharded", action="store_true",
                    help="world > 1, p2p: owner-computes decode (GTC_DECODE_SHARDED, SURVEY 8(f) #4)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


# ------------------------------------------------------------------ helpers
def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms in the background."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.marks = []

    def start(self):
        if os.environ.get("BENCH_NO_SMI"):  # diagnostics: no sampler
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self):
        self.marks.append(time.time())

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        t0, t1 = (self.marks + [0, 0])[:2] if len(self.marks) >= 2 else (0, 1e30)
        inside = [r for t, r in self.rows if t0 <= t <= t1 + 0.2] or [r for _, r in self.rows]
        sm = [float(r[1]) for r in inside if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in inside if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in inside for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside)}


def n_grad_buffers(n):
    """Gradients rotate over 3 buffers (LSTM-AM sizes: g + r > L2 every step);
    one buffer is already 32x the L2 at 1e9 params."""
    return N_GRAD_BUFFERS if n < 100_000_000 else 1


def make_inputs(n, tau, rho, rank, world):
    """Per-rank synthetic inputs (host): LSTM-shaped gradients applied in
    rotation, calibrated so the STATIONARY density is rho
    (synth.sigma_for_cycle_density), a stationary residual
    (synth.steady_residual: the density holds from the first step) and the
    replicated weights w0."""
    nb = n_grad_buffers(n)
    corr = 0.5 if world > 1 else 0.0
    sigma = synth.sigma_for_cycle_density(rho, tau, synth.mean_abs_scale(n), nb, corr)
    grads = [synth.lstm_gradient(n, sigma, synth.BASE_SEED, t, rank, corr) for t in range(nb)]
    r0 = synth.steady_residual(grads, tau, synth.rank_seed(rank))
    w0 = synth.normal(n, synth.BASE_SEED, 0, 11) * np.float32(0.05)  # replicated weights
    return grads, r0, w0


def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        affinity = len(os.sched_getaffinity(0))
    except AttributeError:
        affinity = os.cpu_count()
    return {"cpu_model": model, "nproc": os.cpu_count(), "affinity": affinity}


# ------------------------------------------------------------------ oracle legs
def oracle_step_args(args_accum, mu, n):
    """(accum_mode, extra kwargs) of oracle.step for --accum."""
    import oracle

    if args_accum == "momentum":
        return oracle.ACCUM_MOMENTUM, {"buf": np.zeros(n, np.float32), "mu": mu}
    return oracle.ACCUM_WEIGHTS, {}


def cpu_oracle_run(n_full, tau, rho, cmp, alpha, budget_s, world=1, inputs=None, accum="weights", mu=0.9):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload."""
    import oracle

    cores = 1  # oracle.step is single-threaded
    n = n_full
    grads, r0, w0 = inputs if inputs is not None else make_inputs(n, tau, rho, 0, 1)
    gs = [grads[t % len(grads)] for t in range(len(grads))]
    rs = [r0.copy() for _ in range(world)]
    w = w0.copy()
    mode = oracle.CMP_GT if cmp == "gt" else oracle.CMP_GE
    amode, akw = oracle_step_args(accum, mu, n)
    steps, t_used = 0, 0.0
    while t_used < budget_s or steps < 1:
        g = [gs[steps % len(gs)]] * world
        t0 = time.perf_counter()
        oracle.step(g, rs, w, tau, mode, alpha, amode, **akw)
        t_used += time.perf_counter() - t0
        steps += 1
        if steps >= 200:
            break
    value = world * n * steps / t_used
    return dict({"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                 "sample": f"{steps} full steps of the {n}-param workload x {world} simulated worker(s) "
                           f"(oracle.step: encode+aggregate+apply, single thread), {t_used:.1f} s"}, **cpu_info())


def run_reference(args):
    rank, local_rank, world = dist_env()
    if rank != 0:
        return 0
    import oracle

    wl = WORKLOADS[args.workload]
    n_full = wl["n"]
    # per-step sample sized so warmup+steps finish in about a minute
    per_param = 8e-9
    budget = 60.0
    n = int(min(n_full, max(65_536, budget / max(1, args.steps + args.warmup) / per_param)))
    grads, r0, w0 = make_inputs(n, args.tau, args.rho, 0, 1)
    mode = oracle.CMP_GT if args.cmp == "gt" else oracle.CMP_GE
    rs = [r0.copy() for _ in range(world)]
    w = w0.copy()
    amode, akw = oracle_step_args(args.accum, args.mu, n)
    for t in range(args.warmup):
        oracle.step([grads[t % len(grads)]] * world, rs, w, args.tau, mode, args.alpha, amode, **akw)
    t0 = time.perf_counter()
    for t in range(args.steps):
        oracle.step([grads[t % len(grads)]] * world, rs, w, args.tau, mode, args.alpha, amode, **akw)
    dt = time.perf_counter() - t0
    value = world * n * args.steps / dt
    sample = f"each step: {n} of {n_full} params x {world} simulated worker(s), oracle.step single thread"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": args.workload, "n_params": n_full, "sample_params": n,
                                        "tau": args.tau, "rho_target": args.rho, "cmp": args.cmp,
                                        "apply": "ACCUM_MOMENTUM" if args.accum == "momentum" else "ACCUM_WEIGHTS"},
        "cpu_baseline": dict({"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
                             **cpu_info()),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


class NvlinkCounters:
    """NVLink data counters of one GPU (NVML field values, KiB), sampled
    around the timed region; None where the driver does not expose them."""

    TX, RX = 138, 139  # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX

    def __init__(self, gpu_index):
        self.h = None
        self.err = None
        if os.environ.get("BENCH_NO_NVML"):  # diagnostics: no counters
            self.err = "disabled (BENCH_NO_NVML)"
            return
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        except Exception as e:  # no NVML: report why
            self.err = f"nvml: {e}"

    def read(self):
        if self.h is None:
            return None
        try:
            vals = self.nv.nvmlDeviceGetFieldValues(self.h, [self.TX, self.RX])
            out = []
            for v in vals:
                if v.nvmlReturn != 0:
                    self.err = f"field {v.fieldId}: nvml return {v.nvmlReturn}"
                    return None
                out.append(int(v.value.ullVal))
            return out
        except Exception as e:
            self.err = f"nvml read: {e}"
            return None

    @staticmethod
    def delta(a, b):
        if a is None or b is None:
            return None
        return {"tx_bytes": 1024 * (b[0] - a[0]), "rx_bytes": 1024 * (b[1] - a[1])}


# ------------------------------------------------------------------ GPU leg
def run_gtc(args):
    import torch
    import torch.distributed as dist

    import paper_1904_10584_b200 as gtc

    rank, local_rank, world = dist_env()
    if world != args.gpus and not (world == 1 and args.gpus == 1):
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    wl = WORKLOADS[args.workload]
    n, tau = wl["n"], args.tau
    grads_h, r0_h, w0_h = make_inputs(n, tau, args.rho, rank, world)
    grads = [torch.from_numpy(g).to(dev) for g in grads_h]
    NB = len(grads)
    r = torch.from_numpy(r0_h).to(dev)
    w = torch.from_numpy(w0_h).to(dev)
    # the contiguous message is only built on demand (gtc_message / NCCL mode):
    # at 1e9 params cap it at 5 % of n to save 3 GB per rank
    cap = 0 if n < 100_000_000 or args.exchange == "nccl" else n // 20
    ctx = gtc.GTC(n, tau, rank, world, dev, cmp=args.cmp, exchange=args.exchange, max_words_per_rank=cap,
                  fused_step=not args.split_step, sharded=args.sharded and world > 1)
    stream = torch.cuda.current_stream(dev)
    momentum = args.accum == "momentum"
    amode = gtc.GTC_ACCUM_MOMENTUM if momentum else gtc.GTC_ACCUM_WEIGHTS
    if momentum:
        mbuf = torch.zeros(n, dtype=torch.float32, device=dev)
        ctx.bind_momentum(mbuf, args.mu)

    def allmax(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def step(t):
        ctx.encode(grads[t % NB], r)
        ctx.exchange()
        ctx.decode_apply(w, args.alpha, amode)

    for t in range(3):  # the separate calls once (and the buffers of both step parities)
        step(t)
    torch.cuda.synchronize()
    stepf = ctx.stepper(grads, r, w, args.alpha, amode, stream)
    # one kernel per gtc_step?  (world 1: the fused encode+apply; world > 1,
    # p2p: the fused encode+exchange+decode kernel, step_p2p.cu)
    l0 = ctx.kernel_launches()
    stepf(0)
    torch.cuda.synchronize()
    one_kernel = ctx.kernel_launches() - l0 == 1
    assert ctx.check() == gtc.GTC_OK

    # Timed region: K steps through the one-call C entry point (gtc_step: one
    # fused kernel at world 1 and, p2p, at world > 1).  With more than one
    # kernel per step (NCCL exchange, --split-step, momentum at world > 1)
    # every EV_EVERY-th step runs as the three separate calls with CUDA events
    # between them (per-phase durations).
    K = args.steps
    EV_EVERY = 8
    inst = [] if one_kernel else [t for t in range(K) if t % EV_EVERY == 0]
    ev = {t: [torch.cuda.Event(enable_timing=True) for _ in range(4)] for t in inst}
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.6)
    # the W warm-up steps run right before the timed region
    for t in range(max(3, args.warmup)):
        stepf(t)
    torch.cuda.synchronize()
    launches0 = ctx.kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    e_start.record(stream)
    for t in range(K):
        if t in ev:
            e = ev[t]
            e[0].record(stream)
            ctx.encode(grads[t % NB], r)
            e[1].record(stream)
            ctx.exchange()
            e[2].record(stream)
            ctx.decode_apply(w, args.alpha, amode)
            e[3].record(stream)
        else:
            stepf(t)
    e_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks.mark()
    launches = ctx.kernel_launches() - launches0
    time.sleep(0.3)
    clocks.stop()
    # device-side faults (GTC_EPEER, GTC_ENONFINITE) are sticky: a faulted
    # run is not a measurement
    status = int(allmax([float(ctx.check())])[0])
    if status != gtc.GTC_OK:
        raise SystemExit(f"bench: timed steps faulted on some rank: {gtc.gtc_strerror(status)}")

    ms_local = e_start.elapsed_time(e_end)
    phases = None
    if inst:
        phases = [sum(ev[t][i].elapsed_time(ev[t][i + 1]) for t in inst) / len(inst) for i in range(3)]

    # NVLink data counters (NVML) bracket a SEPARATE, untimed pass of K steps:
    # an NVML NVLink field read stalls a running p2p job for ~10 ms
    # (profiles/r02/nvml_stall: 130.1 us/step over 200 steps with the read
    # inside the timed region, 75.8 without)
    nv_delta, nvl_err = None, "world 1"
    if world > 1:
        nvl = NvlinkCounters(local_rank)
        nvl0 = nvl.read()
        if -allmax([-(1.0 if nvl0 is not None else 0.0)])[0] > 0.5:  # every rank reads them
            for t in range(K):
                stepf(t)
            torch.cuda.synchronize()
        nv_delta = NvlinkCounters.delta(nvl0, nvl.read())
        nvl_err = nvl.err

    # density over the timed steps' regime (untimed: the inputs are
    # stationary, so the next M steps sample the same distribution)
    M = min(K, 64)
    ks = []
    for t in range(K, K + M):
        stepf(t)
        ks.append(ctx.last_counts())  # waits
    k_rank = [kk[rank if world > 1 else 0] for kk in ks]
    k_mean = float(np.mean(k_rank))
    k_all_mean = [float(np.mean([kk[m] for kk in ks])) for m in range(world)]

    # unfused breakdown (untimed by the step metric): the encode kernel alone
    # and the exchange + decode alone (separate calls), CUDA events on the stream
    brk = None
    if one_kernel:
        B = 64
        eb = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(B)]
        if world > 1:
            dist.barrier()
        for t in range(B):
            eb[t][0].record(stream)
            ctx.encode(grads[t % NB], r)
            eb[t][1].record(stream)
            ctx.exchange()
            ctx.decode_apply(w, args.alpha, amode)
            eb[t][2].record(stream)
        torch.cuda.synchronize()
        bt = allmax([sum(e[0].elapsed_time(e[1]) for e in eb) / B, sum(e[1].elapsed_time(e[2]) for e in eb) / B])
        brk = {"encode_only_ms": bt[0], "decode_only_ms": bt[1]}

    # touched set of one step (decode's algorithmic bytes; the sector floor)
    cnt = torch.empty(n, dtype=torch.int8, device=dev)
    ctx.encode(grads[K % NB], r)
    ctx.exchange()
    ctx.decode_apply(w, args.alpha, amode, cnt)
    nz = torch.nonzero(cnt).flatten()
    nnz_c = int(nz.numel())
    sectors_c = int(torch.unique_consecutive(nz // 8).numel())  # distinct 32-byte sectors of the target
    del cnt, nz

    # residual-aliased gradient: the caller's backward
    # accumulates into r, then gtc_step(grad = NULL) encodes at 8 B/param
    # instead of 12.  Stand-in backward: torch's r.add_(g).  The step's time
    # is (add_ + gtc_step(NULL) loop) - (add_ loop), each loop timed whole
    # (per-step events would stall the stream and hide nothing less).
    GN = 64
    sp = stream.cuda_stream
    lib = gtc.load_library()
    rp, wp = r.data_ptr(), w.data_ptr()

    def loop(with_step):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for t in range(GN):
            r.add_(grads[t % NB])
            if with_step:
                lib.gtc_step(ctx.ctx, None, rp, wp, args.alpha, amode, sp)
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / GN

    loop(True)  # warm
    add_ms = allmax([loop(False)])[0]
    both_ms = allmax([loop(True)])[0]
    gn_ms = both_ms - add_ms
    assert ctx.check() == gtc.GTC_OK

    ms, = allmax([ms_local])
    ms_per_step = ms / K
    if phases is not None:
        phases = allmax(phases)

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        pinned = [torch.from_numpy(g).pin_memory() for g in grads_h]
        k_host = torch.zeros(1, dtype=torch.int64).pin_memory()
        gdev = torch.empty(n, dtype=torch.float32, device=dev)
        E = args.e2e_steps
        for t in range(2):
            gdev.copy_(pinned[t % NB], non_blocking=True)
            ctx.step(gdev, r, w, args.alpha, amode)
            k_host.copy_(ctx.local_count_tensor(), non_blocking=True)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for t in range(E):
            gdev.copy_(pinned[t % NB], non_blocking=True)
            ctx.step(gdev, r, w, args.alpha, amode)
            k_host.copy_(ctx.local_count_tensor(), non_blocking=True)
            stream.synchronize()
            _ = int(k_host[0])
        s1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = allmax([s0.elapsed_time(s1) / E])[0]
        e2e = {"value": world * n / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 8,
               "ms_per_step": e2e_ms,
               "note": "pinned host gradient -> device copy + gtc_step + k read back, per step"}
        del gdev
        assert ctx.check() == gtc.GTC_OK

    if rank != 0:
        ctx.close()  # collective at world > 1 (quiesce)
        dist.barrier()
        dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel
    peak, peak_src = measured_peaks()
    T = math.ceil(n / gtc.GTC_TILE)
    k = k_mean
    K_all = sum(k_all_mean)
    nvl_bytes = 0.0
    rmw = 16 * n if momentum else 8 * (k if world == 1 else nnz_c)
    rmw_floor = 16 * n if momentum else 64 * sectors_c  # 32-byte sectors read + written
    if world == 1:
        # the fused step kernel: stream g, r -> r (12 B/param), words (4 k),
        # tags (8 B/tile), target read-modify-write of the k touched elements
        base = 12 * n + 4 * k + 8 * T
        kernel_name = "gtc_encode_tile_kernel (fused apply, world 1)"
    elif one_kernel:
        # the fused p2p step kernel, local HBM: the encode (12 n + 4 k + 8 T),
        # this rank's words and tags read back by the decode (4 k + 8 T), the
        # pushed records landing here ((N-1) records), the target RMW
        base = 12 * n + 8 * k + 16 * T
        nvl_bytes = 4 * (K_all - k) + 16 * (world - 1) * T  # records: 16-byte header + entries
        kernel_name = "gtc_step_ticket_kernel (fused encode + exchange + decode + apply)"
    else:
        base = 12 * n + 4 * k + 8 * T
        rmw = rmw_floor = 0
        kernel_name = "gtc_encode_tile_kernel"
    alg_bytes = base + rmw
    floor_bytes = base + rmw_floor
    kern_ms = ms_per_step if one_kernel else phases[0]
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    # DRAM traffic per launch from the committed warm, back-to-back ncu capture
    traffic, traffic_src, loopback_traffic = None, None, None
    tpath = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            key = f"{args.workload}/n{world}/{args.accum}/{'fused' if one_kernel else 'split'}"
            if key in tj and tj[key].get("rho_target") == args.rho:
                traffic, traffic_src = tj[key]["dram_bytes_per_launch"], tj[key]["source"]
        except Exception:
            traffic = None
    if traffic is None and world > 1 and one_kernel:
        # ncu never wraps a multi-rank run: the committed capture of this
        # kernel is its loopback-group form (both ranks on one GPU), per rank
        try:
            with open(tpath) as f:
                lb = json.load(f).get(f"loopback_{args.workload}/n{world}/{args.accum}/fused")
            if lb and lb.get("rho_target") == args.rho:
                traffic_src = ("not this run: " + lb["source"] + ", per rank of a world-%d loopback group on one "
                               "GPU (dram_traffic_loopback_per_rank)" % world)
                loopback_traffic = lb["dram_bytes_per_launch"]
        except Exception:
            pass
    roofline = {"bound": "hbm", "kernel": kernel_name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "alg_bytes_per_launch": alg_bytes, "ms_per_launch": kern_ms, "peak_source": peak_src,
                "sector_floor_bytes_per_launch": floor_bytes,
                "frac_sector_floor": floor_bytes / (kern_ms * 1e-3) / 1e9 / peak,
                "touched_elements": nnz_c, "touched_sectors": sectors_c,
                "share_of_step": kern_ms / ms_per_step}
    if loopback_traffic is not None:
        roofline["dram_traffic_loopback_per_rank"] = loopback_traffic
    if world > 1:
        roofline["nvlink"] = {
            "bytes_per_step_per_rank": nvl_bytes if one_kernel else 4 * (world - 1) * max(k_all_mean),
            "frac_of_900GBs": (nvl_bytes if one_kernel else 4 * (world - 1) * max(k_all_mean))
            / (ms_per_step * 1e-3) / 900e9,
            "frac_of_770GBs_measured_peer_copy": (nvl_bytes if one_kernel else 4 * (world - 1) * max(k_all_mean))
            / (ms_per_step * 1e-3) / 770e9,
            "counters_timed_region": None if nv_delta is None else
            {kk: v / K for kk, v in nv_delta.items()},  # per step
            "counters_note": "NVML NVLink data counters of rank 0's GPU over a separate untimed pass of K steps, "
                             "per step" if nv_delta is not None else (nvl_err or "unavailable")}
    gn_bytes = base - 4 * n + rmw  # grad = NULL: no 4 n gradient read
    line = {
        "metric": METRIC, "value": world * n / (ms_per_step * 1e-3), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": args.workload, "desc": wl["desc"], "n_params": n, "tau": tau,
                   "rho_target": args.rho, "rho_measured_mean": k / n,
                   "rho_measured_min": min(k_rank) / n, "rho_measured_max": max(k_rank) / n,
                   "rho_note": f"k per step of rank {rank} over {M} steps after the timed region (same stationary "
                               "inputs: steady-state residual, gradients in rotation)",
                   "cmp": args.cmp, "parallelism": f"dp{world}",
                   "apply": f"ACCUM_MOMENTUM (mu={args.mu})" if momentum else "ACCUM_WEIGHTS",
                   "exchange": ctx.exchange_mode() + (" sharded (owner-computes)" if args.sharded and world > 1
                                                      else ""),
                   "step": "one kernel" if one_kernel else "separate kernels",
                   "l2": f"inputs larger than L2: g rotates over {NB} buffer(s), "
                         f"g+r = {8 * n / 2**20:.0f} MiB per step vs 126 MB L2"},
        "roofline": roofline,
        "kernels": {"phases_ms": None if phases is None else
                    {"encode": phases[0], "exchange": phases[1], "decode_apply": phases[2]},
                    "unfused_breakdown": brk, "k_per_rank_mean": k_all_mean, "nnz_counts": nnz_c},
        "grad_null": {"ms_per_step": gn_ms, "alg_bytes_per_launch": gn_bytes,
                      "achieved_GBs": gn_bytes / (gn_ms * 1e-3) / 1e9,
                      "frac": gn_bytes / (gn_ms * 1e-3) / 1e9 / peak,
                      "params_per_s": world * n / (gn_ms * 1e-3),
                      "backward_standin_ms": add_ms,
                      "note": "gtc_step(grad=NULL) after the caller's backward accumulated into r: "
                              "(r.add_(g) + gtc_step(NULL)) loop minus r.add_(g) loop, per step"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_oracle_run(n, tau, args.rho, args.cmp, args.alpha, args.cpu_seconds,
                             inputs=(grads_h, r0_h.copy(), w0_h.copy()), accum=args.accum, mu=args.mu)
    if e2e is not None:
        line["e2e"] = e2e
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    ctx.close()  # collective at world > 1 (quiesce)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_bmuf(args):
    """The paper's other trainer: one BMUF-NBM sync step,
    timed over K steps; it runs once per block of 100 mini-batches
    (PAPER.md:249).  p2p (default): one kernel reads shard r of every rank's
    model over NVLink, applies Eqs. (1)-(4) and stores Wg into every model;
    nccl: reduce-scatter + fused Eqs. (1)-(4) on the shard + all-gather."""
    import torch
    import torch.distributed as dist

    import paper_1904_10584_b200 as gtc

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = WORKLOADS[args.workload]["n"]
    eta = args.bmuf_eta if args.bmuf_eta is not None else 1.0 - 1.0 / max(world, 2)
    zeta = gtc.bmuf_zeta(args.bmuf_C, world, eta)
    w0 = torch.from_numpy(synth.normal(n, synth.BASE_SEED, 0, 11)).to(dev)
    b = gtc.BMUF(n, eta, zeta, rank, world, dev, w_init=w0, exchange=args.exchange)
    w = b.local_buffer()
    w[:n].copy_(w0)
    w[:n].add_(torch.from_numpy(synth.normal(n, synth.rank_seed(rank), 1) * np.float32(1e-3)).to(dev))
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(3, args.warmup)):
        b.sync(w)
    torch.cuda.synchronize()
    K = args.steps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.6)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    e0.record(stream)
    for _ in range(K):
        b.sync(w)
    e1.record(stream)
    torch.cuda.synchronize()
    b.check()
    if world > 1:
        dist.barrier()
    clocks.mark()
    time.sleep(0.3)
    clocks.stop()
    ms = torch.tensor([e0.elapsed_time(e1) / K], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = ms.item()
    if rank == 0:
        peak, peak_src = measured_peaks()
        # own HBM per rank: read + write Wg, Delta and the own model's shard
        # (nccl: the reduced sum in place of the model); NVLink per rank:
        # (N-1) shards in + (N-1) shards out, as reduce-scatter + all-gather
        hbm_bytes = 24 * b.shard
        nvl = 2 * (world - 1) * 4 * b.shard
        design = ("one kernel: rank-ordered double mean of shard r over NVLink peer reads -> Eqs. (1)-(4) -> "
                  "Wg stored into every rank's model (device-side flags, no NCCL)" if b.workspace is not None else
                  "in-place NCCL reduce-scatter -> fused Eqs. (1)-(4) on the rank's shard -> in-place NCCL "
                  "all-gather")
        line = {
            "metric": "params/sec BMUF-NBM sync step (Eqs. 1-4)", "value": world * n / (ms * 1e-3),
            "unit": "params/s", "n_gpus": world, "steps": K, "warmup": max(3, args.warmup), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "algo": "bmuf",
            "config": {"workload": args.workload, "n_params": n, "eta": eta, "zeta": zeta, "C": args.bmuf_C,
                       "shard": b.shard, "exchange": b.exchange, "design": design},
            "bytes_per_step": {"hbm_kernel": hbm_bytes, "nvlink_per_rank": nvl},
            "achieved_GBs_if_hbm_only": (hbm_bytes + (2 * 4 * b.shard * (world - 1) if world > 1 else 0))
            / (ms * 1e-3) / 1e9, "peak": peak, "peak_source": peak_src,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    b.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.algo == "bmuf":
        return run_bmuf(args)
    return run_gtc(args)


if __name__ == "__main__":
    sys.exit(main())
