"""torchrun diagnostic of the fused p2p step (GTC_DECODE_TRACE=1): per-CTA
phase times of one traced step at the LSTM-AM size, on every rank.

The production library carries no trace code; build a traced one and select it:
    python tools/build_variant.py /tmp/trace.so GTC_STEP_TRACE
    GTC_LIB=/tmp/trace.so GTC_DECODE_TRACE=1 torchrun ... tools/step_trace.py
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_10584_b200 as gtc  # noqa: E402
import synth  # noqa: E402


def report(rank, tr):
    t = tr.reshape(-1, 6).astype(np.int64)
    ncta = int(np.max(np.nonzero(t[:, 0])[0])) + 1
    t = t[:ncta]
    dec = (t[:, 5] >> 16) & 1 == 1          # decodes a tile
    donly = (t[:, 5] >> 17) & 1 == 1        # decode-only tail CTA
    ticketed = True
    ph = t[:, :5].astype(np.float64)
    base = ph[:, 0].min()
    st, en = (ph[:, 0] - base) / 1e3, (ph[:, 4] - base) / 1e3
    kind = "ticketed" if ticketed else "grouped"
    print(f"[rank {rank}] {kind} grid {ncta} ({int(dec.sum())} decoding CTAs, {int(donly.sum())} decode-only): "
          f"kernel span {en.max():.1f} us; start-order violations (>1us): "
          f"{int(np.sum(st[1:] + 1.0 < np.maximum.accumulate(st)[:-1]))}", flush=True)
    if "TRACE_US_PER_STEP" in os.environ:
        print(f"  step - span (launch gap): {float(os.environ['TRACE_US_PER_STEP']) - en.max():.1f} us", flush=True)
    life = en - st
    enc = ~donly if ticketed else ~dec
    print(f"  encoding CTAs life p50/p90 {np.median(life[enc]):.2f}/{np.percentile(life[enc], 90):.2f}", flush=True)
    if dec.any():
        w = (ph[dec, 1] - ph[dec, 0]) / 1e3
        c = (ph[dec, 2] - ph[dec, 1]) / 1e3
        a = (ph[dec, 4] - ph[dec, 2]) / 1e3
        print(f"  decoding CTAs life p50/p90 {np.median(life[dec]):.2f}/{np.percentile(life[dec], 90):.2f} | "
              f"ready p50/p90/max {np.median(w):.2f}/{np.percentile(w, 90):.2f}/{w.max():.2f} counts p50/p90 "
              f"{np.median(c):.2f}/{np.percentile(c, 90):.2f} rest p50/p90 {np.median(a):.2f}/"
              f"{np.percentile(a, 90):.2f}", flush=True)
        if ticketed and (ph[dec, 3] > 0).all():
            e3 = (ph[dec, 3] - ph[dec, 2]) / 1e3
            a3 = (ph[dec, 4] - ph[dec, 3]) / 1e3
            print(f"    rest = entries+push p50/p90 {np.median(e3):.2f}/{np.percentile(e3, 90):.2f} + apply stores "
                  f"p50/p90 {np.median(a3):.2f}/{np.percentile(a3, 90):.2f}", flush=True)
    if donly.any():
        print(f"  decode-only CTAs life p50/p90 {np.median(life[donly]):.2f}/{np.percentile(life[donly], 90):.2f}; "
              f"first start {st[donly].min():.1f} us", flush=True)
    q = [int(ncta * i / 10) for i in range(10)] + [ncta - 1]
    print("  start at CTA-index deciles:", [round(float(st[i]), 1) for i in q], flush=True)
    print("  end   at CTA-index deciles:", [round(float(en[i]), 1) for i in q], flush=True)
    print(f"  kernel first start (globaltimer) {int(ph[:, 0].min())}; last encode end {en[enc].max():.1f} us",
          flush=True)
    tail = np.nonzero(dec)[0][-int(os.environ.get("TRACE_TAIL", "12")):]
    for i in tail:
        print(f"    cta {i}: start {st[i]:.1f} ready {(ph[i, 1] - base) / 1e3:.1f} counts {(ph[i, 2] - base) / 1e3:.1f} "
              f"end {en[i]:.1f}", flush=True)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    n, tau = synth.LSTM_AM_PARAMS, 8.0
    import bench  # the bench's stationary inputs (density 1 % from the first step)

    gh, rh, wh = bench.make_inputs(n, tau, float(os.environ.get("TRACE_RHO", "0.01")), rank, world)
    grads = [torch.from_numpy(g).to(dev) for g in gh]
    r = torch.from_numpy(rh).to(dev)
    w = torch.from_numpy(wh).to(dev)
    ctx = gtc.GTC(n, tau, rank, world, dev)
    f = ctx.stepper(grads, r, w, -1e-3)
    for t in range(50):
        f(t)
    torch.cuda.synchronize()
    dist.barrier()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    K = int(os.environ.get("TRACE_STEPS", "200"))
    for t in range(K):
        f(t)
    e1.record(s)
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / K
    print(f"[rank {rank}] {us:.1f} us/step over {K} steps (trace stores on)", flush=True)
    os.environ["TRACE_US_PER_STEP"] = f"{us}"
    dist.barrier()
    tr = gtc.gtc_debug_step_trace()
    for rr in range(world):
        if rr == rank:
            report(rank, tr)
        dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
