"""torchrun diagnostic of the fused p2p step (GTC_DECODE_TRACE=1): per-CTA
phase times of one traced step at the LSTM-AM size, on every rank."""
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
    dec = (t[:, 5] >> 16) & 1 == 1
    ph = t[:, :5].astype(np.float64)
    base = ph[:, 0].min()
    st, en = (ph[:, 0] - base) / 1e3, (ph[:, 4] - base) / 1e3
    print(f"[rank {rank}] grid {ncta} ({int(dec.sum())} decode CTAs): kernel span {en.max():.1f} us; "
          f"blockIdx order violations (>1us): {int(np.sum(st[1:] + 1.0 < np.maximum.accumulate(st)[:-1]))}", flush=True)
    life = en - st
    e = ~dec
    print(f"  encode CTAs life p50/p90 {np.median(life[e]):.2f}/{np.percentile(life[e], 90):.2f}", flush=True)
    w = (ph[dec, 1] - ph[dec, 0]) / 1e3
    c = (ph[dec, 2] - ph[dec, 1]) / 1e3
    a = (ph[dec, 4] - ph[dec, 2]) / 1e3
    print(f"  decode CTAs life p50/p90 {np.median(life[dec]):.2f}/{np.percentile(life[dec], 90):.2f} | tagwait p50/p90/max "
          f"{np.median(w):.2f}/{np.percentile(w, 90):.2f}/{w.max():.2f} counts p50/p90 {np.median(c):.2f}/"
          f"{np.percentile(c, 90):.2f} apply p50/p90 {np.median(a):.2f}/{np.percentile(a, 90):.2f}", flush=True)
    q = [int(ncta * i / 10) for i in range(10)] + [ncta - 1]
    print("  start at blockIdx deciles:", [round(float(st[i]), 1) for i in q], flush=True)
    print("  end   at blockIdx deciles:", [round(float(en[i]), 1) for i in q], flush=True)
    print(f"  kernel first start (globaltimer) {int(ph[:, 0].min())}; last encode end {en[e].max():.1f} us", flush=True)
    tail = np.nonzero(dec)[0][-int(os.environ.get("TRACE_TAIL", "12")):]
    for i in tail:
        print(f"    cta {i}: start {st[i]:.1f} tags {(ph[i, 1] - base) / 1e3:.1f} counts {(ph[i, 2] - base) / 1e3:.1f} "
              f"end {en[i]:.1f}", flush=True)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    n, tau = synth.LSTM_AM_PARAMS, 8.0
    sigma = synth.sigma_for_density(0.01, tau, synth.mean_abs_scale(n))
    grads = [torch.from_numpy(synth.lstm_gradient(n, sigma, synth.BASE_SEED, t, rank, 0.5)).to(dev) for t in range(3)]
    r = torch.from_numpy(synth.uniform(n, -tau, tau, synth.rank_seed(rank))).to(dev)
    w = torch.zeros(n, device=dev)
    ctx = gtc.GTC(n, tau, rank, world, dev)
    f = ctx.stepper(grads, r, w, -1e-3)
    for t in range(50):
        f(t)
    torch.cuda.synchronize()
    tr = gtc.gtc_debug_step_trace()
    for rr in range(world):
        if rr == rank:
            report(rank, tr)
        dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
