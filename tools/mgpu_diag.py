"""torchrun diagnostic: decode time with the peers certainly done (barrier
between encode and decode) vs. the normal pipelined step."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_10584_b200 as gtc  # noqa: E402
import synth  # noqa: E402


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
    ctx = gtc.GTC(n, tau, rank, world, dev, exchange=os.environ.get("GTC_EXCHANGE", "p2p"))
    s = torch.cuda.current_stream()
    for t in range(20):
        ctx.step(grads[t % 3], r, w, -1e-3)
    torch.cuda.synchronize()
    K = 200
    dec, enc = [], []
    for t in range(K):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(s)
        ctx.encode(grads[t % 3], r)
        e[1].record(s)
        ctx.exchange()
        torch.cuda.synchronize()
        dist.barrier()
        e[2].record(s)
        ctx.decode_apply(w, -1e-3)
        e[3].record(s)
        torch.cuda.synchronize()
        enc.append(e[0].elapsed_time(e[1]))
        dec.append(e[2].elapsed_time(e[3]))
    f = ctx.stepper(grads, r, w, -1e-3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    e0.record(s)
    for t in range(1000):
        f(t)
    e1.record(s)
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / 1000
    print(f"rank {rank}: encode {1e3 * sum(enc) / K:.1f} us, decode-after-barrier {1e3 * sum(dec) / K:.1f} us, "
          f"pipelined step {1e3 * step:.1f} us", flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__" and os.environ.get("DIAG_TRACE") != "1":
    main()


def trace_report(tag, tr, ncta):
    import numpy as np

    t = tr[: ncta * 6].reshape(ncta, 6).astype(np.int64)
    t = t[t[:, 0] > 0]
    base = t[:, 0].min()
    rel = (t - base) / 1e3
    ph = np.diff(t, axis=1) / 1e3
    names = ["wait", "tags", "counts", "list", "apply"]
    s = ", ".join(f"{nm} med {np.median(ph[:, i]):.1f} p90 {np.percentile(ph[:, i], 90):.1f}" for i, nm in enumerate(names))
    st = rel[:, 0]
    en = rel[:, 5]
    print(f"[{tag}] CTAs {len(t)}: start p10/p50/p90/max {np.percentile(st, 10):.1f}/{np.percentile(st, 50):.1f}/"
          f"{np.percentile(st, 90):.1f}/{st.max():.1f} us, end p50/max {np.percentile(en, 50):.1f}/{en.max():.1f} us; "
          f"by blockIdx: first-8 start {st[:8].round(1).tolist()}, last-8 start {st[-8:].round(1).tolist()}; {s}",
          flush=True)


def traced():
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
    for t in range(30):
        ctx.step(grads[t % 3], r, w, -1e-3)
    torch.cuda.synchronize()
    ncta = 4096
    tr = gtc.gtc_debug_decode_trace()
    if rank == 0:
        trace_report(f"pipelined N={world}", tr, ncta)
    ctx.encode(grads[0], r)
    ctx.exchange()
    torch.cuda.synchronize()
    dist.barrier()
    ctx.decode_apply(w, -1e-3)
    torch.cuda.synchronize()
    tr = gtc.gtc_debug_decode_trace()
    if rank == 0:
        trace_report(f"after barrier N={world}", tr, ncta)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__" and os.environ.get("DIAG_TRACE") == "1":
    traced()
