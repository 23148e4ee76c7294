"""Diagnose the grad = NULL step time (world 1): the gtc_step(NULL) kernel
alone, with the stand-in backward (r += g) between steps, bracketed per step
and over the whole loop."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1904_10584_b200 as gtc  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    n, tau = bench.WORKLOADS["lstm_am"]["n"], 8.0
    gh, rh, wh = bench.make_inputs(n, tau, 0.01, 0, 1)
    grads = [torch.from_numpy(g).to(dev) for g in gh]
    r, w = torch.from_numpy(rh).to(dev), torch.from_numpy(wh).to(dev)
    ctx = gtc.GTC(n, tau)
    s = torch.cuda.current_stream()
    sp = s.cuda_stream
    lib = gtc.load_library()

    def null_step():
        lib.gtc_step(ctx.ctx, None, r.data_ptr(), w.data_ptr(), -1e-3, 0, sp)

    def timed(fn, K=200):
        for t in range(10):
            fn(t)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for t in range(K):
            fn(t)
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K * 1e3

    add_only = timed(lambda t: r.add_(grads[t % 3]))
    add_step = timed(lambda t: (r.add_(grads[t % 3]), null_step()))
    grad_step = timed(lambda t: lib.gtc_step(ctx.ctx, grads[t % 3].data_ptr(), r.data_ptr(), w.data_ptr(), -1e-3,
                                             0, sp))
    null_only = timed(lambda t: null_step())
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(64)]
    for t in range(64):
        r.add_(grads[t % 3])
        evs[t][0].record(s)
        null_step()
        evs[t][1].record(s)
    torch.cuda.synchronize()
    per = sum(a.elapsed_time(b) for a, b in evs) / 64 * 1e3
    print(f"us/step: add_ only {add_only:.1f} | add_ + step(NULL) {add_step:.1f} | step(grad) {grad_step:.1f} | "
          f"step(NULL) back to back {null_only:.1f} | step(NULL) bracketed {per:.1f}")


if __name__ == "__main__":
    main()
