#!/usr/bin/env python
"""The fused p2p step of a LOOPBACK group (all ranks on one GPU, one launch per
step: gtc_step_group) at the LSTM-AM size -- for ncu captures of the world > 1
kernel (ncu never wraps a multi-rank command) and quick checks on a one-GPU box.
Not a bench number: the ranks share one GPU's HBM and SMs.

    python tools/loopback_bench.py [--world 2] [--steps 200] [--rho 0.01] [--split]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1904_10584_b200 as gtc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--rho", type=float, default=0.01)
    ap.add_argument("--workload", default="lstm_am")
    ap.add_argument("--split", action="store_true", help="separate calls instead of the fused group kernel")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n, tau, W = bench.WORKLOADS[a.workload]["n"], 8.0, a.world
    ins = [bench.make_inputs(n, tau, a.rho, r, W) for r in range(W)]
    grads = [[torch.from_numpy(g).to(dev) for g in x[0]] for x in ins]
    rs = [torch.from_numpy(x[1]).to(dev) for x in ins]
    ws = [torch.from_numpy(ins[0][2]).to(dev) for _ in range(W)]
    grp = gtc.LoopbackGroup(n, tau, W, dev)
    NB = len(grads[0])

    def step(t):
        g = [grads[r][t % NB] for r in range(W)]
        if a.split:
            grp.split_step(g, rs, ws, -1e-3)
        else:
            grp.step(g, rs, ws, -1e-3)

    for t in range(a.warmup):
        step(t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(a.steps):
        step(t)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    assert grp.check() == [gtc.GTC_OK] * W
    ks = grp.ranks[0].last_counts()
    print(json.dumps({"tool": "loopback_bench", "world": W, "n": n, "ms_per_step": ms,
                      "params_per_s_all_ranks": W * n / (ms * 1e-3), "k": ks, "split": a.split}))
    grp.close()


if __name__ == "__main__":
    main()
