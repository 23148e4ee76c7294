"""Small exerciser of every kernel path for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): ragged sizes, both comparison modes,
fused world-1 step, counting decode with dump, simulated messages, packing,
and a world-2 loopback group (the ticketed fused step, the split p2p calls
and the owner-computes decode) on one GPU."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_10584_b200 as gtc  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    for n in (1, 4097, 3 * 4096 + 1234, 100_003):
        for cmp in ("gt", "ge"):
            tau = 1.0
            g = torch.from_numpy(synth.normal(n, 1, n) * np.float32(0.8)).to(dev)
            r = torch.from_numpy(synth.uniform(n, -tau, tau, 2, n)).to(dev)
            w = torch.zeros(n, device=dev)
            cnt = torch.empty(n, dtype=torch.int8, device=dev)
            ctx = gtc.GTC(n, tau, cmp=cmp, max_sim_msgs=3)
            ctx.step(g, r, w, -0.5)                          # fused world-1 step
            ctx.encode(g, r)
            ctx.exchange()
            ctx.decode_apply(w, 0.5, gtc.GTC_ACCUM_UPDATE, cnt)  # counting kernel + dump
            ctx.encode(None, r)
            ctx.exchange()
            ctx.decode_apply(w, 0.5)                          # single-message kernel
            m = ctx.read_message()                            # packing kernels
            md = torch.from_numpy(m.view(np.int32).copy()).to(dev)
            ctx.decode_apply_msgs([md, md[: max(0, md.numel() // 2)], md], w, 1.0, gtc.GTC_ACCUM_WEIGHTS, cnt)
            assert ctx.check() in (gtc.GTC_OK, gtc.GTC_ENONFINITE)
            ctx.close()
    for n in (4097, 3 * 4096 + 1234):
        for sharded in (False, True):
            tau = 1.0
            grp = gtc.LoopbackGroup(n, tau, 2, dev, sharded=sharded)
            gs = [torch.from_numpy(synth.normal(n, 1, n, r) * np.float32(0.8)).to(dev) for r in range(2)]
            rs = [torch.from_numpy(synth.uniform(n, -tau, tau, 2, n, r)).to(dev) for r in range(2)]
            ws = [torch.zeros(n, device=dev) for _ in range(2)]
            if not sharded:
                grp.step(gs, rs, ws, -0.5)                    # ticketed fused kernel, one launch
            grp.split_step(gs, rs, ws, -0.5)                  # separate p2p calls (or owner count + apply)
            assert grp.check() == [gtc.GTC_OK] * 2
            grp.close()
    torch.cuda.synchronize()
    print("sanitize smoke done")


if __name__ == "__main__":
    main()
