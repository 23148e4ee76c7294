"""One rank of the multi-GPU GTC parity run (launched by torchrun from
tests/test_multigpu.py).  Every rank can regenerate every other rank's seeded
inputs, so each rank runs the full N-worker oracle step itself and checks:
  - every rank's message as received through the NCCL exchange (bit-exact),
  - k per rank, the integer counts, the residual and the weights (bit-exact),
  - the replicas: all ranks hold bitwise-identical weights after every step.
"""
import hashlib
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_1904_10584_b200 as gtc  # noqa: E402
import synth  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    n = int(os.environ.get("GTC_N", 1_000_003))
    steps = int(os.environ.get("GTC_STEPS", 4))
    cmp = os.environ.get("GTC_CMP", "gt")
    exchange = os.environ.get("GTC_EXCHANGE", "p2p")
    tau = 8.0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ctx = gtc.GTC(n, tau, rank, world, dev, cmp=cmp, exchange=exchange)
    assert ctx.exchange_mode() == exchange, ctx.exchange_mode()

    r0 = [synth.uniform(n, -tau, tau, synth.rank_seed(w)) for w in range(world)]
    w0 = synth.normal(n, 99)
    r_or = [r.copy() for r in r0]
    w_or = w0.copy()
    rd = torch.from_numpy(r0[rank].copy()).to(dev)
    wd = torch.from_numpy(w0.copy()).to(dev)
    cnt = torch.empty(n, dtype=torch.int8, device=dev)
    mode = oracle.CMP_GT if cmp == "gt" else oracle.CMP_GE
    for t in range(steps):
        gs = [synth.correlated_gradient(n, 4.0, synth.BASE_SEED, t, w) for w in range(world)]
        ctx.encode(torch.from_numpy(gs[rank]).to(dev), rd)
        st = ctx.exchange()
        assert st == gtc.GTC_OK, st
        assert ctx.check() == gtc.GTC_OK
        ctx.decode_apply(wd, -0.5, gtc.GTC_ACCUM_WEIGHTS, cnt)
        torch.cuda.synchronize()
        om, oc, _ = oracle.step(gs, r_or, w_or, tau, mode, -0.5, oracle.ACCUM_WEIGHTS)
        assert ctx.last_counts() == [m.size for m in om], (ctx.last_counts(), [m.size for m in om])
        for w in range(world):
            got = ctx.read_message(w)
            assert np.array_equal(got, om[w]), f"rank {rank} step {t}: message of rank {w}"
        assert np.array_equal(rd.cpu().numpy().view(np.uint32), r_or[rank].view(np.uint32)), "residual"
        assert np.array_equal(cnt.cpu().numpy().astype(np.int32), oc), "counts"
        wh = wd.cpu().numpy()
        assert np.array_equal(wh.view(np.uint32), w_or.view(np.uint32)), "weights"
        h = hashlib.sha256(wh.tobytes()).hexdigest()
        hs = [None] * world
        dist.all_gather_object(hs, h)
        assert len(set(hs)) == 1, f"replicas differ at step {t}"
    # the one-call step (p2p: pipelined encode/decode chunks on two streams)
    for t in range(steps, 2 * steps):
        gs = [synth.correlated_gradient(n, 4.0, synth.BASE_SEED, t, w) for w in range(world)]
        st = ctx.step(torch.from_numpy(gs[rank]).to(dev), rd, wd, -0.5, gtc.GTC_ACCUM_WEIGHTS)
        assert st == gtc.GTC_OK, st
        torch.cuda.synchronize()
        oracle.step(gs, r_or, w_or, tau, mode, -0.5, oracle.ACCUM_WEIGHTS)
        assert np.array_equal(rd.cpu().numpy().view(np.uint32), r_or[rank].view(np.uint32)), f"step {t}: residual"
        wh = wd.cpu().numpy()
        assert np.array_equal(wh.view(np.uint32), w_or.view(np.uint32)), f"step {t}: weights (gtc_step)"
        hs = [None] * world
        dist.all_gather_object(hs, hashlib.sha256(wh.tobytes()).hexdigest())
        assert len(set(hs)) == 1, f"replicas differ at step {t} (gtc_step)"
    assert ctx.check() == gtc.GTC_OK
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(f"MULTIGPU OK world={world} n={n} steps={steps} cmp={cmp} exchange={exchange}")


if __name__ == "__main__":
    main()
