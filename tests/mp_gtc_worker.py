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
    accum = os.environ.get("GTC_ACCUM", "weights")
    momentum = accum == "momentum"
    gmode = {"weights": gtc.GTC_ACCUM_WEIGHTS, "update": gtc.GTC_ACCUM_UPDATE, "momentum": gtc.GTC_ACCUM_MOMENTUM}[accum]
    omode = {"weights": oracle.ACCUM_WEIGHTS, "update": oracle.ACCUM_UPDATE, "momentum": oracle.ACCUM_MOMENTUM}[accum]
    mu = 0.9
    tau = 8.0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    sharded = os.environ.get("GTC_SHARDED") == "1"
    ctx = gtc.GTC(n, tau, rank, world, dev, cmp=cmp, exchange=exchange, sharded=sharded)
    assert ctx.exchange_mode() == exchange, ctx.exchange_mode()

    r0 = [synth.uniform(n, -tau, tau, synth.rank_seed(w)) for w in range(world)]
    w0 = synth.normal(n, 99)
    r_or = [r.copy() for r in r0]
    w_or = w0.copy()
    rd = torch.from_numpy(r0[rank].copy()).to(dev)
    wd = torch.from_numpy(w0.copy()).to(dev)
    cnt = torch.empty(n, dtype=torch.int8, device=dev)
    mode = oracle.CMP_GT if cmp == "gt" else oracle.CMP_GE
    buf_or = np.zeros(n, np.float32)
    bd = torch.zeros(n, dtype=torch.float32, device=dev)
    if momentum:
        ctx.bind_momentum(bd, mu)

    def check_buf(what):
        if momentum:
            assert np.array_equal(bd.cpu().numpy().view(np.uint32), buf_or.view(np.uint32)), what
    for t in range(steps):
        gs = [synth.correlated_gradient(n, 4.0, synth.BASE_SEED, t, w) for w in range(world)]
        ctx.encode(torch.from_numpy(gs[rank]).to(dev), rd)
        st = ctx.exchange()
        assert st == gtc.GTC_OK, st
        assert ctx.check() == gtc.GTC_OK
        ctx.decode_apply(wd, -0.5, gmode, cnt)
        torch.cuda.synchronize()
        om, oc, _ = oracle.step(gs, r_or, w_or, tau, mode, -0.5, omode, buf=buf_or, mu=mu)
        check_buf(f"rank {rank} step {t}: momentum buffer")
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
    # the one-call step (p2p: one fused encode+exchange+decode kernel); odd steps start the ranks
    # at different times so the in-kernel waits on peers' tiles are exercised
    for t in range(steps, 2 * steps):
        gs = [synth.correlated_gradient(n, 4.0, synth.BASE_SEED, t, w) for w in range(world)]
        g_dev = torch.from_numpy(gs[rank]).to(dev)
        if t % 2 == 1:
            torch.cuda._sleep(int(1e6 * ((rank + t) % world)))
        st = ctx.step(g_dev, rd, wd, -0.5, gmode)
        assert st == gtc.GTC_OK, st
        torch.cuda.synchronize()
        assert ctx.check() == gtc.GTC_OK
        om, _, _ = oracle.step(gs, r_or, w_or, tau, mode, -0.5, omode, buf=buf_or, mu=mu)
        check_buf(f"rank {rank} step {t}: momentum buffer (gtc_step)")
        assert ctx.last_counts() == [m.size for m in om], (ctx.last_counts(), [m.size for m in om])
        for w in range(world):
            assert np.array_equal(ctx.read_message(w), om[w]), f"rank {rank} step {t}: message of rank {w} (gtc_step)"
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
        print(f"MULTIGPU OK world={world} n={n} steps={steps} cmp={cmp} exchange={exchange} momentum={momentum} "
              f"sharded={sharded}")





def bmuf_main():
    """One rank of the multi-GPU BMUF check (GTC_MODE=bmuf)."""
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    n = int(os.environ.get("GTC_N", 1_000_003))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    exchange = os.environ.get("GTC_EXCHANGE", "p2p")
    eta = 1.0 - 1.0 / world
    zeta = 1.0  # Eq. (5) with C = 1
    w0 = synth.normal(n, 5)
    b = gtc.BMUF(n, eta, zeta, rank, world, dev, w_init=torch.from_numpy(w0).to(dev), exchange=exchange)
    wg_h, d_h = w0.copy(), np.zeros(n, np.float32)
    w = b.local_buffer()
    eps = np.float64(2.0 ** -24)
    lo = rank * b.shard
    hi = min(n, lo + b.shard)
    for t in range(4):
        ws_h = [(wg_h + synth.normal(n, 20 + i, t) * np.float32(0.01)).astype(np.float32) for i in range(world)]
        w[:n].copy_(torch.from_numpy(ws_h[rank]))
        if t % 2 == 1:  # ranks arrive at different times: the device-side waits must hold
            torch.cuda._sleep(int(2e6 * rank))
        b.sync(w)
        torch.cuda.synchronize()
        b.check()
        got = w[:n].cpu().numpy()
        if exchange == "p2p":  # rank-ordered double mean: bit-exact with the oracle
            wg_o, d_o = wg_h.copy(), d_h.copy()
            oracle.bmuf_step([x.copy() for x in ws_h], wg_o, d_o, eta, zeta)
            assert np.array_equal(got.view(np.uint32), wg_o.view(np.uint32)), f"rank {rank} step {t}: Wg differs"
            assert np.array_equal(b.delta[: hi - lo].cpu().numpy().view(np.uint32), d_o[lo:hi].view(np.uint32)), \
                f"rank {rank} step {t}: Delta differs"
            assert np.array_equal(b.wg[: hi - lo].cpu().numpy().view(np.uint32), wg_o[lo:hi].view(np.uint32))
        wg_prev = wg_h.astype(np.float64)
        d_prev = d_h.astype(np.float64)
        mean_abs = np.mean(np.abs(np.stack(ws_h).astype(np.float64)), axis=0)
        oracle.bmuf_step([x.copy() for x in ws_h], wg_h, d_h, eta, zeta)
        # Error bound from every rounding of Eqs. (1)-(4), with NCCL summing in
        # its own order: |dWbar| <= (N-1) eps mean|W| + eps |Wbar| (sum, division);
        # G, Delta and Wg add one relative eps per operation on their operands;
        # the mean's error reaches Wg through zeta and (1 + eta).
        G = np.abs(np.mean(np.stack(ws_h).astype(np.float64), axis=0) - wg_prev)
        d_new = np.abs(d_h.astype(np.float64))
        e_wbar = (world - 1) * eps * mean_abs + eps * (mean_abs + G)
        e_d = zeta * (e_wbar + eps * G) + 2 * eps * (eta * np.abs(d_prev) + zeta * G) + eps * d_new
        tol = (1 + eta) * e_d + 3 * eps * (np.abs(wg_prev) + (1 + eta) * d_new) \
            + 2 * np.spacing(np.abs(wg_h)).astype(np.float64)
        err = np.abs(got.astype(np.float64) - wg_h.astype(np.float64))
        bad = np.argmax(err - tol)
        assert np.all(err <= tol), f"rank {rank} step {t}: err {err[bad]} vs tol {tol[bad]} at {bad}"
        wg_h = got.copy()  # continue from the device state (each step checked on its own)
        d_dev = b.delta[: hi - lo].cpu().numpy()
        d_h[lo:hi] = d_dev  # likewise for Delta
        hs = [None] * world
        dist.all_gather_object(hs, hashlib.sha256(got.tobytes()).hexdigest())
        assert len(set(hs)) == 1, f"ranks disagree on Wg at step {t}"
    if exchange == "p2p":
        # back-to-back steps with device-side local updates and no host sync:
        # the push / ready handshake alone orders them
        wg_o, d_o = wg_h.copy(), d_h.copy()
        ws_o = [wg_o.copy() for _ in range(world)]
        w[:n].copy_(torch.from_numpy(wg_h))
        for t in range(3):
            x = [(synth.normal(n, 40 + i, t) * np.float32(0.01)).astype(np.float32) for i in range(world)]
            w[:n].add_(torch.from_numpy(x[rank]).to(dev, non_blocking=True))
            torch.cuda._sleep(int(1e6 * ((rank + t) % world)))
            b.sync(w)
            ws_o = [(ws_o[i] + x[i]).astype(np.float32) for i in range(world)]
            oracle.bmuf_step(ws_o, wg_o, d_o, eta, zeta)
            ws_o = [wg_o.copy() for _ in range(world)]
        torch.cuda.synchronize()
        b.check()
        assert np.array_equal(w[:n].cpu().numpy().view(np.uint32), wg_o.view(np.uint32)), \
            f"rank {rank}: back-to-back steps differ from the oracle"
    b.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(f"BMUF OK world={world} n={n} exchange={exchange}")


if __name__ == "__main__":
    if os.environ.get("GTC_MODE") == "bmuf":
        bmuf_main()
    else:
        main()
