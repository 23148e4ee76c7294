"""Multi-process host logic on CPU (gloo, world_size 2, 127.0.0.1).

Covers what the N > 1 path does outside the kernels:
  - the NCCL unique-id broadcast of the binding (rank 0 -> all) over a
    torch.distributed group,
  - the exchange protocol of gtc_exchange: all-gather
    of (k, flags), pad every message to max_k, all-gather, strip each rank's
    padding by its k -- run here with the oracle's messages so that every rank
    ends with all N messages and the same counts as a single-process N-worker
    oracle step ("communicates the sparse update to all other workers and
    conversely receives all sparse updates"),
  - max-over-ranks timing reduction used by bench.py.
"""
import hashlib
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_uid(rank, world, port, out):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1904_10584_b200 as gtc

    _init(rank, world, port)
    uid = gtc.broadcast_unique_id(rank)
    allu = [None] * world
    dist.all_gather_object(allu, uid)
    out[rank] = int(len(set(allu)) == 1 and len(uid) == 128)
    dist.destroy_process_group()


def _worker_protocol(rank, world, port, out):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import synth

    _init(rank, world, port)
    n, tau = 200_003, 8.0
    gs = [synth.correlated_gradient(n, 4.0, synth.BASE_SEED, 0, w) for w in range(world)]
    r = synth.uniform(n, -tau, tau, synth.rank_seed(rank))
    words, nf = oracle.encode(gs[rank], r.copy(), tau)
    # 1. (k, flags) of every rank
    kx = torch.tensor([words.size, int(nf)], dtype=torch.int64)
    kx_all = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(kx_all, kx)
    ks = [int(t[0]) for t in kx_all]
    max_k = max(ks)
    # 2. padded all-gather of the words, padding stripped by k_r
    pad = torch.zeros(max_k, dtype=torch.int64)
    pad[: words.size] = torch.from_numpy(words.astype(np.int64))
    recv = [torch.zeros(max_k, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(recv, pad)
    msgs = [recv[w][: ks[w]].numpy().astype(np.uint32) for w in range(world)]
    counts = oracle.decode_counts(msgs, n)
    target = synth.normal(n, 3)
    oracle.apply(counts, target, tau, -0.5, oracle.ACCUM_WEIGHTS)
    # single-process reference: the N-worker oracle step
    rs = [synth.uniform(n, -tau, tau, synth.rank_seed(w)) for w in range(world)]
    t_ref = synth.normal(n, 3)
    om, oc, _ = oracle.step(gs, rs, t_ref, tau, oracle.CMP_GT, -0.5, oracle.ACCUM_WEIGHTS)
    ok = all(np.array_equal(msgs[w], om[w]) for w in range(world))
    ok &= np.array_equal(counts, oc) and np.array_equal(target.view(np.uint32), t_ref.view(np.uint32))
    # replicas equal across ranks
    h = [None] * world
    dist.all_gather_object(h, hashlib.sha256(target.tobytes()).hexdigest())
    ok &= len(set(h)) == 1
    # max-over-ranks timing reduction (bench.py)
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ok &= float(t) == float(world)
    out[rank] = int(ok)
    dist.destroy_process_group()


def _run(fn, world=2):
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(fn, args=(world, port, out), nprocs=world, join=True)
    return [out[r] for r in range(world)]


def test_unique_id_broadcast_gloo():
    assert _run(_worker_uid) == [1, 1]


def test_exchange_protocol_gloo():
    assert _run(_worker_protocol) == [1, 1]
