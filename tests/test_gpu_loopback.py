"""World > 1 parity on ONE GPU: the loopback group (GTC_LOOPBACK).

Rows a6 (exchange, "Each worker communicates the sparse update to
all other workers and conversely receives all sparse updates") and f1 (the
device-initiated exchange fused into decode) of SURVEY.md Sec. 8, proved on a
one-GPU box: `world` contexts live in this process and every rank's peers are
the other contexts' workspaces (plain device pointers instead of CUDA-IPC
mappings).  The kernels are the production ones:

  - split path: every rank's gtc_encode (loopback: followed by the publish
    kernel), gtc_exchange, then gtc_decode_apply -- the flag-gated decode
    reading the peers' stamped tiles in place (no kernel ever waits on one not
    yet queued); with GTC_DECODE_SHARDED the owner count (gtc_exchange) and
    the list apply (gtc_decode_apply);
  - fused path: gtc_step_group, the one-kernel encode -> push -> decode ->
    apply step of EVERY rank as ONE launch (ticket g is CTA g/world of rank
    g%world, so no launch waits on another launch).

Every rank's message, k, integer counts, residual, weights (or momentum
buffer) and the replica hash are compared with an N-worker oracle step
(bit-exact).  In the fused path the counts are read back through
GTC_ACCUM_UPDATE into a zero buffer with tau a power of two: fl(0 + fl(c*tau))
= c*tau exactly.
"""
import hashlib
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1904_10584_b200 as gtc  # noqa: E402

DEV = torch.device("cuda", 0)
CMP = {"gt": oracle.CMP_GT, "ge": oracle.CMP_GE}
GMODE = {"weights": gtc.GTC_ACCUM_WEIGHTS, "update": gtc.GTC_ACCUM_UPDATE, "momentum": gtc.GTC_ACCUM_MOMENTUM}
OMODE = {"weights": oracle.ACCUM_WEIGHTS, "update": oracle.ACCUM_UPDATE, "momentum": oracle.ACCUM_MOMENTUM}


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def bits(t):
    return t.detach().cpu().numpy().view(np.uint32)


def grads_for(kind, n, tau, t, world):
    if kind == "correlated":  # counts of +-2 .. +-N and cancellations
        return [synth.correlated_gradient(n, 4.0, synth.BASE_SEED, t, w) for w in range(world)]
    if kind == "dense":  # >> kPushCap = 512 entries per tile: the pull-over path
        return [synth.correlated_gradient(n, 3.0 * tau, synth.BASE_SEED, t, w) for w in range(world)]
    if kind == "dyadic":
        return [synth.dyadic_gradient(n, 3.0, tau, synth.BASE_SEED, t, w) for w in range(world)]
    raise ValueError(kind)


class Run:
    """Device state of a loopback group plus the oracle's mirror of it."""

    def __init__(self, n, tau, world, cmp, accum, mu=0.9, seed=0, sharded=False):
        self.n, self.tau, self.world, self.cmp, self.accum, self.mu = n, tau, world, cmp, accum, mu
        self.grp = gtc.LoopbackGroup(n, tau, world, DEV, cmp=cmp, sharded=sharded)
        self.r_or = [synth.uniform(n, -tau, tau, synth.rank_seed(w), seed) for w in range(world)]
        self.w_or = synth.normal(n, 99 + seed)
        if accum == "update":
            self.w_or[:] = 0.0
        self.rd = [to_dev(r) for r in self.r_or]
        self.wd = [to_dev(self.w_or) for _ in range(world)]  # one replica per rank
        self.buf_or = np.zeros(n, np.float32)
        self.bd = [torch.zeros(n, dtype=torch.float32, device=DEV) for _ in range(world)]
        if accum == "momentum":
            self.grp.bind_momentum(self.bd, mu)

    def oracle_step(self, gs, alpha):
        if self.accum == "update":
            self.w_or[:] = 0.0
        return oracle.step(gs, self.r_or, self.w_or, self.tau, CMP[self.cmp], alpha, OMODE[self.accum],
                           buf=self.buf_or, mu=self.mu)

    def check(self, om, oc, what, counts=None):
        grp, world = self.grp, self.world
        for r in range(world):
            assert grp.ranks[r].last_counts() == [m.size for m in om], f"{what}: k seen by rank {r}"
            for m in range(world):
                got = grp.ranks[r].read_message(m)
                assert np.array_equal(got, om[m]), f"{what}: message of rank {m} as seen by rank {r}"
            assert np.array_equal(bits(self.rd[r]), self.r_or[r].view(np.uint32)), f"{what}: residual {r}"
            wh = self.wd[r].cpu().numpy()
            assert np.array_equal(wh.view(np.uint32), self.w_or.view(np.uint32)), f"{what}: weights of rank {r}"
            if self.accum == "momentum":
                assert np.array_equal(bits(self.bd[r]), self.buf_or.view(np.uint32)), f"{what}: momentum {r}"
            if counts is not None:
                assert np.array_equal(counts[r].cpu().numpy().astype(np.int32), oc), f"{what}: counts of rank {r}"
        if self.accum == "update":
            # fused path: tau is a power of two, so target / tau is the count
            got_c = (self.wd[0].cpu().numpy() / np.float32(self.tau)).astype(np.int64)
            assert np.array_equal(got_c, oc.astype(np.int64)), f"{what}: counts via the update buffer"
        hs = {hashlib.sha256(w.cpu().numpy().tobytes()).hexdigest() for w in self.wd}
        assert len(hs) == 1, f"{what}: replicas differ"
        for r, st in enumerate(grp.check()):
            assert st == gtc.GTC_OK, f"{what}: rank {r} flags {st}"

    def zero_update_targets(self):
        if self.accum == "update":
            for w in self.wd:
                w.zero_()

    def close(self):
        self.grp.close()


# ------------------------------------------------------------------ split path (flag-gated decode)
@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("cmp", ["gt", "ge"])
@pytest.mark.parametrize("accum", ["weights", "update", "momentum"])
def test_loopback_split_parity(world, cmp, accum):
    n, tau, alpha = 1_000_003, 8.0, -0.5
    run = Run(n, tau, world, cmp, accum)
    counts = [torch.empty(n, dtype=torch.int8, device=DEV) for _ in range(world)]
    for t in range(4):
        gs = grads_for("correlated" if t % 2 == 0 else "dyadic", n, tau, t, world)
        run.zero_update_targets()
        sts = run.grp.split_step([to_dev(g) for g in gs], run.rd, run.wd, alpha, GMODE[accum], counts_out=counts)
        assert all(st == gtc.GTC_OK for st in sts)
        torch.cuda.synchronize()
        om, oc, _ = run.oracle_step(gs, alpha)
        run.check(om, oc, f"split world={world} step {t}", counts)
    run.close()


# ------------------------------------------------------------------ owner-computes (sharded) decode
@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("accum", ["weights", "update", "momentum"])
def test_loopback_sharded_parity(world, accum):
    """GTC_DECODE_SHARDED: each owner counts its tile range
    from every rank's message and publishes per-tile (index, count) lists;
    every rank applies every list.  Bit-identical to the replicated decode and
    the oracle, counts_out included (odd n: a ragged last tile)."""
    n, tau, alpha = 1_000_003, 8.0, -0.5
    run = Run(n, tau, world, "gt" if world != 3 else "ge", accum, sharded=True)
    counts = [torch.empty(n, dtype=torch.int8, device=DEV) for _ in range(world)]
    for t in range(4):
        gs = grads_for("correlated" if t % 2 == 0 else "dense", n, tau, t, world)
        run.zero_update_targets()
        run.grp.split_step([to_dev(g) for g in gs], run.rd, run.wd, alpha, GMODE[accum], counts_out=counts)
        torch.cuda.synchronize()
        om, oc, _ = run.oracle_step(gs, alpha)
        run.check(om, oc, f"sharded world={world} step {t}", counts)
    # gtc_step on a sharded context of a loopback group is refused like any
    # loopback gtc_step; without counts_out the sparse list apply runs
    for t in range(4, 6):
        gs = grads_for("correlated", n, tau, t, world)
        run.zero_update_targets()
        run.grp.split_step([to_dev(g) for g in gs], run.rd, run.wd, alpha, GMODE[accum])
        torch.cuda.synchronize()
        om, oc, _ = run.oracle_step(gs, alpha)
        run.check(om, oc, f"sharded world={world} step {t} (no counts)")
    run.close()


def test_loopback_sharded_tiny_and_more_ranks_than_tiles():
    """Owner ranges of 0 tiles (n < world tiles) and a one-tile vector."""
    for n in (1, 4097, 3 * 4096 + 5):
        run = Run(n, 2.0, 4, "gt", "weights", sharded=True)
        for t in range(2):
            gs = grads_for("correlated", n, 2.0, t, 4)
            run.grp.split_step([to_dev(g) for g in gs], run.rd, run.wd, -0.5)
            torch.cuda.synchronize()
            om, oc, _ = run.oracle_step(gs, -0.5)
            run.check(om, oc, f"sharded tiny n={n} step {t}")
        run.close()


# ------------------------------------------------------------------ fused one-kernel step
@pytest.mark.parametrize("world,lag,accum,cmp", [
    (2, None, "weights", "gt"), (2, "1", "update", "ge"), (2, "7", "weights", "gt"),
    (3, "64", "update", "gt"), (3, None, "momentum", "ge"),
    (4, "5", "weights", "ge"), (4, None, "update", "gt"), (4, "9", "momentum", "gt"),
])
def test_loopback_fused_parity(world, lag, accum, cmp, monkeypatch):
    """gtc_step_group: the fused kernel of every rank in one launch, with the
    default decode lag and with short lags (CTAs then wait on tiles
    still being encoded: stamped entries, re-polls)."""
    if lag is not None:
        monkeypatch.setenv("GTC_FUSED_LAG", lag)
    n, tau, alpha = 1_000_003, 8.0, -0.5
    run = Run(n, tau, world, cmp, accum)
    for t in range(4):
        gs = grads_for("correlated" if t % 2 == 0 else "dyadic", n, tau, t, world)
        run.zero_update_targets()
        st = run.grp.step([to_dev(g) for g in gs], run.rd, run.wd, alpha, GMODE[accum])
        assert st == gtc.GTC_OK
        torch.cuda.synchronize()
        om, oc, _ = run.oracle_step(gs, alpha)
        run.check(om, oc, f"fused world={world} lag={lag} step {t}")
    run.close()


@pytest.mark.parametrize("world", [2, 4])
def test_loopback_fused_dense_tiles_pull_over(world, monkeypatch):
    """Tiles far denser than the pushed record (> 512 entries): the decode
    pulls the rest from the owner's segmented buffer."""
    monkeypatch.setenv("GTC_FUSED_LAG", "3")
    n, tau = 300_007, 8.0
    run = Run(n, tau, world, "gt", "update")
    for t in range(3):
        gs = grads_for("dense", n, tau, t, world)
        run.zero_update_targets()
        assert run.grp.step([to_dev(g) for g in gs], run.rd, run.wd, 1.0, gtc.GTC_ACCUM_UPDATE) == gtc.GTC_OK
        torch.cuda.synchronize()
        om, oc, _ = run.oracle_step(gs, 1.0)
        assert max(m.size for m in om) > 0.2 * n  # many tiles beyond kPushCap
        run.check(om, oc, f"dense world={world} step {t}")
    run.close()


@pytest.mark.parametrize("world", [5, 8])
@pytest.mark.parametrize("path", ["fused", "split", "sharded"])
def test_loopback_up_to_8_ranks(world, path, monkeypatch):
    """World 5 and 8 (kFusedMaxRanks): the N = 8 configs of BASELINE.json
    cannot run on the harness's at most 4 GPUs, so their code paths -- 8
    ranks' records per decode, speculative windows of 32 entries per rank and
    the overflow rounds beyond them, 7 pushes per tile, 8 owners -- are
    checked here, bit-exact against the N-worker oracle."""
    n, tau = 150_011, 8.0
    run = Run(n, tau, world, "gt", "weights", sharded=(path == "sharded"))
    kinds = ["correlated", "dense", "dyadic"]
    for t in range(3):
        if path == "fused":
            monkeypatch.setenv("GTC_FUSED_LAG", ["5", "1", "40"][t])
        gs = grads_for(kinds[t], n, tau, t, world)
        gd = [to_dev(g) for g in gs]
        if path == "fused":
            assert run.grp.step(gd, run.rd, run.wd, -0.5) == gtc.GTC_OK
        else:
            run.grp.split_step(gd, run.rd, run.wd, -0.5)
        torch.cuda.synchronize()
        om, oc, _ = run.oracle_step(gs, -0.5)
        run.check(om, oc, f"{path} world={world} step {t} ({kinds[t]})")
    run.close()


def test_loopback_fused_grid_changes_between_steps(monkeypatch):
    """The ticket counter wraps to 0 at the end of every launch, so
    consecutive fused steps with different grids (T + L CTAs, L changed by
    GTC_FUSED_LAG) each hand out tickets 0 .. T + L - 1: a leftover count
    would give CTAs out-of-range tickets and skip tiles."""
    n, tau, world = 400_009, 8.0, 2
    run = Run(n, tau, world, "gt", "weights")
    for t, lag in enumerate(["3", "97", None, "1", "40", None]):
        if lag is None:
            monkeypatch.delenv("GTC_FUSED_LAG", raising=False)
        else:
            monkeypatch.setenv("GTC_FUSED_LAG", lag)
        gs = grads_for("correlated", n, tau, t, world)
        assert run.grp.step([to_dev(g) for g in gs], run.rd, run.wd, -0.5) == gtc.GTC_OK
        torch.cuda.synchronize()
        om, oc, _ = run.oracle_step(gs, -0.5)
        run.check(om, oc, f"lag {lag} step {t}")
    run.close()


def test_loopback_alternating_fused_and_split(monkeypatch):
    """Fused and split steps interleaved: the push records of a parity whose
    last step was split are cleared before the next fused step of it."""
    monkeypatch.setenv("GTC_FUSED_LAG", "2")
    n, tau, world = 200_003, 8.0, 3
    run = Run(n, tau, world, "gt", "weights")
    for t, kind in enumerate(["fused", "split", "split", "fused", "fused", "split", "fused"]):
        gs = grads_for("correlated", n, tau, t, world)
        gd = [to_dev(g) for g in gs]
        if kind == "fused":
            assert run.grp.step(gd, run.rd, run.wd, -0.25) == gtc.GTC_OK
        else:
            run.grp.split_step(gd, run.rd, run.wd, -0.25)
        torch.cuda.synchronize()
        om, oc, _ = run.oracle_step(gs, -0.25)
        run.check(om, oc, f"{kind} step {t}")
    run.close()


def test_loopback_fused_grad_null_and_ragged():
    """grad = NULL (residual already holds r + g) and a ragged last tile."""
    n, tau, world = 3 * gtc.GTC_TILE * 8 + 1234, 8.0, 2
    run = Run(n, tau, world, "ge", "weights")
    for t in range(3):
        gs = grads_for("correlated", n, tau, t, world)
        for r in range(world):
            run.rd[r].add_(to_dev(gs[r]))  # the caller's backward accumulated into r
        assert run.grp.step(None, run.rd, run.wd, -0.5) == gtc.GTC_OK
        torch.cuda.synchronize()
        for r in range(world):  # the oracle's grad=NULL: r already holds fl(r + g)
            run.r_or[r][:] = (run.r_or[r] + gs[r]).astype(np.float32)
        om, oc, _ = oracle.step(None, run.r_or, run.w_or, tau, oracle.CMP_GE, -0.5, oracle.ACCUM_WEIGHTS)
        run.check(om, oc, f"grad-null step {t}")
    run.close()


def test_loopback_lstm_am_size_fused_world4():
    """C3 at the paper's LSTM-AM size (24,286,575 params), world 4, one launch."""
    n, tau, world = synth.LSTM_AM_PARAMS, 8.0, 4
    sigma = synth.sigma_for_density(0.01, tau, synth.mean_abs_scale(n))
    run = Run(n, tau, world, "gt", "weights")
    for t in range(2):
        gs = [synth.lstm_gradient(n, sigma, synth.BASE_SEED, t, w, 0.5) for w in range(world)]
        assert run.grp.step([to_dev(g) for g in gs], run.rd, run.wd, -1e-3) == gtc.GTC_OK
        torch.cuda.synchronize()
        om, oc, _ = run.oracle_step(gs, -1e-3)
        run.check(om, oc, f"lstm_am world=4 step {t}")
    run.close()


@pytest.mark.parametrize("rho", [0.0001, 0.01, 0.1])
def test_loopback_config4_density_sweep_fused_world8(rho):
    """C4 (BASELINE.json configs[3]: density 0.01 %-10 %, 8 workers) through the
    fused one-kernel step itself: a world-8 loopback group at the LSTM-AM
    size, one step per density, bit-exact against the 8-worker oracle."""
    n, tau, world = synth.LSTM_AM_PARAMS, 8.0, 8
    sigma = synth.sigma_for_density(rho, tau, synth.mean_abs_scale(n))
    run = Run(n, tau, world, "gt", "weights")
    gs = [synth.lstm_gradient(n, sigma, synth.BASE_SEED, 0, w, 0.5) for w in range(world)]
    assert run.grp.step([to_dev(g) for g in gs], run.rd, run.wd, -1e-3) == gtc.GTC_OK
    torch.cuda.synchronize()
    om, oc, _ = run.oracle_step(gs, -1e-3)
    assert abs(sum(m.size for m in om) / (world * n) - rho) < 0.5 * rho  # the intended density regime
    run.check(om, oc, f"lstm_am world=8 rho={rho}")
    run.close()


# ------------------------------------------------------------------ failure semantics
def test_loopback_fused_missing_peer_raises_epeer_everywhere(monkeypatch):
    """A rank that never shows up (debug bit): the others time out, and EVERY
    rank's gtc_check reports GTC_EPEER (gtc.h: the step is incomplete)."""
    monkeypatch.setenv("GTC_PEER_TIMEOUT_MS", "200")
    n, tau, world = 100_003, 8.0, 3
    grp = gtc.LoopbackGroup(n, tau, world, DEV)
    gs = grads_for("correlated", n, tau, 0, world)
    rd = [to_dev(synth.uniform(n, -tau, tau, w)) for w in range(world)]
    wd = [torch.zeros(n, dtype=torch.float32, device=DEV) for _ in range(world)]
    assert grp.step([to_dev(g) for g in gs], rd, wd, 1.0, gtc.GTC_ACCUM_WEIGHTS, debug_flags=1 << 1) == gtc.GTC_OK
    torch.cuda.synchronize()
    assert grp.check() == [gtc.GTC_EPEER] * world
    assert grp.check() == [gtc.GTC_OK] * world  # reported once, then cleared
    grp.close()


def test_loopback_split_missing_peer_applies_nothing(monkeypatch):
    """Separate calls: rank 1 never publishes.  Every CTA of rank 0's decode
    waits for every rank's ready flag before touching the target, so nothing is
    applied, and both ranks report GTC_EPEER."""
    monkeypatch.setenv("GTC_PEER_TIMEOUT_MS", "200")
    n, tau, world = 100_003, 8.0, 2
    grp = gtc.LoopbackGroup(n, tau, world, DEV)
    g0 = to_dev(grads_for("correlated", n, tau, 0, world)[0])
    r0 = to_dev(synth.uniform(n, -tau, tau, 3))
    w0 = to_dev(synth.normal(n, 4))
    w_before = bits(w0).copy()
    grp.ranks[0].encode(g0, r0)
    grp.ranks[0].exchange()
    grp.ranks[0].decode_apply(w0, -0.5)
    torch.cuda.synchronize()
    assert np.array_equal(bits(w0), w_before)
    assert grp.ranks[0].check() == gtc.GTC_EPEER
    assert grp.ranks[1].check() == gtc.GTC_EPEER
    grp.close()


def test_loopback_api_errors():
    n, tau = 10_000, 8.0
    a = gtc.GTC(n, tau, 0, 2, DEV, loopback=True)
    b = gtc.GTC(n, tau, 1, 2, DEV, loopback=True)
    r = torch.zeros(n, dtype=torch.float32, device=DEV)
    with pytest.raises(gtc.GTCError) as e:  # not connected yet
        a.encode(r, r)
    assert e.value.status == gtc.GTC_ESTATE
    with pytest.raises(gtc.GTCError) as e:  # ranks out of order
        gtc.gtc_connect_loopback([b.ctx, a.ctx])
    assert e.value.status == gtc.GTC_EINVAL
    gtc.gtc_connect_loopback([a.ctx, b.ctx])
    with pytest.raises(gtc.GTCError) as e:  # one rank's whole step would wait on the others
        a.step(r, r, r)
    assert e.value.status == gtc.GTC_EUNSUPPORTED
    c = gtc.GTC(n + 1, tau, 1, 2, DEV, loopback=True)
    with pytest.raises(gtc.GTCError) as e:  # sizes differ
        gtc.gtc_connect_loopback([a.ctx, c.ctx])
    assert e.value.status == gtc.GTC_EINVAL
    for x in (a, b, c):
        x.close()


def test_peer_timeout_env_is_per_context(monkeypatch):
    monkeypatch.setenv("GTC_PEER_TIMEOUT_MS", "1")
    grp = gtc.LoopbackGroup(50_000, 8.0, 2, DEV)
    monkeypatch.delenv("GTC_PEER_TIMEOUT_MS")
    # a correct step never times out even with a 1 ms budget when every
    # rank is queued before any decode (separate calls)
    n = 50_000
    rd = [torch.zeros(n, dtype=torch.float32, device=DEV) for _ in range(2)]
    wd = [torch.zeros(n, dtype=torch.float32, device=DEV) for _ in range(2)]
    g = [to_dev(x) for x in grads_for("correlated", n, 8.0, 0, 2)]
    grp.split_step(g, rd, wd)
    torch.cuda.synchronize()
    assert grp.check() == [gtc.GTC_OK, gtc.GTC_OK]
    grp.close()
    assert "GTC_PEER_TIMEOUT_MS" not in os.environ
