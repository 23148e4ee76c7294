"""Model check of the stale-entry protocol of the p2p exchange (DESIGN.md
Sec. 7; csrc/tile_encode.cuh, csrc/step_p2p.cu, gtc.cu step_fused_p2p).

Readers accept an entry of a tile slot (the owner's segmented buffer) or of a
pushed record (a peer's push region) as soon as it carries this step's stamp,
with no fence on the writer's side, so the protocol is only correct if no
slot can hold an OLD entry with the current stamp at the moment a step starts
writing.  The writers' rules that guarantee it:
  - a step writes entries [0, k) and clears [k, prev_k) of its parity's slot;
  - a fused step's record copy covers [0, roundup4(min(max(k, prev_k), cap)))
    (zeros beyond k), and the first fused step after a non-fused step of the
    same parity clears the whole record first.
This test replays those rules over random sequences of fused / separate steps
and counts, with a deliberately SHORT stamp period (5 instead of 524,287) so
that any rule slip lets an old entry alias the current stamp within a few
steps.  It checks that, at the start of every step, no entry position the
readers will accept holds a pre-existing value with the current stamp.  The
negative controls show the check has teeth: dropping either clearing rule
makes it fail."""
import random

import pytest

PERIOD = 5          # stamp(e) = e % PERIOD + 1 (the library: 524287, odd like this)
TILE = 64           # entries per slot (the library: 4096)
CAP = 16            # pushed entries per record (the library: 512)


def stamp(e):
    return e % PERIOD + 1


def run(steps, seed, clear_seg=True, clear_record_range=True, reset_dirty_records=True):
    rng = random.Random(seed)
    seg = [[0] * TILE for _ in range(2)]       # (stamp) per entry, per parity
    tag_k = [0, 0]                             # last count written per parity
    rec = [[0] * CAP for _ in range(2)]        # this rank's record on a peer, per parity
    clean = [True, True]
    violations = 0
    for e in range(1, steps + 1):
        p = e & 1
        k = rng.choice([0, 1, 3, 5, 15, 16, 17, 40, TILE]) if rng.random() < 0.5 else rng.randrange(TILE + 1)
        fused = rng.random() < 0.6
        s = stamp(e)
        prev = tag_k[p]
        # readers of this step accept positions [0, k) of the slot and
        # [0, min(k, CAP)) of the record: none may already carry stamp s
        violations += sum(1 for j in range(k) if seg[p][j] == s)
        if fused and not clean[p] and reset_dirty_records:
            rec[p] = [0] * CAP
        if fused:
            violations += sum(1 for j in range(min(k, CAP)) if rec[p][j] == s)
        # the writes of step e
        for j in range(k):
            seg[p][j] = s
        if clear_seg:
            for j in range(k, prev):
                seg[p][j] = 0
        if fused:
            clr = min(max(k, prev), CAP) if clear_record_range else min(k, CAP)
            clr4 = (clr + 3) // 4 * 4
            for j in range(min(clr4, CAP)):
                rec[p][j] = s if j < k else 0
            clean[p] = True
        else:
            clean[p] = False
        tag_k[p] = k
    return violations


@pytest.mark.parametrize("seed", range(8))
def test_protocol_never_accepts_a_stale_entry(seed):
    assert run(20000, seed) == 0


def test_negative_controls():
    """Each clearing rule is necessary: without it old entries alias."""
    assert sum(run(20000, s, clear_seg=False) for s in range(4)) > 0
    assert sum(run(20000, s, clear_record_range=False) for s in range(4)) > 0
    assert sum(run(20000, s, reset_dirty_records=False) for s in range(4)) > 0


def test_library_stamp_period_is_odd_and_nonzero():
    # the real stamp function (tile_encode.cuh entry_stamp): e % 524287 + 1
    assert 524287 % 2 == 1 and 524287 < (1 << 19)
