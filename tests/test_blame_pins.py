"""Pins of the NEXT-4 event-level blame oracle (oracle.blame; DESIGN.md §10e readings EB1-EB6),
CPU only. The definition is ours (the paper's insight P:L139-140: victims "only lag because they are
waiting for the faulty peer"), so it is pinned by hand-derived chains and a cycle, by wait
conservation against the analysis' own per-rank wait sums, and by the DES generator's injected
throttles (the throttled rank must carry the largest inflicted wait)."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from helpers import AR, C

NONE, CYCLE = 2**64 - 1, 2**64 - 2


def test_chain_through_a_victim():
    # rank 0 computes 100 then joins c0 = {0,1}; rank 1 waits 90 for it, then joins c1 = {1,2}
    # where rank 2 waits 190 for rank 1. Rank 1's lateness in c1 comes from its wait in c0, so both
    # waits are blamed on rank 0's compute event (event 0).
    tr = tg.from_events(1, 1, 3, [[0, 1], [1, 2]], [
        [(C, 0, 100), (AR, 0, 10, 0)],
        [(C, 0, 10), (AR, 0, 100, 0), (AR, 0, 10, 1)],
        [(C, 0, 10), (AR, 0, 200, 1)],
    ])
    b = oracle.blame(tr)
    assert b["bl_root"].tolist() == [NONE, NONE, NONE, 0, NONE, NONE, 0]
    assert b["bl_inflicted"].tolist() == [280, 0, 0]
    assert b["bl_self"].tolist() == [0, 0, 0]
    assert b["bl_suffered"].tolist() == [0, 90, 190]
    assert b["bl_n_waiting"] == 2 and b["bl_n_cyclic"] == 0


def test_self_blame_and_first_event_root():
    # rank 1's first event is a collective it arrives last to (no wait); its next collective waits
    # for rank 0, whose previous event is that same first collective of rank 0 -> root is rank 0's
    # first event (a communication event with no predecessor). Rank 0 then waits on rank 1 whose
    # previous event is rank 1's own compute -> inflicted on rank 1.
    tr = tg.from_events(1, 1, 2, [[0, 1]], [
        [(AR, 0, 50, 0), (C, 0, 30), (AR, 0, 5, 0), (AR, 0, 40, 0)],
        [(AR, 0, 10, 0), (AR, 0, 20, 0), (C, 0, 70), (AR, 0, 5, 0)],
    ])
    b = oracle.blame(tr)
    # instances: #0 (50 | 10) rank 0 waits 40, last = 1, Le = event 4 (rank 1's first) -> root 4
    #            #1 (5 | 20)  rank 1 waits 15, last = 0, Le = event 2 -> pred = event 1 (compute)
    #            #2 (40 | 5)  rank 0 waits 35, last = 1, Le = event 7 -> pred = event 6 (compute)
    assert b["bl_root"].tolist() == [4, NONE, NONE, 6, NONE, 1, NONE, NONE]
    assert b["bl_inflicted"].tolist() == [15, 75]
    assert b["bl_suffered"].tolist() == [75, 15]


def test_cycle_is_unattributed():
    # c0 and c1 have the same members; rank 0 runs c0 then c1, rank 1 runs c1 then c0 and each
    # arrives last to the collective the other waits in: the pointers form a cycle.
    tr = tg.from_events(1, 1, 2, [[0, 1], [0, 1]], [
        [(AR, 0, 10, 0), (AR, 0, 2, 1)],
        [(AR, 0, 10, 1), (AR, 0, 2, 0)],
    ])
    b = oracle.blame(tr)
    assert b["bl_root"].tolist() == [CYCLE, NONE, CYCLE, NONE]
    assert b["bl_unattributed"].tolist() == [8, 8]
    assert b["bl_inflicted"].tolist() == [0, 0] and b["bl_n_cyclic"] == 2


def test_no_waits():
    tr = tg.from_events(1, 1, 2, [[0, 1]], [[(C, 0, 10), (AR, 0, 5, 0)], [(C, 0, 10), (AR, 0, 5, 0)]])
    b = oracle.blame(tr)
    assert b["bl_n_waiting"] == 0 and not b["bl_inflicted"].any() and (b["bl_root"] == NONE).all()


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_wait_conservation(seed):
    """Every waiting nanosecond is blamed exactly once; per rank, the suffered wait is the analysis'
    own per-rank wait sum (A3 rk_sum_wait)."""
    tr = tg.generate(tg.GenConfig(2, 2, 2, 2, 4, 4, seed=seed, faults=[tg.Fault(tg.THROTTLE, seed, factor=2.0)]))
    b = oracle.blame(tr)
    tot = int(b["bl_suffered"].sum())
    assert tot == int(b["bl_inflicted"].sum() + b["bl_self"].sum() + b["bl_unattributed"].sum())
    assert np.array_equal(b["bl_suffered"], b["rk_sum_wait"])
    w = b["bl_root"] != NONE
    assert int(w.sum()) == b["bl_n_waiting"]
    assert int(b["ev_wait"][w].astype(np.uint64).sum()) == tot


@pytest.mark.parametrize("tp,pp,dp,src", [(2, 2, 2, 5), (2, 2, 2, 2), (2, 1, 4, 6), (1, 2, 4, 3), (4, 2, 2, 9)])
def test_injected_throttle_is_the_top_source(tp, pp, dp, src):
    """DES ground truth: the throttled rank (x2.5 on every kernel) inflicts the most wait."""
    tr = tg.generate(tg.GenConfig(tp, pp, dp, 2, max(pp, 4), 4, seed=7, faults=[tg.Fault(tg.THROTTLE, src, factor=2.5)]))
    b = oracle.blame(tr)
    assert int(np.argmax(b["bl_inflicted"])) == src
    assert b["bl_n_cyclic"] == 0


def test_roots_are_compute_or_first_events():
    tr = tg.generate(tg.GenConfig(2, 2, 2, 2, 4, 3, seed=4))
    b = oracle.blame(tr)
    ro = tr.rank_offsets.astype(np.int64)
    firsts = set(ro[:-1].tolist())
    for e in np.flatnonzero(b["bl_root"] < CYCLE):
        x = int(b["bl_root"][e])
        assert (tr.kind_op[x] & 7) == 0 or x in firsts
