"""Pins of the oracle's timeline alignment (NEXT-1; DESIGN.md
readings AL1-AL6), -m "not gpu". Each case is fixed by something other than the oracle's code: the
SPEC worked examples, exact recovery of constant clock offsets, the generator's hidden true clock
(skew + 10 ppm drift) within the drift x anchor-gap bound, and invariants (identity without skew,
reference invariance up to one shift, per-rank monotonicity)."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from tracegen import configs
from helpers import AR, C, SEND, RECV


def _with_start(tr, start):
    from dataclasses import replace
    return replace(tr, start_ns=np.ascontiguousarray(start, dtype=np.int64))


def test_spec_uniform_skew_one_allreduce():
    """two ranks, rank 1's clock uniformly +500 us ahead, one AllReduce -> offset -500 us."""
    # true timeline: rank 0 computes 1000 ns, rank 1 1500 ns; the AllReduce ends for both at 3000 ns
    tr = tg.from_events(1, 1, 2, [[0, 1]], [[(C, 0, 1000), (AR, 0, 2000, 0)], [(C, 0, 1500), (AR, 0, 1500, 0)]])
    start = tr.start_ns.copy()
    start[2:] += 500_000
    o = oracle.align(_with_start(tr, start), 0)
    assert o["al_status"] == 0
    assert list(o["al_level"]) == [0, 1] and list(o["al_nanchor"]) == [0, 1]
    np.testing.assert_array_equal(o["al_start"], tr.start_ns)
    assert list(o["al_residual"]) == [0, 0]


def test_spec_single_rank_zero_offset():
    """a single rank aligns to itself (zero offset, residual 0)."""
    tr = tg.from_events(1, 1, 1, [[0]], [[(C, 0, 10), (AR, 0, 5, 0), (C, 0, 7)]])
    o = oracle.align(_with_start(tr, tr.start_ns + 12345), 0)
    np.testing.assert_array_equal(o["al_start"], tr.start_ns + 12345)
    assert list(o["al_level"]) == [0] and list(o["al_residual"]) == [0]


def test_unreached_rank_keeps_local_clock():
    """S:L271 errors: a rank sharing no collective instance (P2P only, AL1) is not aligned."""
    tr = tg.from_events(1, 1, 2, [], [[(C, 0, 10), (SEND, 0, 5, 1, 64)], [(C, 0, 12), (RECV, 0, 3, 0, 64)]])
    start = tr.start_ns + np.array([0, 0, 999, 999])
    o = oracle.align(_with_start(tr, start), 0)
    assert list(o["al_level"]) == [0, -1]
    np.testing.assert_array_equal(o["al_start"], start)


def test_decreasing_anchor_ends_rejected():
    """AL3: collective ends must not decrease along a rank's program order."""
    tr = tg.from_events(1, 1, 2, [[0, 1]], [[(AR, 0, 100, 0), (AR, 0, 100, 0)], [(AR, 0, 100, 0), (AR, 0, 100, 0)]])
    start = tr.start_ns.copy()
    start[1] = start[0] - 500  # rank 0's second all-reduce ends before its first
    assert oracle.align(_with_start(tr, start), 0)["al_status"] == -9


def _skew_free(cfg):
    cfg.clock_skew = False
    return tg.generate(cfg, ground_truth=True)


def test_identity_without_skew():
    """Skew-free DES: every member of a collective ends at the same true time, so every anchor
    offset is 0 and the aligned timeline is the recorded one."""
    tr = _skew_free(configs.c1(seed=3, iterations=4))
    assert np.array_equal(tr.start_ns, tr.gt_true_start)
    o = oracle.align(tr, 0)
    assert o["al_status"] == 0 and (o["al_level"] >= 0).all()
    np.testing.assert_array_equal(o["al_start"], tr.start_ns)
    assert (o["al_residual"] == 0).all()


@pytest.mark.parametrize("ref", [0, 5])
def test_constant_offsets_recovered_exactly(ref):
    """Pure per-rank clock offsets (no drift): every rank maps onto the reference's clock exactly,
    i.e. aligned = true + c_ref; two references differ by one global shift."""
    tr = _skew_free(configs.c1(seed=4, iterations=4))
    W = tr.world
    c = np.random.default_rng(7).integers(-2_000_000, 2_000_000, W)
    rank_of_ev = np.repeat(np.arange(W), np.diff(tr.rank_offsets).astype(np.int64))
    o = oracle.align(_with_start(tr, tr.gt_true_start + c[rank_of_ev]), ref)
    assert o["al_status"] == 0
    np.testing.assert_array_equal(o["al_start"], tr.gt_true_start + c[ref])


def test_drift_bound_and_monotone():
    """Generator clocks: offset U[-2 ms, 2 ms] + drift U[-10, 10] ppm (tracegen). Against the
    reference rank's clock of the true time, a rank at BFS level k is within
    k * (2e-5 * G + 2 ns) where G is the longest interval a rank's offset is interpolated or
    extrapolated over (anchor gaps and the spans before the first / after the last anchor)."""
    tr = tg.generate(configs.c1(seed=5, iterations=6), ground_truth=True)
    o = oracle.align(tr, 0)
    assert o["al_status"] == 0
    W, ro = tr.world, tr.rank_offsets
    true, loc = tr.gt_true_start.astype(np.float64), tr.start_ns.astype(np.float64)
    r0 = slice(int(ro[0]), int(ro[1]))
    a, b = np.polyfit(true[r0], loc[r0], 1)  # the reference's clock: loc = a * true + b
    err = np.abs(o["al_start"].astype(np.float64) - (a * true + b))
    span = float(tr.start_ns.max() - tr.start_ns.min())  # no anchor gap exceeds the trace span
    for r in range(W):
        sl = slice(int(ro[r]), int(ro[r + 1]))
        k = int(o["al_level"][r])
        assert k >= 0
        assert err[sl].max() <= k * (2e-5 * span + 2) + 2, (r, err[sl].max())
        assert (np.diff(o["al_start"][sl]) >= 0).all()  # S:L288 monotonicity
    raw = np.abs(loc - (a * true + b))
    assert raw.max() > 50 * err.max()  # the skew was real (ms) and alignment removed it (tens of us)
