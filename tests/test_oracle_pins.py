"""Pins for the oracle (-m "not gpu"): the oracle is checked against things other than itself —
SPEC.md's worked examples (tests/golden/spec_examples.json), closed forms, brute-force
enumeration of match sets, the generator's DES ground truth, and invariants — chosen so that a
plausible slip (dropped term, wrong index/sign, transposed operand) fails at least one of them.
"""
import itertools
import random

import numpy as np
import pytest

import oracle
import tracegen as tg
from tracegen import configs
from helpers import AR, C, RECV, SEND, case_trace, dp_trace, groups_by, load_golden, tiny_gen

NONE32 = 0xFFFFFFFF
F_VALID, F_UNIQUE = 8, 16
V_NONE, V_COMPUTE, V_LINK, V_BOTH, V_EXON, V_INSUFF = range(6)
L_CLEAN, L_SRC_RANK, L_SRC_LINK, L_VICTIM, L_UNATTR = range(5)


# ---------------------------------------------------------------- SPEC worked examples
@pytest.mark.parametrize("case", load_golden("spec_examples.json")["cases"], ids=lambda c: c["name"])
def test_spec_examples(case):
    tr = case_trace(case)
    o = oracle.run(tr)
    ex = case["expect"]
    for k in ("n_instances", "n_incomplete", "n_payload_mismatch", "status"):
        if k in ex:
            assert o[k] == ex[k], (k, case["cite"])
    for k in ("in_k", "in_dmin", "in_dmax", "in_payload", "in_npresent", "in_last", "lk_n"):
        if k in ex:
            assert list(o[k]) == ex[k], (k, case["cite"])
    if "lk_med_bw" in ex:
        assert o["lk_med_bw"][0] == pytest.approx(ex["lk_med_bw"][0], rel=1e-15)
    if "in_flags_valid" in ex:
        assert [int(bool(f & F_VALID)) for f in o["in_flags"]] == ex["in_flags_valid"]
    if "inst_members" in ex:
        for i, mem in enumerate(ex["inst_members"]):
            ev = np.nonzero(o["ev_inst"] == i)[0]
            ranks = sorted(int(np.searchsorted(tr.rank_offsets, e, side="right") - 1) for e in ev)
            assert ranks == mem


# ---------------------------------------------------------------- brute-force match enumeration
def _random_tiny(rng: random.Random):
    """Consistent tiny trace: a random global call sequence projected onto each rank."""
    W = rng.choice([2, 3, 4])
    comms = []
    for _ in range(rng.randint(1, 3)):
        k = rng.randint(2, W)
        comms.append(sorted(rng.sample(range(W), k)))
    ranks = [[] for _ in range(W)]
    cnt = [0] * W
    for _ in range(rng.randint(3, 10)):
        if rng.random() < 0.6:
            c = rng.randrange(len(comms))
            if any(cnt[m] >= 6 for m in comms[c]):
                continue
            for m in comms[c]:
                ranks[m].append((AR, 0, rng.randint(1, 9) * 1000, c, 0, 0, 0))
                cnt[m] += 1
        else:
            s, d = rng.sample(range(W), 2)
            if cnt[s] >= 6 or cnt[d] >= 6:
                continue
            pl = rng.choice([64, 128])
            ranks[s].append((SEND, 0, rng.randint(1, 9) * 1000, d, pl, 0, 0))
            ranks[d].append((RECV, 0, rng.randint(1, 9) * 1000, s, pl, 0, 0))
            cnt[s] += 1
            cnt[d] += 1
        if rng.random() < 0.3:
            r = rng.randrange(W)
            ranks[r].append((C, 1, 500, 0, 0, 0, 0))
    return tg.from_events(W, 1, 1, comms, ranks)


def _brute_force_matchings(tr, limit=5000):
    """All order-consistent (acyclic) assignments of comm events to instances, one event per
    member per instance. Channels are re-derived here from the raw columns."""
    W = tr.world
    kinds = tr.kind_op & 7
    ev_rank = np.repeat(np.arange(W), np.diff(tr.rank_offsets).astype(np.int64))
    comms = [list(tr.comm_members[int(tr.comm_offsets[c]):int(tr.comm_offsets[c + 1])]) for c in range(tr.n_comms)]
    per_chan = {}  # channel -> {member rank: [events in order]}
    for e in range(tr.n_events):
        k, r, x = int(kinds[e]), int(ev_rank[e]), int(tr.comm[e])
        if k == 0:
            continue
        ch = ("p", r, x) if k == SEND else ("p", x, r) if k == RECV else ("c", x)
        per_chan.setdefault(ch, {}).setdefault(r, []).append(e)
    chan_opts = []
    for ch, mem in per_chan.items():
        members = list(ch[1:]) if ch[0] == "p" else comms[ch[1]]
        lists = [mem.get(int(m), []) for m in members]
        n = len(lists[0])
        assert all(len(lst) == n for lst in lists)
        opts = []
        for perms in itertools.product(*[list(itertools.permutations(lst)) for lst in lists[1:]]):
            opts.append([tuple([lists[0][i]] + [p[i] for p in perms]) for i in range(n)])
        chan_opts.append(opts)
    total = 1
    for opts in chan_opts:
        total *= len(opts)
    if total > limit:
        return None
    results = []
    for combo in itertools.product(*chan_opts):
        inst_of = {}
        for insts in combo:
            for inst in insts:
                for e in inst:
                    inst_of[e] = inst
        # happens-before graph over instances from each rank's program order
        adj = {}
        for r in range(W):
            seq = [inst_of[e] for e in range(int(tr.rank_offsets[r]), int(tr.rank_offsets[r + 1])) if kinds[e] != 0]
            for a, b in zip(seq, seq[1:]):
                adj.setdefault(a, set()).add(b)
        color = {}

        def cyclic(u):
            color[u] = 1
            for v in adj.get(u, ()):
                if color.get(v) == 1 or (v not in color and cyclic(v)):
                    return True
            color[u] = 2
            return False

        if not any(cyclic(u) for u in list(adj) if u not in color):
            results.append({frozenset(i) for insts in combo for i in insts})
    return results


@pytest.mark.parametrize("seed", range(40))
def test_bruteforce_unique_matching(seed):
    """P:L131 'a single pass ... matches': on a consistent trace exactly one order-consistent
    match set exists, and it is the oracle's."""
    rng = random.Random(seed)
    sols = None
    while sols is None:  # redraw traces whose enumeration space is too large
        tr = _random_tiny(rng)
        sols = _brute_force_matchings(tr)
    o = oracle.run(tr)
    assert o["status"] == 0 and o["n_incomplete"] == 0
    assert len(sols) == 1
    mine = groups_by(o["ev_inst"], (tr.kind_op & 7) != 0)
    assert mine == sols[0]


def test_truncated_trace_prefix_is_maximal():
    """unequal counts -> the oracle keeps the common prefix complete and reports the rest."""
    ranks = [[(AR, 0, 100, 0, 0, 0, 0)] * 3, [(AR, 0, 100, 0, 0, 0, 0)] * 2, [(AR, 0, 100, 0, 0, 0, 0)] * 3]
    tr = tg.from_events(3, 1, 1, [[0, 1, 2]], ranks)
    o = oracle.run(tr)
    assert o["status"] == 1 and o["n_incomplete"] == 1 and o["n_instances"] == 3
    assert list(o["in_npresent"]) == [3, 3, 2]
    assert [bool(f & F_VALID) for f in o["in_flags"]] == [True, True, False]


# ---------------------------------------------------------------- DES ground truth
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_partition_equals_ground_truth(seed):
    """matched instances equal the simulator's true instances exactly."""
    tr = tiny_gen(seed=seed, tp=2, pp=4, dp=2, layers=2, mb=6, iters=3)
    o = oracle.run(tr)
    comm = (tr.kind_op & 7) != 0
    assert o["status"] == 0
    assert groups_by(o["ev_inst"], comm) == groups_by(tr.gt_inst, comm)


def test_wait_closed_form_vs_true_clock():
    """A3 closed form: with no clock skew, the generator's hidden true clock gives
    wait_m = true_start(last arriver) - true_start(m), and dmin = end - last arrival."""
    tr = tiny_gen(seed=4, tp=2, pp=2, dp=2, layers=2, mb=4, iters=2, skew=False)
    o = oracle.run(tr)
    ev_rank = np.repeat(np.arange(tr.world), np.diff(tr.rank_offsets).astype(np.int64))
    comm = np.nonzero((tr.kind_op & 7) != 0)[0]
    by_inst = {}
    for e in comm:
        by_inst.setdefault(int(o["ev_inst"][e]), []).append(int(e))
    for i, evs in by_inst.items():
        assert o["in_flags"][i] & F_VALID
        starts = {int(ev_rank[e]): int(tr.gt_true_start[e]) for e in evs}
        last = int(o["in_last"][i])
        ends = {int(tr.gt_true_start[e]) + int(tr.dur_ns[e]) for e in evs}
        assert len(ends) == 1  # end-simultaneity holds in the DES
        for e in evs:
            assert o["ev_wait"][e] == starts[last] - int(tr.gt_true_start[e])
        assert o["in_dmin"][i] == ends.pop() - max(starts.values())


def test_decomposition_invariants():
    tr = tiny_gen(seed=5, tp=2, pp=2, dp=2, layers=2, mb=4, iters=3)
    o = oracle.run(tr)
    comm = np.nonzero((tr.kind_op & 7) != 0)[0]
    ev_rank = np.repeat(np.arange(tr.world), np.diff(tr.rank_offsets).astype(np.int64))
    tot = {}
    for e in comm:
        i = int(o["ev_inst"][e])
        if ev_rank[e] == o["in_last"][i]:
            assert o["ev_wait"][e] == 0  # wait_L = 0
        tot[i] = tot.get(i, 0) + int(tr.dur_ns[e]) - int(o["ev_wait"][e])
    for i, v in tot.items():  # sum_m (dur_m - wait_m) = |I| * dmin
        assert v == o["in_npresent"][i] * int(o["in_dmin"][i])
    # per-rank sums are the column sums
    for r in range(tr.world):
        sl = slice(int(tr.rank_offsets[r]), int(tr.rank_offsets[r + 1]))
        k = (tr.kind_op[sl] & 7)
        assert o["rk_sum_compute"][r] == int(tr.dur_ns[sl][k == 0].astype(np.uint64).sum())
        assert o["rk_sum_wait"][r] == int(o["ev_wait"][sl][k != 0].astype(np.uint64).sum())


def test_clock_skew_invariance():
    """Reading R5: the analysis is clock-free; the same trace with any per-rank offset/drift of
    start_ns gives byte-identical outputs (P:L118 local GPU clocks)."""
    tr = tiny_gen(seed=6, tp=2, pp=2, dp=2, layers=2, mb=4, iters=3, faults=[tg.Fault(tg.THROTTLE, 3, factor=2.0)])
    o1 = oracle.run(tr)
    rng = np.random.default_rng(0)
    offs = rng.integers(-2_000_000, 2_000_000, tr.world)
    ev_rank = np.repeat(np.arange(tr.world), np.diff(tr.rank_offsets).astype(np.int64))
    tr.start_ns = tr.start_ns + offs[ev_rank] + (tr.start_ns * 1e-5).astype(np.int64)
    o2 = oracle.run(tr)
    for k in o1:
        if isinstance(o1[k], np.ndarray):
            assert np.array_equal(o1[k], o2[k]), k
        else:
            assert o1[k] == o2[k], k


# ---------------------------------------------------------------- stage 1
def test_stage1_dp1_empty():
    """dp_size == 1 -> empty stats."""
    tr = dp_trace([[1000] * 20])
    o = oracle.run(tr)
    assert o["wd_total"].sum() == 0 and o["wd_cand"].sum() == 0


def test_stage1_one_of_four_at_2x():
    """4 DP peers, one rank's every kernel 2x median -> that rank's slow_fraction == 1.0."""
    base = [1_000_000 + 1000 * j for j in range(20)]
    durs = [base, base, [2 * x for x in base], base]
    o = oracle.run(dp_trace(durs, extra_comm=False))
    assert list(o["wd_frac"]) == [0.0, 0.0, 1.0, 0.0]
    assert list(o["wd_cand"]) == [0, 0, 1, 0]
    assert list(o["wd_total"]) == [20] * 4


def test_stage1_loo_median_closed_forms():
    """Leave-one-out lower median (reading R8/R15) in closed form: dp=2 -> the other peer;
    dp=3 -> the smaller of the other two; dp=4 -> the middle of the other three."""
    o = oracle.run(dp_trace([[100], [700]], extra_comm=False))
    assert list(o["ev_ref"]) == [700, 100]
    o = oracle.run(dp_trace([[100], [700], [400]], extra_comm=False))
    assert list(o["ev_ref"]) == [400, 100, 100]
    o = oracle.run(dp_trace([[100], [700], [400], [900]], extra_comm=False))
    assert list(o["ev_ref"]) == [700, 400, 700, 400]


def test_stage1_thresholds_exact():
    """slow iff dur > 1.5 ref AND dur - ref > 50 us, evaluated exactly at the edges."""
    ref = 200_000
    o = oracle.run(dp_trace([[ref], [300_000], [300_001]], extra_comm=False))  # dp=3: refs = min(other two)
    # rank1: 300000 vs ref 200000 -> 1.5x exactly: not slow; rank2: 300001 -> slow
    assert list(o["ev_slow"]) == [0, 0, 1]
    o = oracle.run(dp_trace([[80_000], [80_000], [120_001]], extra_comm=False))  # margin 40001 < 50 us
    assert list(o["ev_slow"]) == [0, 0, 0]


def test_stage1_op_mismatch_common_prefix():
    """S:L334 + reading R9: peers whose kernel sequences differ are compared on the common prefix."""
    ranks = [[(C, 1, 100), (C, 2, 100), (C, 3, 100)], [(C, 1, 100), (C, 5, 100), (C, 3, 100)]]
    tr = tg.from_events(1, 1, 2, [], ranks)
    o = oracle.run(tr)
    assert list(o["cl_J"]) == [1] and list(o["cl_mismatch"]) == [1]
    assert list(o["wd_total"]) == [1, 1]


def test_stage1_monotonicity():
    """increasing one event's duration never decreases its rank's slow count and never
    increases another rank's."""
    rng = np.random.default_rng(3)
    durs = [list(rng.integers(100_000, 200_000, 30)) for _ in range(5)]
    o1 = oracle.run(dp_trace(durs, extra_comm=False))
    for trial in range(20):
        r, j = int(rng.integers(5)), int(rng.integers(30))
        d2 = [list(x) for x in durs]
        d2[r][j] = int(d2[r][j]) + int(rng.integers(1, 400_000))
        o2 = oracle.run(dp_trace(d2, extra_comm=False))
        assert o2["wd_slow"][r] >= o1["wd_slow"][r]
        for q in range(5):
            if q != r:
                assert o2["wd_slow"][q] <= o1["wd_slow"][q]


def test_stage1_downclock_unique_candidate():
    """topo(2,2,2), rank 5 downclocked x1.8 -> rank 5 is the unique candidate."""
    tr = tiny_gen(seed=2, tp=2, pp=2, dp=2, layers=4, mb=8, iters=3, faults=[tg.Fault(tg.THROTTLE, 5, factor=1.8)])
    o = oracle.run(tr)
    assert list(np.nonzero(o["wd_cand"])[0]) == [5]


# ---------------------------------------------------------------- stage 2
def _tp_pair_trace(late_always: bool, n=20):
    """2 ranks in one TP group (dp=2 peers on other ranks make rank 0 a stage-1 candidate)."""
    # topology tp=2, dp=2: ranks 0,1 = TP group of dp0; ranks 2,3 = TP group of dp1
    comms = [[0, 1], [2, 3]]
    ranks = []
    for r in range(4):
        evs = []
        for j in range(n):
            slow = (r == 0)
            evs.append((C, 1, 2_000_000 if slow else 1_000_000))
            grp = 0 if r < 2 else 1
            if r == 0:
                d = 150_000 if late_always else 1_150_000
            elif r == 1:
                d = 1_150_000 if late_always else 150_000
            else:
                d = 150_000 + (r - 2) * 10
            evs.append((AR, 1, d, grp))
        ranks.append(evs)
    return tg.from_events(2, 1, 2, comms, ranks)


def test_stage2_latest_in_all():
    """candidate latest in all 20 of its TP allreduces by > margin -> fraction 1.0, root cause."""
    o = oracle.run(_tp_pair_trace(True))
    assert o["wd_cand"][0] == 1
    assert o["wl_joined"][0] == 20 and o["wl_late"][0] == 20 and o["wl_late_frac"][0] == 1.0
    assert o["wl_verdict"][0] == V_COMPUTE


def test_stage2_never_latest():
    """candidate never latest -> fraction 0, exonerated by this stage."""
    o = oracle.run(_tp_pair_trace(False))
    assert o["wd_cand"][0] == 1 and o["wl_late"][0] == 0
    assert o["wl_verdict"][0] == V_EXON


def test_stage2_insufficient():
    """candidate joins < min_samples collectives -> Insufficient, not exonerated."""
    o = oracle.run(_tp_pair_trace(True, n=10), oracle.Config(min_samples=10))
    assert o["wd_cand"][0] == 1 and o["wl_joined"][0] == 10 and o["wl_verdict"][0] == V_COMPUTE
    o = oracle.run(_tp_pair_trace(True, n=10), oracle.Config(min_samples=11))
    assert o["wd_cand"][0] == 0  # total_ops 10 < 11: not even a candidate


def test_stage2_downclock_fractions():
    """simulated downclock on rank 5 -> late_start_fraction(5) >= 0.7 while others < 0.3."""
    tr = tg.generate(configs.c1(seed=3))
    o = oracle.run(tr)
    lf = o["wl_late_frac"]
    assert lf[5] >= 0.7
    assert all(lf[r] < 0.3 for r in range(8) if r != 5)


# ---------------------------------------------------------------- stage 3
def test_stage3_degraded_link():
    """rank 2's egress link degraded x0.5 -> median warm-up bw on (2->3 stage) ~ 0.5x
    median of the other links, within 10%; LinkSlow flagged on exactly that link."""
    # pp=4, tp=1, dp=1 -> ranks are stages; rank 1 -> rank 2 degraded (a forward link)
    cfg = tg.GenConfig(1, 4, 1, 2, 12, 4, seed=7, faults=[tg.Fault(tg.LINK_DEGRADE, 1, 2, factor=0.5)])
    o = oracle.run(tg.generate(cfg))
    fwd = [i for i in range(len(o["lk_src"])) if o["lk_dir"][i] == 0]
    bw = {(int(o["lk_src"][i]), int(o["lk_dst"][i])): o["lk_med_bw"][i] for i in fwd}
    others = [v for k, v in bw.items() if k != (1, 2)]
    assert abs(bw[(1, 2)] / np.median(others) - 0.5) < 0.05
    slow = [(int(o["lk_src"][i]), int(o["lk_dst"][i])) for i in range(len(o["lk_src"])) if o["lk_slow"][i]]
    assert slow == [(1, 2)]
    assert o["wl_verdict"][1] == V_LINK


def test_stage3_warmup_rule():
    """Reading R13: warm-up samples are used when >= min_samples, else all samples."""
    cfg = tg.GenConfig(1, 4, 1, 2, 12, 4, seed=7)
    tr = tg.generate(cfg)
    o = oracle.run(tr)
    for i in range(len(o["lk_src"])):
        s = int(o["lk_src"][i])
        if o["lk_dir"][i] == 0:
            # warm-up sends per iteration on stage s: (PP-s-1) + 1 (first steady send) -> x4 iterations
            nw = (4 - s - 1 + 1) * 4
            assert o["lk_used_warm"][i] == (1 if nw >= 10 else 0)
            assert o["lk_n"][i] == (nw if nw >= 10 else 12 * 4)
        else:
            assert o["lk_used_warm"][i] == 0 and o["lk_n"][i] == 12 * 4


# ---------------------------------------------------------------- diagnose
@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_healthy_no_root_causes(seed):
    tr = tiny_gen(seed=seed, tp=2, pp=4, dp=2, layers=2, mb=8, iters=3)
    o = oracle.run(tr)
    assert o["wd_cand"].sum() == 0 and o["wl_verdict"].sum() == 0 and o["lk_slow"].sum() == 0
    assert set(o["lb_label"]) == {L_CLEAN}


@pytest.mark.parametrize("factor", [1.5, 2.0, 3.0])
def test_single_downclock_exactly_that_rank(factor):
    tr = tiny_gen(seed=11, tp=2, pp=4, dp=2, layers=3, mb=8, iters=3, faults=[tg.Fault(tg.THROTTLE, 9, factor=factor)])
    o = oracle.run(tr)
    roots = [r for r in range(16) if o["wl_verdict"][r] in (V_COMPUTE, V_BOTH)]
    assert roots == [9]
    assert o["lb_label"][9] == L_SRC_RANK
    assert all(o["lb_label"][r] in (L_VICTIM, L_CLEAN) for r in range(16) if r != 9)


def test_victim_exoneration_cascade():
    """S:L370 + C5 shape: collateral slowdown of the source's TP peers makes them stage-1
    candidates; stage 2 must exonerate them (they are victims, not sources)."""
    src = 8 + 0
    peers = [9, 10, 11]
    faults = [tg.Fault(tg.THROTTLE, src, factor=2.5)] + [tg.Fault(tg.THROTTLE, p, factor=1.8, prob=0.4) for p in peers]
    tr = tg.generate(tg.GenConfig(4, 2, 2, 4, 8, 4, seed=3, faults=faults))
    o = oracle.run(tr)
    assert o["wl_verdict"][src] == V_COMPUTE
    for p in peers:
        assert o["wd_cand"][p] == 1
        assert o["wl_verdict"][p] == V_EXON
        assert o["lb_label"][p] == L_VICTIM and o["lb_root_rank"][p] == src


def test_link_only():
    """injected link degrade only -> zero compute candidates, one LinkSlow rank."""
    cfg = tg.GenConfig(2, 4, 2, 2, 8, 4, seed=5, faults=[tg.Fault(tg.LINK_DEGRADE, 4, 8, factor=0.5)])
    o = oracle.run(tg.generate(cfg))
    assert o["wd_cand"].sum() == 0
    assert list(np.nonzero(o["wl_link_slow"])[0]) == [4]
    assert o["lb_label"][8] == L_SRC_LINK and o["lb_root_src"][8] == 4


# ---------------------------------------------------------------- walk (A7-A8; definition is ours)
def _chain_trace():
    """Hand-built chain: rank 0 slow (candidate via DP peer 3); rank 1 waits on 0 (comm A), rank 2
    waits on 1 (comm B). Topology tp=3, dp=2: ranks 0-2 TP group 0, ranks 3-5 TP group 1."""
    comms = [[0, 1], [1, 2], [0, 1, 2], [3, 4, 5]]
    n = 12
    ranks = [[] for _ in range(6)]
    for j in range(n):
        ranks[0] += [(C, 1, 2_000_000), (AR, 1, 150_000, 2), (AR, 1, 150_000, 0)]
        ranks[1] += [(C, 1, 1_000_000), (AR, 1, 1_150_000, 2), (AR, 1, 900_000, 0), (AR, 1, 150_000, 1)]
        ranks[2] += [(C, 1, 1_000_000), (AR, 1, 1_150_000, 2), (AR, 1, 700_000, 1)]
        for r in (3, 4, 5):
            ranks[r] += [(C, 1, 1_000_000), (AR, 1, 150_000 + r, 3)]
    return tg.from_events(3, 1, 2, comms, ranks)


def test_walk_chain_depths():
    o = oracle.run(_chain_trace())
    assert o["wl_verdict"][0] == V_COMPUTE
    assert list(o["lb_label"][:3]) == [L_SRC_RANK, L_VICTIM, L_VICTIM]
    assert list(o["lb_depth"][:3]) == [0, 1, 1]  # rank 2 also waits on 0 directly via comm 2
    assert list(o["lb_root_rank"][:3]) == [0, 0, 0]


def test_walk_two_level_chain():
    """A slow -> B waits on A -> C waits only on B => depths 1, 2."""
    comms = [[0, 1], [1, 2], [0, 3]]
    ranks = [[] for _ in range(4)]
    for j in range(12):
        ranks[0] += [(C, 1, 2_000_000), (AR, 1, 150_000, 0)]
        ranks[1] += [(C, 1, 1_000_000), (AR, 1, 1_150_000, 0), (AR, 1, 150_000, 1)]
        ranks[2] += [(C, 1, 1_000_000), (AR, 1, 500_000, 1)]
        ranks[3] += [(C, 1, 1_000_000)]
    # dp=2 pairs: (0,?) -> use tp=2, dp=2: ranks 0,1 dp0; ranks 2,3 dp1: peers (0,2), (1,3)
    tr = tg.from_events(2, 1, 2, comms, ranks)
    o = oracle.run(tr)
    assert o["wl_verdict"][0] == V_COMPUTE
    assert o["lb_label"][1] == L_VICTIM and o["lb_depth"][1] == 1
    assert o["lb_label"][2] == L_VICTIM and o["lb_depth"][2] == 2 and o["lb_root_rank"][2] == 0


def test_walk_cycle_unattributed():
    """Ranks that wait only on each other (a 2-cycle) and are not reachable from a root are
    UNATTRIBUTED when the window has a root, CLEAN when it has none."""
    comms = [[2, 3], [0, 1]]
    ranks = [[] for _ in range(4)]
    for j in range(12):
        ranks[0] += [(C, 1, 2_000_000), (AR, 1, 150_000, 1)]
        ranks[1] += [(C, 1, 1_000_000), (AR, 1, 1_150_000, 1)]
        w2, w3 = (400_000, 150_000) if j % 2 else (150_000, 400_000)
        ranks[2] += [(C, 1, 1_000_000), (AR, 1, w2, 0)]
        ranks[3] += [(C, 1, 1_000_000), (AR, 1, w3, 0)]
    tr = tg.from_events(2, 1, 2, comms, ranks)
    o = oracle.run(tr)
    assert o["wl_verdict"][0] == V_COMPUTE
    assert o["lb_label"][2] == L_UNATTR and o["lb_label"][3] == L_UNATTR
    # without the slow rank there is no root -> CLEAN
    ranks[0] = [(C, 1, 1_000_000) if e[0] == C else (AR, 1, 150_000, 1) for e in ranks[0]]
    ranks[1] = [(C, 1, 1_000_000) if e[0] == C else (AR, 1, 150_000, 1) for e in ranks[1]]
    o = oracle.run(tg.from_events(2, 1, 2, comms, ranks))
    assert set(o["lb_label"]) == {L_CLEAN}


# ---------------------------------------------------------------- windows
def test_windows_partial_fault():
    """Reading R18: a throttle on iterations [4,8) of 12 is found in windows 1 only (4-it windows)."""
    tr = tg.generate(tg.GenConfig(2, 2, 2, 3, 8, 12, seed=2, faults=[tg.Fault(tg.THROTTLE, 6, it0=4, it1=8, factor=2.0)]))
    o = oracle.run(tr, oracle.Config(window_iters=4))
    assert o["n_windows"] == 3
    v = o["wl_verdict"].reshape(3, 8)
    assert list(v[:, 6]) == [V_NONE, V_COMPUTE, V_NONE]
    assert v.sum() == V_COMPUTE


def test_schema_errors():
    tr = tg.from_events(2, 1, 1, [[0, 1]], [[(AR, 0, 1, 5)], [(AR, 0, 1, 0)]])
    o = oracle.run(tr)
    assert o["status"] == -2 and o["bad_event"] == 0
    tr = tg.from_events(2, 1, 1, [[0]], [[(AR, 0, 1, 0)], [(AR, 0, 1, 0)]])
    o = oracle.run(tr)
    assert o["status"] == -2 and o["bad_event"] == 1  # rank 1 not a member of comm 0
    tr = tg.from_events(2, 1, 1, [], [[(SEND, 0, 1, 0)], []])
    assert oracle.run(tr)["status"] == -2  # peer == self


# ---------------------------------------------------------------- round-2 pins: branches that only
# GPU-vs-oracle parity checked before (kind mismatch, stage2_mode=1, the pslow segment reset)
F_COMPLETE, F_KIND_OK, F_PAYLOAD_OK, F_VALID = 1, 2, 4, 8


def test_kind_mismatch_is_reported_and_excluded():
    """Reading R2 (occurrence counter per communicator) + S:L209 / S:L232: rank 0
    posts an AllReduce where rank 1 posts an AllGather at occurrence 0 of the same communicator.
    Hand-derived: two instances (k = 0, 1); k = 0 is complete but not kind-consistent, so it is
    reported (n_kind_mismatch = 1, status PARTIAL) and excluded from the decomposition (no waits,
    no transfer); k = 1 is a valid instance whose last arriver is rank 1 (duration 300 < 500)."""
    ag = tg.ALLGATHER
    ranks = [[(AR, 0, 700, 0), (AR, 0, 500, 0)],
             [(ag, 0, 400, 0), (AR, 0, 300, 0)]]
    o = oracle.run(tg.from_events(2, 1, 1, [[0, 1]], ranks))
    assert o["n_instances"] == 2 and o["n_kind_mismatch"] == 1 and o["n_incomplete"] == 0
    assert o["status"] == 1  # SCAN_PARTIAL: reported, never dropped
    f0, f1 = int(o["in_flags"][0]), int(o["in_flags"][1])
    assert f0 & F_COMPLETE and not f0 & F_KIND_OK and not f0 & F_VALID
    assert f1 & F_COMPLETE and f1 & F_KIND_OK and f1 & F_VALID
    assert list(o["ev_inst"]) == [0, 1, 0, 1]
    # waits: instance 0 excluded (0, 0); instance 1: dmin = 300 -> rank 0 waits 200, rank 1 waits 0
    assert list(o["ev_wait"]) == [0, 200, 0, 0]
    assert int(o["in_dmin"][1]) == 300 and int(o["in_dmax"][1]) == 500 and int(o["in_last"][1]) == 1
    assert list(o["rk_sum_wait"]) == [200, 0] and list(o["rk_sum_transfer"]) == [300, 300]


def _segment_trace(reps=10):
    """tp=2, pp=1, dp=2 (TP groups {0,1}, {2,3}; DP classes {0,2}, {1,3}). Rank 0 repeats three
    segments, each two compute ops then a TP all-reduce:
      A = [slow, fast, AR]  (slow op FIRST in the segment; rank 0 arrives last: late)
      B = [fast, fast, AR]  (no slow op;                  rank 1 arrives last)
      D = [fast, slow, AR]  (slow op LAST in the segment;  rank 0 arrives last: late)
    slow = 2 ms vs the DP peer's 1 ms (2 x 2 > 3 x 1 and 1 ms > 50 us: slow); fast = 1 ms.
    A late rank 0 has the shortest all-reduce duration (it arrived last, ends are simultaneous)."""
    S, F = 2_000_000, 1_000_000
    comms = [[0, 1], [2, 3]]
    ranks = [[] for _ in range(4)]
    for _ in range(reps):
        for seg in ("A", "B", "D"):
            c0 = {"A": (S, F), "B": (F, F), "D": (F, S)}[seg]
            late0 = seg != "B"
            ranks[0] += [(C, 1, c0[0]), (C, 2, c0[1]), (AR, 3, 150_000 if late0 else 160_000, 0)]
            ranks[1] += [(C, 1, F), (C, 2, F), (AR, 3, 1_150_000 if late0 else 150_000, 0)]
            for r in (2, 3):  # healthy TP group: equal durations, a tie -> nobody late (R20)
                ranks[r] += [(C, 1, F), (C, 2, F), (AR, 3, 150_000, 1)]
    return tg.from_events(2, 1, 2, comms, ranks)


def test_pslow_is_the_segment_or_reset_at_each_comm_event():
    """P:L149 "because its preceding computation is slower" (reading R11): pslow of a comm
    event = OR of the slow bits of the rank's compute ops since its previous comm event. Hand count
    over 10 x (A, B, D): stage 1 total 60, slow 20 (1/3 > 0.3: candidate). Stage 2 CONDITIONAL
    joins the A and D all-reduces only: joined 20, late 20 -> 1.0 -> ComputeSlow. A sticky pslow
    (no reset) would also join B (30 joined), and a last-op-only reading would miss A (10 joined)."""
    o = oracle.run(_segment_trace())
    assert o["wd_total"][0] == 60 and o["wd_slow"][0] == 20 and o["wd_cand"][0] == 1
    assert o["wl_joined"][0] == 20 and o["wl_late"][0] == 20
    assert o["wl_verdict"][0] == V_COMPUTE


def test_stage2_unconditional_mode():
    """S:L342 literal (stage2_mode = 1): every TP / DP instance a candidate joins counts, whatever
    preceded it. On the same trace: joined 30, late 20 -> 0.667 < 0.7 -> Exonerated. The
    CONDITIONAL default keeps the source (previous test)."""
    o = oracle.run(_segment_trace(), oracle.Config(stage2_mode=1))
    assert o["wd_cand"][0] == 1
    assert o["wl_joined"][0] == 30 and o["wl_late"][0] == 20
    assert abs(o["wl_late_frac"][0] - 20 / 30) < 1e-12
    assert o["wl_verdict"][0] == V_EXON
    # rank 1 (not a candidate) is the unique last arriver of the 10 B all-reduces, but its lag
    # 160 - 150 = 10 us is below the 100 us late margin: joined 30, late 0
    assert o["wl_joined"][1] == 30 and o["wl_late"][1] == 0
