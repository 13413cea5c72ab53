"""Test helpers: hand-built traces and golden fixtures (no method arithmetic here)."""
from __future__ import annotations

import json
import os

import numpy as np

import tracegen as tg

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

C, AR, SEND, RECV = tg.COMPUTE, tg.ALLREDUCE, tg.SEND, tg.RECV


def load_golden(name: str) -> dict:
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def case_trace(case: dict) -> tg.Trace:
    tp, pp, dp = case["topo"]
    return tg.from_events(tp, pp, dp, case["comms"], [[tuple(e) for e in r] for r in case["ranks"]])


def tiny_gen(seed=1, tp=2, pp=2, dp=2, layers=2, mb=4, iters=3, faults=(), skew=True, jitter=0.05):
    return tg.generate(tg.GenConfig(tp, pp, dp, layers, mb, iters, seed=seed, faults=list(faults),
                                    clock_skew=skew, jitter=jitter), ground_truth=True)


def groups_by(ids: np.ndarray, mask: np.ndarray) -> set:
    """Partition of event indices (where mask) by the value of ids -> set of frozensets."""
    idx = np.nonzero(mask)[0]
    d: dict = {}
    for i in idx:
        d.setdefault(int(ids[i]), []).append(int(i))
    return {frozenset(v) for v in d.values()}


def dp_trace(durs_per_rank: list[list[int]], tp=1, pp=1, extra_comm=True):
    """DP-only trace: each rank runs the given compute durations; optional DP all-reduce after
    every compute op (so stage 2 has collectives to count)."""
    dp = len(durs_per_rank)
    comms = [list(range(dp))] if extra_comm else []
    ranks = []
    for r, durs in enumerate(durs_per_rank):
        evs = []
        for j, d in enumerate(durs):
            evs.append((C, j % 16, d, 0, 0, 0, 0))
            if extra_comm:
                evs.append((AR, 0, 1000, 0, 0, 0, 0))
        ranks.append(evs)
    return tg.from_events(tp, pp, dp, comms, ranks)
