"""Host side of the multi-GPU path (row A9), CPU only: iteration slicing, the shard plan, the NCCL
id broadcast, and the premises the shard exchange rests on, checked with the ORACLE on each slice
in a world_size-2 gloo job (no GPU):
  * per-shard channel counts add up to the job-wide counts (X1/X2 numbering),
  * a shard-local instance id maps to the job-wide one as base(c) + pre_s(c) + k (no instance
    straddles an iteration block),
  * per-rank sums and wait-for edge weights are additive over shards (X4 all-reduce).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2507_19845_b200 as ms
import tracegen as tg
from tracegen import configs

from shard_merge import merge


def test_iteration_range_generator_matches_full_trace():
    for cfg in (configs.c1(seed=3, iterations=7), configs.c2(seed=2, iterations=6)):
        full = tg.generate(cfg, with_start=False)
        for b, e in ((0, 2), (2, 5), (5, cfg.iterations)):
            part = tg.generate(cfg, with_start=False, iter_range=(b, e))
            ref = ms.slice_iterations(full, b, e)
            for k in ("dur_ns", "kind_op", "meta", "comm", "payload"):
                assert np.array_equal(getattr(part, k), getattr(ref, k)), (k, b, e)
            assert np.array_equal(part.rank_offsets, ref.rank_offsets)


def test_shard_iterations_partition():
    for n in (1, 7, 10, 1000):
        for g in (1, 2, 3, 8):
            blocks = [ms.shard_iterations(n, g, s) for s in range(g)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(g - 1))
            sz = [e - b for b, e in blocks]
            assert max(sz) - min(sz) <= 1


def test_slice_iterations_handles_partial_tail():
    cfg = configs.c1(seed=1, iterations=4)
    full = tg.generate(cfg, with_start=False)
    # drop the last 5 events of rank 2: its last iteration is partial
    keep = np.ones(full.n_events, bool)
    keep[int(full.rank_offsets[3]) - 5:int(full.rank_offsets[3])] = False
    ro = full.rank_offsets.copy()
    ro[3:] -= 5
    from dataclasses import replace
    t = replace(full, rank_offsets=ro, **{k: getattr(full, k)[keep] for k in ("dur_ns", "kind_op", "meta", "comm", "payload")})
    a, b = ms.slice_iterations(t, 0, 3), ms.slice_iterations(t, 3, 4)
    assert a.n_events + b.n_events == t.n_events
    assert int(b.rank_offsets[3] - b.rank_offsets[2]) == int(full.rank_offsets[3] - full.rank_offsets[2]) // 4 - 5


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = ms.shard_unique_id()
        cfg = configs.c1(seed=7, iterations=9)
        b, e = ms.shard_iterations(cfg.iterations, world, rank)
        tr = tg.generate(cfg, with_start=False, iter_range=(b, e))
        o = oracle.run(tr, oracle.Config())
        keep = ("ch_kind", "ch_a", "ch_b", "ch_nmax", "ch_base", "ev_inst", "ev_wait", "rk_sum_compute", "rk_sum_wait",
                "rk_sum_transfer", "eg_window", "eg_src", "eg_dst", "eg_weight", "in_dmin", "in_dmax", "in_last")
        part = {"uid": uid, "ro": np.asarray(tr.rank_offsets), "o": {k: o[k] for k in keep}}
        parts = [None] * world if rank == 0 else None
        dist.gather_object(part, parts, dst=0)
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_two_shards_premises():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    # one NCCL id broadcast to every rank
    assert len(parts[0]["uid"]) == 128 and all(p["uid"] == parts[0]["uid"] for p in parts)
    full = tg.generate(configs.c1(seed=7, iterations=9), with_start=False)
    of = oracle.run(full, oracle.Config())
    # identical channel lists; counts add up
    for k in ("ch_kind", "ch_a", "ch_b"):
        assert all(np.array_equal(p["o"][k], of[k]) for p in parts), k
    assert np.array_equal(sum(p["o"]["ch_nmax"].astype(np.int64) for p in parts), of["ch_nmax"].astype(np.int64))
    # shard-local instance id -> job-wide id = base(c) + pre_s(c) + k
    pre = np.zeros_like(of["ch_nmax"], dtype=np.int64)
    W = full.world
    for s, p in enumerate(parts):
        loc_base = p["o"]["ch_base"].astype(np.int64)
        ev = p["o"]["ev_inst"].astype(np.int64)
        comm = ev != np.iinfo(np.uint32).max
        ch = np.searchsorted(loc_base, ev[comm], side="right") - 1
        gid = of["ch_base"].astype(np.int64)[ch] + pre[ch] + (ev[comm] - loc_base[ch])
        # the same events in the full trace
        idx = np.concatenate([np.arange(int(full.rank_offsets[r]) + sum(int(q["ro"][r + 1] - q["ro"][r]) for q in parts[:s]),
                                        int(full.rank_offsets[r]) + sum(int(q["ro"][r + 1] - q["ro"][r]) for q in parts[:s + 1]))
                              for r in range(W)])
        assert np.array_equal(gid, of["ev_inst"][idx][comm].astype(np.int64))
        assert np.array_equal(p["o"]["ev_wait"], of["ev_wait"][idx])
        pre += p["o"]["ch_nmax"].astype(np.int64)
    # additive per-rank sums and wait-for edges
    for k in ("rk_sum_compute", "rk_sum_wait", "rk_sum_transfer"):
        assert np.array_equal(sum(p["o"][k] for p in parts), of[k]), k
    def edges(o):
        d = {}
        for s_, t_, w_ in zip(o["eg_src"], o["eg_dst"], o["eg_weight"]):
            d[(int(s_), int(t_))] = d.get((int(s_), int(t_)), 0) + int(w_)
        return d
    tot = {}
    for p in parts:
        for key, v in edges(p["o"]).items():
            tot[key] = tot.get(key, 0) + v
    assert tot == edges(of)
    # the test merge helper reassembles event order
    fake = [{"out": {"ev_inst": p["o"]["ev_inst"], "ch_base": of["ch_base"], "ch_shard_k0": np.zeros(1, np.uint64),
                     "ch_shard_n": np.zeros(1, np.uint32)}, "ro": p["ro"], "res": {"status": 0, "match": {}, "detect": {}, "localize": {}}}
            for p in parts]
    merged, issues = merge(fake)
    assert len(merged["ev_inst"]) == full.n_events

