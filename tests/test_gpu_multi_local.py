"""Sharded analysis on ONE GPU (-m gpu, row A9): G logical shards of the same job, each a sharded
context of an in-process group (scan_create_sharded_local), driven by one host thread each with its
own CUDA stream. The exchange layer (xch.cu) replaces NCCL by host barriers and device copies, so
every step of the sharded path (census, X1 / X2 numbering, the X3 regroup of P2P instance records to
the link owner, the X4 reduction, the stage-2 boundary fix-up and the replicated tail) runs exactly as
on G GPUs. The per-shard exports are reassembled (tests/shard_merge.py) and compared element by
element with the oracle run on the whole trace -- the same cases as tests/multigpu_parity.py."""
import os
import sys
import threading

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import oracle  # noqa: E402
import tracegen as tg  # noqa: E402
from shard_merge import coverage, merge  # noqa: E402
from multigpu_parity import CASES  # noqa: E402

pytestmark = pytest.mark.gpu


def _run_shards(G, cfg, wi, mode, mins, transform):
    import torch
    import paper_2507_19845_b200 as ms
    group = ms.LocalGroup(G)
    streams = [torch.cuda.Stream(0) for _ in range(G)]
    scans = [ms.Scan(0, streams[g].cuda_stream, shards=(G, g, group)) for g in range(G)]
    full = transform(tg.generate(cfg)) if transform is not None else None
    traces = []
    for g in range(G):
        b, e = ms.shard_iterations(cfg.iterations, G, g)
        traces.append(tg.generate(cfg, with_start=False, iter_range=(b, e)) if full is None else
                      ms.slice_iterations(full, b, e))
    d = ms.DetectConfig(window_iters=wi, want_ref=True, min_samples=mins)
    l_ = ms.LocalizeConfig(stage2_mode=mode, min_samples=mins)
    parts = [None] * G

    def work(g):
        part = {"ro": np.asarray(traces[g].rank_offsets), "err": None, "out": None, "res": None}
        try:
            scans[g].load(traces[g])
            part["res"] = scans[g].analyze(d, l_)
            out = scans[g].export_all()
            out["ch_shard_k0"] = scans[g].export("ch_shard_k0")
            out["ch_shard_n"] = scans[g].export("ch_shard_n")
            part["out"] = out
        except ms.ScanError as x:
            part["err"] = (x.status, str(x))
        parts[g] = part

    th = [threading.Thread(target=work, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a shard thread did not finish (exchange deadlock)"
    for s in scans:
        s.close()
    group.close()
    return parts, full


@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("case", CASES[:7] + CASES[7:10], ids=lambda c: c[0])
def test_local_shards_equal_the_oracle(G, case):
    name, mk, wi, mode, mins, transform, expect = case
    cfg = mk()
    if cfg.iterations < G:
        pytest.skip("fewer iterations than shards")
    parts, full = _run_shards(G, cfg, wi, mode, mins, transform)
    if expect is not None:
        errs = [p["err"] for p in parts]
        assert all(e is not None and e[0] == expect for e in errs), f"expected status {expect}, got {errs}"
        return
    errs = [p["err"] for p in parts if p["err"]]
    assert not errs, f"shard errors: {errs}"
    if full is None:
        full = tg.generate(cfg)
    o = oracle.run(full, oracle.Config(window_iters=wi, stage2_mode=mode, min_samples=mins))
    merged, issues = merge(parts)
    assert not issues, "\n".join(issues)
    cov = coverage(parts, int(o["n_instances"]))
    assert (cov == 1).all(), f"instance coverage: {np.unique(cov, return_counts=True)}"
    merged["_res"] = parts[0]["res"]
    from test_gpu_parity import compare
    compare(o, merged)


@pytest.mark.parametrize("G", [2, 3])
def test_local_shards_emit_merges_to_the_whole_document(G):
    """scan_emit_chrome on a sharded context writes the shard's own iteration block with job-wide
    instance ids; merged by (ts, pid, shard order) the shards' event lists are the whole job's document
    (one time-ordered merged trace)."""
    import json
    import torch
    import paper_2507_19845_b200 as ms
    from tracegen import configs
    cfg = configs.c2(iterations=6)
    full = tg.generate(cfg)
    group = ms.LocalGroup(G)
    streams = [torch.cuda.Stream(0) for _ in range(G)]
    scans = [ms.Scan(0, streams[g].cuda_stream, shards=(G, g, group)) for g in range(G)]
    slices = []
    for g in range(G):
        b, e = ms.shard_iterations(cfg.iterations, G, g)
        slices.append(ms.slice_iterations(full, b, e))
    docs, errs = [None] * G, []

    def work(g):
        try:
            scans[g].load(slices[g], start=True)
            scans[g].analyze()
            docs[g] = scans[g].emit_chrome()
        except ms.ScanError as x:
            errs.append((g, x.status, str(x)))

    th = [threading.Thread(target=work, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for s in scans:
        s.close()
    group.close()
    assert not errs, errs
    whole = ms.Scan(0)
    whole.load(full, start=True)
    whole.analyze()
    ref = json.loads(whole.emit_chrome())["traceEvents"]
    whole.close()
    merged = []
    for g, d in enumerate(docs):
        for i, ev in enumerate(json.loads(d)["traceEvents"]):
            merged.append(((ev["ts"], ev["pid"], g, i), ev))
    merged.sort(key=lambda x: x[0])
    assert len(merged) == len(ref)
    assert [ev for _, ev in merged] == ref


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("cfgname", ["c2", "c5"])
def test_local_shards_blame_equals_the_oracle(G, cfgname):
    """scan_blame on a sharded context (collective): chains that leave a shard's iteration block are
    resolved over the earlier shards' per-rank tables; per-rank sums are job-wide and each shard's
    BL_ROOT holds job-wide event ids for its own events -- merged, bit-exact against oracle.blame on
    the whole trace (EB1-EB6)."""
    import paper_2507_19845_b200 as ms
    import torch
    from tracegen import configs
    cfg = configs.c2(iterations=6) if cfgname == "c2" else configs.c5(iterations=6)
    full = tg.generate(cfg)
    o = oracle.blame(full, oracle.Config())
    group = ms.LocalGroup(G)
    streams = [torch.cuda.Stream(0) for _ in range(G)]
    scans = [ms.Scan(0, streams[g].cuda_stream, shards=(G, g, group)) for g in range(G)]
    slices = []
    for g in range(G):
        b, e = ms.shard_iterations(cfg.iterations, G, g)
        slices.append(ms.slice_iterations(full, b, e))
    outs, errs = [None] * G, []

    def work(g):
        try:
            scans[g].load(slices[g])
            scans[g].analyze()
            res = scans[g].blame()
            outs[g] = (res, {k: scans[g].export(k) for k in ("bl_root", "bl_inflicted", "bl_self", "bl_unattributed",
                                                               "bl_suffered")})
        except ms.ScanError as x:
            errs.append((g, x.status, str(x)))

    th = [threading.Thread(target=work, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for s in scans:
        s.close()
    group.close()
    assert not errs, errs
    for g in range(G):
        res, ex = outs[g]
        for k in ("bl_inflicted", "bl_self", "bl_unattributed", "bl_suffered"):
            assert np.array_equal(ex[k], o[k]), (g, k)
        assert res["n_waiting"] == o["bl_n_waiting"] and res["n_cyclic"] == o["bl_n_cyclic"]
        top = int(np.argmax(o["bl_inflicted"])) if o["bl_inflicted"].any() else 0xFFFFFFFF
        assert res["top_rank"] == top
    # job event order: rank-major, each rank's events shard after shard
    parts = []
    for r in range(full.world):
        for g in range(G):
            ro = np.asarray(slices[g].rank_offsets)
            parts.append(outs[g][1]["bl_root"][int(ro[r]):int(ro[r + 1])])
    root = np.concatenate(parts)
    bad = np.nonzero(root != o["bl_root"])[0]
    assert len(bad) == 0, f"bl_root: {len(bad)} diffs, first {bad[:5]}: gpu {root[bad[:5]]} oracle {o['bl_root'][bad[:5]]}"


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("cfgname,ref", [("c2", 0), ("c5", 0), ("c5", 77)])
def test_local_shards_align_equals_the_oracle(G, cfgname, ref):
    """scan_align on a sharded context (collective): BFS levels from the communicators valid on any
    shard, the anchor dedupe carried across shards, interpolation between the anchors of neighbouring
    shards; each shard's aligned starts merged in job order, and the job-wide levels, anchor counts and
    residuals, bit-exact against oracle.align on the whole trace (AL1-AL6)."""
    import paper_2507_19845_b200 as ms
    import torch
    from tracegen import configs
    cfg = configs.c2(iterations=6) if cfgname == "c2" else configs.c5(iterations=6)
    full = tg.generate(cfg)
    o = oracle.align(full, ref)
    assert o["al_status"] == 0
    group = ms.LocalGroup(G)
    streams = [torch.cuda.Stream(0) for _ in range(G)]
    scans = [ms.Scan(0, streams[g].cuda_stream, shards=(G, g, group)) for g in range(G)]
    slices = []
    for g in range(G):
        b, e = ms.shard_iterations(cfg.iterations, G, g)
        slices.append(ms.slice_iterations(full, b, e))
    outs, errs = [None] * G, []

    def work(g):
        try:
            scans[g].load(slices[g], start=True)
            scans[g].analyze()
            res = scans[g].align(ref)
            outs[g] = (res, {k: scans[g].export(k) for k in ms.ALIGN_OUTPUTS})
        except ms.ScanError as x:
            errs.append((g, x.status, str(x)))

    th = [threading.Thread(target=work, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for s in scans:
        s.close()
    group.close()
    assert not errs, errs
    for g in range(G):
        res, ex = outs[g]
        for k in ("al_level", "al_nanchor", "al_residual"):
            bad = np.nonzero(ex[k] != o[k])[0]
            assert len(bad) == 0, f"shard {g} {k}: {len(bad)} diffs, first {bad[:5]}: gpu {ex[k][bad[:5]]} oracle {o[k][bad[:5]]}"
        assert res["n_anchors"] == int(o["al_nanchor"].sum())
    parts = []
    for r in range(full.world):
        for g in range(G):
            ro = np.asarray(slices[g].rank_offsets)
            parts.append(outs[g][1]["al_start"][int(ro[r]):int(ro[r + 1])])
    st = np.concatenate(parts)
    bad = np.nonzero(st != o["al_start"])[0]
    assert len(bad) == 0, f"al_start: {len(bad)} diffs, first {bad[:5]}: gpu {st[bad[:5]]} oracle {o['al_start'][bad[:5]]}"
