"""Multi-GPU parity (row A9), launched by tests/test_gpu_multi.py as
    torchrun --nproc-per-node N tests/multigpu_parity.py
Every rank analyses its iteration block of the same seeded trace through ONE sharded context
(scan_create_sharded + scan_analyze, NCCL exchange); rank 0 gathers the per-shard exports (over a
gloo side group), reassembles them (tests/shard_merge.py) and compares them element by element
with the oracle run on the whole trace. Exit code 0 iff every case passes."""
from __future__ import annotations

import os
import sys
import traceback

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import paper_2507_19845_b200 as ms  # noqa: E402
import tracegen as tg  # noqa: E402
from tracegen import configs  # noqa: E402
from shard_merge import coverage, merge  # noqa: E402


def _c5():
    cfg = configs.c5(iterations=8)
    cfg.faults = [tg.Fault(tg.THROTTLE, 208, it0=2, factor=2.5)] + [
        tg.Fault(tg.THROTTLE, p, it0=2, factor=1.8, prob=0.4) for p in range(209, 216)]
    return cfg


def _drop_event(trace, rank, pos):
    """Full trace with event `pos` of `rank` removed (breaks shard regularity)."""
    keep = np.ones(trace.n_events, bool)
    keep[int(trace.rank_offsets[rank]) + pos] = False
    ro = trace.rank_offsets.copy()
    ro[rank + 1:] -= 1
    from dataclasses import replace
    cols = {k: getattr(trace, k)[keep] for k in ("start_ns", "dur_ns", "kind_op", "meta", "comm", "payload")}
    return replace(trace, rank_offsets=ro, gt_inst=None, gt_true_start=None, **cols)


# name, generator config, window_iters, stage2 mode, min_samples, full-trace transform, expected error
CASES = [
    ("c1_default", lambda: configs.c1(seed=1), 0, 0, 10, None, None),
    ("c1_windows3", lambda: configs.c1(seed=2), 3, 0, 10, None, None),
    ("c1_mode1_windows4", lambda: configs.c1(seed=3), 4, 1, 10, None, None),
    ("c1_uneven_9it_windows7", lambda: configs.c1(seed=4, iterations=9), 7, 0, 5, None, None),
    ("c2_24it_windows5", lambda: configs.c2(seed=1, iterations=24), 5, 0, 10, None, None),
    ("c5_cascade_windows4", _c5, 4, 0, 10, None, None),
    ("irregular_first_shard", lambda: configs.c1(seed=5), 0, 0, 10, lambda t: _drop_event(t, 1, 3), -8),  # SCAN_E_UNSUPPORTED
]


def _random_cfg(seed):
    rng = np.random.default_rng(seed)
    tp, pp, dp = (int(x) for x in rng.integers(1, 5, 3))
    if tp * pp * dp == 1:
        dp = 2
    W = tp * pp * dp
    faults = [tg.Fault(tg.THROTTLE, int(rng.integers(0, W)), it0=int(rng.integers(0, 6)), factor=2.0)]
    if pp > 1:
        faults.append(tg.Fault(tg.LINK_DEGRADE, 0, tp * dp, factor=0.3))
    return tg.GenConfig(tp, pp, dp, int(rng.integers(1, 4)), int(rng.integers(pp, pp + 4)), int(rng.integers(8, 13)),
                        seed=seed, faults=faults)


# random SPMD jobs (TP, PP, DP in 1..4), random windows / stage-2 mode / min samples
CASES += [(f"random_{sd}", (lambda sd=sd: _random_cfg(sd)), int([0, 2, 3, 5][sd % 4]), sd % 2, [3, 10][sd % 2], None, None)
          for sd in range(301, 301 + int(os.environ.get("MS_MULTI_FUZZ_N", "10")))]


def main() -> int:
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    gl = dist.new_group(backend="gloo")
    s = ms.Scan(local, shards=(world, rank, ms.shard_unique_id()))
    failures = []
    for name, mk, wi, mode, mins, transform, expect in CASES:
        cfg = mk()
        full = None
        if transform is None:
            b, e = ms.shard_iterations(cfg.iterations, world, rank)
            tr = tg.generate(cfg, with_start=False, iter_range=(b, e))
        else:
            full = transform(tg.generate(cfg))
            tr = ms.slice_iterations(full, *ms.shard_iterations(cfg.iterations, world, rank))
        d = ms.DetectConfig(window_iters=wi, want_ref=True, min_samples=mins)
        l_ = ms.LocalizeConfig(stage2_mode=mode, min_samples=mins)
        part = {"ro": np.asarray(tr.rank_offsets), "err": None, "out": None, "res": None}
        try:
            s.load(tr)
            part["res"] = s.analyze(d, l_)
            out = s.export_all()
            out["ch_shard_k0"] = s.export("ch_shard_k0")
            out["ch_shard_n"] = s.export("ch_shard_n")
            part["out"] = out
        except ms.ScanError as x:
            part["err"] = (x.status, str(x))
        parts = [None] * world if rank == 0 else None
        dist.gather_object(part, parts, dst=0, group=gl)
        if rank == 0:
            try:
                if expect is not None:
                    errs = [p["err"] for p in parts]
                    assert all(e_ is not None and e_[0] == expect for e_ in errs), f"expected status {expect}, got {errs}"
                else:
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
                print(f"[multigpu x{world}] {name}: ok", flush=True)
            except Exception:
                failures.append(name)
                print(f"[multigpu x{world}] {name}: FAIL\n{traceback.format_exc()}", flush=True)
        dist.barrier(group=gl)
    s.close()
    flag = [len(failures)]
    dist.broadcast_object_list(flag, src=0, group=gl)
    dist.destroy_process_group()
    return 1 if flag[0] else 0


if __name__ == "__main__":
    sys.exit(main())
