"""Randomised GPU parity (-m gpu): many small seeded jobs of the DES generator with random topology
(TP, PP, DP in 1..4, including non-powers of two), random throttles / link faults, random
window lengths and stage-2 modes, optionally truncated so the last iteration is ragged (incomplete
instances, class mismatches). Every case runs through scan_analyze (fused when SPMD, else general)
and through the three-call general path; every exported array must equal the oracle's."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from test_gpu_parity import compare

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(seed)
    tp, pp, dp = (int(x) for x in rng.integers(1, 5, 3))
    if tp * pp * dp == 1:
        dp = 2
    W = tp * pp * dp
    layers, mb, iters = int(rng.integers(1, 4)), int(rng.integers(max(pp, 1), pp + 4)), int(rng.integers(3, 9))
    faults = []
    for _ in range(int(rng.integers(0, 3))):
        faults.append(tg.Fault(tg.THROTTLE, int(rng.integers(0, W)), it0=int(rng.integers(0, iters)),
                               factor=float(rng.choice([1.6, 2.0, 3.0])), prob=float(rng.choice([1.0, 0.5]))))
    if pp > 1 and rng.random() < 0.5:
        s = int(rng.integers(0, pp - 1))
        src = int(rng.integers(0, tp)) + tp * (int(rng.integers(0, dp)) + dp * s)
        faults.append(tg.Fault(tg.LINK_DEGRADE, src, src + tp * dp, factor=0.3))
    cfg = tg.GenConfig(tp, pp, dp, layers, mb, iters, seed=seed, faults=faults)
    tr = tg.generate(cfg)
    if rng.random() < 0.3:  # truncate a few ranks' tails: ragged last iteration
        from dataclasses import replace
        keep = np.ones(tr.n_events, bool)
        ro = tr.rank_offsets.astype(np.int64).copy()
        for r in rng.choice(W, size=min(W, 2), replace=False):
            cut = int(rng.integers(1, 6))
            keep[ro[r + 1] - cut:ro[r + 1]] = False
        nro = np.zeros(W + 1, np.uint64)
        for r in range(W):
            nro[r + 1] = nro[r] + keep[ro[r]:ro[r + 1]].sum()
        tr = replace(tr, rank_offsets=nro, gt_inst=None, gt_true_start=None,
                     **{k: getattr(tr, k)[keep] for k in ("start_ns", "dur_ns", "kind_op", "meta", "comm", "payload")})
    wi = int(rng.choice([0, 0, 2, 3]))
    mode = int(rng.integers(0, 2))
    mins = int(rng.choice([3, 10]))
    return tr, wi, mode, mins


@pytest.mark.parametrize("seed", range(101, 101 + int(__import__("os").environ.get("MS_FUZZ_N", "60"))))
def test_fuzz(seed):
    import paper_2507_19845_b200 as ms
    tr, wi, mode, mins = _case(seed)
    o = oracle.run(tr, oracle.Config(window_iters=wi, stage2_mode=mode, min_samples=mins))
    d = ms.DetectConfig(window_iters=wi, want_ref=True, min_samples=mins)
    l_ = ms.LocalizeConfig(stage2_mode=mode, min_samples=mins)
    for path in ("analyze", "separate"):
        s = ms.Scan(0)
        s.load(tr)
        res = s.analyze(d, l_) if path == "analyze" else s.run(d, l_)
        g = s.export_all()
        g["_res"] = res
        s.close()
        compare(o, g)
