"""GPU parity of the timeline alignment (NEXT-1, scan_align) vs the oracle, -m gpu: aligned start
of every event, BFS level, anchor count and residual of every rank, bit-exact (integer ns
arithmetic on both sides, readings AL1-AL6). Runs after both analysis paths (fused scan_analyze and
the three-call general path) and for two reference ranks."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from tracegen import configs
from helpers import AR, C, RECV, SEND

pytestmark = pytest.mark.gpu


def _gpu_align(trace, ref, path):
    import paper_2507_19845_b200 as ms
    s = ms.Scan(0)
    s.load(trace, start=True)
    if path == "fused":
        s.analyze()
    else:
        s.run()
    res = s.align(ref)
    out = {k: s.export(k) for k in ms.ALIGN_OUTPUTS}
    s.close()
    return res, out


def _check(trace, ref, path):
    o = oracle.align(trace, ref)
    assert o["al_status"] == 0
    res, g = _gpu_align(trace, ref, path)
    for k in ("al_start", "al_level", "al_nanchor", "al_residual"):
        v = o[k]
        assert g[k].shape == v.shape, k
        bad = np.nonzero(g[k] != v)[0]
        assert len(bad) == 0, f"{k}: {len(bad)} diffs, first {bad[:5]}: gpu {g[k][bad[:5]]} oracle {v[bad[:5]]}"
    assert res["n_anchors"] == int(o["al_nanchor"].sum())
    assert res["n_unaligned_ranks"] == int((o["al_level"] < 0).sum())
    assert res["max_residual_ns"] == int(o["al_residual"].max())


@pytest.mark.parametrize("path", ["fused", "general"])
@pytest.mark.parametrize("ref", [0, 5])
def test_c1_skew_drift(path, ref):
    _check(tg.generate(configs.c1(seed=5, iterations=6), ground_truth=True), ref, path)


@pytest.mark.parametrize("path", ["fused", "general"])
def test_c2_skew_drift(path):
    _check(tg.generate(configs.c2(seed=2, iterations=6)), 3, path)


def test_c5_shape():
    _check(tg.generate(configs.c5(seed=1, iterations=3)), 0, "fused")


def test_spec_examples_and_unreached():
    tr = tg.from_events(1, 1, 2, [[0, 1]], [[(C, 0, 1000), (AR, 0, 2000, 0)], [(C, 0, 1500), (AR, 0, 1500, 0)]])
    tr.start_ns[2:] += 500_000
    _check(tr, 0, "general")
    tr2 = tg.from_events(1, 1, 2, [], [[(C, 0, 10), (SEND, 0, 5, 1, 64)], [(C, 0, 12), (RECV, 0, 3, 0, 64)]])
    tr2.start_ns[2:] += 999
    _check(tr2, 0, "general")


def test_decreasing_ends_rejected():
    import paper_2507_19845_b200 as ms
    tr = tg.from_events(1, 1, 2, [[0, 1]], [[(AR, 0, 100, 0), (AR, 0, 100, 0)], [(AR, 0, 100, 0), (AR, 0, 100, 0)]])
    tr.start_ns[1] = tr.start_ns[0] - 500
    assert oracle.align(tr, 0)["al_status"] == -9
    s = ms.Scan(0)
    s.load(tr, start=True)
    s.run()
    with pytest.raises(ms.ScanError) as e:
        s.align(0)
    assert e.value.status == -8


def test_align_requires_start_and_analysis():
    import paper_2507_19845_b200 as ms
    tr = tg.generate(configs.c1(seed=1, iterations=2))
    s = ms.Scan(0)
    s.load(tr)  # no start_ns
    with pytest.raises(ms.ScanError):
        s.align(0)  # before analysis
    s.analyze()
    with pytest.raises(ms.ScanError):
        s.align(0)  # start_ns not loaded


@pytest.mark.parametrize("seed", range(201, 201 + int(__import__("os").environ.get("MS_ALIGN_FUZZ_N", "20"))))
def test_fuzz_alignment(seed):
    """Random small jobs (TP, PP, DP in 1..4) with clock skew + drift, random reference rank."""
    rng = np.random.default_rng(seed)
    tp, pp, dp = (int(x) for x in rng.integers(1, 5, 3))
    if tp * pp * dp == 1:
        dp = 2
    cfg = tg.GenConfig(tp, pp, dp, int(rng.integers(1, 4)), int(rng.integers(pp, pp + 4)), int(rng.integers(2, 6)), seed=seed,
                       faults=[tg.Fault(tg.THROTTLE, int(rng.integers(0, tp * pp * dp)), factor=2.0)])
    _check(tg.generate(cfg), int(rng.integers(0, tp * pp * dp)), "fused" if seed % 2 else "general")


@pytest.mark.parametrize("shift", [12, 29])
def test_extreme_drift_interpolation(shift):
    """One rank's clock runs 2^shift times fast: at 2^12 the offset change between anchors exceeds 2^31
    but stays below 2^50 (the kernels' 64-bit exact interpolation; the other tests run their 32-bit
    one), at 2^29 most intervals exceed 2^50 (their 128-bit fallback); every mode must equal the
    oracle's exact floor (AL4) to the nanosecond."""
    tr = tg.generate(configs.c1(seed=5, iterations=6))
    st = tr.start_ns.copy()
    r = 3
    a, b = int(tr.rank_offsets[r]), int(tr.rank_offsets[r + 1])
    st[a:b] = st[a:b] * (1 << shift) + 12345
    from dataclasses import replace
    _check(replace(tr, start_ns=st), 0, "fused")
