"""GPU parity of the event-level blame (NEXT-4, scan_blame) vs oracle.blame, -m gpu: the root of
every waiting event and the per-rank inflicted / self / unattributed / suffered waits bit-exact,
after both analysis paths (fused scan_analyze and the three-call general path)."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from tracegen import configs
from helpers import AR, C
from test_gpu_fuzz import _case

pytestmark = pytest.mark.gpu

KEYS = ("bl_root", "bl_inflicted", "bl_self", "bl_unattributed", "bl_suffered")


def _check(trace, path="fused", mins=10):
    import paper_2507_19845_b200 as ms
    o = oracle.blame(trace, oracle.Config(min_samples=mins))
    assert o["status"] >= 0
    s = ms.Scan(0)
    s.load(trace)
    d, l_ = ms.DetectConfig(min_samples=mins), ms.LocalizeConfig(min_samples=mins)
    if path == "fused":
        s.analyze(d, l_)
    else:
        s.run(d, l_)
    res = s.blame()
    for k in KEYS:
        g, v = s.export(k), o[k]
        assert g.shape == v.shape, k
        bad = np.nonzero(g != v)[0]
        assert len(bad) == 0, f"{k}: {len(bad)} diffs, first {bad[:5]}: gpu {g[bad[:5]]} oracle {v[bad[:5]]}"
    assert res["n_waiting"] == o["bl_n_waiting"] and res["n_cyclic"] == o["bl_n_cyclic"]
    assert res["total_wait_ns"] == int(o["bl_suffered"].sum())
    top = int(np.argmax(o["bl_inflicted"])) if o["bl_inflicted"].any() else 0xFFFFFFFF
    assert res["top_rank"] == top
    s.close()
    return res


HAND = {
    "chain": tg.from_events(1, 1, 3, [[0, 1], [1, 2]], [
        [(C, 0, 100), (AR, 0, 10, 0)],
        [(C, 0, 10), (AR, 0, 100, 0), (AR, 0, 10, 1)],
        [(C, 0, 10), (AR, 0, 200, 1)]]),
    "first_event": tg.from_events(1, 1, 2, [[0, 1]], [
        [(AR, 0, 50, 0), (C, 0, 30), (AR, 0, 5, 0), (AR, 0, 40, 0)],
        [(AR, 0, 10, 0), (AR, 0, 20, 0), (C, 0, 70), (AR, 0, 5, 0)]]),
    "cycle": tg.from_events(1, 1, 2, [[0, 1], [0, 1]], [
        [(AR, 0, 10, 0), (AR, 0, 2, 1)],
        [(AR, 0, 10, 1), (AR, 0, 2, 0)]]),
    "no_wait": tg.from_events(1, 1, 2, [[0, 1]], [[(C, 0, 10), (AR, 0, 5, 0)], [(C, 0, 10), (AR, 0, 5, 0)]]),
}


@pytest.mark.parametrize("path", ["fused", "general"])
@pytest.mark.parametrize("name", sorted(HAND))
def test_hand_cases(name, path):
    _check(HAND[name], path)


@pytest.mark.parametrize("path", ["fused", "general"])
def test_c1_throttle(path):
    res = _check(tg.generate(configs.c1(seed=3, iterations=6)), path)
    assert res["top_rank"] == 5  # c1's throttled rank


def test_c2_shape():
    _check(tg.generate(configs.c2(seed=2, iterations=3)))


def test_c5_shape():
    _check(tg.generate(configs.c5(seed=1, iterations=3)))


@pytest.mark.parametrize("seed", range(101, 101 + int(__import__("os").environ.get("MS_BLAME_FUZZ_N", "20"))))
def test_fuzz(seed):
    tr, wi, mode, mins = _case(seed)
    _check(tr, "fused" if seed % 2 else "general", mins)


def test_blame_requires_analysis_and_resets():
    import paper_2507_19845_b200 as ms
    s = ms.Scan(0)
    s.load(tg.generate(configs.c1(seed=1, iterations=2)))
    with pytest.raises(ms.ScanError):
        s.blame()
    s.analyze()
    s.blame()
    assert s.export("bl_inflicted").size == 8  # c1: 8 ranks
    s.analyze()  # a new analysis invalidates the blame outputs (size 0, as any output not computed)
    assert s.export("bl_inflicted").size == 0
    s.close()
