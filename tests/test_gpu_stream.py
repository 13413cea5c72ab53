"""GPU parity of the sliding-window stream (NEXT-3, scan_stream_open / scan_stream_push), -m gpu:
after every pushed iteration, each window-level output equals the oracle run from scratch on the
window's events (the last K iterations, one analysis window). Integers / flags bit-exact, f64
reports within 1e-6 relative (as test_gpu_parity)."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from tracegen import configs

pytestmark = pytest.mark.gpu

FLOAT_KEYS = {"wd_frac", "wl_late_frac", "lk_med_bw"}


def _c5_small():
    cfg = configs.c5(iterations=6)
    cfg.faults = [tg.Fault(tg.THROTTLE, 208, it0=1, factor=2.5)] + [
        tg.Fault(tg.THROTTLE, p, it0=1, factor=1.8, prob=0.4) for p in range(209, 216)]
    return cfg


CASES = [
    ("c1_k4", lambda: configs.c1(seed=1), 4, 0, 10),
    ("c1_k3_mode1", lambda: configs.c1(seed=2, iterations=7), 3, 1, 5),
    ("c2_k3", lambda: configs.c2(seed=1, iterations=6), 3, 0, 10),
    ("c5_k3_cascade", _c5_small, 3, 0, 10),
    ("random_tp3_k2", lambda: tg.GenConfig(3, 2, 2, 2, 3, 6, seed=9, faults=[tg.Fault(tg.THROTTLE, 4, it0=2, factor=2.0)]), 2, 0, 3),
]


@pytest.mark.parametrize("name,mk,K,mode,mins", CASES, ids=[c[0] for c in CASES])
def test_stream_window_parity(name, mk, K, mode, mins):
    import paper_2507_19845_b200 as ms
    cfg = mk()
    full = tg.generate(cfg)
    s = ms.Scan(0)
    s.stream_open(full, K, ms.DetectConfig(min_samples=mins), ms.LocalizeConfig(stage2_mode=mode, min_samples=mins))
    for i in range(cfg.iterations):
        res = s.stream_push(ms.slice_iterations(full, i, i + 1))
        lo = max(0, i - K + 1)
        assert res["window"] == i + 1 - lo
        o = oracle.run(ms.slice_iterations(full, lo, i + 1), oracle.Config(stage2_mode=mode, min_samples=mins))
        bad = []
        for k in ms.Scan.STREAM_OUTPUTS:
            v, g = o[k], s.export(k)
            if g.shape != v.shape:
                bad.append(f"{k}: shape {g.shape} vs {v.shape}")
            elif k in FLOAT_KEYS:
                if not np.allclose(g, v, rtol=1e-6, atol=0):
                    bad.append(f"{k}: float diffs")
            elif not np.array_equal(g, v):
                j = np.nonzero(g != v)[0][:5]
                bad.append(f"{k}: {int((g != v).sum())} diffs at {j}: gpu {g[j]} oracle {v[j]}")
        assert not bad, f"push {i} (window {lo}..{i}):\n" + "\n".join(bad)
    s.close()


def test_stream_rejects_other_outputs_and_order():
    import paper_2507_19845_b200 as ms
    full = tg.generate(configs.c1(seed=1, iterations=2))
    s = ms.Scan(0)
    with pytest.raises(ms.ScanError):
        s.stream_push(ms.slice_iterations(full, 0, 1))  # before open
    s.stream_open(full, 2)
    s.stream_push(ms.slice_iterations(full, 0, 1))
    with pytest.raises(ms.ScanError):
        s.export("ev_inst")


@pytest.mark.parametrize("seed", range(401, 401 + int(__import__("os").environ.get("MS_STREAM_FUZZ_N", "8"))))
def test_stream_fuzz(seed):
    """Random SPMD jobs (TP, PP, DP in 1..3), window length, stage-2 mode and throttles: after every
    push the window-level outputs equal the oracle on the window."""
    import paper_2507_19845_b200 as ms
    rng = np.random.default_rng(seed)
    tp, pp, dp = (int(x) for x in rng.integers(1, 4, 3))
    if tp * pp * dp == 1:
        dp = 2
    W = tp * pp * dp
    iters = int(rng.integers(3, 7))
    faults = [tg.Fault(tg.THROTTLE, int(rng.integers(0, W)), it0=int(rng.integers(0, iters)), factor=float(rng.choice([1.8, 2.5])))]
    cfg = tg.GenConfig(tp, pp, dp, int(rng.integers(1, 3)), int(rng.integers(pp, pp + 3)), iters, seed=seed, faults=faults)
    full = tg.generate(cfg)
    K, mode, mins = int(rng.integers(1, 4)), int(rng.integers(0, 2)), int(rng.choice([3, 10]))
    s = ms.Scan(0)
    s.stream_open(full, K, ms.DetectConfig(min_samples=mins), ms.LocalizeConfig(stage2_mode=mode, min_samples=mins))
    for i in range(iters):
        s.stream_push(ms.slice_iterations(full, i, i + 1))
        lo = max(0, i - K + 1)
        o = oracle.run(ms.slice_iterations(full, lo, i + 1), oracle.Config(stage2_mode=mode, min_samples=mins))
        for k in ms.Scan.STREAM_OUTPUTS:
            v, g = o[k], s.export(k)
            assert g.shape == v.shape, (i, k)
            if k in FLOAT_KEYS:
                assert np.allclose(g, v, rtol=1e-6, atol=0), (i, k)
            else:
                assert np.array_equal(g, v), (i, k, np.nonzero(g != v)[0][:5])
    s.close()
