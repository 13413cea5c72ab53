"""Developer check: scan_analyze on a list of shapes against the oracle, naming the fused kernel that
ran (k_stage / k_fused); exits non-zero on the first difference. `python scripts/dev_check.py [names]`."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import tracegen as tg  # noqa: E402
from tracegen import configs  # noqa: E402
import paper_2507_19845_b200 as ms  # noqa: E402

FLOAT = {"wd_frac", "wl_late_frac", "lk_med_bw"}


def c5w():
    cfg = configs.c5(iterations=8)
    cfg.faults = [tg.Fault(tg.THROTTLE, 208, it0=2, factor=2.5)] + [
        tg.Fault(tg.THROTTLE, p, it0=2, factor=1.8, prob=0.4) for p in range(209, 216)]
    return tg.generate(cfg)


CASES = {
    "c2": (lambda: tg.generate(configs.c2(iterations=12)), {}),
    "c3": (lambda: tg.generate(configs.c3(iterations=4)), {}),
    "c3w": (lambda: tg.generate(configs.c3(iterations=4)), {"window_iters": 2, "want_ref": True}),
    "c3m1": (lambda: tg.generate(configs.c3(iterations=4)), {"mode": 1}),
    "c4": (lambda: tg.generate(configs.c4(iterations=3)), {"min_samples": 5}),
    "c5w": (c5w, {"window_iters": 4}),
    "tp4dp8": (lambda: tg.generate(tg.GenConfig(4, 4, 8, 2, 8, 4, seed=3, faults=[tg.Fault(tg.THROTTLE, 37, factor=2.0)])), {}),
    "tp2dp6": (lambda: tg.generate(tg.GenConfig(2, 4, 6, 2, 8, 4, seed=4, faults=[tg.Fault(tg.THROTTLE, 13, factor=2.5)])), {"window_iters": 1}),
    "tp8dp16w1": (lambda: tg.generate(configs.c3(iterations=3)), {"window_iters": 1, "want_ref": True}),
}


def run(name):
    mk, kw = CASES[name]
    tr = mk()
    d = ms.DetectConfig(window_iters=kw.get("window_iters", 0), want_ref=kw.get("want_ref", True), min_samples=kw.get("min_samples", 10))
    l_ = ms.LocalizeConfig(stage2_mode=kw.get("mode", 0), min_samples=kw.get("min_samples", 10))
    oc = oracle.Config(window_iters=kw.get("window_iters", 0), stage2_mode=kw.get("mode", 0), min_samples=kw.get("min_samples", 10))
    t0 = time.time()
    o = oracle.run(tr, oc)
    t1 = time.time()
    s = ms.Scan(0)
    s.load(tr)
    s.analyze(d, l_)  # first call: lazy module loading
    s.set_timing(True)
    res = s.analyze(d, l_)
    kt = s.kernel_timing()
    g = s.export_all()
    s.close()
    bad = []
    for k, v in o.items():
        if not isinstance(v, np.ndarray):
            continue
        if k == "ev_ref" and not kw.get("want_ref", True):
            continue
        gv = g[k]
        if gv.shape != v.shape:
            bad.append(f"{k}: shape {gv.shape} vs {v.shape}")
        elif k in FLOAT:
            if not np.allclose(gv, v, rtol=1e-6, atol=0):
                bad.append(f"{k}: float diffs")
        elif not np.array_equal(gv, v):
            i = np.nonzero(gv != v)[0][:6]
            bad.append(f"{k}: {int((gv != v).sum())} diffs at {i}: gpu {gv[i]} oracle {v[i]}")
    for k in ("n_instances", "n_incomplete", "n_kind_mismatch", "n_payload_mismatch"):
        if res["match"][k] != o[k]:
            bad.append(f"{k}: {res['match'][k]} vs {o[k]}")
    kern = "k_stage" if "k_stage" in kt else ("k_fused" if "k_fused" in kt else "general")
    ms_k = kt.get(kern, (0, 1))[0]
    print(f"{name}: {tr.n_events} events fused={res['fused']} kernel={kern} {ms_k:.3f} ms, oracle {t1 - t0:.1f} s -> "
          f"{'OK' if not bad else 'FAIL'}", flush=True)
    for b in bad:
        print("   ", b, flush=True)
    return not bad


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    ok = True
    for n in names:
        ok &= run(n)
    sys.exit(0 if ok else 1)
