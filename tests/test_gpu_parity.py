"""GPU parity (-m gpu): the CUDA path through the C ABI vs the oracle, element by element, on the
same seeded inputs. Integer / index / flag outputs bit-exact; f64 reports within 1e-6 relative
(BASELINE.json north_star). Sizes span many warp tiles (2048 events) and ragged tails."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from tracegen import configs
from helpers import AR, C, RECV, SEND, case_trace, load_golden

pytestmark = pytest.mark.gpu

FLOAT_KEYS = {"wd_frac", "wl_late_frac", "lk_med_bw"}
SKIP_KEYS = set()


MODE = {"mode": "analyze"}


@pytest.fixture(params=["analyze", "separate"], autouse=True)
def _mode(request):
    """Every parity case runs twice: through scan_analyze (fused SPMD stage-tile pass when the trace
    is SPMD, else the general path) and through scan_match_collectives + scan_detect + scan_localize
    (general path)."""
    MODE["mode"] = request.param
    yield


def _gpu(trace, dcfg=None, lcfg=None, device_ptrs=False):
    import paper_2507_19845_b200 as ms
    s = ms.Scan(0)
    if device_ptrs:
        import torch
        cols = {k: torch.from_numpy(np.ascontiguousarray(getattr(trace, k)).view(np.int16 if getattr(trace, k).dtype == np.uint16 else np.int32)).cuda()
                for k in ("dur_ns", "kind_op", "meta", "comm", "payload")}
        s.load(trace, device_ptrs=True, cols=cols)
    else:
        s.load(trace)
    if MODE["mode"] == "analyze":
        res = s.analyze(dcfg, lcfg)
    else:
        res = s.run(dcfg, lcfg)
        res["fused"] = False
    out = s.export_all()
    out["_res"] = res
    s.close()
    return out


def _cfgs(window_iters=0, want_ref=True, mode=0, min_samples=10):
    import paper_2507_19845_b200 as ms
    d = ms.DetectConfig(window_iters=window_iters, want_ref=want_ref, min_samples=min_samples)
    l_ = ms.LocalizeConfig(stage2_mode=mode, min_samples=min_samples)
    o = oracle.Config(window_iters=window_iters, stage2_mode=mode, min_samples=min_samples)
    return d, l_, o


def compare(o, g):
    res = g["_res"]
    assert res["status"] == o["status"]
    m = res["match"]
    assert m["n_instances"] == o["n_instances"]
    assert m["n_incomplete"] == o["n_incomplete"]
    assert m["n_kind_mismatch"] == o["n_kind_mismatch"]
    assert m["n_payload_mismatch"] == o["n_payload_mismatch"]
    assert m["n_channels"] == o["n_channels"]
    assert res["detect"]["n_windows"] == o["n_windows"]
    bad = []
    for k, v in o.items():
        if not isinstance(v, np.ndarray) or k in SKIP_KEYS:
            continue
        gv = g[k]
        if gv.shape != v.shape:
            bad.append(f"{k}: shape {gv.shape} vs oracle {v.shape}")
            continue
        if k in FLOAT_KEYS:
            if not np.allclose(gv, v, rtol=1e-6, atol=0):
                i = np.nonzero(~np.isclose(gv, v, rtol=1e-6, atol=0))[0][:5]
                bad.append(f"{k}: first diffs at {i}: gpu {gv[i]} oracle {v[i]}")
        elif not np.array_equal(gv, v):
            i = np.nonzero(gv != v)[0][:5]
            bad.append(f"{k}: {int((gv != v).sum())} diffs, first at {i}: gpu {gv[i]} oracle {v[i]}")
    assert not bad, "\n".join(bad)


def _run_both(tr, **kw):
    d, l_, oc = _cfgs(**kw)
    o = oracle.run(tr, oc)
    g = _gpu(tr, d, l_)
    return o, g


@pytest.mark.parametrize("seed", [1, 2])
def test_c1_full(seed):
    """configs[0]: 8-rank TP2xPP2xDP2, 10 iterations, throttled rank 5 (111,280 events, 55 tiles)."""
    o, g = _run_both(tg.generate(configs.c1(seed=seed)))
    compare(o, g)
    assert list(np.nonzero(g["wl_verdict"])[0]) == [5]
    assert g["_res"]["fused"] == (MODE["mode"] == "analyze")


def test_c2_short():
    """configs[1] shape (64 ranks TP8xPP4xDP2, jittered links) on 12 iterations."""
    o, g = _run_both(tg.generate(configs.c2(iterations=12)))
    compare(o, g)
    assert g["_res"]["fused"] == (MODE["mode"] == "analyze")


def test_c5_windows_cascade():
    """configs[4] shape: 512 ranks TP8xPP8xDP8, cascading victims; 4-iteration windows."""
    cfg = configs.c5(iterations=8)
    cfg.faults = [tg.Fault(tg.THROTTLE, 208, it0=2, factor=2.5)] + [
        tg.Fault(tg.THROTTLE, p, it0=2, factor=1.8, prob=0.4) for p in range(209, 216)]
    o, g = _run_both(tg.generate(cfg), window_iters=4)
    compare(o, g)


@pytest.mark.parametrize("mode", [0, 1])
def test_stage2_modes_windows(mode):
    tr = tg.generate(tg.GenConfig(2, 4, 2, 2, 8, 9, seed=3, faults=[tg.Fault(tg.THROTTLE, 9, it0=3, it1=7, factor=2.0),
                                                                    tg.Fault(tg.LINK_DEGRADE, 4, 8, factor=0.5)]))
    o, g = _run_both(tr, window_iters=3, mode=mode, min_samples=4)
    compare(o, g)


@pytest.mark.parametrize("case", load_golden("spec_examples.json")["cases"], ids=lambda c: c["name"])
def test_spec_cases(case):
    o, g = _run_both(case_trace(case))
    compare(o, g)


def test_ragged_and_corrupt():
    """Ragged per-rank lengths, an incomplete instance, a payload mismatch, a kind mismatch,
    ranks with no events, compute-only ranks."""
    rng = np.random.default_rng(5)
    W = 6
    comms = [[0, 1, 2], [3, 4], [0, 5]]
    ranks = [[] for _ in range(W)]
    for it in range(300):
        for r in (0, 1, 2):
            ranks[r].append((C, 1, int(rng.integers(1000, 900000))))
            ranks[r].append((AR if not (it == 7 and r == 1) else tg.ALLGATHER, 0, int(rng.integers(1, 500000)), 0))
        ranks[3].append((C, 2, int(rng.integers(1000, 900000))))
        ranks[3].append((SEND, 0, int(rng.integers(1, 300000)), 4, 4096 if it != 11 else 8))
        ranks[4].append((RECV, 0, int(rng.integers(1, 300000)), 3, 4096))
        if it % 3 == 0:
            ranks[0].append((AR, 0, int(rng.integers(1, 300000)), 2))
            ranks[5].append((AR, 0, int(rng.integers(1, 300000)), 2, 0, 0, it % 7 == 0))
    ranks[2].append((AR, 0, 5, 0))  # one extra -> incomplete instance
    tr = tg.from_events(6, 1, 1, comms, ranks)
    o, g = _run_both(tr)
    assert o["status"] == 1
    compare(o, g)
    assert not g["_res"]["fused"]  # not SPMD: scan_analyze falls back to the general path


def test_schema_error_matches():
    import paper_2507_19845_b200 as ms
    tr = tg.from_events(2, 1, 1, [[0]], [[(AR, 0, 1, 0)], [(C, 0, 1), (AR, 0, 1, 0)]])
    o = oracle.run(tr)
    assert o["status"] == -2
    s = ms.Scan(0)
    s.load(tr)
    with pytest.raises(ms.ScanError) as ei:
        s.analyze() if MODE["mode"] == "analyze" else s.match()
    assert ei.value.status == -2 and f"event {o['bad_event']}" in str(ei.value)


def test_device_pointer_load():
    """Zero-copy load from torch CUDA tensors gives the same results as the host copy path."""
    tr = tg.generate(configs.c1(seed=4, iterations=3))
    d, l_, oc = _cfgs()
    o = oracle.run(tr, oc)
    g = _gpu(tr, d, l_, device_ptrs=True)
    compare(o, g)


def test_rerun_same_context_deterministic():
    import paper_2507_19845_b200 as ms
    tr = tg.generate(configs.c1(seed=2, iterations=4))
    s = ms.Scan(0)
    s.load(tr)
    run = s.analyze if MODE["mode"] == "analyze" else s.run
    run()
    a = s.export_all()
    run()
    b = s.export_all()
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_spmd_violation_falls_back():
    """A trace that is SPMD at load (equal counts, same roles) but whose events disagree with the
    stage template (one op id changed on one rank) fails verification inside the fused pass; the
    call must transparently produce the general path's (oracle-equal) results."""
    tr = tg.generate(configs.c1(seed=3, iterations=3))
    e = int(tr.rank_offsets[6]) + 1000
    assert (tr.kind_op[e] & 7) == 0
    tr.kind_op[e] = (tr.kind_op[e] & 0xF) | (((tr.kind_op[e] >> 4) ^ 5) << 4)
    o, g = _run_both(tr)
    compare(o, g)
    assert not g["_res"]["fused"]


@pytest.mark.parametrize("dp", [3, 5, 6])
def test_fused_odd_dp(dp):
    """Non-power-of-two DP groups (padding of the sorting network)."""
    tr = tg.generate(tg.GenConfig(2, 2, dp, 2, 4, 3, seed=dp, faults=[tg.Fault(tg.THROTTLE, 3, factor=2.0)]))
    o, g = _run_both(tr)
    compare(o, g)


def test_link_median_global_scratch():
    """More samples on a link than the shared-memory capacity of the median kernel (8192)."""
    tr = tg.generate(tg.GenConfig(1, 2, 1, 1, 64, 140, seed=9, faults=[tg.Fault(tg.LINK_JITTER, 0, 1)]))
    o, g = _run_both(tr)
    assert o["lk_n"].max() > 8192
    compare(o, g)


def test_link_median_exact_ties():
    """Zero jitter: every transfer on a link has the same payload and duration, so the median is
    decided by the instance-id tie-break alone."""
    tr = tg.generate(tg.GenConfig(2, 4, 2, 1, 12, 3, seed=2, jitter=0.0, clock_skew=False,
                                  faults=[tg.Fault(tg.LINK_DEGRADE, 2, 6, factor=0.5)]))
    o, g = _run_both(tr)
    compare(o, g)


def test_spmd_comm_violation_falls_back():
    """A collective whose communicator differs from the stage template's role (still a communicator the
    rank belongs to, so the trace stays schema-valid) must be caught by the fused path's comm check."""
    tr = tg.generate(configs.c1(seed=5, iterations=3))
    r = 6
    lo, hi = int(tr.rank_offsets[r]), int(tr.rank_offsets[r + 1])
    kinds = tr.kind_op[lo:hi] & 7
    comms = tr.comm[lo:hi]
    # first TP all-reduce of rank 6 -> its DP communicator (both contain rank 6)
    tp_comm = int(comms[np.nonzero(kinds == 1)[0][0]])
    others = sorted(set(int(c) for c in comms[kinds == 1]) - {tp_comm})
    e = lo + int(np.nonzero((kinds == 1) & (comms == tp_comm))[0][0])
    tr.comm[e] = others[0]
    o, g = _run_both(tr)
    compare(o, g)
    assert not g["_res"]["fused"]


def _gpu_variant(trace, variant, dcfg=None, lcfg=None):
    import paper_2507_19845_b200 as ms
    s = ms.Scan(0)
    s.fused_variant(variant)
    s.load(trace)
    res = s.analyze(dcfg, lcfg)
    out = s.export_all()
    out["_res"] = res
    s.close()
    return out


@pytest.mark.parametrize("name", ["c1", "c2", "c5w", "tp3"])
def test_fused_generic_tile_kernel(name):
    """The generic fused tile kernel (used when TP does not divide 32) against the oracle, also forced on
    the shapes the transposed kernel normally takes."""
    if MODE["mode"] != "analyze":
        pytest.skip("analyze-only")
    kw = {}
    if name == "c1":
        tr = tg.generate(configs.c1(seed=6, iterations=4))
    elif name == "c2":
        tr = tg.generate(configs.c2(iterations=6))
    elif name == "c5w":
        cfg = configs.c5(iterations=6)
        cfg.faults = [tg.Fault(tg.THROTTLE, 208, it0=2, factor=2.5)]
        tr = tg.generate(cfg)
        kw = dict(window_iters=2)
    else:
        tr = tg.generate(tg.GenConfig(3, 2, 4, 2, 6, 3, seed=3, faults=[tg.Fault(tg.THROTTLE, 4, factor=2.0)]))
    d, l_, oc = _cfgs(**kw)
    o = oracle.run(tr, oc)
    for variant in (0, -1):
        g = _gpu_variant(tr, variant, d, l_)
        compare(o, g)
        assert g["_res"]["fused"]


def test_c4_shape():
    """configs[3] shape: 3072 ranks TP8xPP64xDP6 (non-power-of-two DP, 64 stages), a throttled rank
    and a half-bandwidth link; 3 iterations (4.8 M events)."""
    o, g = _run_both(tg.generate(configs.c4(iterations=3)), min_samples=5)
    compare(o, g)


def test_round2_pin_traces():
    """The hand-built traces of the round-2 oracle pins (kind mismatch; the pslow segment reset in
    both stage-2 modes) through both GPU paths."""
    import test_oracle_pins as pins
    ag = tg.ALLGATHER
    km = tg.from_events(2, 1, 1, [[0, 1]], [[(AR, 0, 700, 0), (AR, 0, 500, 0)], [(ag, 0, 400, 0), (AR, 0, 300, 0)]])
    o, g = _run_both(km)
    compare(o, g)
    for mode in (0, 1):
        o, g = _run_both(pins._segment_trace(), mode=mode)
        compare(o, g)
