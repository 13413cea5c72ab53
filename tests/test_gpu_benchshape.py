"""GPU parity at the bench's own kernel shapes and at the u32 limits (-m gpu).

The bench times C3 (TP8 x PP8 x DP16: the transposed fused kernel with a 16-wide sorting network and
four 32-row blocks per lane). The oracle cannot run the whole 1000-iteration job in seconds, but a
few iterations of the SAME shape take the same kernel instantiation, tile geometry and fault mix, so
here EVERY exported array (per event, per instance, per rank, per window, per link, walk, edges) is
compared element by element with `oracle.run` on:
* C3 shape, 4 iterations (3.8 M events; rank 299 throttled on iterations [0, 2), rank 862 on [2, 3),
  jittered forward links leaving stage 4), through both analysis paths, with and without windows;
* C4 shape (3072 ranks TP8 x PP64 x DP6), 8 iterations (12.7 M events);
* the u32 limits: C3-shape durations scaled up to 0xFFFFFFFF, so that one tile's wait sum on one
  wait-for edge passes 2^32 (the carry of the fused kernel's 32-bit shared-memory edge sums) and the
  per-tile compute / wait sums need their high words;
* the K = 50 sliding window over 512 ranks (the streaming bench's configuration), at its first
  full window and its last;
* the general path at C3 shape with one SPMD violation (an op id changed on one rank).
Integers / flags / labels bit-exact, f64 reports within 1e-6 relative (BASELINE.json north_star)."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from tracegen import configs

pytestmark = pytest.mark.gpu

FLOAT_KEYS = {"wd_frac", "wl_late_frac", "lk_med_bw"}


def _gpu(trace, mode, dcfg, lcfg):
    import paper_2507_19845_b200 as ms
    s = ms.Scan(0)
    s.load(trace)
    if mode == "analyze":
        res = s.analyze(dcfg, lcfg)
    else:
        res = s.run(dcfg, lcfg)
        res["fused"] = False
    out = s.export_all()
    out["_res"] = res
    s.close()
    return out


def _cfgs(window_iters=0, want_ref=False, mode=0, min_samples=10):
    import paper_2507_19845_b200 as ms
    return (ms.DetectConfig(window_iters=window_iters, want_ref=want_ref, min_samples=min_samples),
            ms.LocalizeConfig(stage2_mode=mode, min_samples=min_samples),
            oracle.Config(window_iters=window_iters, stage2_mode=mode, min_samples=min_samples))


def compare(o, g, skip=()):
    res = g["_res"]
    assert res["status"] == o["status"]
    m = res["match"]
    for k in ("n_instances", "n_incomplete", "n_kind_mismatch", "n_payload_mismatch", "n_channels"):
        assert m[k] == o[k], k
    assert res["detect"]["n_windows"] == o["n_windows"]
    bad = []
    for k, v in o.items():
        if not isinstance(v, np.ndarray) or k in skip:
            continue
        gv = g[k]
        if gv.shape != v.shape:
            bad.append(f"{k}: shape {gv.shape} vs oracle {v.shape}")
        elif k in FLOAT_KEYS:
            if not np.allclose(gv, v, rtol=1e-6, atol=0):
                i = np.nonzero(~np.isclose(gv, v, rtol=1e-6, atol=0))[0][:5]
                bad.append(f"{k}: first diffs at {i}: gpu {gv[i]} oracle {v[i]}")
        elif not np.array_equal(gv, v):
            i = np.nonzero(gv != v)[0][:5]
            bad.append(f"{k}: {int((gv != v).sum())} diffs, first at {i}: gpu {gv[i]} oracle {v[i]}")
    assert not bad, "\n".join(bad)


@pytest.fixture(scope="module")
def c3_short():
    return tg.generate(configs.c3(iterations=4))


@pytest.mark.parametrize("mode", ["analyze", "separate"])
@pytest.mark.parametrize("wi,want_ref", [(0, False), (2, True)])
def test_c3_shape_every_output(c3_short, mode, wi, want_ref):
    """The bench's k_fused_t<16,4> instantiation (analyze) and the general path (separate) against
    the oracle on every exported array; the 4 iterations hold both throttle windows and the jittered
    links, so stage 1, stage 2, stage 3, the walk and the edges all have non-trivial content."""
    tr = c3_short
    d, l_, oc = _cfgs(window_iters=wi, want_ref=want_ref)
    o = oracle.run(tr, oc)
    assert o["wd_cand"].sum() >= 1 and o["eg_weight"].size > 0 and o["lk_n"].size > 0
    g = _gpu(tr, mode, d, l_)
    assert g["_res"]["fused"] == (mode == "analyze")
    compare(o, g, skip=() if want_ref else ("ev_ref",))  # stage-1 references are exported only on request


def test_c4_shape_eight_iterations():
    """configs[3] shape (3072 ranks TP8 x PP64 x DP6: 48-row blocks, 8-wide sorting network, 64
    stages) over 8 iterations, through scan_analyze (fused)."""
    tr = tg.generate(configs.c4(iterations=8))
    d, l_, oc = _cfgs(min_samples=5, want_ref=True)
    o = oracle.run(tr, oc)
    g = _gpu(tr, "analyze", d, l_)
    assert g["_res"]["fused"]
    compare(o, g)


def _scaled_c3(iterations=3):
    """C3 shape at the u32 limits. Every duration is scaled so the largest is 0xFFFFFFFF, and the TP
    all-reduces of rank 862's TP group (ranks 856-863) get durations near 2^32 on the seven peers and
    ~1 us on rank 862: each such instance then puts a wait of ~2^32 on the edge peer -> 862, about
    36 of them per 128-position tile (the fused kernel's 32-bit shared-memory edge sums carry into
    the 64-bit global weights many times per tile), and the per-rank wait sums pass 2^41. The
    analysis reads only durations (reading R5), so any durations are a valid trace."""
    tr = tg.generate(configs.c3(iterations=iterations))
    d = tr.dur_ns.astype(np.float64) * (0xFFFFFFFF / float(tr.dur_ns.max()))
    tr.dur_ns = np.minimum(np.round(d), 0xFFFFFFFF).astype(np.uint32)
    co = tr.comm_offsets.astype(np.int64)
    grp = list(range(856, 864))
    cid = next(c for c in range(len(co) - 1) if list(tr.comm_members[co[c]:co[c + 1]]) == grp)
    for r in grp:
        lo, hi = int(tr.rank_offsets[r]), int(tr.rank_offsets[r + 1])
        idx = lo + np.flatnonzero(((tr.kind_op[lo:hi] & 7) == 1) & (tr.comm[lo:hi] == cid))
        tr.dur_ns[idx] = (1000 + idx % 7) if r == 862 else (0xFFFFFFFF - idx % 1000)
    tr.dur_ns[np.flatnonzero((tr.kind_op[:100_000] & 7) == 0)[::997]] = 0xFFFFFFFF  # exact maxima
    return tr


@pytest.mark.parametrize("mode", ["analyze", "separate"])
def test_u32_limits(mode):
    tr = _scaled_c3()
    d, l_, oc = _cfgs(want_ref=True)
    o = oracle.run(tr, oc)
    assert int(tr.dur_ns.max()) == 0xFFFFFFFF
    # the per-tile edge sums of the fused kernel overflow 32 bits: the whole-trace weights are far above
    assert int(o["eg_weight"].max()) > 256 * 2**32
    assert int(o["rk_sum_wait"].max()) > 2**41
    g = _gpu(tr, mode, d, l_)
    assert g["_res"]["fused"] == (mode == "analyze")
    compare(o, g)


def test_stream_k50_512_ranks():
    """The streaming bench's configuration (C5: 512 ranks, K = 50): after 100 pushes the window's
    outputs equal the oracle from scratch on iterations [50, 100); also checked at the first full
    window (iterations [0, 50))."""
    import paper_2507_19845_b200 as ms
    cfg = configs.c5(iterations=100)
    full = tg.generate(cfg, with_start=False)
    s = ms.Scan(0)
    K = 50
    s.stream_open(full, K)
    for i in range(cfg.iterations):
        res = s.stream_push(ms.slice_iterations(full, i, i + 1))
        if i not in (K - 1, cfg.iterations - 1):
            continue
        lo = i - K + 1
        assert res["window"] == K
        o = oracle.run(ms.slice_iterations(full, lo, i + 1), oracle.Config())
        bad = []
        for k in ms.Scan.STREAM_OUTPUTS:
            v, gv = o[k], s.export(k)
            if gv.shape != v.shape:
                bad.append(f"{k}: shape {gv.shape} vs {v.shape}")
            elif k in FLOAT_KEYS:
                if not np.allclose(gv, v, rtol=1e-6, atol=0):
                    bad.append(f"{k}: float diffs")
            elif not np.array_equal(gv, v):
                j = np.nonzero(gv != v)[0][:5]
                bad.append(f"{k}: {int((gv != v).sum())} diffs at {j}: gpu {gv[j]} oracle {v[j]}")
        assert not bad, f"window {lo}..{i}:\n" + "\n".join(bad)
        if i == cfg.iterations - 1:
            assert o["wl_verdict"][208] == 1  # the x2.5 source is ComputeSlow in the last window
    s.close()


def test_general_path_c3_shape_with_violation():
    """One op id changed on one rank of the C3 shape: the fused pass must reject the trace and the
    general path must produce the oracle's results on every output."""
    tr = tg.generate(configs.c3(iterations=3))
    r = 300
    lo = int(tr.rank_offsets[r])
    e = lo + int(np.flatnonzero((tr.kind_op[lo:lo + 5000] & 7) == 0)[1234])
    tr.kind_op[e] = (tr.kind_op[e] & 0xF) | ((((tr.kind_op[e] >> 4) ^ 9) & 0xFFF) << 4)
    d, l_, oc = _cfgs(want_ref=True)
    o = oracle.run(tr, oc)
    assert o["cl_mismatch"].sum() >= 1  # the common-prefix rule fired (reading R9)
    g = _gpu(tr, "analyze", d, l_)
    assert not g["_res"]["fused"]
    compare(o, g)
