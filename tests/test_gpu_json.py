"""GPU parity of the Chrome-trace JSON ingest and emit (NEXT-2, scan_ingest_json / scan_emit_chrome)
against oracle/chrome_json.py, -m gpu. Ingest: every loaded column, the communicator table and the
skipped count bit-exact; errors: same kind, and for schema errors the same field and byte offset.
Emit: the merged document byte-exact (local and aligned timestamps). The analysis of an ingested
job equals the oracle's analysis of the oracle-parsed job."""
import json
import os

import numpy as np
import pytest

import oracle
import tracegen as tg
from oracle import chrome_json as cj
from tracegen import chrome, configs
from test_chrome_pins import GOLD, SCHEMA, SYNTAX, _gold_docs, schema_cases
from test_gpu_parity import compare

pytestmark = pytest.mark.gpu

COLS = ("start_ns", "dur_ns", "kind_op", "meta", "comm", "payload", "rank_offsets")


def _ingest(docs, topo, device=False):
    import paper_2507_19845_b200 as ms
    s = ms.Scan(0)
    res = s.ingest_json(docs, *topo, device=device)
    return s, res


def _check_columns(s, res, t, skipped):
    assert res["n_events"] == t.n_events and res["n_skipped"] == skipped and res["n_comms"] == t.n_comms
    for k in COLS:
        g = s.loaded(k)
        v = getattr(t, k)
        assert g.dtype == v.dtype and np.array_equal(g, v), k
    assert np.array_equal(s.loaded("comm_offsets"), t.comm_offsets)
    assert np.array_equal(s.loaded("comm_members"), t.comm_members)


def test_golden():
    exp = json.load(open(os.path.join(GOLD, "chrome_small_expected.json")))
    s, res = _ingest(_gold_docs(), exp["topology"])
    t, skipped = cj.parse(_gold_docs(), *exp["topology"])
    _check_columns(s, res, t, skipped)
    assert s.loaded("start_ns").tolist() == exp["start_ns"]
    s.close()


@pytest.mark.parametrize("messy,device", [(True, False), (False, False), (True, True)])
def test_generator_docs(messy, device):
    cfg = configs.c1(seed=7, iterations=3)
    docs = chrome.rank_documents(tg.generate(cfg), messy=messy, seed=11)
    t, skipped = cj.parse(docs, cfg.tp, cfg.pp, cfg.dp)
    s, res = _ingest(docs, (cfg.tp, cfg.pp, cfg.dp), device=device)
    _check_columns(s, res, t, skipped)
    s.close()


def test_c2_docs_then_analysis_and_emit():
    """64 ranks: ingest == oracle parse; analysis of the ingested job == oracle.run; emit == oracle.emit."""
    cfg = configs.c2(seed=3, iterations=2)
    docs = chrome.rank_documents(tg.generate(cfg), messy=True, seed=2)
    t, skipped = cj.parse(docs, cfg.tp, cfg.pp, cfg.dp)
    s, res = _ingest(docs, (cfg.tp, cfg.pp, cfg.dp))
    _check_columns(s, res, t, skipped)
    o = oracle.run(t, oracle.Config())
    import paper_2507_19845_b200 as ms
    r = s.analyze(ms.DetectConfig(want_ref=True))
    g = s.export_all()
    g["_res"] = r
    compare(o, g)
    assert s.emit_chrome() == cj.emit(t, o["ev_inst"])
    s.close()


@pytest.mark.parametrize("path", ["fused", "general"])
def test_emit_after_binary_load_local_and_aligned(path):
    import paper_2507_19845_b200 as ms
    tr = tg.generate(configs.c1(seed=5, iterations=4))
    o = oracle.run(tr, oracle.Config())
    al = oracle.align(tr, 1)
    s = ms.Scan(0)
    s.load(tr, start=True)
    if path == "fused":
        s.analyze()
    else:
        s.run()
    out = s.emit_chrome()
    assert out == cj.emit(tr, o["ev_inst"])
    s.align(1)
    assert s.emit_chrome(aligned=True) == cj.emit(tr, o["ev_inst"], start=al["al_start"])
    # the merged document re-ingests to the same job (communicators renumbered by first use)
    t2, _ = cj.parse([out], tr.tp, tr.pp, tr.dp)
    s2, res = _ingest([out], (tr.tp, tr.pp, tr.dp))
    _check_columns(s2, res, t2, 0)
    s.close()
    s2.close()


def test_emit_to_device_buffer():
    import torch
    import paper_2507_19845_b200 as ms
    tr = tg.generate(configs.c1(seed=2, iterations=2))
    s = ms.Scan(0)
    s.load(tr, start=True)
    s.analyze()
    host = s.emit_chrome()
    buf = torch.empty(len(host) + 10, dtype=torch.uint8, device="cuda")
    n = s.emit_chrome(dst=buf)
    assert n == len(host) and bytes(buf[:n].cpu().numpy()) == host
    s.close()


@pytest.mark.parametrize("i", range(len(SCHEMA) + 4))
def test_schema_errors(i):
    import paper_2507_19845_b200 as ms
    b, f, off = schema_cases()[i]
    with pytest.raises(ms.JsonTraceError) as e:
        _ingest([b], (1, 1, 2))
    assert (e.value.kind, e.value.field, e.value.offset) == (cj.E_SCHEMA, f, off)


@pytest.mark.parametrize("b", SYNTAX)
def test_syntax_errors(b):
    import paper_2507_19845_b200 as ms
    with pytest.raises(ms.JsonTraceError) as e:
        _ingest([b], (1, 1, 2))
    assert e.value.kind == cj.E_SYNTAX


def test_syntax_beats_schema_and_multi_doc_offsets():
    import paper_2507_19845_b200 as ms
    bad = b'{"traceEvents":[{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":7}]}'
    with pytest.raises(ms.JsonTraceError) as e:
        _ingest([bad, b"[{"], (1, 1, 2))
    assert e.value.kind == cj.E_SYNTAX
    good = b'[{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":0}]'
    with pytest.raises(ms.JsonTraceError) as e:
        _ingest([good, bad], (1, 1, 2))
    assert (e.value.kind, e.value.field, e.value.offset) == (cj.E_SCHEMA, cj.F_PID, len(good) + bad.index(b'{"cat"'))


def test_valid_edge_cases_and_empty():
    s_ = (' \n[ {"ph":"M","ts":"not checked"} , {"cat":"compute","ph":"X","ts":-0,"dur":4294967.295,"pid":1,'
          '"tid":"t","args":{"iter_end":false,"bwd":true,"op":0,"op":4095,"u":{"v":["}",{"w":"\\"]"}]}}},'
          ' {"cat":"compute","ph":"X","ts":-0.5,"dur":0,"pid":1}\t]\r\n')
    docs = [s_.encode(), b"[]", b'{"traceEvents":[]}']
    t, skipped = cj.parse(docs, 1, 1, 2)
    s, res = _ingest(docs, (1, 1, 2))
    _check_columns(s, res, t, skipped)
    s.close()
    s, res = _ingest([], (2, 1, 1))
    assert res["n_events"] == 0 and s.loaded("rank_offsets").tolist() == [0, 0, 0]
    s.close()


@pytest.mark.parametrize("seed", range(301, 311))
def test_fuzz_random_jobs(seed):
    """Random topologies / faults, messy per-rank files: ingest, analysis and emit all match."""
    rng = np.random.default_rng(seed)
    tp, pp, dp = (int(x) for x in rng.integers(1, 4, 3))
    if tp * pp * dp == 1:
        dp = 2
    cfg = tg.GenConfig(tp, pp, dp, int(rng.integers(1, 3)), int(rng.integers(pp, pp + 3)), int(rng.integers(2, 4)),
                       seed=seed, faults=[tg.Fault(tg.THROTTLE, int(rng.integers(0, tp * pp * dp)), factor=2.0)])
    docs = chrome.rank_documents(tg.generate(cfg), messy=True, seed=seed)
    if rng.random() < 0.5:  # files in another order: program order and first use do not depend on it
        docs = docs[::-1]
    t, skipped = cj.parse(docs, tp, pp, dp)
    s, res = _ingest(docs, (tp, pp, dp))
    _check_columns(s, res, t, skipped)
    o = oracle.run(t, oracle.Config(min_samples=3))
    import paper_2507_19845_b200 as ms
    s.analyze(ms.DetectConfig(min_samples=3), ms.LocalizeConfig(min_samples=3))
    assert s.emit_chrome() == cj.emit(t, o["ev_inst"])
    s.close()


@pytest.mark.parametrize("run", [1, 2, 63, 64, 65, 127, 128, 129, 1 << 20])
def test_long_backslash_runs(run):
    """Escapes across 64-byte words: a string holding `run` escaped backslashes (2*run backslash bytes)
    then an escaped quote, inside an unknown args key of the first event, and a second document whose
    first string starts right after a run boundary. The entry escape state of every word comes from a
    scan (no look-back), so a 2 MB run costs the same per byte as any other input."""
    cfg = configs.c1(seed=3, iterations=2)
    docs = chrome.rank_documents(tg.generate(cfg), messy=False, seed=1)
    d0 = docs[0].decode()
    k = d0.index('"args":{') + len('"args":{')
    pad = '"note":"' + '\\\\' * run + '\\"x",'
    docs = [(d0[:k] + pad + d0[k:]).encode()] + list(docs[1:])
    t, skipped = cj.parse(docs, cfg.tp, cfg.pp, cfg.dp)
    s, res = _ingest(docs, (cfg.tp, cfg.pp, cfg.dp))
    _check_columns(s, res, t, skipped)
    s.close()
