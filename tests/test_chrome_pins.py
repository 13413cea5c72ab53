"""Pins of the JSON ingest / emit oracle (oracle/chrome_json.py, NEXT-2; DESIGN.md §10d J1-J12),
CPU only. Not checked against itself: a hand-derived golden fixture, the DES generator's own
columns through its independent per-rank writer, the standard library's json.loads on every
emitted document, and one hand-placed case per schema / syntax error."""
import json
import os

import numpy as np
import pytest

import tracegen as tg
from tracegen import chrome, configs
from oracle import chrome_json as cj

GOLD = os.path.join(os.path.dirname(__file__), "golden")
COLS = ("start_ns", "dur_ns", "kind_op", "meta", "payload")


def _gold_docs():
    return [open(os.path.join(GOLD, f"chrome_small_rank{r}.json"), "rb").read() for r in (0, 1)]


def _canon_comm(t):
    """Per event: the participant list of a collective, the peer of a P2P event, 0 for compute."""
    k = t.kind_op & 7
    co = t.comm_offsets.astype(np.int64)
    return [tuple(int(x) for x in t.comm_members[co[c]:co[c + 1]]) if 1 <= kk <= 4 else int(c)
            for kk, c in zip(k, t.comm)]


def assert_same_trace(a, b):
    assert np.array_equal(a.rank_offsets, b.rank_offsets)
    for k in COLS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert _canon_comm(a) == _canon_comm(b)


def test_golden_columns():
    exp = json.load(open(os.path.join(GOLD, "chrome_small_expected.json")))
    t, skipped = cj.parse(_gold_docs(), *exp["topology"])
    assert skipped == exp["n_skipped"]
    for k in ("rank_offsets",) + COLS + ("comm", "comm_offsets", "comm_members"):
        assert getattr(t, k).tolist() == exp[k], k


def test_golden_emit_bytes():
    exp = json.load(open(os.path.join(GOLD, "chrome_small_expected.json")))
    t, _ = cj.parse(_gold_docs(), *exp["topology"])
    ev_inst = np.array([100, 0xFFFFFFFF, 7, 100, 7, 9], dtype=np.uint32)
    out = cj.emit(t, ev_inst)
    assert out == open(os.path.join(GOLD, "chrome_small_emit.json"), "rb").read()
    json.loads(out)  # a Chrome Tracing document the standard decoder accepts


def test_merged_document_reparses_to_the_same_columns():
    exp = json.load(open(os.path.join(GOLD, "chrome_small_expected.json")))
    t, _ = cj.parse(_gold_docs(), *exp["topology"])
    t2, skipped = cj.parse([cj.emit(t, np.zeros(t.n_events, np.uint32))], *exp["topology"])
    assert skipped == 0
    assert_same_trace(t, t2)


@pytest.mark.parametrize("messy", [True, False])
def test_generator_round_trip(messy):
    """The DES generator's columns -> its per-rank writer -> parse == the generator's columns."""
    cfg = configs.c1(seed=3, iterations=2)
    tr = tg.generate(cfg)
    docs = chrome.rank_documents(tr, messy=messy, seed=5)
    t, skipped = cj.parse(docs, cfg.tp, cfg.pp, cfg.dp)
    assert skipped == (cfg.world if messy else 0)
    assert_same_trace(tr, t)
    # communicator ids are numbered by first use in program order (J4)
    first = []
    for c, k in zip(t.comm, t.kind_op & 7):
        if 1 <= k <= 4 and int(c) not in first:
            first.append(int(c))
    assert first == list(range(t.n_comms))
    # and the merged, annotated document parses back to the same job
    m = cj.emit(t, np.arange(t.n_events, dtype=np.uint32))
    json.loads(m)
    t3, _ = cj.parse([m], cfg.tp, cfg.pp, cfg.dp)
    assert_same_trace(t, t3)


def test_emit_is_time_ordered_with_rank_and_program_tie_break():
    tr = tg.generate(configs.c1(seed=4, iterations=1))
    d = json.loads(cj.emit(tr, np.zeros(tr.n_events, np.uint32)))["traceEvents"]
    key = [(round(e["ts"] * 1000), e["pid"]) for e in d]
    assert key == sorted(key)
    assert len(d) == tr.n_events


E = '{"cat":"all_reduce","ph":"X","ts":1,"dur":2,"pid":0,"args":{"group":[0,1]}}'


def _doc(bad: str) -> tuple[bytes, int]:
    s = '{"traceEvents":[' + E + ", " + bad + "," + E + "]}"
    return s.encode(), s.index(bad)


SCHEMA = [
    ('{"cat":"compute","ph":"X","dur":2,"pid":0}', cj.F_TS),
    ('{"cat":"compute","ph":"X","ts":"1","dur":2,"pid":0}', cj.F_TS),
    ('{"cat":"compute","ph":"X","ts":1.2345,"dur":2,"pid":0}', cj.F_TS),
    ('{"cat":"compute","ph":"X","ts":1e3,"dur":2,"pid":0}', cj.F_TS),
    ('{"cat":"compute","ph":"X","ts":9223372036854775.808,"dur":2,"pid":0}', cj.F_TS),
    ('{"cat":"compute","ph":"X","ts":1,"dur":-1,"pid":0}', cj.F_DUR),
    ('{"cat":"compute","ph":"X","ts":1,"dur":4294967.296,"pid":0}', cj.F_DUR),
    ('{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":2}', cj.F_PID),
    ('{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":1.0}', cj.F_PID),
    ('{"cat":"compute","ph":"X","ts":1,"dur":2}', cj.F_PID),
    ('{"cat":"allreduce","ph":"X","ts":1,"dur":2,"pid":0}', cj.F_CAT),
    ('{"ph":"X","ts":1,"dur":2,"pid":0}', cj.F_CAT),
    ('{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":0,"args":[]}', cj.F_ARGS),
    ('{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":0,"args":{"op":4096}}', cj.F_OP),
    ('{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":0,"args":{"iter_end":2}}', cj.F_ITER_END),
    ('{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":0,"args":{"iter_end":"true"}}', cj.F_ITER_END),
    ('{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":0,"args":{"mb":1024}}', cj.F_MB),
    ('{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":0,"args":{"chunk":8}}', cj.F_CHUNK),
    ('{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":0,"args":{"bwd":"1"}}', cj.F_BWD),
    ('{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":0,"args":{"warmup":null}}', cj.F_WARMUP),
    ('{"cat":"all_gather","ph":"X","ts":1,"dur":2,"pid":0,"args":{"group":[1,0]}}', cj.F_GROUP),
    ('{"cat":"all_gather","ph":"X","ts":1,"dur":2,"pid":0,"args":{"group":[]}}', cj.F_GROUP),
    ('{"cat":"all_gather","ph":"X","ts":1,"dur":2,"pid":0,"args":{"group":[0,2]}}', cj.F_GROUP),
    ('{"cat":"broadcast","ph":"X","ts":1,"dur":2,"pid":0}', cj.F_GROUP),
    ('{"cat":"send","ph":"X","ts":1,"dur":2,"pid":0,"args":{}}', cj.F_PEER),
    ('{"cat":"recv","ph":"X","ts":1,"dur":2,"pid":0,"args":{"peer":2}}', cj.F_PEER),
    ('{"cat":"recv","ph":"X","ts":1,"dur":2,"pid":0,"args":{"peer":1,"bytes":4294967296}}', cj.F_BYTES),
    ('{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":0,"args":{"bytes":-1}}', cj.F_BYTES),
    ('{"cat":"compute","ts":1,"dur":2,"pid":0}', cj.F_PH),
    ('{"cat":"compute","ph":1,"ts":1,"dur":2,"pid":0}', cj.F_PH),
    ('5', cj.F_EVENT),
    ('[]', cj.F_EVENT),
    ('{"cat":"nope","ph":"X","ts":"x","dur":2,"pid":9}', cj.F_TS),  # first failing field in J11 order
]


def schema_cases():
    """(bytes, field, offset) per case; shared with the GPU parity test."""
    out = []
    for bad, f in SCHEMA:
        b, off = _doc(bad)
        out.append((b, f, off))
    out.append((b'{"other":[]}', cj.F_TRACE_EVENTS, 0))
    out.append((b'  {"traceEvents":{}}', cj.F_TRACE_EVENTS, 2))
    out.append((b'{"traceEvents":[],"traceEvents":[]}', cj.F_TRACE_EVENTS, 0))
    s = '{"traceEvents":[' + E + ',{"cat":"x","ph":"X","ts":1,"dur":2,"pid":0},{"ph":"X"}]}'
    out.append((s.encode(), cj.F_CAT, s.index('{"cat":"x"')))  # smallest offset wins
    return out


SYNTAX = [b'{"traceEvents":[{"cat":"compute",}]}', b'[{"ts":01}]', b'[{"a":"\\x"}]', b'[{"a":"abc}]',
          b'[{}] x', b'', b'  ', b'[{"a":tru}]', b'[{"a":"\x01"}]', b'[NaN]', b'[{"a" 1}]', b'[{"a":1}',
          b'[{"a":-}]', b'[{"a":1.}]', b'[{"a":[1,]}]', b'[{"ph":"X",}]', b'[5, 6x]', b'[5,]', b'[{"ph":"M"},]',
          b'[{"ph":"M"} {"ph":"M"}]', b'[{"ph":"M"},[1,]]', b'{"traceEvents":[]', b'{"traceEvents":[]}}',
          rb'[{"a\q":1}]', rb'[{"a":"\u12G4"}]', b'[{"a":{"b" 1}}]', b'[{"a":{"b":1,}}]', b'[]]']


@pytest.mark.parametrize("i", range(len(SCHEMA) + 4))
def test_schema_errors(i):
    b, f, off = schema_cases()[i]
    with pytest.raises(cj.JsonTraceError) as e:
        cj.parse([b], 1, 1, 2)
    assert (e.value.kind, e.value.field, e.value.offset) == (cj.E_SCHEMA, f, off)


@pytest.mark.parametrize("b", SYNTAX)
def test_syntax_errors(b):
    with pytest.raises(cj.JsonTraceError) as e:
        cj.parse([b], 1, 1, 2)
    assert e.value.kind == cj.E_SYNTAX


def test_syntax_error_beats_schema_error_in_an_earlier_document():
    bad_schema, _ = _doc('{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":7}')
    with pytest.raises(cj.JsonTraceError) as e:
        cj.parse([bad_schema, b"[{"], 1, 1, 2)
    assert e.value.kind == cj.E_SYNTAX


def test_valid_edge_cases():
    s = (' \n[ {"ph":"M","ts":"not checked"} , {"cat":"compute","ph":"X","ts":-0,"dur":4294967.295,"pid":1,'
         '"tid":"t","args":{"iter_end":false,"bwd":true,"op":0,"op":4095,"u":{"v":["}",{"w":"\\"]"}]}}},'
         ' {"cat":"compute","ph":"X","ts":-0.5,"dur":0,"pid":1}\t]\r\n')
    t, skipped = cj.parse([s.encode(), b"[]", b'{"traceEvents":[]}'], 1, 1, 2)
    assert skipped == 1
    assert t.rank_offsets.tolist() == [0, 0, 2]
    assert t.start_ns.tolist() == [-500, 0] and t.dur_ns.tolist() == [0, 4294967295]
    assert t.kind_op.tolist() == [0, 4095 << 4] and t.meta.tolist() == [0, 1 << 13]
    assert t.n_comms == 0


def test_empty_input():
    t, skipped = cj.parse([], 2, 1, 1)
    assert t.n_events == 0 and skipped == 0 and t.rank_offsets.tolist() == [0, 0, 0]
    assert cj.emit(t, np.zeros(0, np.uint32)) == b'{"traceEvents":[\n]}\n'


def test_fast_writer_is_the_clean_writer():
    tr = tg.generate(configs.c2(seed=2, iterations=1))
    b, off = chrome.rank_documents_fast(tr)
    docs = chrome.rank_documents(tr, messy=False)
    assert b == b"".join(docs)
    assert [int(x) for x in np.diff(off)] == [len(d) for d in docs]
