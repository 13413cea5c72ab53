"""Mutation fuzz of the JSON ingest (NEXT-2), -m gpu: random single-byte edits (delete / insert /
replace, from a JSON-structural alphabet) of small valid bare-array documents. The GPU ingest and
the oracle must agree on every mutant: both accept with bit-equal columns, or both reject with the
same error kind, and for schema errors the same field and byte offset. The whole input is validated
(reading J10), so edits may land anywhere, including an object root's other members."""
import numpy as np
import pytest

from oracle import chrome_json as cj

pytestmark = pytest.mark.gpu

BASE = [
    b'[{"cat":"all_reduce","ph":"X","ts":1.5,"dur":2,"pid":0,"args":{"group":[0,1],"op":3}},'
    b' {"cat":"compute","ph":"X","ts":0,"dur":10.25,"pid":1,"args":{"mb":2,"bwd":true,"x":[1,{"y":"]\\"}"}]}},'
    b'{"ph":"M","name":"meta"},{"cat":"send","ph":"X","ts":-3,"dur":1,"pid":1,"args":{"peer":0,"bytes":64}}]',
    b'[\n {"name": "a \\u0041", "cat": "recv", "ph": "X", "ts": 7, "dur": 0.001, "pid": 0, "tid": 2,'
    b' "args": {"peer": 1, "bytes": 64, "iter_end": 1}},\n {"cat":"compute","ph":"X","ts":8,"dur":3,"pid":0}\n]',
    b'{"otherData": {"a": [1, 2.5, {"b": "}]"}], "t": true}, "traceEvents": [{"cat":"all_gather","ph":"X",'
    b'"ts":2,"dur":1,"pid":1,"args":{"group":[1],"warmup":0}}, {"cat":"compute","ph":"X","ts":1,"dur":1,"pid":0}],'
    b' "displayTimeUnit": "ns", "n": null}',
]
ALPHABET = b'{}[]:,"\\ 0123456789-.eEtfnXxa'


def _mutants(seed, n):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        b = bytearray(BASE[int(rng.integers(0, len(BASE)))])
        for _ in range(int(rng.integers(1, 3))):
            op, i = int(rng.integers(0, 3)), int(rng.integers(0, len(b)))
            c = ALPHABET[int(rng.integers(0, len(ALPHABET)))]
            if op == 0 and len(b) > 1:
                del b[i]
            elif op == 1:
                b.insert(i, c)
            else:
                b[i] = c
        out.append(bytes(b))
    return out


def _oracle(doc):
    try:
        t, skipped = cj.parse([doc], 1, 1, 2)
        return ("ok", t, skipped)
    except cj.JsonTraceError as e:
        return ("err", e.kind, e.field, e.offset)


def _gpu(doc):
    import paper_2507_19845_b200 as ms
    s = ms.Scan(0)
    try:
        res = s.ingest_json([doc], 1, 1, 2)
        cols = {k: s.loaded(k) for k in ("rank_offsets", "start_ns", "dur_ns", "kind_op", "meta", "comm", "payload",
                                         "comm_offsets", "comm_members")}
        return ("ok", res, cols)
    except ms.JsonTraceError as e:
        return ("err", e.kind, e.field, e.offset)
    finally:
        s.close()


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("MS_JSON_FUZZ_N", "25"))))
def test_mutants_agree(seed):
    bad = []
    for doc in _mutants(seed, 60):
        o, g = _oracle(doc), _gpu(doc)
        if o[0] != g[0]:
            bad.append((doc, o[:1] + (o[1:] if o[0] == "err" else ()), g[:1] + (g[1:] if g[0] == "err" else ())))
            continue
        if o[0] == "err":
            same = o[1] == g[1] and (o[1] == cj.E_SYNTAX or (o[2], o[3]) == (g[2], g[3]))
            if not same:
                bad.append((doc, o, g))
            continue
        t, skipped = o[1], o[2]
        res, cols = g[1], g[2]
        ok = res["n_skipped"] == skipped and all(np.array_equal(cols[k], getattr(t, k)) for k in cols)
        if not ok:
            bad.append((doc, "columns differ", None))
    assert not bad, "\n".join(repr(x) for x in bad[:5])
