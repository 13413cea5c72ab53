"""oracle.chrome_json — plain Python reference of the Chrome-trace JSON ingest and emit (NEXT-2).

TEST INFRASTRUCTURE ONLY (same rule as ``oracle/__init__``): imported by ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs, never by the product path. Shares no code
with ``paper_2507_19845_b200`` (the GPU tokeniser in ``csrc/k_json.cu``).

What it computes, in the paper's order (§3.2):
  * P:L117-118 "every rank has its own recorded event sequence as a JSON file": ``parse`` reads
    one or more JSON documents (Chrome Tracing Format, object ``{"traceEvents":[...]}`` or bare
    array) with the Python standard library decoder, takes the complete ("ph":"X") events and
    their ``tracers.scope`` metadata, and builds the event columns the analysis reads;
  * P:L130-131 "for collective operations we log the global ID list of all participating ranks":
    every distinct participant list becomes one communicator id, numbered in order of first use;
  * P:L119-125 "merges them-ordered by time-into a single JSON file conforming to the Chrome
    Tracing Format ... each rank is mapped to a separate process": ``emit`` writes the merged
    document, events ordered by (timestamp, rank, program order), pid = rank;
  * P:L133 the matched instance of every communication event "stored in the related_sync_op
    attribute": ``emit`` writes it into ``args.related_sync_op``.
Schema, validation order and the byte-exact output format: DESIGN.md §10d, readings J1-J12.

Pins (tests/test_chrome_pins.py): a hand-written golden fixture with hand-derived columns
(tests/golden/chrome_small.json), the seeded DES generator's own columns round-tripped through
its independent per-rank writer (tracegen.chrome), the standard library's ``json.loads`` accepting
every emitted document, emit -> parse round trips, and one case per schema error.
"""
from __future__ import annotations

import json
import re

import numpy as np

KIND_NAMES = ("compute", "all_reduce", "all_gather", "reduce_scatter", "broadcast", "send", "recv")

# error kinds / fields (scan.h SCAN_JSON_* / SCAN_JF_*)
E_SYNTAX, E_SCHEMA = 1, 2
(F_TRACE_EVENTS, F_EVENT, F_PH, F_TS, F_DUR, F_PID, F_CAT, F_ARGS, F_OP, F_ITER_END, F_MB, F_CHUNK,
 F_BWD, F_WARMUP, F_GROUP, F_PEER, F_BYTES) = range(1, 18)


class JsonTraceError(Exception):
    def __init__(self, kind: int, field: int, offset: int, msg: str):
        super().__init__(f"{'syntax' if kind == E_SYNTAX else 'schema'} error at byte {offset} (field {field}): {msg}")
        self.kind, self.field, self.offset = kind, field, offset


class _Num(str):
    """A JSON number kept as its literal text (reading J5: exact decimal conversion)."""


_DEC = json.JSONDecoder(parse_int=_Num, parse_float=_Num, parse_constant=lambda s: (_ for _ in ()).throw(ValueError(s)))
_WS = " \t\n\r"
_USEC = re.compile(r"(-?)(\d+)(?:\.(\d{1,3}))?")


def _ws(s: str, i: int) -> int:
    while i < len(s) and s[i] in _WS:
        i += 1
    return i


def _decode(s: str, i: int, base: int):
    try:
        return _DEC.raw_decode(s, i)
    except (json.JSONDecodeError, ValueError) as e:
        raise JsonTraceError(E_SYNTAX, 0, base + i, str(e)) from None


def _doc_events(s: str, base: int):
    """Elements of the document's event array as (byte offset, value); doc-level schema errors are
    returned as (offset, JsonTraceError) items so they sort with the event errors (reading J11)."""
    i = _ws(s, 0)
    if i == len(s):
        raise JsonTraceError(E_SYNTAX, 0, base + i, "empty document")
    out = []

    def array(i):
        i = _ws(s, i + 1)
        if i < len(s) and s[i] == "]":
            return i + 1
        while True:
            v, j = _decode(s, i, base)
            out.append((base + i, v))
            j = _ws(s, j)
            if j < len(s) and s[j] == ",":
                i = _ws(s, j + 1)
                continue
            if j < len(s) and s[j] == "]":
                return j + 1
            raise JsonTraceError(E_SYNTAX, 0, base + j, "expected , or ] in the event array")

    root = i
    if s[i] == "[":
        i = array(i)
    elif s[i] == "{":
        found = 0
        i = _ws(s, i + 1)
        if i < len(s) and s[i] == "}":
            i += 1
        else:
            while True:
                k, i = _decode(s, i, base)
                if not isinstance(k, str) or isinstance(k, _Num):
                    raise JsonTraceError(E_SYNTAX, 0, base + i, "object key must be a string")
                i = _ws(s, i)
                if i >= len(s) or s[i] != ":":
                    raise JsonTraceError(E_SYNTAX, 0, base + i, "expected :")
                i = _ws(s, i + 1)
                if k == "traceEvents" and i < len(s) and s[i] == "[":
                    found += 1
                    i = array(i)
                else:
                    if k == "traceEvents":
                        found += 2  # present but not an array
                    _, i = _decode(s, i, base)
                i = _ws(s, i)
                if i < len(s) and s[i] == ",":
                    i = _ws(s, i + 1)
                    continue
                if i < len(s) and s[i] == "}":
                    i += 1
                    break
                raise JsonTraceError(E_SYNTAX, 0, base + i, "expected , or } in the root object")
        if found != 1:
            out.insert(0, (base + root, JsonTraceError(E_SCHEMA, F_TRACE_EVENTS, base + root,
                                                       "need exactly one traceEvents array")))
    else:
        raise JsonTraceError(E_SYNTAX, 0, base + i, "document root must be an object or an array")
    if _ws(s, i) != len(s):
        raise JsonTraceError(E_SYNTAX, 0, base + _ws(s, i), "trailing data after the document root")
    return out


def _ns(v, lo: int, hi: int):
    """Chrome "ts"/"dur" microseconds -> integer ns, exact (J5); None if not representable."""
    if not isinstance(v, _Num):
        return None
    m = _USEC.fullmatch(v)
    if not m:
        return None
    ns = int(m.group(2)) * 1000 + int((m.group(3) or "").ljust(3, "0"))
    ns = -ns if m.group(1) else ns
    return ns if lo <= ns <= hi else None


def _int(v, lo: int, hi: int):
    if not isinstance(v, _Num) or not re.fullmatch(r"-?\d+", v):
        return None
    x = int(v)
    return x if lo <= x <= hi else None


def _flag(v):
    if v is True or v is False:
        return int(v)
    return _int(v, 0, 1)


def _event(d, off: int, world: int):
    """Schema of one element (J6-J9): returns None (skipped, "ph" != "X") or the field tuple;
    raises the first failing field in the fixed order F_EVENT, F_PH, ..., F_BYTES (J11)."""
    def fail(f, msg):
        raise JsonTraceError(E_SCHEMA, f, off, msg)
    if not isinstance(d, dict):
        fail(F_EVENT, "event array element is not an object")
    ph = d.get("ph")
    if not isinstance(ph, str) or isinstance(ph, _Num):
        fail(F_PH, "ph missing or not a string")
    if ph != "X":
        return None
    ts = _ns(d.get("ts"), -(1 << 63), (1 << 63) - 1)
    if ts is None:
        fail(F_TS, "ts missing or not microseconds with <= 3 decimals in int64 ns")
    dur = _ns(d.get("dur"), 0, (1 << 32) - 1)
    if dur is None:
        fail(F_DUR, "dur missing, negative, or not microseconds with <= 3 decimals in uint32 ns")
    pid = _int(d.get("pid"), 0, world - 1)
    if pid is None:
        fail(F_PID, "pid missing or not a rank < world")
    cat = d.get("cat")
    if isinstance(cat, _Num) or cat not in KIND_NAMES:
        fail(F_CAT, "cat missing or not an event kind")
    kind = KIND_NAMES.index(cat)
    a = d.get("args", {})
    if not isinstance(a, dict):
        fail(F_ARGS, "args not an object")
    vals = {}
    for f, key, lo, hi in ((F_OP, "op", 0, 4095), (F_ITER_END, "iter_end", 0, 1), (F_MB, "mb", 0, 1023),
                           (F_CHUNK, "chunk", 0, 7), (F_BWD, "bwd", 0, 1), (F_WARMUP, "warmup", 0, 1)):
        if key not in a:
            vals[key] = 0
            continue
        x = _flag(a[key]) if hi == 1 else _int(a[key], lo, hi)
        if x is None:
            fail(f, f"args.{key} out of range / wrong type")
        vals[key] = x
    group, peer = None, 0
    if 1 <= kind <= 4:
        g = a.get("group")
        if not isinstance(g, list) or not g:
            fail(F_GROUP, "collective without a non-empty group list")
        group = []
        for x in g:
            y = _int(x, 0, world - 1)
            if y is None or (group and y <= group[-1]):
                fail(F_GROUP, "group members must be ascending ranks < world")
            group.append(y)
        group = tuple(group)
    elif kind >= 5:
        peer = _int(a.get("peer"), 0, world - 1)
        if peer is None:
            fail(F_PEER, "send/recv without a peer rank < world")
    pay = 0
    if "bytes" in a:
        pay = _int(a["bytes"], 0, (1 << 32) - 1)
        if pay is None:
            fail(F_BYTES, "args.bytes not a uint32")
    ko = kind | (vals["iter_end"] << 3) | (vals["op"] << 4)
    meta = vals["mb"] | (vals["chunk"] << 10) | (vals["bwd"] << 13) | (vals["warmup"] << 14)
    return pid, ts, dur, ko, meta, group, peer, pay


def parse(docs: list[bytes], tp: int, pp: int, dp: int):
    """Per-rank (or merged) JSON documents -> (tracegen.Trace columns, n_skipped).

    Bytes are decoded as Latin-1 so that string positions are byte offsets (J10). Any syntax
    error wins over every schema error (J11); among schema errors the one at the smallest byte
    offset is raised."""
    from tracegen import Trace  # the shared input container (no arithmetic)
    world = tp * pp * dp
    items, base = [], 0
    for b in docs:
        items.extend(_doc_events(b.decode("latin-1"), base))
        base += len(b)
    evs, skipped = [], 0
    for off, v in items:
        if isinstance(v, JsonTraceError):
            raise v
        e = _event(v, off, world)
        if e is None:
            skipped += 1
        else:
            evs.append((off,) + e)
    # program order per rank: by local start time, ties by position in the input (J3)
    evs.sort(key=lambda e: (e[1], e[2], e[0]))
    n = len(evs)
    ro = np.zeros(world + 1, dtype=np.uint64)
    for e in evs:
        ro[e[1] + 1] += 1
    ro = np.cumsum(ro).astype(np.uint64)
    # communicators: distinct participant lists in order of first use in that order (J4)
    comm_id, groups = {}, []
    for e in evs:
        if e[6] is not None and e[6] not in comm_id:
            comm_id[e[6]] = len(groups)
            groups.append(e[6])
    coff = np.zeros(len(groups) + 1, dtype=np.uint64)
    for k, g in enumerate(groups):
        coff[k + 1] = coff[k] + len(g)
    mem = np.array([x for g in groups for x in g], dtype=np.uint32)
    cols = dict(start_ns=np.array([e[2] for e in evs], dtype=np.int64).reshape(n),
                dur_ns=np.array([e[3] for e in evs], dtype=np.uint32).reshape(n),
                kind_op=np.array([e[4] for e in evs], dtype=np.uint16).reshape(n),
                meta=np.array([e[5] for e in evs], dtype=np.uint16).reshape(n),
                comm=np.array([comm_id[e[6]] if e[6] is not None else e[7] for e in evs], dtype=np.uint32).reshape(n),
                payload=np.array([e[8] for e in evs], dtype=np.uint32).reshape(n))
    return Trace(tp, pp, dp, ro, coff, mem, **cols), skipped


def _usec3(ns: int) -> str:
    a = -ns if ns < 0 else ns
    return ("-" if ns < 0 else "") + f"{a // 1000}.{a % 1000:03d}"


def emit(trace, ev_inst, start=None) -> bytes:
    """Merged Chrome Tracing document of the whole job, byte format J12.

    ``ev_inst``: matched instance id per event (UINT32_MAX for compute events), e.g. oracle.run's
    "ev_inst"; ``start``: per-event timestamps to write (default trace.start_ns; pass the aligned
    starts of ``oracle.align`` for the aligned timeline)."""
    start = trace.start_ns if start is None else start
    ro = trace.rank_offsets.astype(np.int64)
    coff, cmem = trace.comm_offsets.astype(np.int64), trace.comm_members
    rank = np.repeat(np.arange(trace.world), np.diff(ro))
    order = sorted(range(trace.n_events), key=lambda i: (int(start[i]), int(rank[i]), i))
    lines = []
    for i in order:
        ko, m = int(trace.kind_op[i]), int(trace.meta[i])
        kind, iend, op = ko & 7, (ko >> 3) & 1, ko >> 4
        args = []
        if op:
            args.append(f'"op":{op}')
        if iend:
            args.append('"iter_end":true')
        for key, v in (("mb", m & 1023), ("chunk", (m >> 10) & 7), ("bwd", (m >> 13) & 1), ("warmup", (m >> 14) & 1)):
            if v:
                args.append(f'"{key}":{v}')
        if 1 <= kind <= 4:
            c = int(trace.comm[i])
            args.append('"group":[' + ",".join(str(int(x)) for x in cmem[coff[c]:coff[c + 1]]) + "]")
        elif kind >= 5:
            args.append(f'"peer":{int(trace.comm[i])}')
        if int(trace.payload[i]):
            args.append(f'"bytes":{int(trace.payload[i])}')
        if kind != 0:
            args.append(f'"related_sync_op":{int(ev_inst[i])}')
        name = KIND_NAMES[kind]
        lines.append(f'{{"name":"{name}","cat":"{name}","ph":"X","ts":{_usec3(int(start[i]))},'
                     f'"dur":{_usec3(int(trace.dur_ns[i]))},"pid":{int(rank[i])},"tid":0,"args":{{{",".join(args)}}}}}')
    return ('{"traceEvents":[' + ",".join("\n" + x for x in lines) + "\n]}\n").encode()
