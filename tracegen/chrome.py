"""tracegen.chrome — per-rank Chrome-trace JSON files of a generated trace (TEST INFRASTRUCTURE,
shared input source; holds none of MegaScan's analysis arithmetic).

Writes what the paper's tracer leaves on disk after training: "every rank has its own recorded
event sequence as a JSON file" (§3.2) with the metadata ``tracers.scope`` attaches
(micro-batch index, communication volume, peer rank) and, for collectives, "the global ID
list of all participating ranks". The schema is DESIGN.md §10d (readings J1-J12).

``messy=True`` (default) varies everything a real writer may vary and a parser must tolerate:
key order, whitespace / indentation, integer vs decimal timestamps, booleans vs 0/1, metadata
("ph":"M") events, unknown keys with nested values whose strings contain brackets, quotes and
escapes, top-level keys before / after "traceEvents", and adjacent events written out of time order.
"""
from __future__ import annotations

import numpy as np

KIND_NAMES = ("compute", "all_reduce", "all_gather", "reduce_scatter", "broadcast", "send", "recv")


def _us(ns: int, rng) -> str:
    """ns -> microseconds as a JSON number with <= 3 fractional digits (exact)."""
    s = "-" if ns < 0 else ""
    a = -ns if ns < 0 else ns
    q, r = divmod(a, 1000)
    if r == 0 and (rng is None or rng.random() < 0.5):
        return f"{s}{q}"
    f = f"{r:03d}"
    if rng is not None and rng.random() < 0.5:
        f = f.rstrip("0") or "0"
    return f"{s}{q}.{f}"


def _dumps_str(x: str) -> str:
    out = ['"']
    for ch in x:
        if ch == '"':
            out.append('\\"')
        elif ch == "\\":
            out.append("\\\\")
        elif ch == "\n":
            out.append("\\n")
        elif ord(ch) < 0x20:
            out.append(f"\\u{ord(ch):04x}")
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def _obj(items, sep_kv, sep_items):
    return "{" + sep_items.join(f'"{k}"{sep_kv}{v}' for k, v in items) + "}"


def rank_documents(trace, messy: bool = True, seed: int = 0) -> list[bytes]:
    """One JSON document per rank, events in program order up to local swaps."""
    rng = np.random.default_rng(seed) if messy else None
    ro = trace.rank_offsets.astype(np.int64)
    coff, cmem = trace.comm_offsets.astype(np.int64), trace.comm_members
    docs = []
    for r in range(trace.world):
        pretty = messy and r % 2 == 1
        kv, it = (": ", ", ") if pretty else (":", ",")
        nl = "\n  " if pretty else ""
        evs = []
        if messy:
            evs.append(_obj([("name", '"process_name"'), ("ph", '"M"'), ("pid", str(r)), ("tid", "0"),
                             ("args", _obj([("name", _dumps_str(f"rank {r}"))], kv, it))], kv, it))
        b, e = int(ro[r]), int(ro[r + 1])
        order = list(range(b, e))
        if messy:  # write some adjacent pairs out of time order (the parser sorts by ts)
            j = 0
            while j + 1 < len(order):
                if rng.random() < 0.05 and trace.start_ns[order[j]] != trace.start_ns[order[j + 1]]:
                    order[j], order[j + 1] = order[j + 1], order[j]
                    j += 2
                else:
                    j += 1
        for i in order:
            ko = int(trace.kind_op[i])
            kind, iend, op = ko & 7, (ko >> 3) & 1, ko >> 4
            m = int(trace.meta[i])
            mb, chunk, bwd, warm = m & 1023, (m >> 10) & 7, (m >> 13) & 1, (m >> 14) & 1
            name = KIND_NAMES[kind]
            if messy and kind == 0:
                name = f'{"bwd" if bwd else "fwd"} mb={mb} "chunk" {chunk}\\{{]}}' if rng.random() < 0.1 else f"layer_{op}"
            args = []
            if op or (messy and rng.random() < 0.3):
                args.append(("op", str(op)))
            if iend or (messy and rng.random() < 0.2):
                args.append(("iter_end", ("true" if iend else "false") if messy and rng.random() < 0.5 else str(iend)))
            for key, v in (("mb", mb), ("chunk", chunk), ("bwd", bwd), ("warmup", warm)):
                if v or (messy and rng.random() < 0.2):
                    args.append((key, str(v)))
            if 1 <= kind <= 4:
                c = int(trace.comm[i])
                args.append(("group", "[" + it.join(str(int(x)) for x in cmem[coff[c]:coff[c + 1]]) + "]"))
            elif kind >= 5:
                args.append(("peer", str(int(trace.comm[i]))))
            if int(trace.payload[i]) or (messy and kind >= 5 and rng.random() < 0.5):
                args.append(("bytes", str(int(trace.payload[i]))))
            if messy and rng.random() < 0.1:
                args.append(("stream", _dumps_str("nccl:0 } ] \" ,")))
            if messy and rng.random() < 0.05:
                args.append(("extra", '{"k": [1, 2.5e3, {"z": "]}\\u0041"}, [], {}], "t": true, "n": null}'))
            if messy:
                rng.shuffle(args)
            items = [("name", _dumps_str(name)), ("cat", f'"{KIND_NAMES[kind]}"'), ("ph", '"X"'),
                     ("ts", _us(int(trace.start_ns[i]), rng)), ("dur", _us(int(trace.dur_ns[i]), rng)),
                     ("pid", str(r)), ("tid", str(0 if kind == 0 else 1)), ("args", _obj(args, kv, it))]
            if messy:
                rng.shuffle(items)
            evs.append(_obj(items, kv, it))
        body = "[" + nl + ("," + nl).join(evs) + ("\n" if pretty else "") + "]"
        top = [("traceEvents", body)]
        if messy and r % 3 == 1:
            top.insert(0, ("otherData", '{"note": "brackets } ] in \\"strings\\"", "list": [1, [2, {}]]}'))
        if messy and r % 3 == 2:
            top.append(("displayTimeUnit", '"ns"'))
        docs.append((_obj(top, kv, it) + ("\n" if messy else "")).encode())
    return docs


def rank_documents_fast(trace, threads: int = 0) -> tuple[bytes, np.ndarray]:
    """``rank_documents(trace, messy=False)`` written by the C++ generator library (multi-threaded),
    already concatenated: (bytes, doc_offsets[W+1])."""
    import ctypes
    from . import _load
    lib = _load()
    f = lib.gen_chrome
    f.restype = ctypes.c_int64
    f.argtypes = [ctypes.c_uint32] + [ctypes.c_void_p] * 11 + [ctypes.c_int]
    cols = [np.ascontiguousarray(a) for a in (trace.rank_offsets, trace.start_ns, trace.dur_ns, trace.kind_op, trace.meta,
                                              trace.comm, trace.payload, trace.comm_offsets, trace.comm_members)]
    ptrs = [c.ctypes.data for c in cols]
    off = np.zeros(trace.world + 1, dtype=np.uint64)
    n = f(trace.world, *ptrs, None, off.ctypes.data, threads)
    buf = np.empty(max(n, 1), dtype=np.uint8)
    f(trace.world, *ptrs, buf.ctypes.data, off.ctypes.data, threads)
    return buf[:n].tobytes(), off


def concat(docs: list[bytes]) -> tuple[bytes, np.ndarray]:
    """Concatenate documents; returns (bytes, doc_offsets[n_docs+1])."""
    off = np.zeros(len(docs) + 1, dtype=np.uint64)
    for i, d in enumerate(docs):
        off[i + 1] = off[i] + len(d)
    return b"".join(docs), off
