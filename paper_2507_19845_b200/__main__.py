"""Command line: the paper's workflow on the GPU (§3.2).

    python -m paper_2507_19845_b200 analyze --tp 2 --pp 2 --dp 2 [--window-iters K] [--align-ref R]
                                            [--emit merged.json] rank0.json rank1.json ...

Per-rank tracer files are parsed on the GPU (scan_ingest_json), analysed (scan_analyze:
matching, decomposition, 3-stage detection, source-vs-victim walk), optionally aligned onto a
reference rank's clock (scan_align), every wait is blamed (scan_blame), and a JSON report goes to
stdout. ``--emit`` writes the merged Chrome Tracing document with related_sync_op (P:L119-125,
P:L133), on the aligned timeline when ``--align-ref`` is given. Exit code 0 on success, 2 on a
rejected input (the report then holds the error).
"""
from __future__ import annotations

import argparse
import json
import sys

import numpy as np

VERDICTS = {0: "none", 1: "compute_slow", 2: "link_slow", 3: "both", 4: "exonerated", 5: "insufficient"}
LABELS = {0: "clean", 1: "source_rank", 2: "source_link", 3: "victim", 4: "unattributed"}


def analyze(args) -> int:
    import paper_2507_19845_b200 as ms
    docs = [open(f, "rb").read() for f in args.files]
    s = ms.Scan(args.device)
    report: dict = {"files": len(docs), "json_bytes": sum(len(d) for d in docs)}
    try:
        ing = s.ingest_json(docs, args.tp, args.pp, args.dp)
    except ms.JsonTraceError as e:
        report["error"] = {"kind": {1: "syntax", 2: "schema"}.get(e.kind, e.kind), "field": e.field,
                           "byte_offset": e.offset, "message": str(e)}
        print(json.dumps(report, indent=1))
        return 2
    except ms.ScanError as e:  # the parsed job fails the load schema (e.g. a rank outside its group)
        report["error"] = {"kind": "scan", "status": e.status, "message": str(e)}
        print(json.dumps(report, indent=1))
        return 2
    report["ingest"] = ing
    try:
        return _analyze_loaded(s, args, report)
    except ms.ScanError as e:  # a rejected job (membership schema, capacity, alignment): exit 2 with the report
        report["error"] = {"kind": "scan", "status": e.status, "message": str(e)}
        print(json.dumps(report, indent=1, default=int))
        return 2
    finally:
        s.close()


def _analyze_loaded(s, args, report) -> int:
    import paper_2507_19845_b200 as ms
    res = s.analyze(ms.DetectConfig(window_iters=args.window_iters), ms.LocalizeConfig())
    report["analysis"] = {"fused": bool(res.get("fused")), "match": res["match"], "detect": res["detect"],
                          "localize": res["localize"]}
    W = args.tp * args.pp * args.dp
    verdict = s.export("wl_verdict").reshape(-1, W)
    label = s.export("lb_label").reshape(-1, W)
    report["windows"] = [
        {"window": w,
         "verdicts": {str(r): VERDICTS.get(int(v), int(v)) for r, v in enumerate(verdict[w]) if v},
         "sources": [r for r, v in enumerate(label[w]) if v in (1, 2)],
         "victims": [r for r, v in enumerate(label[w]) if v == 3]}
        for w in range(verdict.shape[0])]
    lk_slow = s.export("lk_slow")
    if lk_slow.size:
        src, dst, win = s.export("lk_src"), s.export("lk_dst"), s.export("lk_window")
        report["slow_links"] = [{"window": int(win[i]), "src": int(src[i]), "dst": int(dst[i])}
                                for i in np.flatnonzero(lk_slow)]
    if args.align_ref is not None:
        report["alignment"] = s.align(args.align_ref)
    bl = s.blame()
    inflicted = s.export("bl_inflicted")
    top = np.argsort(-inflicted.astype(np.float64), kind="stable")[:args.top]
    report["blame"] = dict(bl, top_inflicting_ranks=[{"rank": int(r), "inflicted_wait_ns": int(inflicted[r])}
                                                     for r in top if inflicted[r]])
    if args.emit:
        doc = s.emit_chrome(aligned=args.align_ref is not None)
        with open(args.emit, "wb") as f:
            f.write(doc)
        report["emitted"] = {"path": args.emit, "bytes": len(doc), "aligned": args.align_ref is not None}
    print(json.dumps(report, indent=1, default=int))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2507_19845_b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    a = sub.add_parser("analyze", help="ingest per-rank JSON traces, analyse, report")
    a.add_argument("files", nargs="+")
    a.add_argument("--tp", type=int, required=True)
    a.add_argument("--pp", type=int, required=True)
    a.add_argument("--dp", type=int, required=True)
    a.add_argument("--window-iters", type=int, default=0, help="analysis window in iterations (0 = whole trace)")
    a.add_argument("--align-ref", type=int, default=None, help="align every rank onto this rank's clock")
    a.add_argument("--emit", default=None, help="write the merged, annotated Chrome Tracing document here")
    a.add_argument("--top", type=int, default=5, help="ranks listed in the blame summary")
    a.add_argument("--device", type=int, default=0)
    args = ap.parse_args(argv)
    return analyze(args)


if __name__ == "__main__":
    sys.exit(main())
