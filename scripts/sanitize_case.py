"""One small pass over every entry point of the library, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): `compute-sanitizer --tool racecheck python scripts/sanitize_case.py c1`.
Runs the fused and the general analysis, alignment, blame, the stream and the JSON ingest / emit on a
small job, and checks the analysis against the oracle (so a run that passes the sanitizer also
passed parity)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import tracegen as tg  # noqa: E402
from tracegen import configs  # noqa: E402
import paper_2507_19845_b200 as ms  # noqa: E402


def main(name: str):
    if name == "c1":
        tr = tg.generate(configs.c1(seed=1, iterations=2))
    elif name == "c2":
        tr = tg.generate(configs.c2(iterations=2))
    elif name == "c3":
        tr = tg.generate(configs.c3(iterations=1))
    else:
        raise SystemExit(f"unknown case {name}")
    ref = oracle.run(tr)
    for general in (False, True):
        s = ms.Scan(0)
        s.load(tr, start=True)
        if general:
            s.force_general(True)
        s.analyze(ms.DetectConfig(want_ref=True))
        got = s.export_all()
        for k, v in ref.items():
            if isinstance(v, np.ndarray):
                ok = np.allclose(got[k], v, rtol=1e-6, atol=0) if v.dtype == np.float64 else np.array_equal(got[k], v)
                assert ok, (name, general, k)
        s.align(0)
        s.blame()
        s.close()
    if name != "c3":
        s = ms.Scan(0)
        s.stream_open(tr, 1)
        for i in range(2):
            s.stream_push(ms.slice_iterations(tr, i, i + 1))
        s.close()
        from tracegen import chrome
        s = ms.Scan(0)
        s.ingest_json(chrome.rank_documents(tr, messy=True, seed=1), tr.tp, tr.pp, tr.dp)
        s.analyze()
        s.emit_chrome()
        s.close()
    print(f"sanitize case {name}: ok ({tr.n_events} events)")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c1")
