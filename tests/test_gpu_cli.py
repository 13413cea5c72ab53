"""The command line (python -m paper_2507_19845_b200 analyze) end to end on the GPU, -m gpu: per-rank
JSON files -> report + merged aligned document, the document byte-exact against the oracle chain
(parse -> run -> align -> emit); a malformed file -> exit code 2 with the error in the report."""
import json
import os
import subprocess
import sys

import pytest

import oracle
import tracegen as tg
from oracle import chrome_json as cj
from tracegen import chrome, configs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cli(args):
    return subprocess.run([sys.executable, "-m", "paper_2507_19845_b200", "analyze", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_cli_report_and_aligned_document(tmp_path):
    cfg = configs.c1(seed=4, iterations=6)
    docs = chrome.rank_documents(tg.generate(cfg), messy=True, seed=3)
    files = []
    for r, d in enumerate(docs):
        f = tmp_path / f"rank{r}.json"
        f.write_bytes(d)
        files.append(str(f))
    out = tmp_path / "merged.json"
    p = _cli(["--tp", "2", "--pp", "2", "--dp", "2", "--align-ref", "0", "--emit", str(out), *files])
    assert p.returncode == 0, p.stderr
    rep = json.loads(p.stdout)
    assert rep["ingest"]["n_events"] > 0 and rep["ingest"]["n_skipped"] == 8
    assert rep["windows"][0]["verdicts"].get("5") in ("compute_slow", "both")  # c1's throttled rank
    assert rep["blame"]["top_rank"] == 5
    t, _ = cj.parse(docs, cfg.tp, cfg.pp, cfg.dp)
    o = oracle.run(t, oracle.Config())
    al = oracle.align(t, 0)
    assert out.read_bytes() == cj.emit(t, o["ev_inst"], start=al["al_start"])


def test_cli_rejects_malformed_file(tmp_path):
    f = tmp_path / "bad.json"
    f.write_bytes(b'{"traceEvents":[{"cat":"compute","ph":"X","ts":1,"dur":2,"pid":9}]}')
    p = _cli(["--tp", "1", "--pp", "1", "--dp", "2", str(f)])
    assert p.returncode == 2
    rep = json.loads(p.stdout)
    assert rep["error"]["kind"] == "schema" and rep["error"]["field"] == cj.F_PID
