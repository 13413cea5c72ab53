"""Quick timing of the JSON ingest / emit leg of bench.py (scan_ingest_json, scan_emit_chrome) alone."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2507_19845_b200 as ms  # noqa: E402

torch.cuda.set_device(0)
r = bench.json_io(ms, torch, 0, torch.cuda.current_stream(0), 5, 3, False)
print(json.dumps({k: r[k] for k in ("value", "ms_per_call", "events_per_s")}))
print(json.dumps(r["kernels"]))
print(json.dumps(r["emit"]))
