"""One analysis of a C3-shape job for profiling (ncu -k regex:k_stage): `python scripts/prof_case.py [iters]`."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import tracegen as tg  # noqa: E402
from tracegen import configs  # noqa: E402
import paper_2507_19845_b200 as ms  # noqa: E402

it = int(sys.argv[1]) if len(sys.argv) > 1 else 100
variant = int(sys.argv[2]) if len(sys.argv) > 2 else -1
cfg = configs.c3(iterations=it)
if len(sys.argv) > 3 and sys.argv[3] == "clean":  # no injected faults (no stage-1 rare path)
    cfg.faults = []
tr = tg.generate(cfg, with_start=False)
dev = {k: torch.from_numpy(np.ascontiguousarray(getattr(tr, k)).view(np.int16 if getattr(tr, k).dtype == np.uint16 else np.int32)).cuda()
       for k in ("dur_ns", "kind_op", "meta", "comm", "payload")}
s = ms.Scan(0)
s.fused_variant(variant)
s.load(tr, device_ptrs=True, cols=dev)
s.analyze()
s.set_timing(True)
for _ in range(3):
    s.analyze()
torch.cuda.synchronize()
print({k: round(v[0] / v[1], 4) for k, v in s.kernel_timing().items()})
