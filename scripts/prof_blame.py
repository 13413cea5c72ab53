"""One analysis + scan_blame of the full C3 job (for ncu -k regex:k_bl_)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import tracegen as tg  # noqa: E402
from tracegen import configs  # noqa: E402
import paper_2507_19845_b200 as ms  # noqa: E402

it = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
tr = tg.generate(configs.c3(iterations=it), with_start=False)
dev = {k: torch.from_numpy(np.ascontiguousarray(getattr(tr, k)).view(np.int16 if getattr(tr, k).dtype == np.uint16 else np.int32)).cuda()
       for k in ("dur_ns", "kind_op", "meta", "comm", "payload")}
s = ms.Scan(0)
s.load(tr, device_ptrs=True, cols=dev)
s.analyze()
s.set_timing(True)
s.blame()
torch.cuda.synchronize()
print({k: round(v[0] / v[1], 3) for k, v in s.kernel_timing().items() if k.startswith("k_bl")})
