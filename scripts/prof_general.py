"""One general-path analysis of the full C3 job (for ncu -k regex:k_event_pass|k_assign ...)."""
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
s.force_general(True)
s.analyze()
s.set_timing(True)
s.analyze()
torch.cuda.synchronize()
print({k: round(v[0] / v[1], 3) for k, v in s.kernel_timing().items() if v[0] / v[1] > 0.2})
