#!/usr/bin/env python3
"""Time one ECM stage-1 launch on a C3-shaped workload (CUDA events, after warm-up); prints JSON.
Used for A/B experiments on kernel variants (not a bench line)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_3809_b200 as eg  # noqa: E402
from workload import ecm_config  # noqa: E402

B1 = int(os.environ.get("B1", 50000))
curves = int(os.environ.get("CURVES", 1 << 20))
L = int(os.environ.get("L", 6))
cfg = ecm_config("C3") if L == 6 else ecm_config("C5")
s = torch.from_numpy(cfg["sigmas"][:curves].copy()).cuda()
eg.ecm_stage1_batch(cfg["N"], L, B1, s[:8192], want=("g",))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r = eg.ecm_stage1_batch(cfg["N"], L, B1, s, want=("g",))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(json.dumps({"tag": os.environ.get("TAG", ""), "L": L, "B1": B1, "curves": curves, "ms": ms,
                  "curves_per_s": curves / ms * 1e3, "flagged": int((r["status"] == 1).sum().item())}))
