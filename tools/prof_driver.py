#!/usr/bin/env python3
"""Single-launch drivers for ncu captures (tools/profile.sh).  Not a benchmark: numbers taken
under a profiler are never reported as bench values."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1310_3809_b200 as eg  # noqa: E402
from workload import ecm_config, mulmod_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("what", choices=["mulmod", "ecm"])
ap.add_argument("--L", type=int, default=6)
ap.add_argument("--count", type=int, default=1 << 24)
ap.add_argument("--iters", type=int, default=256)
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--curves", type=int, default=1 << 16)
ap.add_argument("--B1", type=int, default=50000)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--sliced", action="store_true", help="limb-sliced layout (the bench headline)")
ap.add_argument("--cfg", default="C3", help="ECM config for the modulus and seeds (C1, C3)")
a = ap.parse_args()
torch.cuda.set_device(0)
if a.what == "mulmod":
    x, y, n = (torch.from_numpy(v.T.copy() if a.sliced else v).cuda() for v in mulmod_inputs(a.count, a.L, seed=2))
    fl = a.flags | (eg.ECM_LAYOUT_SLICED if a.sliced else 0)
    for _ in range(a.reps):
        eg.ecm_mulmod_batch(x, y, n, L=a.L, iters=a.iters, flags=fl)
else:
    cfg = ecm_config(a.cfg) if a.L == 6 else ecm_config(L=a.L, nbits=32 * a.L - 2, pbits=64, B1=a.B1,
                                                            curves=a.curves, seed=40 + a.L)
    sig = cfg["sigmas"][: a.curves].copy()
    if a.flags & eg.ECM_CURVE_SMALL:
        sig = (sig % np.uint64((1 << 30) - 1)) + np.uint64(1)
    s = torch.from_numpy(sig).cuda()
    for _ in range(a.reps):
        eg.ecm_stage1_batch(cfg["N"], a.L, a.B1, s, flags=a.flags, want=("g",))
torch.cuda.synchronize()
print("done")
