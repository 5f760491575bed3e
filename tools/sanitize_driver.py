#!/usr/bin/env python3
"""Small invocations of every launch path, for compute-sanitizer (memcheck / racecheck /
initcheck / synccheck): AoS and sliced layouts, ragged tiles, square mode, all REDC variants,
host-buffer staging, ECM_CHECK, every ECM width (one-lane and four-lane kernels), ablation and
prime-ladder variants."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1310_3809_b200 as eg  # noqa: E402
from workload import ecm_config, mulmod_inputs  # noqa: E402

torch.cuda.set_device(0)
for L in (4, 6, 8, 12, 16):
    a, b, n = mulmod_inputs(32 * 3 + 5, L, seed=L, lazy=True)
    A, B, N = (torch.from_numpy(x).cuda() for x in (a, b, n))
    for fl in (0, eg.ECM_SQUARE, eg.ECM_CANONICAL, eg.ECM_CHECK, eg.ECM_REDC_KNOWNLOW, eg.ECM_REDC_BLOCKTHM,
               eg.ECM_REDC_CLASSIC, eg.ECM_REDC_BLOCKTHM | eg.ECM_SQUARE):
        eg.ecm_mulmod_batch(A, B, N, L=L, iters=2, flags=fl)
    S = [torch.from_numpy(x.T.copy()).cuda() for x in (a, b, n)]
    eg.ecm_mulmod_batch(*S, L=L, iters=2, flags=eg.ECM_LAYOUT_SLICED)
    eg.ecm_mulmod_batch(a, b, n, L=L, iters=2, flags=eg.ECM_HOST_BUFFERS)
    cfg = ecm_config(L=L, nbits=32 * L - 2, pbits=30, B1=60, curves=37, seed=L)
    s = torch.from_numpy(cfg["sigmas"]).cuda()
    eg.ecm_stage1_batch(cfg["N"], L, cfg["B1"], s)  # small batch: the 4-lane kernel
    eg.ecm_stage1_batch(cfg["N"], L, cfg["B1"], s, flags=eg.ECM_KERNEL_LANES1)
    seeds = torch.from_numpy((cfg["sigmas"] % np.uint64((1 << 30) - 1)) + np.uint64(1)).cuda()
    for fl in (0, eg.ECM_KERNEL_LANES1):  # the small-parameter family (§8(f) N4), both kernels
        eg.ecm_stage1_batch(cfg["N"], L, cfg["B1"], seeds, flags=eg.ECM_CURVE_SMALL | fl)
    eg.ecm_ladder_batch(cfg["N"], L, 12345, s)
    if L in (6, 8):
        for fl in (eg.ECM_EAGER, eg.ECM_REDC_CLASSIC, eg.ECM_PRIME_LADDERS):
            eg.ecm_stage1_batch(cfg["N"], L, cfg["B1"], s, flags=fl, want=("g",))
    eg.ecm_stage1_batch(cfg["N"], L, cfg["B1"], cfg["sigmas"].copy(), flags=eg.ECM_HOST_BUFFERS)
# CTA-tile streaming kernel (K <= 4): full 256-element tiles through the bulk-copy ring + ragged tail
for L in (6, 16):
    for count, fl in ((256 * 3 + 5, 0), (256 * 3 + 4, eg.ECM_LAYOUT_SLICED), (256 * 3 + 4, eg.ECM_SQUARE)):
        a, b, n = mulmod_inputs(count, L, seed=L + 1, lazy=True)
        if fl & eg.ECM_LAYOUT_SLICED:
            a, b, n = (x.T.copy() for x in (a, b, n))
        A, B, N = (torch.from_numpy(x).cuda() for x in (a, b, n))
        eg.ecm_mulmod_batch(A, B, N, L=L, iters=1, flags=fl | eg.ECM_KERNEL_STREAM)
torch.cuda.synchronize()
print("sanitize driver done")
