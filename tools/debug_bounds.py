#!/usr/bin/env python3
"""Runtime check of the Lemma's lazy bound (reading G3) on real workloads: a debug
build of libecmgpu (-DECM_DEBUG_BOUNDS=1: every Montgomery product traps unless its raw output is
< 2N) runs every kernel path — mulmod at every width x mul/sqr x layout x REDC variant on lazy
operands up to 2N-1, and ECM stage 1 (Suyama and small-parameter curves, both kernels, ablation and
prime-ladder variants) — and any violated bound surfaces as a CUDA error.

    python tools/ecm_ab.py build --L 0 debug "-DECM_DEBUG_BOUNDS=1"     # here, on CPU (~5 min)
    python tools/debug_bounds.py                                        # on the GPU box
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def negative_control():
    """Operands far above 2N (a precondition violation, not checked without ECM_CHECK) must make
    the debug build trap — shows the check is live.  Runs in its own process (a trap ends the
    CUDA context)."""
    import torch
    from paper_1310_3809_b200 import _lib
    _lib.library_path = os.path.join(ROOT, "tools", "_variants", "libecmgpu_debug.so")
    import paper_1310_3809_b200 as eg
    L, count = 6, 256
    n = np.zeros((count, L), np.uint32)
    n[:, 0] = 0xFFFFFFFF  # n = 2^32 - 1 (odd, tiny)
    a = np.full((count, L), 0xFFFFFFFF, np.uint32)
    a[:, L - 1] = 0x3FFFFFFF  # a = b < R/4 but >> 2n
    A, N = torch.from_numpy(a).cuda(), torch.from_numpy(n).cuda()
    eg.ecm_mulmod_batch(A, A, N, L=L, iters=1, flags=eg.ECM_KERNEL_WARP)
    torch.cuda.synchronize()


def main():
    if "--negative" in sys.argv:
        negative_control()
        return
    import subprocess
    neg = subprocess.run([sys.executable, __file__, "--negative"], capture_output=True, text=True)
    trapped = neg.returncode != 0
    import torch
    from paper_1310_3809_b200 import _lib
    _lib.library_path = os.path.join(ROOT, "tools", "_variants", "libecmgpu_debug.so")
    import paper_1310_3809_b200 as eg
    from workload import ecm_config, mulmod_inputs
    torch.cuda.set_device(0)
    done = {"mulmod_products": 0, "ecm_curves": 0}
    count = 256 * 64  # whole tiles: no dead lanes
    for L in (4, 6, 8, 12, 16):
        a, b, n = mulmod_inputs(count, L, seed=90 + L, lazy=True)
        a[:64] = b[:64] = 0
        # extreme operands: 2n - 1 (computed per element in Python ints)
        for i in range(64, 128):
            nv = sum(int(w) << (32 * j) for j, w in enumerate(n[i]))
            v = 2 * nv - 1
            a[i] = b[i] = [(v >> (32 * j)) & 0xFFFFFFFF for j in range(L)]
        A, B, N = (torch.from_numpy(x).cuda() for x in (a, b, n))
        S = [torch.from_numpy(x.T.copy()).cuda() for x in (a, b, n)]
        for v in (eg.ECM_REDC_WORD, eg.ECM_REDC_KNOWNLOW, eg.ECM_REDC_BLOCKTHM, eg.ECM_REDC_CLASSIC,
                  eg.ECM_REDC_KARATSUBA):
            for sq in (0, eg.ECM_SQUARE):
                eg.ecm_mulmod_batch(A, B, N, L=L, iters=64, flags=v | sq)
                eg.ecm_mulmod_batch(*S, L=L, iters=64, flags=v | sq | eg.ECM_LAYOUT_SLICED)
                done["mulmod_products"] += 2 * count * 64
        eg.ecm_mulmod_batch(*S, L=L, iters=1, flags=eg.ECM_LAYOUT_SLICED | eg.ECM_KERNEL_STREAM)
        torch.cuda.synchronize()
        cfg = ecm_config(L=L, nbits=32 * L - 2, pbits=40, B1=2000, curves=2048, seed=95 + L)
        s = torch.from_numpy(cfg["sigmas"]).cuda()
        seeds = torch.from_numpy((cfg["sigmas"] % np.uint64((1 << 30) - 1)) + np.uint64(1)).cuda()
        runs = [(s, 0), (s, eg.ECM_KERNEL_LANES1), (s, eg.ECM_KERNEL_LANES4), (seeds, eg.ECM_CURVE_SMALL),
                (seeds, eg.ECM_CURVE_SMALL | eg.ECM_KERNEL_LANES1)]
        if L in (6, 8):
            runs += [(s, eg.ECM_EAGER), (s, eg.ECM_REDC_KNOWNLOW), (s, eg.ECM_REDC_BLOCKTHM), (s, eg.ECM_REDC_CLASSIC),
                     (s, eg.ECM_PRIME_LADDERS)]
        for sig, fl in runs:
            eg.ecm_stage1_batch(cfg["N"], L, cfg["B1"], sig, flags=fl, want=("g",))
            done["ecm_curves"] += sig.numel()
        torch.cuda.synchronize()
    out = {"lazy_bound_violations": 0, **done, "build": eg.ecm_version(),
           "negative_control_trapped": trapped,
           "negative_control_error": next((ln.strip()[:200] for ln in neg.stderr.splitlines()
                                           if "error" in ln.lower() and "CUDA" in ln), "")}
    print(json.dumps(out))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "debug_bounds.json"), "w") as f:
        f.write(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
