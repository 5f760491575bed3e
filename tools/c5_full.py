#!/usr/bin/env python3
"""C5 end to end on one GPU: ECM stage 1, B1 = 250000, 2^22 curves on the 254-bit composite with a
planted 80-bit factor (the 8-GPU configuration; an 8-rank run computes exactly these curves, one
contiguous eighth per rank).  Event-timed; 16 strided curves checked against the oracle; every
flagged g checked by division.  One JSON line.  Not a bench line.

    python tools/c5_full.py [--curves 4194304] [--out gpurun_out/c5_full.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--curves", type=int, default=None)
    ap.add_argument("--check", type=int, default=16)
    ap.add_argument("--out", default="gpurun_out/c5_full.json")
    a = ap.parse_args()
    import torch
    import oracle
    import paper_1310_3809_b200 as eg
    from workload import ecm_config
    cfg = ecm_config("C5")
    L, B1 = cfg["L"], cfg["B1"]
    curves = a.curves or cfg["curves"]
    sig = torch.from_numpy(cfg["sigmas"][:curves].copy()).cuda()
    eg.ecm_stage1_batch(cfg["N"], L, B1, sig[:1024], want=("g",))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = eg.ecm_stage1_batch(cfg["N"], L, B1, sig, want=("X", "Z", "g"))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = r["status"].cpu().numpy()
    g = r["g"].cpu().numpy()
    flagged = np.nonzero(st == 1)[0]
    bad_g = sum(1 for i in flagged if cfg["N"] % eg.limbs_to_int(g[i]) != 0)
    found_p = sum(1 for i in flagged if eg.limbs_to_int(g[i]) == cfg["p"])
    idx = np.linspace(0, curves - 1, a.check).astype(np.int64)
    k, kb = oracle.stage1_k(B1)
    t0 = time.perf_counter()
    w = oracle.ecm_stage1_mt(cfg["N"], L, k, cfg["sigmas"][idx])
    cpu_s = time.perf_counter() - t0
    mism = 0
    for key in ("X", "Z", "g"):
        got = r[key].cpu().numpy()[idx]
        mism += int((got != w[key]).any(axis=1).sum())
    mism += int((st[idx] != w["status"]).sum())
    per_rank = curves // 8
    shard_flags = [int((st[j * per_rank:(j + 1) * per_rank] == 1).sum()) for j in range(8)]
    out = {"workload": f"C5: {curves} curves, B1={B1}, {cfg['nbits']}-bit N (planted {cfg['pbits']}-bit p), 1 GPU",
           "ms": ms, "curves_per_s": curves / ms * 1e3, "k_bits": kb,
           "modmul_per_s": curves / ms * 1e3 * (kb - 1) * 10,
           "frac": curves / (ms * 1e-3) * (kb - 1) * (18 * L * L + 2 * L) / (148 * 32 * 1965e6),
           "flagged": int(flagged.size), "flagged_g_is_p": found_p, "flagged_g_not_dividing_N": bad_g,
           "flags_per_rank_shard_of_8": shard_flags,
           "oracle_checked": int(a.check), "oracle_mismatches": mism, "oracle_seconds": cpu_s}
    print(json.dumps(out), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        f.write(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
