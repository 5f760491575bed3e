"""A/B of the two ecm_mulmod_batch kernels (CTA-tile streaming vs warp-tile) over chain
length K, layout and width: event-timed on the launching stream, inputs resident in HBM.

    python tools/stream_ab.py [--count 16777216] [--out gpurun_out/stream_ab.json]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=1 << 24)
    ap.add_argument("--out", default="gpurun_out/stream_ab.json")
    ap.add_argument("--widths", default="6,4,8,12,16")
    ap.add_argument("--ks", default=None, help="chain lengths (default 1,2,4,8,16,256 at L=6, else 1,256)")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    import paper_1310_3809_b200 as eg
    from paper_1310_3809_b200 import build
    from workload import mulmod_inputs
    build.build()
    hbm = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6537.3) if os.path.exists("MEASURED_PEAKS.json") else 6537.3
    rows = []

    def timeit(fn, reps):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    for L in [int(w) for w in args.widths.split(",")]:
        count = args.count
        a, b, n = mulmod_inputs(count, L, seed=7)
        A, B, N = (torch.from_numpy(x).cuda() for x in (a, b, n))
        SA, SB, SN = (x.t().contiguous() for x in (A, B, N))
        O, SO = torch.empty_like(A), torch.empty_like(SA)
        Ks = [int(k) for k in args.ks.split(",")] if args.ks else ((1, 2, 4, 8, 16, 256) if L == 6 else (1, 256))
        for K in Ks:
            ref = {}
            for layout in ("aos", "sliced"):
                for kern, kf in (("stream", eg.ECM_KERNEL_STREAM), ("warp", eg.ECM_KERNEL_WARP)):
                    if layout == "aos":
                        fn = lambda: eg.ecm_mulmod_batch(A, B, N, O, L=L, iters=K, flags=kf)  # noqa: E731
                    else:
                        fn = lambda: eg.ecm_mulmod_batch(SA, SB, SN, SO, L=L, iters=K,  # noqa: E731
                                                         flags=kf | eg.ECM_LAYOUT_SLICED)
                    ms = timeit(fn, 20 if K <= 16 else args.reps)
                    res = (O if layout == "aos" else SO.t()).cpu().numpy()
                    key = layout
                    same = None
                    if key in ref:
                        same = bool(np.array_equal(ref[key], res))
                    else:
                        ref[key] = res
                    gbs = count * 16 * L / (ms * 1e-3) / 1e9
                    row = {"L": L, "K": K, "layout": layout, "kernel": kern, "ms": ms,
                           "modmul_per_s": count * K / (ms * 1e-3), "hbm_gbs": gbs, "hbm_frac": gbs / hbm,
                           "fpe_frac": count * K * 2 * L * L / (ms * 1e-3) / 9.30624e12, "equal_other_kernel": same}
                    rows.append(row)
                    print(json.dumps(row), flush=True)
        del A, B, N, SA, SB, SN, O, SO
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
