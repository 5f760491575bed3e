#!/usr/bin/env python3
"""Small-batch ECM stage 1: one-lane vs four-lane kernel over the curve count (the crossover that
sets kCoopMaxCurvesPerSM).  Event-timed on the launching stream after warm-up; one JSON line per
(count, kernel).  Not a bench line.

    python tools/ecm_lat.py [--B1 2000] [--counts 256,1024,...] [--out gpurun_out/ecm_lat.jsonl]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B1", type=int, default=2000)
    ap.add_argument("--L", type=int, default=6)
    ap.add_argument("--counts", default="32,256,1024,2048,4096,4736,6144,8192,16384,32768")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/ecm_lat.jsonl")
    a = ap.parse_args()
    import torch
    import paper_1310_3809_b200 as eg
    from workload import ecm_config
    cfg = ecm_config("C3") if a.L == 6 else ecm_config("C5")
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "a") as f:
        for count in [int(x) for x in a.counts.split(",")]:
            s = torch.from_numpy(cfg["sigmas"][:count].copy()).cuda()
            outs = {}
            for name, fl in (("lanes1", eg.ECM_KERNEL_LANES1), ("lanes4", eg.ECM_KERNEL_LANES4), ("default", 0)):
                r = eg.ecm_stage1_batch(cfg["N"], a.L, a.B1, s, flags=fl, want=("X", "Z", "g"))
                torch.cuda.synchronize()
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.reps + 1)]
                ev[0].record()
                for k in range(a.reps):
                    r = eg.ecm_stage1_batch(cfg["N"], a.L, a.B1, s, flags=fl, want=("X", "Z", "g"))
                    ev[k + 1].record()
                torch.cuda.synchronize()
                ms = min(ev[k].elapsed_time(ev[k + 1]) for k in range(a.reps))
                outs[name] = r
                line = {"L": a.L, "B1": a.B1, "count": count, "kernel": name, "ms": ms,
                        "curves_per_s": count / ms * 1e3,
                        "same_as_lanes1": all(torch.equal(r[k], outs["lanes1"][k]) for k in ("X", "Z", "g", "status"))}
                print(json.dumps(line), flush=True)
                f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
