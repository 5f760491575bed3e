#!/usr/bin/env python3
"""A/B experiments on build-time variants of the ECM ladder kernel (ecm_kernels.cuh knobs).

    python tools/ecm_ab.py build [--L 6] NAME "-DECM_SWAP_BRANCH=1 -DECM_MIN_BLOCKS=7" [NAME2 "FLAGS2" ...]
        compiles csrc/ecm_l<L>.cu and mulmod_l<L>.cu with the flags and links it with the product objects of
        paper_1310_3809_b200/_build into tools/_variants/libecmgpu_NAME.so (here, on CPU)
    python tools/ecm_ab.py time [--curves 1048576,131072] [--B1 50000] [--L 6] NAME ...
        (GPU box) one subprocess per variant ("base" = the product library): event-timed
        ecm_stage1_batch launches on C3-shaped inputs, the outputs compared with the product
        library's on a strided sample; one JSON line per (variant, curves).
Not a bench line: experiments only.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "tools", "_variants")


def build(pairs, L=6):
    """Variant NAME = the product objects with ecm_l<L>.cu and mulmod_l<L>.cu (L = 0: every .cu)
    recompiled with FLAGS."""
    import concurrent.futures as cf
    from paper_1310_3809_b200 import build as B
    B.build()
    os.makedirs(VAR, exist_ok=True)
    objs = sorted(os.path.join(B.BUILD, f) for f in os.listdir(B.BUILD) if f.endswith(".o"))
    # single-width library (small enough to ship several to the GPU box): the dispatchers are rebuilt
    # with -DECM_ONLY_L and only that width's kernels are linked
    srcs = [f"ecm_l{L}.cu", f"mulmod_l{L}.cu", "ecm.cu", "mulmod.cu"] if L else \
        sorted(f for f in os.listdir(B.CSRC) if f.endswith(".cu"))
    if L:
        objs = [o for o in objs if os.path.basename(o)[:-2] in srcs + ["abi.cu"]]
    jobs = []
    for name, flags in pairs:
        for src in srcs:
            o = os.path.join(VAR, f"{src}_{name}.o")
            only = [f"-DECM_ONLY_L={L}"] if L else []
            jobs.append((name, src, o, [B.NVCC, *B.ARCH, *B.CFLAGS, *only, *flags.split(), "-c", os.path.join(B.CSRC, src),
                                        "-o", o]))
    with cf.ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        for (name, src, o, cmd), r in zip(jobs, ex.map(lambda j: subprocess.run(j[3], capture_output=True, text=True),
                                                       jobs)):
            if r.returncode:
                sys.stderr.write(r.stderr)
                raise SystemExit(f"nvcc failed for {name}/{src}")
    for name, _ in pairs:
        lib = os.path.join(VAR, f"libecmgpu_{name}.so")
        link = [os.path.join(VAR, f"{os.path.basename(x)[:-2]}_{name}.o") if os.path.basename(x)[:-2] in srcs else x
                for x in objs]
        r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *link],
                           capture_output=True, text=True)
        if r.returncode:
            raise SystemExit(r.stderr)
        print(lib)


def time_one(name, curves_list, B1, L):
    import numpy as np
    import torch
    from paper_1310_3809_b200 import _lib
    if name != "base":
        _lib.library_path = os.path.join(VAR, f"libecmgpu_{name}.so")
    import paper_1310_3809_b200 as eg
    from workload import ecm_config
    cfg = ecm_config("C3") if L == 6 else ecm_config("C5") if L == 8 else \
        ecm_config(L=L, nbits=32 * L - 2, pbits=64, B1=B1, curves=max(curves_list), seed=40 + L)
    if os.environ.get("AB_MULMOD", "1") == "1":
        from workload import mulmod_inputs
        a, b, n = (torch.from_numpy(v.T.copy()).cuda() for v in mulmod_inputs(1 << 24, L, seed=2))
        out = torch.empty_like(a)
        tags = [("mul", eg.ECM_LAYOUT_SLICED), ("sqr", eg.ECM_LAYOUT_SLICED | eg.ECM_SQUARE)]
        if os.environ.get("AB_AOS") == "1":  # the AoS kernels on the same arrays read as AoS triples
            tags += [("aos_mul", 0), ("aos_sqr", eg.ECM_SQUARE)]
        for tag, fl in tags:
            eg.ecm_mulmod_batch(a, b, n, out, L=L, iters=256, flags=fl)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            reps = int(os.environ.get("AB_REPS", "3"))
            for _ in range(reps):
                eg.ecm_mulmod_batch(a, b, n, out, L=L, iters=256, flags=fl)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            fpe = 2 * L * L if tag.endswith("mul") else (3 * L * L + L) // 2
            print(json.dumps({"variant": name, "mulmod": tag, "L": L, "ms": ms, "modmul_per_s": (1 << 24) * 256 / ms * 1e3,
                              "frac": (1 << 24) * 256 * fpe / (ms * 1e-3) / (148 * 32 * 1965e6),
                              "out_sum": int(out[:, :4096].to(torch.int64).sum().item())}), flush=True)
        del a, b, n, out
    for curves in curves_list:
        s = torch.from_numpy(cfg["sigmas"][:curves].copy()).cuda()
        eg.ecm_stage1_batch(cfg["N"], L, B1, s[:4096], want=("g",))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = eg.ecm_stage1_batch(cfg["N"], L, B1, s, want=("g",))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        idx = np.linspace(0, curves - 1, 64).astype(np.int64)
        print(json.dumps({"variant": name, "L": L, "B1": B1, "curves": curves, "ms": ms,
                          "curves_per_s": curves / ms * 1e3,
                          "g_sample": r["g"].cpu().numpy()[idx].astype(np.int64).sum(axis=1).tolist()[:8],
                          "status_sum": int(r["status"].to(torch.int64).sum().item())}), flush=True)


def main():
    if sys.argv[1] == "build":
        a = sys.argv[2:]
        L = 6
        if a and a[0] == "--L":
            L, a = int(a[1]), a[2:]
        build(list(zip(a[0::2], a[1::2])), L=L)
    elif sys.argv[1] == "time":
        import argparse
        ap = argparse.ArgumentParser()
        ap.add_argument("--curves", default="1048576,131072")
        ap.add_argument("--B1", type=int, default=50000)
        ap.add_argument("--L", type=int, default=6)
        ap.add_argument("names", nargs="+")
        a = ap.parse_args(sys.argv[2:])
        for n in a.names:
            subprocess.run([sys.executable, __file__, "_one", n, a.curves, str(a.B1), str(a.L)], check=False)
    elif sys.argv[1] == "_one":
        time_one(sys.argv[2], [int(x) for x in sys.argv[3].split(",")], int(sys.argv[4]), int(sys.argv[5]))


if __name__ == "__main__":
    main()
