#!/usr/bin/env python3
"""B200 analogue of the paper's Table 5: ECM stage 1 at the
paper's setting — 254-bit N (L = 8), B1 = 8192 — for the REDC forms x {eager, lazy} reduction,
plus the mulmod REDC forms on C2.  Prints one JSON object (bench hygiene: warm-up, CUDA events).
The reduction census per ladder step is structural (DESIGN.md §3 G5): lazy = 8 conditional
reductions (after add/sub only), eager = 8 + 10 (after every product) = 18.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_3809_b200 as eg  # noqa: E402
from workload import ecm_config, mulmod_inputs  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    torch.cuda.set_device(0)
    curves = int(os.environ.get("ABL_CURVES", 1 << 18))
    B1 = int(os.environ.get("ABL_B1", 8192))
    out = {"ecm": {}, "mulmod": {}, "setting": f"L=8 (254-bit N), B1={B1}, {curves} curves; C2 L=6 K=256"}
    cfg = ecm_config(L=8, nbits=254, pbits=64, B1=B1, curves=curves, seed=7)
    s = torch.from_numpy(cfg["sigmas"]).cuda()
    kb = eg.ecm_stage1_kbits(B1)
    names = {eg.ECM_REDC_WORD: "word", eg.ECM_REDC_KNOWNLOW: "knownlow", eg.ECM_REDC_BLOCKTHM: "blockthm",
             eg.ECM_REDC_CLASSIC: "classic"}
    ref = None
    for var, name in names.items():
        for eager, tag in ((eg.ECM_EAGER, "eager"), (0, "lazy")):
            ms = timed(lambda: eg.ecm_stage1_batch(cfg["N"], 8, B1, s, flags=var | eager, want=("g",)), reps=1)
            st = eg.ecm_stage1_batch(cfg["N"], 8, B1, s, flags=var | eager, want=("g",))["status"].cpu()
            if ref is None:
                ref = st
            assert torch.equal(st, ref)
            cps = curves / (ms * 1e-3)
            out["ecm"][f"{name}_{tag}"] = {"ms": ms, "curves_per_s": cps, "modmul_per_s": cps * (kb - 1) * 10,
                                          "reductions_per_step": 18 if eager else 8}
    base = out["ecm"]["classic_eager"]["curves_per_s"]
    for v in out["ecm"].values():
        v["ratio_vs_classic_eager"] = v["curves_per_s"] / base
    # Table 5 proper: the paper's schedule (prime-by-prime ladders, 11 products/step; 128,722
    # products per curve at B1 = 8192 — SURVEY §6) with/without Sections 2.2 and 2.3.
    from workload import ecm_config as _cfg
    prim = {}
    rows = [("without_optimizations", eg.ECM_REDC_CLASSIC | eg.ECM_EAGER),
            ("section_2_2_only", eg.ECM_REDC_CLASSIC),
            ("section_2_3_only", eg.ECM_REDC_BLOCKTHM | eg.ECM_EAGER),
            ("fully_optimized", eg.ECM_REDC_BLOCKTHM),
            ("b200_word_cios_lazy", eg.ECM_REDC_WORD)]
    mulmods_per_curve = 128722 if B1 == 8192 else None
    for name, fl in rows:
        f = fl | eg.ECM_PRIME_LADDERS
        ms = timed(lambda: eg.ecm_stage1_batch(cfg["N"], 8, B1, s, flags=f, want=("g",)), reps=1)
        st = eg.ecm_stage1_batch(cfg["N"], 8, B1, s, flags=f, want=("g",))["status"].cpu()
        assert torch.equal(st, ref)
        cps = curves / (ms * 1e-3)
        prim[name] = {"ms": ms, "curves_per_s": cps,
                      "modmul_per_s": cps * mulmods_per_curve if mulmods_per_curve else None}
    b = prim["without_optimizations"]["curves_per_s"]
    for v in prim.values():
        v["ratio"] = v["curves_per_s"] / b
    out["table5_prime_schedule"] = prim
    out["paper_table5_hd5770"] = {"without_optimizations": 1.0, "section_2_2_only": 1.031,
                                  "section_2_3_only": 1.076, "fully_optimized": 1.112}
    a, b, n = (torch.from_numpy(x).cuda() for x in mulmod_inputs(1 << 24, 6, seed=2))
    for var, name in list(names.items()) + [(eg.ECM_REDC_KARATSUBA, "karatsuba")]:
        for sq in (0, eg.ECM_SQUARE):
            ms = timed(lambda: eg.ecm_mulmod_batch(a, b, n, L=6, iters=256, flags=var | sq))
            out["mulmod"][f"{name}{'_sqr' if sq else ''}"] = {"ms": ms, "modmul_per_s": (1 << 24) * 256 / (ms * 1e-3)}
    del a, b, n
    # the paper's second Theorem (Karatsuba-level REDC, 2 instead of 3 half-size products for q*N,
    # PAPER.md:262-274) against the word-serial CIOS across widths
    out["width_karatsuba"] = {}
    for Lw in (6, 8, 12, 16):
        cnt = 1 << 23
        a, b, n = (torch.from_numpy(x).cuda() for x in mulmod_inputs(cnt, Lw, seed=4))
        row = {}
        for var, name in ((eg.ECM_REDC_WORD, "word"), (eg.ECM_REDC_KARATSUBA, "karatsuba")):
            for sq in (0, eg.ECM_SQUARE):
                ms = timed(lambda: eg.ecm_mulmod_batch(a, b, n, L=Lw, iters=64, flags=var | sq))
                row[f"{name}{'_sqr' if sq else ''}"] = cnt * 64 / (ms * 1e-3)
        out["width_karatsuba"][f"L{Lw}"] = row
        del a, b, n
    print(json.dumps(out))


if __name__ == "__main__":
    main()
