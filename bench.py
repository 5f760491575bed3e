#!/usr/bin/env python3
"""bench.py — throughput of the paper's hot path on B200 (arXiv 1310.3809).

Default (N = 1): config C2 of BASELINE.json — 2^24 independent (a, b, N) triples of 192-bit
(L = 6) operands in the limb-sliced layout, K = 256 chained lazy Montgomery products per
triple; one step = one ecm_mulmod_batch over the whole batch (inputs resident in HBM,
1.15 GiB > L2).  Metric:
192-bit modmul/s.  The same JSON line carries ECM stage-1 curves/s on config C3 (B1 = 50000,
2^20 curves, 190-bit N) measured in the same run (`ecm`), the roofline of the dominant
kernel, the CPU oracle baseline, clocks sampled during the timed region, and the end-to-end
number through the public API with host buffers.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--no-ecm]
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N ...; mulmod shards are independent
replicas (weak scaling, no collective); ECM shards the 2^20 curves by contiguous ranges and
all-gathers the per-curve status bytes over NCCL (strong scaling).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

L = 6
C2_COUNT = 1 << 24
C2_ITERS = 256
FPE_MUL = 2 * L * L                      # 32x32->64 partial products per L-limb product
FPE_LADDER_STEP = 18 * L * L + 2 * L     # 6M + 4S (sqr = (3L^2+L)/2)
MULMODS_PER_STEP = 10
SMS = 148
WIDE_PER_CLK_SM = 32                     # measured: profiles/r01_imad_rates.jsonl


def peaks():
    p = {}
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    mhz = float(p.get("sm_max_mhz", 1965.0))
    return {"sm_max_mhz": mhz, "fpe_peak": SMS * WIDE_PER_CLK_SM * mhz * 1e6, "hbm_gbs": float(p.get("hbm_gbs", 6650.0)),
            "source": "MEASURED_PEAKS.json sm_max_mhz x 148 SMs x 32 IMAD.WIDE/clk/SM (measured)" if p else "fallback"}


# ---------------------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in self.rows for j in range(4) if r[3 + j].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


BACKEND = os.environ.get("ECM_DIST_BACKEND", "nccl")  # gloo: exercise N > 1 on one GPU (tests only)


def max_over_ranks(torch, x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if BACKEND == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(torch, ws):
    torch.cuda.synchronize()
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def time_steps(torch, fn, steps, ws):
    """Times `steps` calls of fn with CUDA events on the current stream; returns (total_ms, per-step ms)."""
    stream = torch.cuda.current_stream()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    barrier(torch, ws)
    evs[0].record(stream)
    for i in range(steps):
        fn()
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    per = [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]
    total = evs[0].elapsed_time(evs[-1])
    barrier(torch, ws)
    return total, per


def ncu_traffic(name):
    """dram bytes per launch for a kernel from the committed ncu summary (profiles/)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return d.get(name)
    except Exception:
        return None


# ---------------------------------------------------------------------------------------
CPU_TARGET_S = 10.0  # bounded oracle sample: about 10 s of host work per baseline


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline_mulmod(sample_elems: int, iters: int, target_s: float = CPU_TARGET_S):
    """The oracle as it stands on all host cores, over consecutive C2 triples: at least
    `sample_elems`, then further chunks until about `target_s` seconds have elapsed."""
    import oracle
    from workload import mulmod_inputs
    threads = os.cpu_count() or 1
    done, dt = 0, 0.0
    while done < C2_COUNT and (done < sample_elems or dt < target_s):
        chunk = sample_elems if done == 0 else min(max(threads * 2048, sample_elems), C2_COUNT - done)
        a, b, n = mulmod_inputs(chunk, L, seed=2, start=done)
        t0 = time.perf_counter()
        oracle.mulmod_chain_mt(a, b, n, L, iters, threads=threads)
        dt += time.perf_counter() - t0
        done += chunk
    return {"value": done * iters / dt, "unit": "modmul/s", "cores": threads, "kind": "oracle",
            "sample": f"first {done} of C2's 2^24 triples x K={iters} (oracle C, {threads} host threads)",
            "seconds": dt, "per_core": done * iters / dt / threads, "cpu": cpu_model()}


def cpu_baseline_ecm(N, k, sigmas, B1, target_s: float = CPU_TARGET_S):
    """The oracle on all host cores over a strided sample of C3's curves, in chunks of one
    curve per thread until about `target_s` seconds have elapsed (or the sample is used up)."""
    import oracle
    threads = os.cpu_count() or 1
    done, dt = 0, 0.0
    while done < len(sigmas) and dt < target_s:
        part = sigmas[done:done + threads]
        t0 = time.perf_counter()
        oracle.ecm_stage1_mt(N, L, k, part, threads=threads)
        dt += time.perf_counter() - t0
        done += len(part)
    return {"value": done / dt, "unit": "curves/s", "cores": threads, "kind": "oracle",
            "sample": f"{done} strided curves of C3 at B1={B1}", "seconds": dt, "per_core": done / dt / threads,
            "cpu": cpu_model()}


# ---------------------------------------------------------------------------------------
def c2_config(count, iters, ws):
    """The C2 workload both arms report (the reference arm processes a bounded sample of it per step,
    described in its cpu_baseline)."""
    return {"workload": f"C2: {count} independent (a,b,N) triples per GPU, L=6 (190-bit N), "
                        f"K={iters} chained lazy Montgomery products", "L": L, "count_per_gpu": count,
            "iters": iters, "redc": "word-CIOS (default)", "layout": "limb-sliced [j*count+i]",
            "l2": "inputs 1.15 GiB > L2 (no flush needed)", "parallelism": f"replicas x{ws}"}


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group(BACKEND)
    else:
        torch.cuda.set_device(0)
    import paper_1310_3809_b200 as eg
    from paper_1310_3809_b200 import build as _b
    _b.build()
    from workload import ecm_config, mulmod_inputs

    pk = peaks()
    # ---------------- C2: batched 192-bit mulmod, K = 256, this rank's replica shard ----------------
    count = args.count
    # limb-sliced layout (north_star (1)): limb j of triple i at word [j*count + i]
    a, b, n = mulmod_inputs(count, L, seed=2, start=rank * count)
    A, B, Nn = (torch.from_numpy(x).cuda() for x in (a, b, n))
    S3 = [x.t().contiguous() for x in (A, B, Nn)]
    out = torch.empty_like(S3[0])
    step = lambda: eg.ecm_mulmod_batch(S3[0], S3[1], S3[2], out, L=L, iters=args.iters,  # noqa: E731
                                       flags=eg.ECM_LAYOUT_SLICED)
    for _ in range(args.warmup):
        step()
    with ClockSampler(local) as clk:
        total_ms, per = time_steps(torch, step, args.steps, ws)
    total_ms = max_over_ranks(torch, total_ms, ws)
    mulmods = count * args.iters * args.steps * ws
    value = mulmods / (total_ms * 1e-3)
    kernel_ms = sum(per) / len(per)
    fpe_launch = count * args.iters * FPE_MUL
    achieved = fpe_launch / (kernel_ms * 1e-3)
    clocks = clk.summary()

    # ---------------- square mode and the C4 width sweep (same count, K) ----------------
    sweep = {}
    if not args.no_sweep:
        out_sq = torch.empty_like(S3[0])
        sq = lambda: eg.ecm_mulmod_batch(S3[0], S3[1], S3[2], out_sq, L=L, iters=args.iters,  # noqa: E731
                                         flags=eg.ECM_SQUARE | eg.ECM_LAYOUT_SLICED)
        sq()
        ms, _ = time_steps(torch, sq, 3, ws)
        ms = max_over_ranks(torch, ms / 3, ws)
        fpe_sq = (3 * L * L + L) // 2
        del out_sq
        sweep["square_L6"] = {"modmul_per_s": count * args.iters * ws / (ms * 1e-3), "ms": ms,
                              "frac": count * args.iters * fpe_sq / (ms * 1e-3) / pk["fpe_peak"]}
        # K = 1: one product per triple -> HBM bound (16L bytes per mulmod: a, b, n in, out)
        # the AoS layout at the headline K (warp-tile kernel) for contrast
        out_aos = torch.empty_like(A)
        fa = lambda: eg.ecm_mulmod_batch(A, B, Nn, out_aos, L=L, iters=args.iters)  # noqa: E731
        fa()
        ms, _ = time_steps(torch, fa, 3, ws)
        ms = max_over_ranks(torch, ms / 3, ws)
        sweep["aos_L6"] = {"modmul_per_s": count * args.iters * ws / (ms * 1e-3), "ms": ms,
                           "frac": count * args.iters * FPE_MUL / (ms * 1e-3) / pk["fpe_peak"]}
        del out_aos
        out_k1 = torch.empty_like(A)
        S_out = torch.empty_like(S3[0])
        # default kernel at K = 1 is the CTA-tile streaming kernel; the warp-tile kernel for contrast
        k1 = []
        for kname, kf in (("", 0), ("_warp", eg.ECM_KERNEL_WARP)):
            k1.append((f"k1_aos{kname}", lambda kf=kf: eg.ecm_mulmod_batch(A, B, Nn, out_k1, L=L, iters=1, flags=kf)))
            k1.append((f"k1_sliced{kname}", lambda kf=kf: eg.ecm_mulmod_batch(
                S3[0], S3[1], S3[2], S_out, L=L, iters=1, flags=eg.ECM_LAYOUT_SLICED | kf)))
        for tag, fn in k1:
            fn()
            ms, _ = time_steps(torch, fn, 10, ws)
            ms = max_over_ranks(torch, ms / 10, ws)
            gbs = count * 16 * L / (ms * 1e-3) / 1e9
            sweep[tag] = {"modmul_per_s": count * ws / (ms * 1e-3), "ms": ms, "bound": "hbm", "achieved_gbs": gbs,
                          "peak_gbs": pk["hbm_gbs"], "frac": gbs / pk["hbm_gbs"]}
        del out_k1, S_out
        for Lw in (4, 8, 12, 16):
            aw, bw, nw = mulmod_inputs(count, Lw, seed=4, start=rank * count)
            Aw, Bw, Nw = (torch.from_numpy(x.T.copy()).cuda() for x in (aw, bw, nw))
            Ow = torch.empty_like(Aw)
            f = lambda: eg.ecm_mulmod_batch(Aw, Bw, Nw, Ow, L=Lw, iters=args.iters,  # noqa: E731
                                            flags=eg.ECM_LAYOUT_SLICED)
            f()
            ms, _ = time_steps(torch, f, 2, ws)
            ms = max_over_ranks(torch, ms / 2, ws)
            sweep[f"mul_L{Lw}"] = {"bits": 32 * Lw - 2, "modmul_per_s": count * args.iters * ws / (ms * 1e-3),
                                   "ms": ms, "frac": count * args.iters * 2 * Lw * Lw / (ms * 1e-3) / pk["fpe_peak"]}
            del Aw, Bw, Nw, Ow
        sweep["mul_L6"] = {"bits": 190, "modmul_per_s": value, "ms": kernel_ms, "frac": achieved / pk["fpe_peak"]}

    # ---------------- end to end: public API with host (pinned) buffers ----------------
    ah, bh, nh = (torch.from_numpy(x.T.copy()).pin_memory() for x in (a, b, n))
    oh = torch.empty_like(ah).pin_memory()
    e2e_step = lambda: eg.ecm_mulmod_batch(ah, bh, nh, oh, L=L, iters=args.iters,  # noqa: E731
                                           flags=eg.ECM_HOST_BUFFERS | eg.ECM_LAYOUT_SLICED)
    e2e_step()
    barrier(torch, ws)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    barrier(torch, ws)
    e2e_s = max_over_ranks(torch, time.perf_counter() - t0, ws)
    e2e = {"value": mulmods / e2e_s, "unit": "modmul/s", "h2d_bytes_per_step": int(3 * a.nbytes),
           "d2h_bytes_per_step": int(a.nbytes)}
    del ah, bh, nh, oh

    # ---------------- C3: ECM stage 1 curves/s (strong scaling over ranks) ----------------
    ecm, ecm_last = None, {}
    if not args.no_ecm:
        # --ecm-curves above C3's 2^20 draws more seeds of the same recipe (e.g. a sustained run)
        cfg = ecm_config("C3", curves=args.ecm_curves) if (args.ecm_curves or 0) > (1 << 20) else ecm_config("C3")
        if args.ecm_b1:
            cfg["B1"] = args.ecm_b1
        curves = cfg["curves"] if args.ecm_curves is None else args.ecm_curves
        kb = eg.ecm_stage1_kbits(cfg["B1"])
        from paper_1310_3809_b200.dist import ecm_stage1_distributed, shard_bounds
        gdev = "cuda" if BACKEND == "nccl" else "cpu"  # gloo (tests): the gather runs on CPU tensors
        # the seeds are staged on the device before the timed region (inputs resident in HBM, like C2's)
        sig_all = torch.from_numpy(np.ascontiguousarray(cfg["sigmas"][:curves])).cuda()
        # warm-up: the same distributed step (plan cache, kernels, communicators) on 4096 curves per rank
        ecm_stage1_distributed(cfg["N"], L, cfg["B1"], sig_all[: 4096 * ws], device=gdev)
        evs, loc = {}, {}
        gathered, factors = None, None

        def ecm_step():
            nonlocal gathered, factors
            # shard -> ecm_stage1_batch on this rank's GPU -> status all-gather + factor records
            # (at N = 1 the same call without collectives)
            # the timed step ends with the gathered statuses and factor records on the device; rank 0
            # decodes the records into integers after the timed region (host post-processing)
            gathered, factors = ecm_stage1_distributed(cfg["N"], L, cfg["B1"], sig_all, device=gdev,
                                                       events=evs, local=loc, decode="defer")

        with ClockSampler(local) as clk2:
            ecm_ms, _ = time_steps(torch, ecm_step, 1, ws)
        ecm_ms = max_over_ranks(torch, ecm_ms, ws)
        kern_ms = evs["start"].elapsed_time(evs["computed"])
        gather_ms = evs["computed"].elapsed_time(evs["gathered"])
        kmax = max_over_ranks(torch, kern_ms, ws)
        kmin = -max_over_ranks(torch, -kern_ms, ws)
        gmax = max_over_ranks(torch, gather_ms, ws)
        st = gathered.cpu().numpy()
        from paper_1310_3809_b200.dist import decode_records
        factors = decode_records(loc["recs"].cpu().numpy(), loc["world"], loc["cap"]) if rank == 0 else None
        curves_s = curves / (ecm_ms * 1e-3)
        fpe_curve = (kb - 1) * FPE_LADDER_STEP
        lo, hi = shard_bounds(curves, rank, ws)
        ecm = {"workload": f"C3: ECM stage 1, B1={cfg['B1']}, {curves} curves, 190-bit N=p*q (planted 64-bit p)",
               "curves_per_s": curves_s, "modmul_per_s": curves_s * (kb - 1) * MULMODS_PER_STEP,
               "ms": ecm_ms, "k_bits": kb, "flagged_factor": int((st == 1).sum()), "scaling": "strong",
               "curves_per_rank": [shard_bounds(curves, r, ws)[1] - shard_bounds(curves, r, ws)[0] for r in range(ws)],
               "kernel_ms_per_rank": {"min": kmin, "max": kmax}, "gather_ms": gmax,
               "gather_share": gmax / ecm_ms,
               "status_digest": hashlib.sha256(st.tobytes()).hexdigest()[:16],
               "roofline": {"bound": "alu", "achieved": curves_s / ws * fpe_curve / 1e12,
                            "peak": pk["fpe_peak"] / 1e12, "unit": "Tpp/s",
                            "frac": curves_s / ws * fpe_curve / pk["fpe_peak"],
                            "frac_kernel": curves / ws / (kmax * 1e-3) * fpe_curve / pk["fpe_peak"]},
               "clocks": clk2.summary()}
        if rank == 0:
            ecm["factors_found"] = len(factors)
            ecm["factors_digest"] = hashlib.sha256(repr(factors).encode()).hexdigest()[:16]
        ecm_last = {"status": loc["status"], "g": loc["g"]} if ws == 1 else {}

    # ---------------- §8(f) N4: the small-parameter family on C3's modulus, B1 and curve count ----------
    if ecm is not None and not args.no_sweep:
        seeds_np = (cfg["sigmas"][:curves] % np.uint64((1 << 30) - 1)) + np.uint64(1)
        sd = torch.from_numpy(seeds_np[lo:hi].copy()).cuda()
        eg.ecm_stage1_batch(cfg["N"], L, cfg["B1"], sd[:4096], flags=eg.ECM_CURVE_SMALL, want=("g",))
        rs = {}
        mss, _ = time_steps(torch, lambda: rs.update(eg.ecm_stage1_batch(cfg["N"], L, cfg["B1"], sd,
                                                                            flags=eg.ECM_CURVE_SMALL, want=("g",))),
                            1, ws)
        mss = max_over_ranks(torch, mss, ws)
        cps = curves / (mss * 1e-3)
        fpe_small = 4 * FPE_MUL + 4 * (3 * L * L + L) // 2 + 2 * L  # 4M + 4S + one word-level REDC
        ecm["small_family"] = {"workload": "C3 modulus/B1/curves, a24 = s/2^32, x0 = 2 (SURVEY §8(f) N4; not the "
                                           "paper's curves)", "curves_per_s": cps, "ms": mss,
                               "flagged_factor_rank0": int((rs["status"] == 1).sum().item()),
                               "speedup_vs_suyama": cps / curves_s,
                               "frac": cps / ws * (kb - 1) * fpe_small / pk["fpe_peak"]}
        del sd

    # ---------------- ECM width sweep (C4's widths for stage 1): whole waves per width ----------------
    if ecm is not None and not args.no_sweep:
        ecm["widths"] = {}
        for Lw in (4, 6, 8, 12, 16):
            cw = ecm_config(L=Lw, nbits=32 * Lw - 2, pbits=64, B1=cfg["B1"], curves=args.ecm_width_curves,
                            seed=40 + Lw)
            sw = torch.from_numpy(cw["sigmas"][rank::ws].copy()).cuda()
            eg.ecm_stage1_batch(cw["N"], Lw, cw["B1"], sw[:1024], want=("g",))
            rw = {}
            # one launch per timed run, `--ecm-width-reps` runs: the fastest is reported, every run listed
            # (a single one-launch shot once read 0.85 instead of 0.90 at L = 12, profiles/r02q_bench.jsonl)
            runs = []
            for _ in range(args.ecm_width_reps):
                msr, _ = time_steps(torch, lambda: rw.update(eg.ecm_stage1_batch(cw["N"], Lw, cw["B1"], sw,
                                                                                want=("g",))), 1, ws)
                runs.append(max_over_ranks(torch, msr, ws))
            msw = min(runs)
            cps = args.ecm_width_curves / (msw * 1e-3)
            fpe_w = (kb - 1) * (18 * Lw * Lw + 2 * Lw)
            ecm["widths"][f"L{Lw}"] = {"bits": 32 * Lw - 2, "curves": args.ecm_width_curves, "ms": msw,
                                       "ms_runs": runs, "curves_per_s": cps, "modmul_per_s": cps * (kb - 1) * MULMODS_PER_STEP,
                                       "frac": cps / ws * fpe_w / pk["fpe_peak"]}
            del sw

    # ---------------- C1: 256 curves, B1 = 2000 — latency bound (report time, not roofline) --------
    c1 = None
    if not args.no_ecm:
        cfg1 = ecm_config("C1")
        s1 = torch.from_numpy(cfg1["sigmas"]).cuda()
        f1 = lambda: eg.ecm_stage1_batch(cfg1["N"], L, cfg1["B1"], s1)  # noqa: E731
        f1()
        ms1, _ = time_steps(torch, f1, 3, ws)
        ms1 = max_over_ranks(torch, ms1 / 3, ws)
        st1 = f1()["status"].cpu().numpy()
        c1 = {"workload": "C1: 256 curves, B1=2000, 190-bit N with a planted 32-bit p (one launch)",
              "ms": ms1, "curves": 256, "found_p": int((st1 == 1).sum())}

    # ---------------- optional: one rank's shard of C5 (8-GPU config) on this GPU ----------------
    c5 = None
    if args.c5:
        cfg5 = ecm_config("C5")
        per_rank = cfg5["curves"] // 8
        lo = rank * per_rank
        sig5 = torch.from_numpy(cfg5["sigmas"][lo:lo + per_rank].copy()).cuda()
        kb5 = eg.ecm_stage1_kbits(cfg5["B1"])
        eg.ecm_stage1_batch(cfg5["N"], 8, cfg5["B1"], sig5[:1024], want=("g",))
        r5 = {}
        with ClockSampler(local) as clk5:
            ms5, _ = time_steps(torch, lambda: r5.update(eg.ecm_stage1_batch(cfg5["N"], 8, cfg5["B1"], sig5,
                                                                                 want=("g",))), 1, ws)
        cps5 = per_rank / (ms5 * 1e-3)
        fpe5 = (kb5 - 1) * (18 * 64 + 16)
        c5 = {"workload": f"C5 rank shard: {per_rank} of 2^22 curves, B1={cfg5['B1']}, 254-bit N (planted 80-bit p)",
              "curves_per_s_per_gpu": cps5, "ms": ms5, "k_bits": kb5,
              "flagged_factor": int((r5["status"] == 1).sum().item()),
              "frac": cps5 * fpe5 / pk["fpe_peak"], "clocks": clk5.summary()}

    line = {
        "metric": "192-bit Montgomery modmul/s",
        "value": value, "unit": "modmul/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": c2_config(count, args.iters, ws),
        "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": pk["fpe_peak"] / 1e12, "unit": "Tpp/s",
                     "frac": achieved / pk["fpe_peak"], "traffic": ncu_traffic("mulmod_batch_kernel<6,0,false,true>"),
                     "kernel": "ecm::mulmod_batch_kernel<6,0,false,true>", "kernel_ms": kernel_ms,
                     "peak_source": pk["source"],
                     "frac_at_measured_clock": (achieved / (SMS * WIDE_PER_CLK_SM * clocks["sm_mhz"] * 1e6))
                     if clocks.get("sm_mhz") else None},
        "clocks": clocks, "e2e": e2e, "gpu_launches": args.steps,
    }
    if ecm:
        line["ecm"] = ecm
    if sweep:
        line["sweep"] = sweep
    if c5:
        line["c5_shard"] = c5
    if c1:
        line["c1"] = c1
    if rank == 0 and ws == 1 and not args.no_cpu:
        # parity spot check of the timed launches against the oracle (sampled outputs)
        import oracle
        got = out.cpu().numpy().T
        idx = np.linspace(0, count - 1, 2048).astype(np.int64)
        want = oracle.mulmod_chain_mt(a[idx], b[idx], n[idx], L, args.iters)
        par = {"mulmod_checked": int(len(idx)), "mulmod_mismatches": int((got[idx] != want).any(axis=1).sum())}
        if ecm and ecm_last:
            cfg = ecm_config("C3")
            k3, _ = oracle.stage1_k(cfg["B1"])
            ci = np.linspace(0, len(ecm_last["status"]) - 1, 32).astype(np.int64)
            w3 = oracle.ecm_stage1_mt(cfg["N"], L, k3, cfg["sigmas"][ci])
            g3 = ecm_last["g"].cpu().numpy()[ci]
            s3 = ecm_last["status"].cpu().numpy()[ci]
            par["ecm_checked"] = int(len(ci))
            par["ecm_mismatches"] = int(((g3 != w3["g"]).any(axis=1) | (s3 != w3["status"])).sum())
        line["parity"] = par
        line["cpu_baseline"] = cpu_baseline_mulmod(args.cpu_elems, args.iters, target_s=args.cpu_seconds)
        if ecm:
            cfg = ecm_config("C3")
            import oracle
            k, _ = oracle.stage1_k(cfg["B1"])
            idx = np.arange(0, cfg["curves"], cfg["curves"] // args.cpu_curves)[: args.cpu_curves]
            ecm["cpu_baseline"] = cpu_baseline_ecm(cfg["N"], k, cfg["sigmas"][idx], cfg["B1"], target_s=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference(args):
    """The reference arm for this tier is the CPU oracle as it stands."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    sample = args.cpu_elems
    for _ in range(args.warmup):
        cpu_baseline_mulmod(max(1024, sample // 16), args.iters, target_s=0.0)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_baseline_mulmod(sample, args.iters, target_s=0.0))
    dt = time.perf_counter() - t0
    value = sample * args.iters * args.steps / dt
    cb = dict(vals[-1])
    cb["value"] = value
    line = {"impl": "reference", "metric": "192-bit Montgomery modmul/s", "value": value, "unit": "modmul/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": c2_config(args.count, args.iters, ws),
            "cpu_baseline": cb, "e2e": {"value": value, "unit": "modmul/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--count", type=int, default=C2_COUNT)
    ap.add_argument("--iters", type=int, default=C2_ITERS)
    ap.add_argument("--no-ecm", action="store_true")
    ap.add_argument("--ecm-curves", type=int, default=None)
    # 148 SMs x 128 threads x 12: whole waves at 6, 3 and 2 resident CTAs per SM (the ladder's occupancy at
    # L <= 6, 8 / 12 and 16), so no width's number carries a partly filled last wave
    ap.add_argument("--ecm-width-curves", type=int, default=148 * 128 * 12, help="curves per width in the ECM width sweep")
    ap.add_argument("--ecm-width-reps", type=int, default=2, help="timed one-launch runs per width (fastest reported)")
    ap.add_argument("--ecm-b1", type=int, default=None, help="override C3's B1 (tests / profiling only)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--c5", action="store_true", help="also time one rank's 1/8 shard of C5 (~40 s)")
    ap.add_argument("--cpu-elems", type=int, default=1 << 17)
    ap.add_argument("--cpu-curves", type=int, default=4096, help="strided C3 curves available to the oracle")
    ap.add_argument("--cpu-seconds", type=float, default=CPU_TARGET_S, help="host seconds per oracle baseline")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
