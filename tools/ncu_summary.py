#!/usr/bin/env python3
"""Summarise ncu CSV exports (tools/profile.sh): key raw metrics of one capture, and the
per-opcode stall attribution from the source page (SASS view).

    ncu_summary.py raw    gpurun_out/TAG_ncu_NAME_raw.csv
    ncu_summary.py source gpurun_out/TAG_ncu_NAME_source.csv
    ncu_summary.py traffic gpurun_out/TAG_ncu_NAME_raw.csv   -> dram bytes per launch
"""
import csv
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_issued.sum",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    for k in KEYS:
        if k in d:
            print(f"{k:75s} {d[k][0]:10s} {d[k][1]}")
    stalls = {h: float(v.replace(",", "")) for h, (u, v) in d.items()
              if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")}
    print("top stalls (warps per issue):")
    for h, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]:
        print(f"   {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {v:.3f}")
    return d


def traffic(path):
    d = raw.__wrapped__(path) if hasattr(raw, "__wrapped__") else None
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    dd = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        u, v = dd[k]
        tot += float(v.replace(",", "")) * UNIT[u]
    print(int(tot))


def source(path):
    rows = list(csv.reader(open(path)))
    # find header row containing "Source" / "Warp Stall Sampling"
    hi = next(i for i, r in enumerate(rows) if any("Stall" in c for c in r) and any("Source" in c for c in r))
    hdr = rows[hi]
    src = hdr.index("Source")
    samp_cols = [i for i, c in enumerate(hdr) if c.startswith("Warp Stall Sampling (All")]
    reason_cols = [i for i, c in enumerate(hdr) if c.startswith("stall_") or c.endswith("(stall)")]
    by_op = defaultdict(float)
    total = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= src or not r[src].strip():
            continue
        op = r[src].strip().split()[0]
        if op.startswith("@"):
            op = r[src].strip().split()[1]
        try:
            v = float(r[samp_cols[0]].replace(",", "")) if samp_cols else 0.0
        except ValueError:
            v = 0.0
        by_op[op.split(".")[0] if op.startswith(("IMAD.WIDE", "IMAD.HI")) is False else op] += v
        total += v
    print(f"stall samples by opcode (total {total:.0f}):")
    for op, v in sorted(by_op.items(), key=lambda x: -x[1])[:15]:
        print(f"   {op:22s} {v:10.0f}  {v / max(total, 1):6.1%}")


if __name__ == "__main__":
    {"raw": raw, "source": source, "traffic": traffic}[sys.argv[1]](sys.argv[2])
