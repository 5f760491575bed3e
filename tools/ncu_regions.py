#!/usr/bin/env python3
"""Attribute an ECM kernel's ncu stall samples (and executed instructions) to setup / ladder / tail.

    python tools/ncu_regions.py <source.csv> [--json]

<source.csv> is `ncu -i X.ncu-rep --page source --csv` of one ecm_stage1 launch (SASS rows with
addresses).  The ladder loop is the backward branch whose body holds the most IMAD.WIDE; every
instruction before it is setup (Brent-Suyama curve and the D^{-1} xgcd), every instruction after
it is the tail (out of Montgomery form, gcd(Z, N), affine x, stores).  The xgcd loops are the
backward uniform branches (BRA.U) outside the ladder.  Reported per region: share of the warp
stall samples (time) and of the executed warp instructions.
"""
import csv
import json
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    hdr = rows[hdr_i]
    ix = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr):
            continue
        try:
            addr = int(r[ix["Address"]], 16)
        except ValueError:
            continue

        def num(col):
            try:
                return float(r[ix[col]] or 0)
            except (KeyError, ValueError):
                return 0.0
        out.append({"addr": addr, "sass": r[ix["Source"]].strip(),
                    "samples": num("Warp Stall Sampling (All Samples)"),
                    "inst": num("Instructions Executed")})
    return sorted(out, key=lambda x: x["addr"])


def regions(ins):
    best = None
    loops = []
    for x in ins:
        m = re.search(r"BRA(\.U)?\s.*?0x([0-9a-f]+)", x["sass"])
        if m and int(m.group(2), 16) < x["addr"]:
            lo, hi = int(m.group(2), 16), x["addr"]
            w = sum("IMAD.WIDE" in y["sass"] for y in ins if lo <= y["addr"] <= hi)
            loops.append((lo, hi, w, bool(m.group(1))))
            if best is None or w > best[2]:
                best = (lo, hi, w)
    lo, hi, _ = best
    xg = [(a, b) for a, b, w, uni in loops if uni and not (lo <= a <= hi)]
    return lo, hi, xg


def main():
    ins = load(sys.argv[1])
    lo, hi, xg = regions(ins)
    tot_s = sum(x["samples"] for x in ins) or 1.0
    tot_i = sum(x["inst"] for x in ins) or 1.0
    res = {}
    for name, pred in (("setup", lambda a: a < lo), ("ladder", lambda a: lo <= a <= hi), ("tail", lambda a: a > hi),
                       ("xgcd", lambda a: any(p <= a <= q for p, q in xg))):
        s = sum(x["samples"] for x in ins if pred(x["addr"]))
        i = sum(x["inst"] for x in ins if pred(x["addr"]))
        res[name] = {"stall_sample_share": s / tot_s, "inst_share": i / tot_i}
    res["ladder_addr"] = [hex(lo), hex(hi)]
    res["xgcd_loop_addr"] = [[hex(a), hex(b)] for a, b in xg]
    if "--json" in sys.argv:
        print(json.dumps(res))
    else:
        for k, v in res.items():
            print(k, v)


if __name__ == "__main__":
    main()
