#!/usr/bin/env python3
"""Count SASS opcodes per kernel in a cubin / executable / .so (cuobjdump -sass).

Used to check the instruction mix of the Montgomery kernels before spending GPU time
(IMAD-family vs ALU instructions per mulmod).
usage: sass_count.py FILE [--kernel REGEX] [--min N] [--full]
"""
import argparse
import re
import subprocess
import sys
from collections import Counter, OrderedDict


def parse(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    funcs = OrderedDict()
    cur = None
    ins = re.compile(r"^\s+/\*[0-9a-f]{4,}\*/\s+(.*?)\s*;")
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = ins.match(line)
        if m and cur is not None:
            text = m.group(1)
            toks = text.split()
            if toks and toks[0].startswith("@"):
                toks = toks[1:]
            addr = int(re.match(r"^\s+/\*([0-9a-f]+)\*/", line).group(1), 16)
            funcs[cur].append((toks[0] if toks else "?", text, addr))
    return funcs


def demangle(names):
    try:
        r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
        return r.stdout.splitlines()
    except Exception:
        return names


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("file")
    ap.add_argument("--kernel", default=".")
    ap.add_argument("--min", type=int, default=1)
    ap.add_argument("--full", action="store_true", help="print the full opcode (with modifiers)")
    ap.add_argument("--loop", action="store_true",
                    help="count only the smallest backward-branch loop body that contains IMAD.WIDE (the hot loop)")
    a = ap.parse_args()
    funcs = parse(a.file)
    names = list(funcs)
    for raw, dem in zip(names, demangle(names)):
        if not re.search(a.kernel, dem) and not re.search(a.kernel, raw):
            continue
        body = funcs[raw]
        if a.loop:
            # hot loop = the smallest backward-branch region holding >= 80% of the IMAD.WIDE/HI of
            # the richest region (the outer grid-stride loop contains it but also the prologue)
            regions = []
            for k, (op, text, addr) in enumerate(body):
                m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", text)
                if op.startswith("BRA") and m and int(m.group(1), 16) < addr:
                    tgt = int(m.group(1), 16)
                    region = [b for b in body if tgt <= b[2] <= addr]
                    w = sum(b[0].startswith(("IMAD.WIDE", "IMAD.HI")) for b in region)
                    regions.append((w, len(region), region))
            if regions:
                wmax = max(r[0] for r in regions)
                body = min((r for r in regions if r[0] >= 0.8 * wmax), key=lambda r: r[1])[2]
            else:
                body = []
        c = Counter()
        for op, _, _ in body:
            key = op if a.full else op.split(".")[0]
            c[key] += 1
        total = sum(c.values())
        print(f"== {dem}  (total {total})")
        for k, v in c.most_common():
            if v >= a.min:
                print(f"   {v:7d}  {k}")


if __name__ == "__main__":
    sys.exit(main())
