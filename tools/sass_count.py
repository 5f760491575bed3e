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
            funcs[cur].append((toks[0] if toks else "?", text))
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
    a = ap.parse_args()
    funcs = parse(a.file)
    names = list(funcs)
    for raw, dem in zip(names, demangle(names)):
        if not re.search(a.kernel, dem) and not re.search(a.kernel, raw):
            continue
        c = Counter()
        for op, _ in funcs[raw]:
            key = op if a.full else op.split(".")[0]
            c[key] += 1
        total = sum(c.values())
        print(f"== {dem}  (total {total})")
        for k, v in c.most_common():
            if v >= a.min:
                print(f"   {v:7d}  {k}")


if __name__ == "__main__":
    sys.exit(main())
