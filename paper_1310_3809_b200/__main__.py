"""Command-line interface (mirroring SPEC S:500-566 for this path).

    python -m paper_1310_3809_b200 factor --n HEX [--b1 B1] [--curves C] [--seed S] [--L L]
                                          [--schedule full|primes] [--family suyama|small]
                                          [--format text|jsonl]
    python -m paper_1310_3809_b200 mulmod --L L --count C --iters K [--seed S] [--square]
    python -m paper_1310_3809_b200 version

`factor` runs ECM stage 1 on the GPU (ecm_stage1_batch) with `curves` Suyama seeds derived from
`seed` and prints every proper factor found (each checked by division on the host).
Exit codes: 0 factor found / ok, 1 input error, 2 no factor found.  Hex input is big-endian,
lowercase or uppercase, no prefix required.
"""
from __future__ import annotations

import argparse
import json
import sys

EXIT_OK, EXIT_INPUT, EXIT_NOFACTOR = 0, 1, 2


def _pick_L(n: int) -> int | None:
    for L in (4, 6, 8, 12, 16):
        if n.bit_length() <= 32 * L - 2:
            return L
    return None


def cmd_factor(a) -> int:
    import numpy as np
    import torch

    import paper_1310_3809_b200 as eg
    from workload import sigmas as make_sigmas

    try:
        n = int(a.n.lower().removeprefix("0x"), 16)
    except ValueError:
        print("error: --n must be hexadecimal", file=sys.stderr)
        return EXIT_INPUT
    if n < 3 or n % 2 == 0:
        print("error: n must be odd and >= 3", file=sys.stderr)
        return EXIT_INPUT
    L = a.L or _pick_L(n)
    if L is None or n.bit_length() > 32 * L - 2:
        print("error: n is wider than 510 bits (L = 16, two spare bits)", file=sys.stderr)
        return EXIT_INPUT
    if a.b1 < 2 or a.curves < 1:
        print("error: need B1 >= 2 and curves >= 1", file=sys.stderr)
        return EXIT_INPUT
    sig = make_sigmas(a.seed, a.curves)
    flags = eg.ECM_PRIME_LADDERS if a.schedule == "primes" else 0
    if a.family == "small":  # §8(f) N4 curves: seeds in [1, 2^30)
        if a.schedule == "primes":
            print("error: --family small needs --schedule full", file=sys.stderr)
            return EXIT_INPUT
        sig = (sig % np.uint64((1 << 30) - 1)) + np.uint64(1)
        flags |= eg.ECM_CURVE_SMALL
    if torch.cuda.is_available():
        r = eg.ecm_stage1_batch(n, L, a.b1, torch.from_numpy(sig).cuda(), flags=flags, want=("g",))
        status = r["status"].cpu().numpy()
        g = r["g"].cpu().numpy()
    else:
        print("error: no CUDA device (there is no CPU fallback)", file=sys.stderr)
        return EXIT_INPUT
    found = {}
    for i in np.nonzero((status == 1) | (status == 4))[0]:
        d = eg.limbs_to_int(g[i])
        if 1 < d < n and n % d == 0:  # every reported factor is checked by division
            found.setdefault(d, (int(i), int(sig[i])))
    if a.format == "jsonl":
        print(json.dumps({"n": hex(n), "B1": a.b1, "curves": a.curves, "L": L,
                          "factors": [{"factor": hex(d), "curve": c, "sigma": s} for d, (c, s) in sorted(found.items())],
                          "status_counts": {int(k): int(v) for k, v in zip(*np.unique(status, return_counts=True))}}))
    else:
        for d, (c, s) in sorted(found.items()):
            print(f"factor {d} (0x{d:x}) from curve {c}, sigma {s}")
        if not found:
            print(f"no factor found with {a.curves} curves at B1 = {a.b1}")
    return EXIT_OK if found else EXIT_NOFACTOR


def cmd_mulmod(a) -> int:
    import torch

    import paper_1310_3809_b200 as eg
    from workload import mulmod_inputs

    if a.L not in (4, 6, 8, 12, 16) or a.count < 1 or a.iters < 1:
        print("error: L in {4,6,8,12,16}, count >= 1, iters >= 1", file=sys.stderr)
        return EXIT_INPUT
    x, y, n = (torch.from_numpy(v).cuda() for v in mulmod_inputs(a.count, a.L, seed=a.seed))
    flags = eg.ECM_SQUARE if a.square else 0
    eg.ecm_mulmod_batch(x, y, n, L=a.L, iters=a.iters, flags=flags)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    eg.ecm_mulmod_batch(x, y, n, L=a.L, iters=a.iters, flags=flags)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(json.dumps({"L": a.L, "count": a.count, "iters": a.iters, "square": a.square, "ms": ms,
                      "modmul_per_s": a.count * a.iters / ms * 1e3}))
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1310_3809_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    f = sub.add_parser("factor", help="ECM stage 1 on the GPU")
    f.add_argument("--n", required=True, help="hex, big-endian")
    f.add_argument("--b1", type=int, default=8192)
    f.add_argument("--curves", type=int, default=1024)
    f.add_argument("--seed", type=int, default=1)
    f.add_argument("--L", type=int, default=None)
    f.add_argument("--schedule", choices=["full", "primes"], default="full")
    f.add_argument("--family", choices=["suyama", "small"], default="suyama",
                   help="curve family: the paper's Brent-Suyama curves, or the small-parameter family")
    f.add_argument("--format", choices=["text", "jsonl"], default="text")
    m = sub.add_parser("mulmod", help="time one batched Montgomery chain")
    m.add_argument("--L", type=int, default=6)
    m.add_argument("--count", type=int, default=1 << 20)
    m.add_argument("--iters", type=int, default=256)
    m.add_argument("--seed", type=int, default=2)
    m.add_argument("--square", action="store_true")
    sub.add_parser("version")
    a = ap.parse_args(argv)
    if a.cmd == "factor":
        return cmd_factor(a)
    if a.cmd == "mulmod":
        return cmd_mulmod(a)
    import paper_1310_3809_b200 as eg
    print(eg.ecm_version())
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
