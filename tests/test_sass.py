"""SASS-level checks of the built library (CPU only: cuobjdump reads the sm_100a cubins, no GPU).

They pin the instruction-mix facts DESIGN.md §6 builds its rooflines on, so a compiler or source
change that silently re-introduces work on the IMAD.WIDE pipe fails here instead of in a bench line:
  * every cubin is sm_100a, with no PTX for a JIT fallback;
  * C2's kernel (mulmod_batch_kernel<6, WORD, multiply, sliced>): 2L^2 = 72 IMAD.WIDE/HI products and
    L = 6 IMAD (the m_i = t_0 n0' of the CIOS rows) per product in the hot loop — n0' is
    re-read from its shared slot, not rematerialised by a Newton iteration — no spills;
  * square mode: (3L^2 + L)/2 = 57 products and 6 IMAD per square, no IMAD.X carry adds on the fma pipe;
  * the ECM ladder step at L = 6 (6 multiplies + 4 squares): 660 products, 60 IMAD, no
    local-memory traffic; and no data-dependent branch outside the ladder loop: every
    other branch is warp-uniform (BRA.U) or an EXIT.
"""
import os
import re
import shutil
import subprocess

import pytest

CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
pytestmark = pytest.mark.skipif(not os.path.exists(CUOBJDUMP), reason="cuobjdump not available")

C2_MUL = "_ZN3ecm19mulmod_batch_kernelILi6ELi0ELb0ELb1EEEvPKjS2_S2_Pjmjj"
C2_SQR = "_ZN3ecm19mulmod_batch_kernelILi6ELi0ELb1ELb1EEEvPKjS2_S2_Pjmjj"
LADDER6 = "_ZN3ecm17ecm_stage1_kernelILi6ELi0ELb0ELb0ELi0EEEvNS_9EcmParamsEPKjjPKmmPjS6_S6_PhS6_j"
MULMOD = "_ZN3ecm19mulmod_batch_kernelILi{L}ELi0ELb{sq}ELb1EEEvPKjS2_S2_Pjmjj"
LADDER = "_ZN3ecm17ecm_stage1_kernelILi{L}ELi0ELb0ELb0ELi0EEEvNS_9EcmParamsEPKjjPKmmPjS6_S6_PhS6_j"
PRODUCT = ("IMAD.WIDE", "IMAD.HI")


@pytest.fixture(scope="module")
def lib():
    from paper_1310_3809_b200 import build
    return build.build()


def sass(lib, fn):
    out = subprocess.run([CUOBJDUMP, "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
    ins = []
    for line in out.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?)\s*;", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    assert ins, f"{fn} not found in {lib}"
    return ins


def opcode(text):
    t = text.split()
    return t[1] if t[0].startswith("@") else t[0]


def hot_loop(ins, min_products):
    """The smallest backward-branch loop body holding at least `min_products` products."""
    best, span = None, None
    for addr, text in ins:
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", text)
        if m and int(m.group(1), 16) < addr:
            body = [t for a, t in ins if int(m.group(1), 16) <= a <= addr]
            n = sum(opcode(t).startswith(PRODUCT) for t in body)
            if n >= min_products and (best is None or len(body) < len(best)):
                best, span = body, (int(m.group(1), 16), addr)
    assert best is not None
    hot_loop.span = span
    return best


def mix(body):
    ops = [opcode(t) for t in body]
    return {
        "products": sum(o.startswith(PRODUCT) for o in ops),
        "imad": sum(o == "IMAD" for o in ops),
        "imad_x": sum(o == "IMAD.X" for o in ops),
        "local": sum(o.startswith(("LDL", "STL")) for o in ops),
        "lds": sum(o.startswith("LDS") for o in ops),
    }


def test_every_cubin_is_sm100a_without_ptx(lib):
    elfs = subprocess.run([CUOBJDUMP, "-lelf", lib], capture_output=True, text=True).stdout.split("\n")
    elfs = [e for e in elfs if e.strip()]
    assert elfs and all("sm_100a" in e for e in elfs), elfs
    ptx = subprocess.run([CUOBJDUMP, "-lptx", lib], capture_output=True, text=True)
    assert ".ptx" not in ptx.stdout


def test_c2_multiply_loop_mix(lib):
    m = mix(hot_loop(sass(lib, C2_MUL), 200))
    n = m["products"] // 72
    assert n >= 2 and m["products"] == 72 * n, m
    assert m["imad"] == 6 * n, m  # the m_i only: no Newton iteration for n0' inside the loop
    assert m["lds"] == n, m       # n0' re-read from its shared slot once per product
    assert m["imad_x"] == 0 and m["local"] == 0, m


def test_c2_square_loop_mix(lib):
    m = mix(hot_loop(sass(lib, C2_SQR), 200))
    n = m["products"] // 57
    assert n >= 2 and m["products"] == 57 * n, m
    assert m["imad"] == 6 * n and m["imad_x"] == 0 and m["local"] == 0, m


def test_ladder_step_mix_and_uniform_branches(lib):
    ins = sass(lib, LADDER6)
    body = hot_loop(ins, 600)
    m = mix(body)
    assert 660 <= m["products"] <= 662, m  # 6 * 72 + 4 * 57 (+ at most a scheduling duplicate)
    assert m["imad"] == 60 and m["local"] == 0, m
    # the ladder loop's span: from its first to its last instruction (back edge)
    lo, hi = hot_loop.span
    for a, t in ins:
        op = opcode(t)
        if not op.startswith("BRA") or lo - 0x200 <= a <= hi + 0x200:
            continue  # the ladder's own entry guards and back edge (k_bits: a kernel parameter)
        target = int(re.search(r"0x([0-9a-f]+)", t.split("BRA", 1)[1]).group(1), 16)
        if target == a:  # the trailing self-branch after EXIT
            continue
        assert op.startswith("BRA.U") or t.startswith("BRA"), (hex(a), t)


@pytest.mark.parametrize("L", (4, 6, 8, 12, 16))
def test_every_width_products_per_step_and_spills(lib, L):
    """Every width's default chains and ladder: 2L^2 / (3L^2+L)/2 products per multiply / square, 6
    multiplies + 4 squares = 18L^2 + 2L per ladder step, no local memory in the mulmod loops; the ladder
    loops spill only at L = 12 (held to 168 registers for 3 CTAs/SM): a few words per step."""
    for sq, per in ((0, 2 * L * L), (1, (3 * L * L + L) // 2)):
        m = mix(hot_loop(sass(lib, MULMOD.format(L=L, sq=sq)), 2 * per))
        assert m["products"] % per == 0 and m["imad"] == L * (m["products"] // per), (sq, m)
        assert m["local"] == 0, (sq, m)
    m = mix(hot_loop(sass(lib, LADDER.format(L=L)), 18 * L * L))
    step = 18 * L * L + 2 * L
    assert step <= m["products"] <= step + 2 and m["imad"] == 10 * L, m
    assert m["local"] <= (8 if L == 12 else 0), m
