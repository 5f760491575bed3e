"""C-ABI library: loads on a CPU-only host, exports every symbol include/ecmgpu.h declares,
and rejects bad arguments before touching the device (no compute calls here)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_1310_3809_b200 import build
    build.build()
    from paper_1310_3809_b200 import _lib
    return _lib


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ecmgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ecm_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("ecm_mulmod_batch", "ecm_stage1_batch"):
        assert required in names


def test_library_exports_every_declared_symbol(L):
    lib = ctypes.CDLL(L.library_path)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(L.EXPORTS)


def test_strerror_and_version(L):
    lib = L.lib()
    for s in range(8):
        assert lib.ecm_strerror(s)
    assert lib.ecm_version().startswith(b"libecmgpu sm_100a")


def test_kbits_plan_host_side(L):
    lib = L.lib()
    assert lib.ecm_stage1_kbits(10) == 12       # k(10) = 2520
    assert lib.ecm_stage1_kbits(2000) == 2878
    assert lib.ecm_stage1_kbits(1) == 0


def test_argument_errors_before_any_device_work(L):
    lib = L.lib()
    buf = np.zeros(64, np.uint32)
    p = ctypes.c_void_p(buf.ctypes.data)
    # unsupported L, count 0, null pointers, unknown flags, iters 0
    assert lib.ecm_mulmod_batch(p, p, p, p, 4, 5, 1, 0, None) == 1
    assert lib.ecm_mulmod_batch(p, p, p, p, 0, 6, 1, 0, None) == 1
    assert lib.ecm_mulmod_batch(p, p, p, p, (1 << 62) + 1, 6, 1, 0, None) == 1  # size overflow guard
    assert lib.ecm_mulmod_batch(None, p, p, p, 4, 6, 1, 0, None) == 1
    assert lib.ecm_mulmod_batch(p, None, p, p, 4, 6, 1, 0, None) == 1
    assert lib.ecm_mulmod_batch(p, p, p, p, 4, 6, 1, 1 << 20, None) == 1
    assert lib.ecm_mulmod_batch(p, p, p, p, 4, 6, 0, 0, None) == 1
    N = np.zeros(6, np.uint32)
    Np = N.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
    sig = np.full(4, 6, np.uint64)
    sp = ctypes.c_void_p(sig.ctypes.data)
    st = np.zeros(4, np.uint8)
    stp = ctypes.c_void_p(st.ctypes.data)
    N[0] = 10  # even
    assert lib.ecm_stage1_batch(Np, 6, 100, sp, 4, None, None, None, stp, None, 0, None) == 2
    N[0] = 11
    N[5] = 1 << 30  # 191 bits > 32*6-2
    assert lib.ecm_stage1_batch(Np, 6, 100, sp, 4, None, None, None, stp, None, 0, None) == 3
    N[5] = 0
    assert lib.ecm_stage1_batch(Np, 6, 1, sp, 4, None, None, None, stp, None, 0, None) == 4
    assert lib.ecm_stage1_batch(Np, 7, 100, sp, 4, None, None, None, stp, None, 0, None) == 1
    N16 = np.zeros(16, np.uint32)
    N16[0] = 11
    assert lib.ecm_stage1_batch(N16.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), 10, 100, sp, 4,
                                None, None, None, stp, None, 0, None) == 1  # no L = 10
    # ablation variants exist for L = 6, 8 only
    assert lib.ecm_stage1_batch(N16.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), 16, 100, sp, 4,
                                None, None, None, stp, None, 0x40, None) == 1
    # stage-1 kernel choice: not both; the 4-lane kernel only for the default lazy full-k ladder;
    # not a mulmod flag
    assert lib.ecm_stage1_batch(Np, 6, 100, sp, 4, None, None, None, stp, None, 0x6000, None) == 1
    assert lib.ecm_stage1_batch(Np, 6, 100, sp, 4, None, None, None, stp, None, 0x2000 | 0x40, None) == 1
    assert lib.ecm_stage1_batch(Np, 6, 100, sp, 4, None, None, None, stp, None, 0x2000 | 0x80, None) == 1
    assert lib.ecm_stage1_batch(Np, 6, 100, sp, 4, None, None, None, stp, None, 0x2000 | (3 << 8), None) == 1
    assert lib.ecm_mulmod_batch(p, p, p, p, 4, 6, 1, 0x2000, None) == 1
    assert lib.ecm_mulmod_batch(p, p, p, p, 4, 6, 1, 0x4000, None) == 1
    # small-parameter family: default ladder only; not a mulmod flag
    assert lib.ecm_stage1_batch(Np, 6, 100, sp, 4, None, None, None, stp, None, 0x8000 | 0x40, None) == 1
    assert lib.ecm_stage1_batch(Np, 6, 100, sp, 4, None, None, None, stp, None, 0x8000 | 0x80, None) == 1
    assert lib.ecm_stage1_batch(Np, 6, 100, sp, 4, None, None, None, stp, None, 0x8000 | (1 << 8), None) == 1
    assert lib.ecm_mulmod_batch(p, p, p, p, 4, 6, 1, 0x8000, None) == 1
    kw = np.array([5], np.uint32)
    kp = kw.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
    assert lib.ecm_ladder_batch(Np, 6, kp, 4, sp, 4, None, None, None, stp, None, 0, None) == 4  # k_bits wrong


def test_product_package_never_imports_oracle():
    """The product path shares no code with oracle/ (DESIGN.md §2)."""
    pkg = os.path.join(ROOT, "paper_1310_3809_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("no oracle", ""), f
