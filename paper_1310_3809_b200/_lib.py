"""ctypes loader for libecmgpu.so: signatures mirror include/ecmgpu.h exactly.

Fails loudly (ImportError/OSError) when the library has not been built; there is no
fallback implementation anywhere in this package.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(HERE, "libecmgpu.so")

ECM_CANONICAL = 0x1
ECM_SQUARE = 0x2
ECM_LAYOUT_SLICED = 0x4
ECM_CHECK = 0x8
ECM_HOST_BUFFERS = 0x10
ECM_NO_XAFF = 0x20
ECM_EAGER = 0x40
ECM_PRIME_LADDERS = 0x80
ECM_REDC_WORD = 0 << 8
ECM_REDC_KNOWNLOW = 1 << 8
ECM_REDC_BLOCKTHM = 2 << 8
ECM_REDC_CLASSIC = 3 << 8
ECM_REDC_KARATSUBA = 4 << 8
ECM_KERNEL_STREAM = 0x800
ECM_KERNEL_WARP = 0x1000
ECM_KERNEL_LANES4 = 0x2000
ECM_KERNEL_LANES1 = 0x4000
ECM_CURVE_SMALL = 0x8000

# every symbol include/ecmgpu.h declares (checked by tests/test_abi.py)
EXPORTS = ("ecm_mulmod_batch", "ecm_stage1_batch", "ecm_ladder_batch", "ecm_stage1_kbits",
           "ecm_strerror", "ecm_version")


class EcmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(library_path):
            raise OSError(f"{library_path} is missing: run `python -m paper_1310_3809_b200.build` "
                          "(there is no CPU fallback)")
        L = ctypes.CDLL(library_path)
        vp, sz, u32, u64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint64
        u32p = ctypes.POINTER(ctypes.c_uint32)
        L.ecm_mulmod_batch.argtypes = [vp, vp, vp, vp, sz, ctypes.c_int, u32, u32, vp]
        L.ecm_mulmod_batch.restype = ctypes.c_int
        L.ecm_stage1_batch.argtypes = [u32p, ctypes.c_int, u64, vp, sz, vp, vp, vp, vp, vp, u32, vp]
        L.ecm_stage1_batch.restype = ctypes.c_int
        L.ecm_ladder_batch.argtypes = [u32p, ctypes.c_int, u32p, u32, vp, sz, vp, vp, vp, vp, vp, u32, vp]
        L.ecm_ladder_batch.restype = ctypes.c_int
        L.ecm_stage1_kbits.argtypes = [u64]
        L.ecm_stage1_kbits.restype = u32
        L.ecm_strerror.argtypes = [ctypes.c_int]
        L.ecm_strerror.restype = ctypes.c_char_p
        L.ecm_version.argtypes = []
        L.ecm_version.restype = ctypes.c_char_p
        _lib = L
    return _lib
