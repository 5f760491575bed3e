"""paper_1310_3809_b200 — Python binding of libecmgpu (include/ecmgpu.h).

Argument marshalling only: every step of the hot path runs in the sm_100a kernels of
``libecmgpu.so``.  PyTorch supplies device memory and streams.  There is no CPU fallback: if
the library is missing or no CUDA device is present, calls raise.

Functions (same names as the C ABI):
    ecm_mulmod_batch(a, b, n, out=None, *, L, iters=1, flags=0, stream=None) -> out
    ecm_stage1_batch(N, L, B1, sigmas, *, flags=0, stream=None, want=("X","Z","g","xaff")) -> dict
    ecm_ladder_batch(N, L, k, sigmas, *, flags=0, stream=None) -> dict
    ecm_stage1_kbits(B1) -> int
Tensors are uint32 limb arrays shaped (count, L) (AoS) or (L, count) (ECM_LAYOUT_SLICED),
on the current CUDA device; with ECM_HOST_BUFFERS they are CPU tensors / numpy arrays.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from ._lib import (  # noqa: F401  (flag constants re-exported)
    ECM_CANONICAL, ECM_SQUARE, ECM_LAYOUT_SLICED, ECM_CHECK, ECM_HOST_BUFFERS, ECM_NO_XAFF, ECM_EAGER, ECM_PRIME_LADDERS,
    ECM_REDC_WORD, ECM_REDC_KNOWNLOW, ECM_REDC_BLOCKTHM, ECM_REDC_CLASSIC, ECM_REDC_KARATSUBA,
    ECM_KERNEL_STREAM, ECM_KERNEL_WARP, ECM_KERNEL_LANES4, ECM_KERNEL_LANES1, ECM_CURVE_SMALL,
    EcmError, lib, library_path,
)

__all__ = [
    "ecm_mulmod_batch", "ecm_stage1_batch", "ecm_ladder_batch", "ecm_stage1_kbits", "ecm_version",
    "EcmError", "lib", "library_path", "int_to_limbs", "limbs_to_int",
]


def int_to_limbs(x: int, L: int) -> np.ndarray:
    if x < 0 or x >> (32 * L):
        raise ValueError("value does not fit in L limbs")
    return np.array([(x >> (32 * i)) & 0xFFFFFFFF for i in range(L)], dtype=np.uint32)


def limbs_to_int(a) -> int:
    a = np.asarray(a, dtype=np.uint32).reshape(-1)
    return sum(int(w) << (32 * i) for i, w in enumerate(a))


def _torch():
    import torch
    return torch


def _ptr(t):
    """Device/host pointer of a torch tensor or numpy array (no copies)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return ctypes.c_void_p(t.ctypes.data)
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        torch = _torch()
        if torch.cuda.is_available():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        return ctypes.c_void_p(0)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _check(st: int, what: str):
    if st != 0:
        raise EcmError(st, f"{what}: {lib().ecm_strerror(st).decode()}")


def _count(t, L):
    n = t.numel() if hasattr(t, "numel") else t.size
    if n % L:
        raise ValueError("size is not a multiple of L")
    return n // L


def _validate(t, name: str, *, host: bool, dtype: str, numel: int | None = None, shape=None):
    """Raise ValueError unless `t` is a contiguous array of `dtype` ("uint32" / "uint64" / "uint8")
    with `numel` elements (and `shape`, if given) that lives where the call expects it: host memory
    (numpy or a CPU tensor) with ECM_HOST_BUFFERS, else a CUDA tensor on the current device."""
    if isinstance(t, np.ndarray):
        if t.dtype != np.dtype(dtype):
            raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")
        if not host:
            raise ValueError(f"{name}: host array without ECM_HOST_BUFFERS (a device tensor is required)")
        n, shp = t.size, tuple(t.shape)
    else:
        torch = _torch()
        if not isinstance(t, torch.Tensor):
            raise ValueError(f"{name}: expected a torch tensor or numpy array, got {type(t).__name__}")
        if t.dtype != getattr(torch, dtype):
            raise ValueError(f"{name}: dtype {t.dtype}, expected torch.{dtype}")
        if host and t.is_cuda:
            raise ValueError(f"{name}: CUDA tensor with ECM_HOST_BUFFERS (host memory is required)")
        if not host:
            if not t.is_cuda:
                raise ValueError(f"{name}: CPU tensor without ECM_HOST_BUFFERS (a CUDA tensor is required)")
            if t.device.index != torch.cuda.current_device():
                raise ValueError(f"{name}: on {t.device}, but the current device is cuda:{torch.cuda.current_device()}")
        n, shp = t.numel(), tuple(t.shape)
    if numel is not None and n != numel:
        raise ValueError(f"{name}: {n} elements, expected {numel}")
    if shape is not None and shp != tuple(shape):
        raise ValueError(f"{name}: shape {shp}, expected {tuple(shape)}")


def ecm_mulmod_batch(a, b, n, out=None, *, L: int, iters: int = 1, flags: int = 0, stream=None):
    """out_i = x_iters with x_0 = a_i, x_{t+1} = REDC(x_t * b_i) (or x_t^2 with ECM_SQUARE) mod n_i."""
    count = _count(a, L)
    host = bool(flags & ECM_HOST_BUFFERS)
    shape = tuple(a.shape)
    _validate(a, "a", host=host, dtype="uint32", numel=count * L)
    if not (flags & ECM_SQUARE):
        if b is None:
            raise ValueError("b is required unless ECM_SQUARE")
        _validate(b, "b", host=host, dtype="uint32", numel=count * L, shape=shape)
    _validate(n, "n", host=host, dtype="uint32", numel=count * L, shape=shape)
    if out is None:
        if isinstance(a, np.ndarray):
            out = np.empty_like(a)
        else:
            out = _torch().empty_like(a)
    _validate(out, "out", host=host, dtype="uint32", numel=count * L, shape=shape)
    st = lib().ecm_mulmod_batch(_ptr(a), _ptr(b), _ptr(n), _ptr(out), count, L, iters, flags, _stream(stream))
    _check(st, "ecm_mulmod_batch")
    return out


def _alloc(like_host: bool, shape, dtype_np, device=None):
    if like_host:
        return np.zeros(shape, dtype_np)
    torch = _torch()
    tdt = {np.uint32: torch.uint32, np.uint8: torch.uint8}[dtype_np]
    return torch.empty(shape, dtype=tdt, device=device or "cuda")


def _run_curves(fn, N, L, args, sigmas, flags, stream, want):
    host = bool(flags & ECM_HOST_BUFFERS)
    _validate(sigmas, "sigmas", host=host, dtype="uint64")
    count = sigmas.numel() if hasattr(sigmas, "numel") else sigmas.size
    Nl = int_to_limbs(int(N), L)
    dev = None if host else sigmas.device
    outs = {k: (_alloc(host, (count, L), np.uint32, dev) if k in want else None) for k in ("X", "Z", "g", "xaff")}
    status = _alloc(host, (count,), np.uint8, dev)
    if "xaff" not in want:
        flags |= ECM_NO_XAFF
    st = fn(Nl.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), L, *args, _ptr(sigmas), count,
            _ptr(outs["X"]), _ptr(outs["Z"]), _ptr(outs["g"]), _ptr(status), _ptr(outs["xaff"]), flags,
            _stream(stream))
    _check(st, fn.__name__)
    res = {k: v for k, v in outs.items() if v is not None}
    res["status"] = status
    return res


def ecm_stage1_batch(N: int, L: int, B1: int, sigmas, *, flags: int = 0, stream=None,
                     want=("X", "Z", "g", "xaff")):
    """ECM stage 1 for every sigma (uint64 tensor on the device, or numpy with ECM_HOST_BUFFERS)."""
    return _run_curves(lib().ecm_stage1_batch, N, L, (ctypes.c_uint64(B1),), sigmas, flags, stream, want)


def ecm_ladder_batch(N: int, L: int, k: int, sigmas, *, flags: int = 0, stream=None,
                     want=("X", "Z", "g", "xaff")):
    """[k]P for an explicit scalar k >= 1 (diagnostic entry point)."""
    bits = int(k).bit_length()
    nw = max(1, (bits + 31) // 32)
    kw = int_to_limbs(int(k), nw)
    keep = kw  # keep alive during the call
    args = (kw.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), ctypes.c_uint32(bits))
    r = _run_curves(lib().ecm_ladder_batch, N, L, args, sigmas, flags, stream, want)
    del keep
    return r


def ecm_stage1_kbits(B1: int) -> int:
    return int(lib().ecm_stage1_kbits(B1))


def ecm_version() -> str:
    return lib().ecm_version().decode()
