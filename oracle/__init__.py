"""CPU oracle for arXiv 1310.3809's hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1310_3809_b200``) never imports it and shares no code with it.

This module is argument marshalling (numpy <-> ctypes) around ``oracle/liboracle.so``,
compiled from ``oracle/oracle.c`` (plain C, see the header there for the paper
citations).  Integers are little-endian uint32 limb arrays, ``L`` limbs per element.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, no target-specific flags)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.run(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC", "-o", tmp, _SRC], check=True)
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.orc_mul.argtypes = [_u32p, _u32p, _u32p, ctypes.c_int]
        L.orc_nprime.argtypes = [_u32p, _u32p, ctypes.c_int]
        L.orc_redc_raw.argtypes = [_u32p, _u32p, _u32p, _u32p, ctypes.c_int]
        L.orc_redc.argtypes = [_u32p, _u32p, _u32p, _u32p, ctypes.c_int]
        L.orc_mulmod_chain.argtypes = [_u32p, _u32p, _u32p, _u32p, ctypes.c_size_t, ctypes.c_int,
                                       ctypes.c_uint32, ctypes.c_int, ctypes.c_int]
        L.orc_add_lazy.argtypes = [_u32p, _u32p, _u32p, _u32p, ctypes.c_int]
        L.orc_sub_lazy.argtypes = [_u32p, _u32p, _u32p, _u32p, ctypes.c_int]
        L.orc_stage1_k.argtypes = [ctypes.c_uint64, _u32p, ctypes.c_size_t]
        L.orc_stage1_k.restype = ctypes.c_uint32
        L.orc_ecm_stage1.argtypes = [_u32p, ctypes.c_int, _u32p, ctypes.c_uint32, _u64p, ctypes.c_size_t,
                                     _u32p, _u32p, _u32p, _u8p, _u32p]
        L.orc_ecm_stage1.restype = ctypes.c_int
        L.orc_ecm_stage1_small.argtypes = L.orc_ecm_stage1.argtypes
        L.orc_ecm_stage1_small.restype = ctypes.c_int
        L.orc_ecm_stage1_primes.argtypes = [_u32p, ctypes.c_int, ctypes.c_uint64, _u64p, ctypes.c_size_t,
                                            _u32p, _u32p, _u32p, _u8p, _u32p]
        L.orc_ecm_stage1_primes.restype = ctypes.c_int
        L.orc_suyama.argtypes = [_u32p, ctypes.c_int, ctypes.c_uint64, _u32p, _u32p, _u32p]
        L.orc_suyama.restype = ctypes.c_int
        L.orc_ladder_trace.argtypes = [_u32p, ctypes.c_int, _u32p, ctypes.c_uint32, ctypes.c_uint64, _u32p]
        L.orc_ladder_trace.restype = ctypes.c_int
        _lib = L
    return _lib


# ---------------------------------------------------------------------------------------
# int <-> limbs (marshalling only)
# ---------------------------------------------------------------------------------------
def to_limbs(x: int, L: int) -> np.ndarray:
    if x < 0 or x >> (32 * L):
        raise ValueError("value does not fit in L limbs")
    return np.array([(x >> (32 * i)) & 0xFFFFFFFF for i in range(L)], dtype=np.uint32)


def from_limbs(a) -> int:
    a = np.asarray(a, dtype=np.uint32).reshape(-1)
    return sum(int(w) << (32 * i) for i, w in enumerate(a))


def _p(a: np.ndarray, t=_u32p):
    return a.ctypes.data_as(t)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


# ---------------------------------------------------------------------------------------
# wrappers
# ---------------------------------------------------------------------------------------
def mul(a: int, b: int, L: int) -> int:
    t = np.zeros(2 * L, np.uint32)
    A, B = to_limbs(a, L), to_limbs(b, L)
    lib().orc_mul(_p(A), _p(B), _p(t), L)
    return from_limbs(t)


def nprime(n: int, L: int) -> int:
    out = np.zeros(L, np.uint32)
    N = to_limbs(n, L)
    lib().orc_nprime(_p(N), _p(out), L)
    return from_limbs(out)


def redc_raw(T: int, n: int, L: int) -> int:
    out = np.zeros(L, np.uint32)
    Tl, N = to_limbs(T, 2 * L), to_limbs(n, L)
    np_ = to_limbs(nprime(n, L), L)
    lib().orc_redc_raw(_p(Tl), _p(N), _p(np_), _p(out), L)
    return from_limbs(out)


def redc(T: int, n: int, L: int) -> int:
    out = np.zeros(L, np.uint32)
    Tl, N = to_limbs(T, 2 * L), to_limbs(n, L)
    np_ = to_limbs(nprime(n, L), L)
    lib().orc_redc(_p(Tl), _p(N), _p(np_), _p(out), L)
    return from_limbs(out)


def add_lazy(x: int, y: int, n: int, L: int) -> int:
    out = np.zeros(L, np.uint32)
    lib().orc_add_lazy(_p(to_limbs(x, L)), _p(to_limbs(y, L)), _p(to_limbs(n, L)), _p(out), L)
    return from_limbs(out)


def sub_lazy(x: int, y: int, n: int, L: int) -> int:
    out = np.zeros(L, np.uint32)
    lib().orc_sub_lazy(_p(to_limbs(x, L)), _p(to_limbs(y, L)), _p(to_limbs(n, L)), _p(out), L)
    return from_limbs(out)


def mulmod_chain(a: np.ndarray, b: np.ndarray, n: np.ndarray, L: int, iters: int,
                 square: bool = False, canonical: bool = False) -> np.ndarray:
    """AoS arrays of shape (count, L) or flat (count*L,).  Returns (count, L) uint32."""
    a, b, n = _u32(a), _u32(b), _u32(n)
    count = a.size // L
    out = np.zeros((count, L), np.uint32)
    lib().orc_mulmod_chain(_p(a), _p(b), _p(n), _p(out), count, L, iters, int(square), int(canonical))
    return out


def stage1_k(B1: int) -> tuple[int, int]:
    """k = prod p^e (p^e <= B1 < p^(e+1)); returns (k, bitlen(k))."""
    cap = max(4, int(B1 * 1.5 / 32) + 8)   # bits(k) ~ 1.44 B1
    w = np.zeros(cap, np.uint32)
    bits = lib().orc_stage1_k(B1, _p(w), cap)
    if bits == 0:
        raise ValueError("bad B1")
    return from_limbs(w), int(bits)


def k_words(k: int) -> tuple[np.ndarray, int]:
    bits = k.bit_length()
    nw = (bits + 31) // 32
    return to_limbs(k, nw), bits


def ecm_stage1(N: int, L: int, k: int, sigmas, want_xaff: bool = True, family: str = "suyama"):
    """Returns dict of numpy arrays X, Z, g (count, L), status (count,), xaff (count, L).
    family "suyama" (the paper's curves) or "small" (§8(f) N4: a24 = s/2^32, x0 = 2)."""
    sig = np.ascontiguousarray(np.asarray(sigmas, dtype=np.uint64))
    count = sig.size
    kw, kb = k_words(k)
    Nl = to_limbs(N, L)
    X = np.zeros((count, L), np.uint32)
    Z = np.zeros((count, L), np.uint32)
    g = np.zeros((count, L), np.uint32)
    st = np.zeros(count, np.uint8)
    xa = np.zeros((count, L), np.uint32)
    fn = {"suyama": lib().orc_ecm_stage1, "small": lib().orc_ecm_stage1_small}[family]
    rc = fn(_p(Nl), L, _p(kw), kb, _p(sig, _u64p), count, _p(X), _p(Z), _p(g),
            _p(st, _u8p), _p(xa) if want_xaff else None)
    if rc != 0:
        raise ValueError("orc_ecm_stage1: bad arguments")
    return {"X": X, "Z": Z, "g": g, "status": st, "xaff": xa}


def ecm_stage1_primes(N: int, L: int, B1: int, sigmas):
    """Paper-comparable schedule: prime-by-prime ladders (see oracle.h)."""
    sig = np.ascontiguousarray(np.asarray(sigmas, dtype=np.uint64))
    count = sig.size
    Nl = to_limbs(N, L)
    X, Z, g, xa = (np.zeros((count, L), np.uint32) for _ in range(4))
    st = np.zeros(count, np.uint8)
    rc = lib().orc_ecm_stage1_primes(_p(Nl), L, B1, _p(sig, _u64p), count, _p(X), _p(Z), _p(g), _p(st, _u8p), _p(xa))
    if rc != 0:
        raise ValueError("orc_ecm_stage1_primes: bad arguments")
    return {"X": X, "Z": Z, "g": g, "status": st, "xaff": xa}


def suyama(N: int, L: int, sigma: int):
    x0 = np.zeros(L, np.uint32)
    a24 = np.zeros(L, np.uint32)
    g = np.zeros(L, np.uint32)
    st = lib().orc_suyama(_p(to_limbs(N, L)), L, sigma, _p(x0), _p(a24), _p(g))
    return st, from_limbs(x0), from_limbs(a24), from_limbs(g)


def ladder_trace(N: int, L: int, k: int, sigma: int):
    """Canonical normal-domain (X0, Z0, X1, Z1) after the initial doubling and each step."""
    kw, kb = k_words(k)
    tr = np.zeros((kb, 4, L), np.uint32)
    st = lib().orc_ladder_trace(_p(to_limbs(N, L)), L, _p(kw), kb, sigma, _p(tr))
    if st < 0:
        raise ValueError("bad arguments")
    if st:
        return st, None
    out = [[from_limbs(tr[s, j]) for j in range(4)] for s in range(kb)]
    return 0, out


# ---------------------------------------------------------------------------------------
# host-thread fan-out (marshalling only: chunks of independent elements / curves)
# ---------------------------------------------------------------------------------------
def _pool_map(fn, chunks, threads):
    import concurrent.futures as cf
    if threads <= 1 or len(chunks) <= 1:
        return [fn(c) for c in chunks]
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:  # ctypes releases the GIL
        return list(ex.map(fn, chunks))


def mulmod_chain_mt(a, b, n, L, iters, square=False, canonical=False, threads=None):
    a, b, n = (np.ascontiguousarray(x, dtype=np.uint32).reshape(-1, L) for x in (a, b, n))
    threads = threads or os.cpu_count() or 1
    count = a.shape[0]
    step = max(1, -(-count // (threads * 4)))
    idx = [(s, min(count, s + step)) for s in range(0, count, step)]
    parts = _pool_map(lambda r: mulmod_chain(a[r[0]:r[1]], b[r[0]:r[1]], n[r[0]:r[1]], L, iters, square, canonical),
                      idx, threads)
    return np.concatenate(parts, axis=0)


def ecm_stage1_primes_mt(N, L, B1, sigmas, threads=None):
    sig = np.asarray(sigmas, dtype=np.uint64)
    threads = threads or os.cpu_count() or 1
    count = sig.size
    step = max(1, -(-count // (threads * 2)))
    idx = [(s, min(count, s + step)) for s in range(0, count, step)]
    parts = _pool_map(lambda r: ecm_stage1_primes(N, L, B1, sig[r[0]:r[1]]), idx, threads)
    return {key: np.concatenate([p[key] for p in parts], axis=0) for key in parts[0]}


def ecm_stage1_mt(N, L, k, sigmas, threads=None, family="suyama"):
    sig = np.asarray(sigmas, dtype=np.uint64)
    threads = threads or os.cpu_count() or 1
    count = sig.size
    step = max(1, -(-count // (threads * 2)))
    idx = [(s, min(count, s + step)) for s in range(0, count, step)]
    parts = _pool_map(lambda r: ecm_stage1(N, L, k, sig[r[0]:r[1]], family=family), idx, threads)
    return {key: np.concatenate([p[key] for p in parts], axis=0) for key in parts[0]}
