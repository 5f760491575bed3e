"""Input recipes.  No method arithmetic lives here.

Randomness is a counter-based splitmix64: word i of stream (seed, tag) is
``mix(base(seed, tag) + (i + 1) * GAMMA)``, so any element can be regenerated alone and the
arrays are identical on every machine.  Integers are little-endian uint32 limbs.
"""
from __future__ import annotations

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def _mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _base(seed: int, tag: int) -> int:
    return _mix((seed * 0x2545F4914F6CDD1D + tag * GAMMA + 0x632BE59BD9B4E019) & M64)


def splitmix64(seed: int, i: int, tag: int = 0) -> int:
    """Word i of the (seed, tag) stream."""
    return _mix((_base(seed, tag) + (i + 1) * GAMMA) & M64)


def splitmix64_array(seed: int, start: int, count: int, tag: int = 0) -> np.ndarray:
    """Words start..start+count-1 of the (seed, tag) stream as uint64 (vectorised)."""
    with np.errstate(over="ignore"):
        idx = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(_base(seed, tag)) + idx * np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


# ---------------------------------------------------------------------------------------
# primes for planted factors (input generation only)
# ---------------------------------------------------------------------------------------
_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71)


def is_probable_prime(n: int) -> bool:
    if n < 2:
        return False
    for p in _MR_BASES:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _MR_BASES:  # deterministic below 3.3e24; error < 4^-20 above
        x = pow(a, d, n)
        if x == 1 or x == n - 1:
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def _rand_below(seed: int, tag: int, ctr: list, bound: int) -> int:
    nb = bound.bit_length()
    while True:
        words = (nb + 63) // 64
        v = 0
        for _ in range(words):
            v = (v << 64) | splitmix64(seed, ctr[0], tag)
            ctr[0] += 1
        v &= (1 << nb) - 1
        if v < bound:
            return v


def random_prime(lo: int, hi: int, seed: int, tag: int = 7) -> int:
    """First probable prime drawn uniformly from [lo, hi) by the (seed, tag) stream."""
    ctr = [0]
    while True:
        c = lo + _rand_below(seed, tag, ctr, hi - lo)
        if is_probable_prime(c):
            return c


# ---------------------------------------------------------------------------------------
# batched mulmod inputs (configs C2 / C4)
# ---------------------------------------------------------------------------------------
def _words(seed, tag, start, count):
    return (splitmix64_array(seed, start, count, tag) & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def mulmod_inputs(count: int, L: int, bits: int | None = None, seed: int = 2, lazy: bool = False,
                  start: int = 0, chunk: int = 1 << 20):
    """(a, b, n) as (count, L) uint32 arrays for elements start..start+count-1.

    n_i: uniform odd with bitlen exactly ``bits`` (default 32L-2, reading G14);
    a_i, b_i: random limbs with top limb drawn below n_i's top limb, so a_i, b_i < n_i.
    lazy=True adds n_i to a_i and b_i on a random per-element bit, exercising [0, 2n_i).
    """
    if bits is None:
        bits = 32 * L - 2
    if not (32 * (L - 1) < bits <= 32 * L - 2):
        raise ValueError("bits must satisfy 32(L-1) < bits <= 32L-2")
    tb = bits - 32 * (L - 1)  # significant bits in the top limb, 1..30
    a = np.empty((count, L), np.uint32)
    b = np.empty((count, L), np.uint32)
    n = np.empty((count, L), np.uint32)
    for c0 in range(0, count, chunk):
        m = min(chunk, count - c0)
        e0 = start + c0
        nw = _words(seed, 2, e0 * L, m * L).reshape(m, L)
        nw[:, L - 1] = (nw[:, L - 1] >> np.uint32(32 - tb)) | np.uint32(1 << (tb - 1))
        nw[:, 0] |= np.uint32(1)
        top = nw[:, L - 1].astype(np.uint64)
        for arr, tag in ((a, 0), (b, 1)):
            w = _words(seed, tag, e0 * L, m * L).reshape(m, L)
            r = splitmix64_array(seed, e0, m, 16 + tag)
            w[:, L - 1] = (r % top).astype(np.uint32)
            if lazy:
                sel = (splitmix64_array(seed, e0, m, 32 + tag) & np.uint64(1)).astype(bool)
                carry = np.zeros(m, np.uint64)
                s = w.astype(np.uint64)
                addend = nw.astype(np.uint64) * sel[:, None].astype(np.uint64)
                for j in range(L):
                    t = s[:, j] + addend[:, j] + carry
                    s[:, j] = t & np.uint64(0xFFFFFFFF)
                    carry = t >> np.uint64(32)
                w = s.astype(np.uint32)
            arr[c0:c0 + m] = w
        n[c0:c0 + m] = nw
    return a, b, n


# ---------------------------------------------------------------------------------------
# ECM configs (C1 / C3 / C5)
# ---------------------------------------------------------------------------------------
def sigmas(seed: int, count: int, start: int = 0) -> np.ndarray:
    """sigma_i = 6 + (splitmix64(seed, i) mod 2^62) (reading G10)."""
    r = splitmix64_array(seed, start, count, tag=3)
    return (r & np.uint64((1 << 62) - 1)) + np.uint64(6)


ECM_CONFIGS = {
    # name: (L, bitlen(N), bits of planted p (None = ~32-bit p in [2^31,2^32)), B1, curves, seed)
    "C1": dict(L=6, nbits=190, pbits=32, B1=2000, curves=256, seed=1),
    "C3": dict(L=6, nbits=190, pbits=64, B1=50000, curves=1 << 20, seed=3),
    "C5": dict(L=8, nbits=254, pbits=80, B1=250000, curves=1 << 22, seed=5),
}

MULMOD_CONFIGS = {
    "C2": dict(L=6, count=1 << 24, seed=2, iters=(1, 16, 256)),
    "C4": dict(Ls=(4, 6, 8, 12), count=1 << 24, seed=4, iters=256),
}


def ecm_config(name: str | None = None, *, L=None, nbits=None, pbits=None, B1=None, curves=None,
               seed=None) -> dict:
    """N = p*q with a planted pbits-bit prime p and bitlen(N) = nbits exactly; sigmas.

    Returns dict(N, p, q, L, B1, sigmas, seed, ...)."""
    cfg = dict(ECM_CONFIGS[name]) if name else {}
    for k, v in dict(L=L, nbits=nbits, pbits=pbits, B1=B1, curves=curves, seed=seed).items():
        if v is not None:
            cfg[k] = v
    s, nb, pb = cfg["seed"], cfg["nbits"], cfg["pbits"]
    p = random_prime(1 << (pb - 1), 1 << pb, s, tag=7)
    lo = -(-(1 << (nb - 1)) // p)  # ceil(2^(nb-1)/p)
    hi = ((1 << nb) - 1) // p + 1
    q = random_prime(lo, hi, s, tag=8)  # p*q in [2^(nb-1), 2^nb) by the choice of [lo, hi)
    assert (p * q).bit_length() == nb and q != p
    cfg.update(N=p * q, p=p, q=q, sigmas=sigmas(s, cfg["curves"]))
    cfg["name"] = name
    return cfg


# ---------------------------------------------------------------------------------------
# Width-limit worst cases: moduli at and near R/4 = 2^(32L-2), the largest
# the two spare bits allow, and operands at the ends of the lazy domain [0, 2N).
# ---------------------------------------------------------------------------------------
def edge_moduli(L: int, seed: int = 60) -> list[int]:
    """Odd moduli with bitlen <= 32L-2 where the carry bounds are tightest: 2^(32L-2)-1 (N just
    below R/4), 2^(32L-2)-3, top limb 0x3fffffff with seeded random lower limbs, the smallest
    full-width N = 2^(32L-3)+1, and the tiny moduli 3 and 5."""
    top = 1 << (32 * L - 2)
    r = int(splitmix64(seed, L, tag=9)) | (int(splitmix64(seed, L, tag=10)) << 64)
    low = (r | (r << 128) | (r << 256) | (r << 384)) & ((1 << (32 * (L - 1))) - 1)
    return [top - 1, top - 3, (0x3FFFFFFF << (32 * (L - 1))) | low | 1, (top >> 1) + 1, 3, 5]


def edge_mulmod_inputs(L: int, reps: int = 2, seed: int = 60):
    """(a, b, n) (count, L) uint32 arrays: every modulus of edge_moduli(L) with every ordered pair
    of operands from {0, 1, N-1, N, 2N-2, 2N-1} (all < 2N), the whole list repeated `reps` times
    so that a batch spans full tiles and a ragged tail."""
    rows = []
    for N in edge_moduli(L, seed):
        ops = sorted({0, 1, N - 1, N, 2 * N - 2, 2 * N - 1})
        rows += [(x, y, N) for x in ops for y in ops]
    rows = rows * reps

    def limbs(v):
        return [(v >> (32 * j)) & 0xFFFFFFFF for j in range(L)]
    a = np.array([limbs(x) for x, _, _ in rows], np.uint32)
    b = np.array([limbs(y) for _, y, _ in rows], np.uint32)
    n = np.array([limbs(N) for _, _, N in rows], np.uint32)
    return a, b, n


def near_max_composite(L: int, pbits: int = 32, seed: int = 61) -> tuple[int, int, int]:
    """(N, p, q): N = p*q with a planted pbits-bit prime p and q the largest prime with
    p*q < 2^(32L-2), so N sits just below R/4."""
    p = random_prime(1 << (pbits - 1), 1 << pbits, seed, tag=11)
    q = ((1 << (32 * L - 2)) - 1) // p
    q -= 1 - (q & 1)
    while not is_probable_prime(q):
        q -= 2
    return p * q, p, q
