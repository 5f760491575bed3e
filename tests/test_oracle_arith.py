"""Pins for the oracle's multiprecision / Montgomery routines.

Everything here checks oracle/ against something other than itself: Python's arbitrary
precision integers (product, modular inverse by pow), the defining property of REDC
(T + qN = out*R with 0 <= q < R, unique), brute force on tiny moduli, closed forms of the
multiplication chains, and the bounds the paper prints in its Lemma.
"""
import random

import numpy as np
import pytest

from workload import mulmod_inputs

LS = (1, 2, 4, 6, 8, 12, 16)


def rnd_mod(rng, L, bits=None):
    bits = bits or 32 * L - 2
    return rng.getrandbits(bits) | (1 << (bits - 1)) | 1


@pytest.mark.parametrize("L", LS)
def test_mul_schoolbook_matches_python(orc, L):
    rng = random.Random(L)
    for _ in range(200):
        a, b = rng.getrandbits(32 * L), rng.getrandbits(32 * L)
        assert orc.mul(a, b, L) == a * b
    full = (1 << (32 * L)) - 1
    assert orc.mul(full, full, L) == full * full
    assert orc.mul(0, full, L) == 0


@pytest.mark.parametrize("L", LS)
def test_nprime_definition(orc, L):
    """m * m' = -1 (mod R)."""
    rng = random.Random(100 + L)
    R = 1 << (32 * L)
    for _ in range(100):
        n = rng.getrandbits(32 * L) | 1
        np_ = orc.nprime(n, L)
        assert 0 <= np_ < R and (n * np_ + 1) % R == 0
    assert (13 * orc.nprime(13, 1) + 1) % (1 << 32) == 0


def test_spec_examples_tiny(orc):
    """SPEC examples re-derived with the oracle's R = 2^32: m=13."""
    R = 1 << 32
    Rinv = pow(R, -1, 13)
    # redc(1) = R^{-1} mod 13; to_mont(1) = R mod 13 squares to itself
    assert orc.redc(1, 13, 1) == Rinv % 13
    one_m = R % 13
    assert orc.redc(one_m * one_m, 13, 1) == one_m


@pytest.mark.parametrize("L", (1, 2))
def test_redc_brute_force_tiny_moduli(orc, L):
    """Brute force on tiny N (< 2^16 held in L limbs): R^{-1} found by search."""
    rng = random.Random(7 + L)
    R = 1 << (32 * L)
    for _ in range(60):
        n = rng.randrange(3, 1 << 16) | 1
        rinv = next(r for r in range(n) if (r * (R % n)) % n == 1)  # brute-force search
        for _ in range(20):
            x, y = rng.randrange(2 * n), rng.randrange(2 * n)
            out = orc.redc_raw(x * y, n, L)
            assert out % n == x * y * rinv % n
            assert out < 2 * n
            assert orc.redc(x * y, n, L) == x * y * rinv % n


@pytest.mark.parametrize("L", (4, 6, 8, 12, 16))
def test_redc_raw_is_the_unique_definition(orc, L):
    """out*R = T + q*N for the unique q in [0, R): the raw lazy value."""
    rng = random.Random(200 + L)
    R = 1 << (32 * L)
    for _ in range(300):
        n = rnd_mod(rng, L)
        x, y = rng.randrange(2 * n), rng.randrange(2 * n)
        T = x * y
        out = orc.redc_raw(T, n, L)
        q, rem = divmod(out * R - T, n)
        assert rem == 0 and 0 <= q < R
        assert out < 2 * n                                  # Lemma with R >= 4N (reading G3)
        assert orc.redc(T, n, L) == T * pow(R, -1, n) % n  # canonical, step 3


@pytest.mark.parametrize("L", (4, 6, 8))
def test_lemma_bounds(orc, L):
    """Lemma: a,b < 2R' -> redc <= R'+m < 2R'; a,b < 3R' -> < 13/4 R'."""
    rng = random.Random(300 + L)
    for _ in range(300):
        bits = rng.randrange(32 * (L - 1) + 1, 32 * L - 1)
        n = rnd_mod(rng, L, bits)
        Rp = 1 << n.bit_length()
        a, b = rng.randrange(2 * Rp), rng.randrange(2 * Rp)
        assert orc.redc_raw(a * b, n, L) <= Rp + n
        a, b = rng.randrange(3 * Rp), rng.randrange(3 * Rp)
        assert 4 * orc.redc_raw(a * b, n, L) < 13 * Rp
        a = b = 2 * Rp - 1  # worst case of claim 1
        assert orc.redc_raw(a * b, n, L) <= Rp + n


@pytest.mark.parametrize("L", (4, 6, 8, 12))
def test_lazy_add_sub(orc, L):
    rng = random.Random(400 + L)
    for _ in range(300):
        n = rnd_mod(rng, L)
        x, y = rng.randrange(2 * n), rng.randrange(2 * n)
        s, d = orc.add_lazy(x, y, n, L), orc.sub_lazy(x, y, n, L)
        assert 0 <= s < 2 * n and (s - x - y) % n == 0
        assert 0 <= d < 2 * n and (d - x + y) % n == 0
    n = rnd_mod(rng, L)
    assert orc.add_lazy(2 * n - 1, 2 * n - 1, n, L) == 2 * n - 2
    assert orc.sub_lazy(0, 2 * n - 1, n, L) == 1


def _ints(arr):
    return [sum(int(w) << (32 * j) for j, w in enumerate(row)) for row in arr]


@pytest.mark.parametrize("L", (4, 6, 8, 12))
@pytest.mark.parametrize("square", (False, True))
def test_chain_closed_form(orc, L, square):
    """Canonical x_K = a (b R^-1)^K (mul) and a^(2^K) R^-(2^K - 1) (sqr) mod N (§8(c) c2)."""
    K = 20 if square else 57
    a, b, n = mulmod_inputs(64, L, seed=11 + L, lazy=True)
    raw = orc.mulmod_chain(a, b, n, L, K, square=square, canonical=False)
    can = orc.mulmod_chain(a, b, n, L, K, square=square, canonical=True)
    R = 1 << (32 * L)
    for ai, bi, ni, r, c in zip(_ints(a), _ints(b), _ints(n), _ints(raw), _ints(can)):
        Ri = pow(R, -1, ni)
        if square:
            want = pow(ai, 1 << K, ni) * pow(Ri, (1 << K) - 1, ni) % ni
        else:
            want = ai * pow(bi * Ri % ni, K, ni) % ni
        assert c == want
        assert r < 2 * ni and r % ni == want


def test_chain_raw_single_step_definition(orc):
    """K = 1 raw outputs equal the unique REDC value of a*b, element by element."""
    L = 6
    a, b, n = mulmod_inputs(500, L, seed=5, lazy=True)
    raw = orc.mulmod_chain(a, b, n, L, 1)
    R = 1 << (32 * L)
    for ai, bi, ni, r in zip(_ints(a), _ints(b), _ints(n), _ints(raw)):
        q, rem = divmod(r * R - ai * bi, ni)
        assert rem == 0 and 0 <= q < R


def test_inputs_in_domain():
    """The generator's recipe: bitlen(n) = 32L-2, n odd, a,b < n (or < 2n when lazy)."""
    for L in (4, 6, 8, 12):
        for lazy in (False, True):
            a, b, n = mulmod_inputs(300, L, seed=9, lazy=lazy)
            for ai, bi, ni in zip(_ints(a), _ints(b), _ints(n)):
                assert ni & 1 and ni.bit_length() == 32 * L - 2
                bound = 2 * ni if lazy else ni
                assert ai < bound and bi < bound
    # counter-based: a slice regenerates identically
    a, b, n = mulmod_inputs(100, 6, seed=3)
    a2, b2, n2 = mulmod_inputs(10, 6, seed=3, start=50)
    assert np.array_equal(a[50:60], a2) and np.array_equal(n[50:60], n2)


@pytest.mark.parametrize("L", (4, 6, 8, 12, 16))
@pytest.mark.parametrize("square", (False, True))
def test_chain_width_limit_edges(orc, L, square):
    """The width-limit worst cases the GPU tests use (workload.edge_mulmod_inputs: N at and just
    below R/4, the smallest full-width N, N = 3, 5; operands 0, 1, N-1, N, 2N-2, 2N-1): the raw
    single step is the unique REDC value (out R = T + qN, 0 <= q < R, out < 2N) and the K = 3
    chain's canonical value matches the closed form."""
    from workload import edge_mulmod_inputs
    a, b, n = edge_mulmod_inputs(L, reps=1)
    R = 1 << (32 * L)
    raw1 = orc.mulmod_chain(a, b, n, L, 1, square=square)
    can3 = orc.mulmod_chain(a, b, n, L, 3, square=square, canonical=True)
    for ai, bi, ni, r, c in zip(_ints(a), _ints(b), _ints(n), _ints(raw1), _ints(can3)):
        T = ai * ai if square else ai * bi
        q, rem = divmod(r * R - T, ni)
        assert rem == 0 and 0 <= q < R and r < 2 * ni
        Ri = pow(R, -1, ni)
        want = pow(ai, 8, ni) * pow(Ri, 7, ni) % ni if square else ai * pow(bi * Ri % ni, 3, ni) % ni
        assert c == want
