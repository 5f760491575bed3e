"""Pins for the oracle's ECM stage 1.

Independent anchors: k = lcm(1..B1) (math.lcm) and SPEC's k(10) = 2520; brute-force point
counts over small prime fields (Suyama curves have 12 | #E); the textbook affine group law
on B y^2 = x^3 + A x^2 + x (with y, Montgomery 1987) for [s]P and for the order of P; the
x-only ladder invariant; planted-factor recovery; divisibility of every reported g.
"""
import math
import random

import numpy as np
import pytest

from workload import ecm_config, random_prime

SMALL_PRIMES = [p for p in range(101, 1200) if all(p % d for d in range(2, int(p ** 0.5) + 1))]


# --------------------------------------------------------------------------------------
# independent affine group law (Python ints) on B y^2 = x^3 + A x^2 + x over Z/pZ
# --------------------------------------------------------------------------------------
O = None


def aff_add(P, Q, A, B, p):
    if P is O:
        return Q
    if Q is O:
        return P
    x1, y1 = P
    x2, y2 = Q
    if x1 == x2:
        if (y1 + y2) % p == 0:
            return O
        lam = (3 * x1 * x1 + 2 * A * x1 + 1) * pow(2 * B * y1, -1, p) % p
    else:
        lam = (y2 - y1) * pow(x2 - x1, -1, p) % p
    x3 = (B * lam * lam - A - x1 - x2) % p
    y3 = (lam * (x1 - x3) - y1) % p
    return (x3, y3)


def aff_mul(s, P, A, B, p):
    R, Q = O, P
    while s:
        if s & 1:
            R = aff_add(R, Q, A, B, p)
        Q = aff_add(Q, Q, A, B, p)
        s >>= 1
    return R


def curve_of(orc, p, sigma):
    """(A, B, x0) with P = (x0, 1) on B y^2 = x^3 + A x^2 + x, A = 4 a24 - 2."""
    st, x0, a24, _ = orc.suyama(p, 1, sigma)
    if st:
        return None
    A = (4 * a24 - 2) % p
    B = (x0 ** 3 + A * x0 * x0 + x0) % p
    if B == 0 or (A * A - 4) % p == 0:
        return None
    return A, B, x0


def count_points(A, B, p):
    """#E(F_p) by brute force: 1 (infinity) + sum over x of #{y : B y^2 = f(x)}."""
    Binv = pow(B, -1, p)
    n = 1
    for x in range(p):
        r = (x * x * x + A * x * x + x) * Binv % p
        if r == 0:
            n += 1
        elif pow(r, (p - 1) // 2, p) == 1:
            n += 2
    return n


# --------------------------------------------------------------------------------------
def test_stage1_k_is_lcm(orc):
    assert orc.stage1_k(10) == (2520, 12)
    assert orc.stage1_k(2)[0] == 2
    for B1 in (3, 17, 100, 2000, 8192):
        k, bits = orc.stage1_k(B1)
        assert k == math.lcm(*range(1, B1 + 1)) and bits == k.bit_length()


def test_stage1_k_bitlens(orc):
    want = {B1: math.lcm(*range(1, B1 + 1)).bit_length() for B1 in (2000, 8192, 50000)}
    for B1, bl in want.items():
        assert orc.stage1_k(B1)[1] == bl
    assert want[2000] == 2878 and want[8192] == 11797 and want[50000] == 72115


@pytest.mark.parametrize("p", SMALL_PRIMES[::12])
def test_suyama_group_order_divisible_by_12(orc, p):
    """Brent-Suyama curves have 12 | #E(F_p) (reading G10); P = (x0, 1) is on the curve."""
    seen = 0
    for sigma in range(6, 30):
        c = curve_of(orc, p, sigma)
        if c is None:
            continue
        A, B, x0 = c
        assert (B * 1 - (x0 ** 3 + A * x0 * x0 + x0)) % p == 0
        assert count_points(A, B, p) % 12 == 0
        seen += 1
    assert seen > 10


@pytest.mark.parametrize("p", SMALL_PRIMES[3::25])
def test_ladder_matches_affine_group_law(orc, p):
    """x([s]P) from the oracle's ladder == affine double-and-add, s = 1..60;
    Z == 0 exactly when ord(P) | s, and [#E]P = O."""
    for sigma in (6, 7, 11, 23):
        c = curve_of(orc, p, sigma)
        if c is None:
            continue
        A, B, x0 = c
        P = (x0, 1)
        nE = count_points(A, B, p)
        for s in list(range(1, 61)) + [nE]:
            r = orc.ecm_stage1(p, 1, s, [sigma])
            X, Z = orc.from_limbs(r["X"][0]), orc.from_limbs(r["Z"][0])
            Q = aff_mul(s, P, A, B, p)
            if Q is O:
                assert Z == 0 and r["status"][0] == 2 and orc.from_limbs(r["g"][0]) == p
            else:
                assert Z != 0 and r["status"][0] == 0
                assert X * pow(Z, -1, p) % p == Q[0]
                assert orc.from_limbs(r["xaff"][0]) == Q[0]


def _invariant(st, A, xd, zd, N):
    X0, Z0, X1, Z1 = st
    t1 = (X0 * Z1 - X1 * Z0) ** 2 * xd * xd
    t2 = 2 * ((X0 * X1 + Z0 * Z1) * (X0 * Z1 + X1 * Z0) + 2 * A * X0 * X1 * Z0 * Z1) * xd * zd
    t3 = (X0 * X1 - Z0 * Z1) ** 2 * zd * zd
    return (t1 - t2 + t3) % N


def test_ladder_step_invariant_composite(orc):
    """R1 - R0 = P after every ladder step, modulo a composite N (§8(c) c6 (i))."""
    cfg = ecm_config("C1")
    N, L = cfg["N"], cfg["L"]
    k, _ = orc.stage1_k(300)
    for sigma in cfg["sigmas"][:3]:
        st, x0, a24, _ = orc.suyama(N, L, int(sigma))
        assert st == 0
        A = (4 * a24 - 2) % N
        st, trace = orc.ladder_trace(N, L, k, int(sigma))
        assert st == 0 and len(trace) == k.bit_length()
        for state in trace:
            assert _invariant(state, A, x0, 1, N) == 0
        # a corrupted state must break it (the test can fail)
        bad = list(trace[5])
        bad[0] = (bad[0] + 1) % N
        assert _invariant(bad, A, x0, 1, N) != 0


def test_ladder_prefix_states_are_multiples(orc):
    """State after j steps is ([m]P, [m+1]P) with m the top j+1 bits of k (small p)."""
    p = 1009
    c = curve_of(orc, p, 9)
    A, B, x0 = c
    k = 0b1011001110101
    st, trace = orc.ladder_trace(p, 1, k, 9)
    bits = k.bit_length()
    for j, (X0, Z0, X1, Z1) in enumerate(trace):
        m = k >> (bits - 1 - j)
        for (X, Z), mult in (((X0, Z0), m), ((X1, Z1), m + 1)):
            Q = aff_mul(mult, (x0, 1), A, B, p)
            if Q is O:
                assert Z == 0
            else:
                assert X * pow(Z, -1, p) % p == Q[0]


def test_c1_planted_factor_and_affine_x(orc):
    """C1: about 10% of curves find p; every g divides N; affine x on
    status-0 curves equals an independent affine double-and-add over Z/NZ."""
    cfg = ecm_config("C1")
    N, L, p = cfg["N"], cfg["L"], cfg["p"]
    k, _ = orc.stage1_k(cfg["B1"])
    r = orc.ecm_stage1(N, L, k, cfg["sigmas"])
    st = r["status"]
    found = int((st == 1).sum())
    assert 10 <= found <= 45, found
    for i in np.nonzero(st == 1)[0]:
        g = orc.from_limbs(r["g"][i])
        assert N % g == 0 and g == p
    checked = 0
    for i in np.nonzero(st == 0)[0][:4]:
        sigma = int(cfg["sigmas"][i])
        _, x0, a24, _ = orc.suyama(N, L, sigma)
        A = (4 * a24 - 2) % N
        B = (x0 ** 3 + A * x0 * x0 + x0) % N
        Q = aff_mul(k, (x0, 1), A, B, N)  # an inversion failure would raise: none expected
        assert orc.from_limbs(r["xaff"][i]) == Q[0]
        X, Z = orc.from_limbs(r["X"][i]), orc.from_limbs(r["Z"][i])
        assert X * pow(Z, -1, N) % N == Q[0]
        checked += 1
    assert checked == 4


def test_setup_degenerate_sigma(orc):
    """u = sigma^2 - 5 = 0 mod N -> status 3; = 0 mod one prime only -> status 4 (§8(b))."""
    # 15^2 - 5 = 220 = 20 * 11
    st, _, _, g = orc.suyama(11, 1, 15)
    assert st == 3 and g == 11
    st, _, _, g = orc.suyama(143, 1, 15)
    assert st == 4 and g == 11
    k, _ = orc.stage1_k(50)
    r = orc.ecm_stage1(143, 1, k, [15])
    assert r["status"][0] == 4 and orc.from_limbs(r["g"][0]) == 11
    assert orc.from_limbs(r["X"][0]) == 0 and orc.from_limbs(r["Z"][0]) == 0


def test_planted_prime_generator():
    cfg = ecm_config("C3")
    assert cfg["N"].bit_length() == 190 and cfg["p"].bit_length() == 64
    assert cfg["N"] == cfg["p"] * cfg["q"]
    assert len(cfg["sigmas"]) == 1 << 20 and int(cfg["sigmas"].min()) >= 6
    assert random_prime(100, 200, 1) == random_prime(100, 200, 1)


def test_prime_schedule_same_point(orc):
    """The paper-comparable prime-by-prime schedule computes the same [k]P: affine x and status
    equal the full-k ladder's (formula-free, reading G9b); X:Z differ by a projective factor."""
    cfg = ecm_config(L=6, nbits=190, pbits=32, B1=400, curves=40, seed=9)
    k, _ = orc.stage1_k(cfg["B1"])
    a = orc.ecm_stage1(cfg["N"], 6, k, cfg["sigmas"])
    b = orc.ecm_stage1_primes(cfg["N"], 6, cfg["B1"], cfg["sigmas"])
    assert np.array_equal(a["status"], b["status"])
    assert np.array_equal(a["xaff"], b["xaff"])
    assert (a["status"] == 1).any()
    ok = np.nonzero(a["status"] == 0)[0]
    assert not np.array_equal(a["X"][ok], b["X"][ok])  # projective representatives differ
    N = cfg["N"]
    for i in ok[:5]:
        X1, Z1 = orc.from_limbs(a["X"][i]), orc.from_limbs(a["Z"][i])
        X2, Z2 = orc.from_limbs(b["X"][i]), orc.from_limbs(b["Z"][i])
        assert (X1 * Z2 - X2 * Z1) % N == 0


@pytest.mark.parametrize("p", [1009, 2003])
def test_prime_schedule_small_field(orc, p):
    """Prime-by-prime ladders over F_p agree with affine [k]P for k = lcm(1..B1)."""
    B1 = 30
    k, _ = orc.stage1_k(B1)
    for sigma in (6, 7, 11):
        c = curve_of(orc, p, sigma)
        if c is None:
            continue
        A, B, x0 = c
        r = orc.ecm_stage1_primes(p, 1, B1, [sigma])
        Q = aff_mul(k, (x0, 1), A, B, p)
        if Q is O:
            assert r["status"][0] == 2
        else:
            assert r["status"][0] == 0 and orc.from_limbs(r["xaff"][0]) == Q[0]


# --------------------------------------------------------------------------------------
# small-parameter family (reading G16): a24 = s / 2^32 mod N, x0 = 2
# --------------------------------------------------------------------------------------
def small_curve(p, s):
    """(A, B) with P = (2, 1) on B y^2 = x^3 + A x^2 + x, A = 4 a24 - 2, a24 = s / 2^32 mod p."""
    a24 = s * pow(1 << 32, -1, p) % p
    A = (4 * a24 - 2) % p
    B = (8 + 4 * A + 2) % p
    if B == 0 or (A * A - 4) % p == 0:
        return None
    return A, B


@pytest.mark.parametrize("p", SMALL_PRIMES[5::30])
def test_small_family_matches_affine_group_law(orc, p):
    """x([m]P) of the small-parameter family's ladder == the affine group law on the curve through
    P = (2, 1), m = 1..40 and m = #E (Z = 0 exactly when ord(P) | m)."""
    seen = 0
    for s in (1, 2, 3, 17, 1000, (1 << 29) + 3, (1 << 30) - 1):
        c = small_curve(p, s)
        if c is None:
            continue
        A, B = c
        P = (2, 1)
        nE = count_points(A, B, p)
        for m in list(range(1, 41)) + [nE]:
            r = orc.ecm_stage1(p, 1, m, [s], family="small")
            X, Z = orc.from_limbs(r["X"][0]), orc.from_limbs(r["Z"][0])
            Q = aff_mul(m, P, A, B, p)
            if Q is O:
                assert Z == 0 and r["status"][0] == 2 and orc.from_limbs(r["g"][0]) == p
            else:
                assert Z != 0 and r["status"][0] == 0
                assert X * pow(Z, -1, p) % p == Q[0] == orc.from_limbs(r["xaff"][0])
        seen += 1
    assert seen >= 4


def test_small_family_seed_range_and_planted_factor(orc):
    """Seeds outside [1, 2^30) are rejected per curve (status 3, g = N); on C1's modulus the
    family finds the planted 32-bit prime on some curves, and every g divides N."""
    cfg = ecm_config("C1")
    N, p = cfg["N"], cfg["p"]
    k, _ = orc.stage1_k(cfg["B1"])
    r = orc.ecm_stage1(N, 6, k, [0, 1 << 30, (1 << 62) + 5], family="small")
    assert list(r["status"]) == [3, 3, 3]
    assert all(orc.from_limbs(g) == N for g in r["g"])
    seeds = np.arange(1, 257, dtype=np.uint64) * 4099
    r = orc.ecm_stage1_mt(N, 6, k, seeds, family="small")
    found = r["status"] == 1
    assert found.sum() >= 5
    for g, st in zip(r["g"], r["status"]):
        gi = orc.from_limbs(g)
        assert N % gi == 0
        if st == 1:
            assert gi == p
