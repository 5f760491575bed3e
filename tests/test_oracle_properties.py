"""Property-based pins of the oracle (hypothesis): randomised operands and moduli of every width,
checked against Python integers.  Complements tests/test_oracle_arith.py's seeded cases."""
import pytest
from hypothesis import given, settings, strategies as st


@st.composite
def modulus_and_operands(draw):
    L = draw(st.sampled_from([1, 2, 3, 4, 6, 8, 12, 16]))
    bits = draw(st.integers(min_value=2, max_value=32 * L - 2))
    n = draw(st.integers(min_value=1 << (bits - 1), max_value=(1 << bits) - 1)) | 1
    if n < 3:
        n = 3
    x = draw(st.integers(min_value=0, max_value=2 * n - 1))
    y = draw(st.integers(min_value=0, max_value=2 * n - 1))
    return L, n, x, y


@settings(max_examples=400, deadline=None)
@given(modulus_and_operands())
def test_redc_raw_property(orc, case):
    L, n, x, y = case
    R = 1 << (32 * L)
    out = orc.redc_raw(x * y, n, L)
    q, rem = divmod(out * R - x * y, n)
    assert rem == 0 and 0 <= q < R and out < 2 * n
    assert orc.redc(x * y, n, L) == x * y * pow(R, -1, n) % n


@settings(max_examples=300, deadline=None)
@given(modulus_and_operands())
def test_lazy_add_sub_property(orc, case):
    L, n, x, y = case
    s, d = orc.add_lazy(x, y, n, L), orc.sub_lazy(x, y, n, L)
    assert 0 <= s < 2 * n and (s - x - y) % n == 0
    assert 0 <= d < 2 * n and (d - x + y) % n == 0


@settings(max_examples=200, deadline=None)
@given(st.sampled_from([1, 2, 4, 6, 8, 12, 16]), st.data())
def test_mul_and_nprime_property(orc, L, data):
    a = data.draw(st.integers(min_value=0, max_value=(1 << (32 * L)) - 1))
    b = data.draw(st.integers(min_value=0, max_value=(1 << (32 * L)) - 1))
    assert orc.mul(a, b, L) == a * b
    n = a | 1
    assert (n * orc.nprime(n, L) + 1) % (1 << (32 * L)) == 0
