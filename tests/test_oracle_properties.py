"""Property-based pins of the oracle (hypothesis, CPU): over random widths and ranges the
oracle must agree with what Eq.(4) and the accept rule fix mathematically.

* w <= 26, any accepted pair of any valid range: every step of Eq.(4) before the division is
  exact in binary64, so the oracle's q is the correctly rounded value of the exact rational
  (2^w (x1 - a0) + x2 - b) / (2^w (a - a0) - b)  (R1/R8) -- Python's
  float(Fraction) is that rounding;
* that value lies strictly inside (0, 1) (R12) and is monotone in (x1, x2) (Eq.(4) is an
  increasing affine map of z = x1 + k x2, Eq.(1));
* the accept rule is exactly a0 < x1 < a (R3);
* w in 27..32: q within the rounding bound of the exact E (at w = 32, full range:
  2^-53 + 2^-54 + 2^-62).
"""
from fractions import Fraction

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st


@st.composite
def ranges(draw, wmin=1, wmax=26):
    w = draw(st.integers(wmin, wmax))
    wb = draw(st.integers(1, w))                  # x2 width <= w (b < 2^w, R5)
    b = (1 << wb) - 1
    # bitlen(a): with bitlen(a) + w <= 53, z = x1 + k x2, C, D and z - C are exact (w <= 26)
    wa = draw(st.integers(2, 32 if w >= 27 else min(32, 53 - w)))
    a = draw(st.integers(max(2, 1 << (wa - 1)), (1 << wa) - 1))
    a0 = draw(st.integers(0, a - 2))
    x1 = draw(st.integers(a0 + 1, a - 1))         # an accepted x1
    x2 = draw(st.integers(0, b))
    return dict(w=w, a0=a0, a=a, b0=0, b=b), x1, x2


def exact(p, x1, x2):
    w = p["w"]
    return Fraction((x1 - p["a0"]) * (1 << w) + x2 - p["b"], (p["a"] - p["a0"]) * (1 << w) - p["b"])


@settings(max_examples=400, deadline=None)
@given(ranges())
def test_eq4_is_the_rounded_exact_rational(orc_h, case):
    p, x1, x2 = case
    e = exact(p, x1, x2)
    q = orc_h.map_pairs(p, [x1], [x2])[0]
    assert 0 < e < 1
    assert q == float(e), (p, x1, x2)


@settings(max_examples=300, deadline=None)
@given(ranges(), st.integers(0, 3), st.integers(0, 3))
def test_eq4_is_monotone(orc_h, case, d1, d2):
    p, x1, x2 = case
    y1, y2 = min(x1 + d1, p["a"] - 1), min(x2 + d2, p["b"])
    q0, q1 = orc_h.map_pairs(p, [x1, y1], [x2, y2])
    assert q1 >= q0


@settings(max_examples=400, deadline=None)
@given(ranges(27, 32))
def test_eq4_error_bound_wide(orc_h, case):
    """w >= 27: z, C and z - C each round once (half an ulp of a value below 2^bitlen(a)), D
    once (relative 2^-53) and the quotient once: |q - E| <= 3 2^(bitlen(a) - 54) / D +
    E 2^-52 + 2^-54 -- at w = 32 on the full range the 2^-53 + 2^-54 + 2^-62 of DESIGN.md."""
    p, x1, x2 = case
    q = Fraction(orc_h.map_pairs(p, [x1], [x2])[0])
    e = exact(p, x1, x2)
    d = Fraction(p["a"] - p["a0"]) - Fraction(p["b"], 1 << p["w"])
    bound = Fraction(3 * 2 ** p["a"].bit_length(), 2**54) / d + e / 2**52 + Fraction(1, 2**54)
    assert abs(q - e) <= bound, (p, x1, x2)


@settings(max_examples=300, deadline=None)
@given(ranges(1, 32), st.integers(0, 2**32 - 1))
def test_accept_rule(orc_h, case, x1):
    p, _, _ = case
    assert orc_h.accept(p, x1) == (p["a0"] < x1 < p["a"])


@pytest.fixture(scope="module")
def orc_h():
    import oracle
    oracle.build()
    return oracle
