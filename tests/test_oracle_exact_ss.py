"""Pins of the oracle's output intervals, max radius and certification on whole
multiplications, against an independent exact-rational recomputation of the
paper's method (tests/exact_ss.py: P:143-155 recursive FFT, P:251-253 and
P:264-265 interval operations with every endpoint rounded from the exact
rational, P:203-211 fast convolution, P:97 inverse, R10 radius).

Every output interval (all N of them) and the max radius must be equal as
numbers (+0 == -0), so a dropped or rescaled radius term (/4 instead of /2,
width instead of radius, the imaginary part ignored) or a changed certify rule
fails here.  The radius of the used coefficients is also pinned at N <= 4,
where every twiddle is exact (1, i, -1, -i) and all arithmetic on digits is
exact, so the radius must be exactly 0.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_1006_0405_b200 import inputs

from .exact import ru64
from .exact_ss import ExactSS


def to_int(d):
    return int.from_bytes(bytes(np.asarray(d, np.uint8)), "little")


# Pairs whose largest radius lies in an IMAGINARY part (found by search over
# random digit pairs; the test re-establishes the property exactly below).
IMAG_DOMINATED = [
    ([176, 0, 0, 0, 0], [152, 19, 67, 4, 35]),
    ([0, 207, 0, 223, 0], [0, 241, 0, 240, 0]),
    ([214, 0, 0, 0, 0, 0, 0, 0], [175, 43, 130, 20, 6, 73, 142, 25]),
    ([0, 0, 0, 244, 0, 244, 0, 0], [0, 0, 0, 201, 0, 228, 0, 0]),
]


def _check_against_exact(a, b, prec):
    E = ExactSS(prec)
    o = oracle.ivmul(a, b, prec=prec, want_intervals=True, want_coeffs=True)
    for p in range(a.shape[0]):
        r = E.multiply(a[p].tolist(), b[p].tolist())
        n = a.shape[1]
        assert o["N"] == r["N"]
        got = o["intervals"][p].astype(np.float64)
        assert np.array_equal(got, r["intervals"]), (prec, a[p], b[p])
        assert o["max_radius"][p] == r["max_radius"], (prec, o["max_radius"][p], r["max_radius"])
        # certified iff every used coefficient holds exactly one integer
        # and its imaginary part only 0; then the product is exact
        used = r["intervals"][:2 * n - 1]
        want_cert = all(np.ceil(lo) == np.floor(hi) and np.ceil(il) == 0 and np.floor(ih) == 0
                        for lo, hi, il, ih in used)
        assert bool(o["cert"][p]) == want_cert
        if want_cert:
            assert to_int(o["prod"][p]) == to_int(a[p]) * to_int(b[p])
            assert o["first_bad"][p] == -1
        else:
            assert (o["prod"][p] == 0).all() and o["first_bad"][p] >= 0


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n", [3, 4, 5, 6, 7, 8])  # N = 8 (n = 3, 4) and 16 (n = 5 .. 8)
def test_whole_multiply_matches_exact_recomputation(prec, n):
    kinds = np.array([0, 0, 1, 2, 3, 0])
    a, b = inputs.pair_digits(0x5EED + n, np.arange(len(kinds)), n, kinds)
    _check_against_exact(a, b, prec)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_imaginary_part_radius_counts(prec):
    """Pairs whose max radius comes from an imaginary part: the oracle's max
    radius must equal the exact recomputation's, i.e. include that part."""
    E = ExactSS(prec)
    for x, y in IMAG_DOMINATED:
        r = E.multiply(x, y)
        if prec == "f64":
            assert r["radius_im"] > r["radius_re"]
        a, b = np.array([x], np.uint8), np.array([y], np.uint8)
        _check_against_exact(a, b, prec)


def test_fp32_uncertified_pairs_match_exact_recomputation():
    """binary32 at n = 8 with large digits: wide enough not to certify, so the
    first-failing index and the zero-filled product are pinned too."""
    a = np.full((2, 8), 255, np.uint8)
    b = np.full((2, 8), 255, np.uint8)
    b[1, ::2] = 254
    o = oracle.ivmul(a, b, prec="f32")
    E = ExactSS("f32")
    for p in range(2):
        r = E.multiply(a[p].tolist(), b[p].tolist())
        assert o["max_radius"][p] == r["max_radius"]
    _check_against_exact(a, b, "f32")


def test_radius_exactly_zero_when_every_twiddle_is_exact():
    """N <= 4 (n <= 2): twiddles 1, i, -1, -i are exact and every operation on
    digit-valued data is exact, so every interval is a point: radius 0."""
    vals = [0, 1, 2, 127, 128, 254, 255]
    g = np.array([(p, q) for p in vals for q in vals], np.uint8)
    a = np.repeat(g, len(g), axis=0)
    b = np.tile(g, (len(g), 1))
    r = oracle.ivmul(a, b, want_intervals=True)
    assert r["N"] == 4
    assert (r["max_radius"] == 0).all()
    assert (r["intervals"][..., 0] == r["intervals"][..., 1]).all()
    assert r["cert"].all()


def test_max_radius_definition():
    """DESIGN.md R10: max over both parts of RU(hi - lo)/2; NaN -> inf."""
    iv = np.array([[0.0, 1.0, 0.0, 0.0], [2.0, 2.0, -0.25, 0.25]])
    assert oracle.max_radius(iv) == 0.5
    iv[1, 2:] = [-1.0, 1.0]
    assert oracle.max_radius(iv) == 1.0  # the imaginary part is the larger
    # an inexact difference is rounded UP: 1 - (-2^-60) -> next double above 1
    lo = -2.0 ** -60
    iv = np.array([[lo, 1.0, 0.0, 0.0]])
    want = ru64(Fraction(1) - Fraction(lo)) / 2
    assert want > 0.5 and oracle.max_radius(iv) == want
    assert oracle.max_radius(np.array([[np.nan, 1.0, 0.0, 0.0]])) == np.inf
    assert oracle.max_radius(np.zeros((3, 4))) == 0.0
    # binary32 twin: endpoints widened exactly, difference rounded up in binary64
    f = np.array([[np.float32(-2.0 ** -40), np.float32(1.0), 0, 0]], np.float32)
    assert oracle.max_radius(f, "f32") == ru64(Fraction(1) + Fraction(2 ** -40)) / 2
