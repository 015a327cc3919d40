"""Pins for the circular-containment-set oracle (oracle/ivm_oracle_disc.c;
P:290, reading R15), checked against things the oracle does not
compute itself: exact rational arithmetic (fractions), Python int products,
closed forms, and the exact DFT of special vectors.

A plausible slip in the disc rules (a dropped a.r*b.r or |c| r term, a missing
rounding term, a wrong sign in the conjugate or the butterfly) makes one of the
containment checks fail: they test points on the boundary of the input discs,
not only the centers.
"""
import math
from fractions import Fraction as F

import numpy as np
import pytest

import oracle



def exact_product_digits(a, b):
    """Python int product as 2n little-endian base-256 digits."""
    z = int.from_bytes(bytes(a), "little") * int.from_bytes(bytes(b), "little")
    return np.frombuffer(z.to_bytes(2 * len(a), "little"), np.uint8)


def _in_disc(z, d):
    """exact z = (re, im) Fractions inside disc d = (cr, ci, r) (floats)."""
    dr, di = z[0] - F(d[0]), z[1] - F(d[1])
    return dr * dr + di * di <= F(d[2]) * F(d[2])


def _boundary_points(d, k=8):
    """exact rational points on (just inside) the circle of disc d."""
    pts = [(F(d[0]), F(d[1]))]
    for j in range(k):
        # rational point on the unit circle: ((1-t^2)/(1+t^2), 2t/(1+t^2)), shrunk by 1 - 2^-40
        t = F(math.tan(math.pi * j / k / 2)).limit_denominator(10 ** 6) if j else F(0)
        den = 1 + t * t
        ux, uy = (1 - t * t) / den, 2 * t / den
        for sx, sy in ((1, 1), (-1, 1), (1, -1), (-1, -1)):
            s = F(d[2]) * (1 - F(1, 2 ** 40))
            pts.append((F(d[0]) + sx * s * ux, F(d[1]) + sy * s * uy))
    return pts


def _random_discs(rng, k, scale):
    c = rng.standard_normal((k, 2)) * scale
    r = np.abs(rng.standard_normal(k)) * scale * 10.0 ** rng.integers(-12, 0, k)
    return np.column_stack([c, r])


@pytest.mark.parametrize("op", ["add", "sub", "mul"])
def test_disc_primitives_contain_every_point_product(op):
    rng = np.random.default_rng(11)
    a = _random_discs(rng, 60, 1e3)
    b = _random_discs(rng, 60, 1e2)
    res = oracle.disc_op(op, a, b)
    f = {"add": lambda x, y: (x[0] + y[0], x[1] + y[1]),
         "sub": lambda x, y: (x[0] - y[0], x[1] - y[1]),
         "mul": lambda x, y: (x[0] * y[0] - x[1] * y[1], x[0] * y[1] + x[1] * y[0])}[op]
    for i in range(a.shape[0]):
        pa, pb = _boundary_points(a[i], 4), _boundary_points(b[i], 4)
        for za in pa[::3]:
            for zb in pb[::3]:
                assert _in_disc(f(za, zb), res[i]), (op, i)


@pytest.mark.parametrize("op", ["add", "mul"])
def test_disc_primitives_are_not_loose(op):
    """The radius stays within the R15 formula's own bound (a factor-2 slack
    would flag e.g. a doubled term)."""
    rng = np.random.default_rng(12)
    a = _random_discs(rng, 200, 1e3)
    b = _random_discs(rng, 200, 1e2)
    res = oracle.disc_op(op, a, b)
    U = 2.0 ** -52
    for i in range(a.shape[0]):
        ca, cb = complex(a[i, 0], a[i, 1]), complex(b[i, 0], b[i, 1])
        if op == "add":
            bound = a[i, 2] + b[i, 2] + U * 2 * (abs(ca) + abs(cb)) * 1.5
        else:
            bound = (abs(ca) * b[i, 2] + abs(cb) * a[i, 2] + a[i, 2] * b[i, 2]
                     + U * 8 * abs(ca) * abs(cb)) * (1 + 1e-12)
        assert res[i, 2] <= bound, (op, i, res[i], bound)
        assert res[i, 2] >= a[i, 2] if op == "add" else True


def test_disc_conjugate():
    a = np.array([[1.5, -2.25, 0.125], [0.0, 3.0, 1.0]])
    r = oracle.disc_op("conj", a, a)
    assert np.array_equal(r, np.array([[1.5, 2.25, 0.125], [0.0, -3.0, 1.0]]))


def test_disc_fft_impulse_and_constant():
    """P:143-155 on discs: FFT(e_0) = all ones, FFT(1,...,1) = (N, 0, ..., 0),
    exactly contained, with radii near zero."""
    N = 64
    e0 = np.zeros((N, 3))
    e0[0, 0] = 1.0
    out = oracle.disc_fft(e0)
    for k in range(N):
        assert _in_disc((F(1), F(0)), out[k])
    # closed form of R15 here: every stage adds E + w 0 = E exactly, and the
    # sum rule charges U |E| = 2^-52 (plus the 2^-1000 guards): radius log2(N) 2^-52
    assert np.all(out[:, 0] == 1.0) and np.all(out[:, 1] == 0.0)
    assert np.allclose(out[:, 2], 6 * 2.0 ** -52, rtol=1e-12, atol=0)
    ones = np.zeros((N, 3))
    ones[:, 0] = 1.0
    out = oracle.disc_fft(ones)
    assert _in_disc((F(N), F(0)), out[0])
    for k in range(1, N):
        assert _in_disc((F(0), F(0)), out[k])
    assert out[:, 2].max() < 1e-12


def test_disc_fft_contains_exact_dft():
    """Random punctual integer vectors: the exact DFT (evaluated with exact
    rational cos/sin enclosures is not needed: |exact - center| is bounded by
    the radius, checked with mpmath at 60 digits)."""
    import mpmath
    mpmath.mp.dps = 60
    rng = np.random.default_rng(13)
    N = 32
    x = np.zeros((N, 3))
    x[:, 0] = rng.integers(0, 256, N)
    for inverse in (0, 1):
        out = oracle.disc_fft(x, inverse)
        sgn = -1 if inverse else 1
        for k in range(N):
            s = mpmath.fsum(int(x[j, 0]) * mpmath.expjpi(sgn * mpmath.mpf(2 * j * k) / N) for j in range(N))
            d = mpmath.sqrt((s.real - out[k, 0]) ** 2 + (s.imag - out[k, 1]) ** 2)
            assert d <= out[k, 2], (inverse, k)


def test_disc_multiply_certified_products_are_exact():
    rng = np.random.default_rng(14)
    for n in (1, 2, 3, 17, 100, 257, 1000):
        a = rng.integers(0, 256, (6, n), dtype=np.uint8)
        b = rng.integers(0, 256, (6, n), dtype=np.uint8)
        a[0] = 255
        b[0] = 255
        r = oracle.disc_mul(a, b)
        assert r["cert"].all(), n
        for p in range(6):
            assert np.array_equal(r["prod"][p], exact_product_digits(a[p], b[p])), (n, p)


def test_disc_multiply_all_255_closed_form():
    """(256^n - 1)^2 = [1, 0 x (n-1), 254, 255 x (n-1)] (little-endian)."""
    n = 3000
    a = np.full((1, n), 255, np.uint8)
    r = oracle.disc_mul(a, a)
    want = np.concatenate([[1], np.zeros(n - 1), [254], np.full(n - 1, 255)]).astype(np.uint8)
    assert r["cert"][0] and np.array_equal(r["prod"][0], want)


def test_disc_multiply_brute_force_two_digit_pairs():
    ds = [0, 1, 2, 127, 128, 254, 255]
    pairs = [(x0, x1, y0, y1) for x0 in ds for x1 in ds for y0 in ds for y1 in ds]
    a = np.array([[p[0], p[1]] for p in pairs], np.uint8)
    b = np.array([[p[2], p[3]] for p in pairs], np.uint8)
    r = oracle.disc_mul(a, b)
    assert r["cert"].all()
    for i, p in enumerate(pairs):
        z = (p[0] + 256 * p[1]) * (p[2] + 256 * p[3])
        assert int.from_bytes(bytes(r["prod"][i]), "little") == z


def test_disc_output_discs_contain_the_exact_coefficients():
    """Containment of every convolution coefficient in its output disc,
    imaginary part 0 included, for uniform, all-255 and sparse operands."""
    rng = np.random.default_rng(15)
    n = 300
    a = rng.integers(0, 256, (3, n), dtype=np.uint8)
    b = rng.integers(0, 256, (3, n), dtype=np.uint8)
    a[1] = 255
    b[1] = 255
    a[2] *= (rng.random(n) < 0.1).astype(np.uint8)
    r = oracle.disc_mul(a, b, want_discs=True)
    for p in range(3):
        c = np.convolve(a[p].astype(np.int64), b[p].astype(np.int64))
        d = r["discs"][p]
        for i in range(2 * n - 1):
            assert _in_disc((F(int(c[i])), F(0)), d[i]), (p, i)


def test_disc_radius_is_tighter_than_rectangles_at_large_n():
    """The paper's motivation for circular sets: rotations do not wrap.
    Recorded, not assumed: at n = 4096 the disc radius is below the rectangle's."""
    rng = np.random.default_rng(16)
    n = 4096
    a = rng.integers(0, 256, (2, n), dtype=np.uint8)
    b = rng.integers(0, 256, (2, n), dtype=np.uint8)
    d = oracle.disc_mul(a, b)
    r = oracle.ivmul(a, b)
    assert d["cert"].all() and r["cert"].all()
    assert (d["max_radius"] < r["max_radius"]).all()
