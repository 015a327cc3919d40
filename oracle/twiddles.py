"""Optimal interval enclosures of the roots of unity -- ORACLE side.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

omega_N^j = e^{2 pi i j / N} (§2.2 Def.), as the tightest
machine intervals [RD(cos), RU(cos)] + i [RD(sin), RU(sin)].  The paper
builds omega by the recurrence of P:163 and says "other efficient methods of
computing omega are also available"; reading R2 explains why
the optimal enclosure is used instead.  The values come from mpmath at 320 bits
and are rounded to binary64 / binary32 by EXACT rational comparison, with a
rigorous error allowance; an entry whose rounding cannot be decided raises.

The table is built independently of the CUDA path's planner (which uses
__float128 in C++); both must agree bit for bit (a cross-check in tests).
"""
from __future__ import annotations

import functools
import math
from fractions import Fraction

import mpmath
import numpy as np

_PREC_BITS = 320
_EPS = Fraction(1, 2 ** 300)  # |mpmath value - true value| bound (generous)


def _exact(x: mpmath.mpf) -> Fraction:
    sign, man, exp, _ = mpmath.mpf(x)._mpf_
    man = -int(man) if sign else int(man)
    exp = int(exp)
    return Fraction(man * 2 ** exp) if exp >= 0 else Fraction(man, 2 ** (-exp))


def _rd64(q: Fraction) -> float:
    f = float(q)  # correctly rounded to nearest
    if Fraction(f) > q:
        f = math.nextafter(f, -math.inf)
    return f


def _ru64(q: Fraction) -> float:
    f = float(q)
    if Fraction(f) < q:
        f = math.nextafter(f, math.inf)
    return f


def _rd32(q: Fraction) -> np.float32:
    c = np.float32(float(q))
    while Fraction(float(c)) > q:
        c = np.nextafter(c, np.float32(-np.inf))
    while Fraction(float(np.nextafter(c, np.float32(np.inf)))) <= q:
        c = np.nextafter(c, np.float32(np.inf))
    return c


def _ru32(q: Fraction) -> np.float32:
    c = np.float32(float(q))
    while Fraction(float(c)) < q:
        c = np.nextafter(c, np.float32(np.inf))
    while Fraction(float(np.nextafter(c, np.float32(-np.inf)))) >= q:
        c = np.nextafter(c, np.float32(-np.inf))
    return c


def enclose(q: Fraction, prec: str, exact: bool = False):
    """[RD, RU] of a real known to lie in [q - eps, q + eps] (or exactly q)."""
    rd, ru = (_rd64, _ru64) if prec == "f64" else (_rd32, _ru32)
    if exact:
        return rd(q), ru(q)
    lo1, lo2 = rd(q - _EPS), rd(q + _EPS)
    hi1, hi2 = ru(q - _EPS), ru(q + _EPS)
    if lo1 != lo2 or hi1 != hi2:
        raise ArithmeticError("twiddle rounding undecidable at this precision")
    return lo1, hi1


def _cos_sin_exact(j: int, N: int):
    """(cos, sin) of 2 pi j / N for j in the first octant, as Fractions."""
    with mpmath.workprec(_PREC_BITS):
        theta = 2 * mpmath.pi * j / N
        return _exact(mpmath.cos(theta)), _exact(mpmath.sin(theta))


@functools.lru_cache(maxsize=16)
def twiddle_table(N: int, prec: str = "f64") -> np.ndarray:
    """Array [N][4] = (re.lo, re.hi, im.lo, im.hi) enclosing omega_N^j, j < N.

    The first octant j <= N/8 is evaluated; the rest follows from the exact
    symmetries cos(pi/2 - t) = sin t, cos(t + pi/2) = -sin t, ... which commute
    with directed rounding (RD(-x) = -RU(x)).  Entries at j = 0, N/4, N/2,
    3N/4 are exact (1, i, -1, -i: PAPER.md:163 omega_1 = 1, omega_2 = -1,
    omega_4 = i).
    """
    assert N >= 1 and N & (N - 1) == 0
    dtype = np.float64 if prec == "f64" else np.float32
    out = np.zeros((N, 4), dtype=dtype)
    if N == 1:
        out[0] = (1, 1, 0, 0)
        return out
    # first-quadrant values c(j) = cos(2 pi j/N), s(j) = sin, j in [0, N/4]
    q = N // 4
    cq = {}
    if N >= 4:
        for j in range(0, N // 8 + 1):
            if j == 0:
                c = (dtype(1), dtype(1)); s = (dtype(0), dtype(0))
            elif N >= 8 and 8 * j == N:  # pi/4: cos = sin, irrational
                cx, sx = _cos_sin_exact(j, N)
                c = enclose(cx, prec); s = c
            else:
                cx, sx = _cos_sin_exact(j, N)
                c = enclose(cx, prec); s = enclose(sx, prec)
            cq[j] = (c, s)
        for j in range(N // 8 + 1, q + 1):  # mirror: angle pi/2 - t
            c, s = cq[q - j]
            cq[j] = (s, c)
    for j in range(N):
        if N == 2:
            out[j] = (1, 1, 0, 0) if j == 0 else (-1, -1, 0, 0)
            continue
        quad, r = divmod(j, q)
        (clo, chi), (slo, shi) = cq[r]
        if quad == 0:    # ( c,  s)
            out[j] = (clo, chi, slo, shi)
        elif quad == 1:  # angle t + pi/2: (-s, c)
            out[j] = (-shi, -slo, clo, chi)
        elif quad == 2:  # t + pi: (-c, -s)
            out[j] = (-chi, -clo, -shi, -slo)
        else:            # t + 3pi/2: (s, -c)
            out[j] = (slo, shi, -chi, -clo)
    return out


def direct_enclosure(N: int, j: int, prec: str = "f64"):
    """Enclosure of omega_N^j evaluated directly at angle 2 pi j/N (no symmetry).

    Used by the pins to check entries of every octant independently.
    """
    if (4 * j) % N == 0:
        quarter = (4 * j) // N % 4
        return [(1, 1, 0, 0), (0, 0, 1, 1), (-1, -1, 0, 0), (0, 0, -1, -1)][quarter]
    with mpmath.workprec(_PREC_BITS + 40):
        theta = 2 * mpmath.pi * j / N
        c, s = _exact(mpmath.cos(theta)), _exact(mpmath.sin(theta))
    lo, hi = enclose(c, prec)
    slo, shi = enclose(s, prec)
    return (lo, hi, slo, shi)
