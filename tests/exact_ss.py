"""An exact-rational recomputation of the paper's interval multiply (tests only).

Written independently of oracle/ (no shared code, tables or constants) to pin
the oracle's radius and certification on whole small multiplications:

- twiddles omega_N^j = e^{2 pi i j/N} as [RD, RU] of cos/sin, from
  mpmath at 256 bits, the quarter-turn values 0, +-1 exact;
- the real interval operations of P:251-253, every endpoint the exact rational
  result rounded down / up (tests/exact.py), the product the min / max of the
  four endpoint products;
- the complex operations of P:264-265;
- the recursive Cooley-Tukey FFT of P:143-155 in the paper's order
  (step 10: out_i = Xe_{i mod n/2} + omega^i * Xo_{i mod n/2});
- the fast convolution of P:203-211 (forward, pointwise, inverse with the
  conjugate roots, then 1/N);
- the radius of DESIGN.md R10: RU(hi - lo)/2 over both parts of the 2n-1 used
  coefficients.

Slow (Fractions everywhere): meant for N <= 16.
"""
from __future__ import annotations

from fractions import Fraction

import mpmath
import numpy as np

from .exact import rd32, rd64, ru32, ru64

F = lambda x: Fraction(float(x))


def _mp_frac(x) -> Fraction:
    x = mpmath.mpf(x)
    man, exp = abs(x).man_exp  # |x| = man * 2^exp
    man, exp = int(man), int(exp)
    q = Fraction(man * 2 ** exp) if exp >= 0 else Fraction(man, 2 ** (-exp))
    return -q if x < 0 else q


class ExactSS:
    def __init__(self, prec: str = "f64"):
        self.prec = prec
        self.rd, self.ru = (rd64, ru64) if prec == "f64" else (rd32, ru32)

    # ---- P:251-253 ----
    def iadd(self, a, b):
        return (self.rd(F(a[0]) + F(b[0])), self.ru(F(a[1]) + F(b[1])))

    def isub(self, a, b):
        return (self.rd(F(a[0]) - F(b[1])), self.ru(F(a[1]) - F(b[0])))

    def imul(self, a, b):
        ps = [F(x) * F(y) for x in a for y in b]
        return (self.rd(min(ps)), self.ru(max(ps)))

    # ---- P:264-265 ----
    def cadd(self, z, w):
        return (self.iadd(z[0], w[0]), self.iadd(z[1], w[1]))

    def cmul(self, z, w):
        return (self.isub(self.imul(z[0], w[0]), self.imul(z[1], w[1])),
                self.iadd(self.imul(z[0], w[1]), self.imul(z[1], w[0])))

    @staticmethod
    def conj(z):
        return (z[0], (-z[1][1], -z[1][0]))

    # ---- omega_N^j, optimal enclosure ----
    def twiddle(self, j: int, N: int):
        j %= N
        if (4 * j) % N == 0:  # 1, i, -1, -i: exact
            c, s = [(1, 0), (0, 1), (-1, 0), (0, -1)][4 * j // N]
            return ((float(c), float(c)), (float(s), float(s)))
        with mpmath.workprec(256):
            t = 2 * mpmath.pi * j / N
            c, s = _mp_frac(mpmath.cos(t)), _mp_frac(mpmath.sin(t))
        # 256-bit values are within 2^-250 of the truth; none of these
        # irrational cos/sin lies that close to a binary64/32 number
        return ((self.rd(c), self.ru(c)), (self.rd(s), self.ru(s)))

    # ---- P:143-155, recursive, literally ----
    def fft(self, x, N_total: int, inverse: bool):
        n = len(x)
        if n == 1:
            return [x[0]]
        h = n // 2
        Xe = self.fft(x[0::2], N_total, inverse)
        Xo = self.fft(x[1::2], N_total, inverse)
        out = []
        for i in range(n):
            w = self.twiddle(i * (N_total // n), N_total)
            if inverse:
                w = self.conj(w)
            out.append(self.cadd(Xe[i % h], self.cmul(w, Xo[i % h])))
        return out

    # ---- P:203-211 + P:97 ----
    def multiply(self, a, b):
        n = len(a)
        N = 1
        while N < 2 * n - 1:
            N *= 2
        zero = (0.0, 0.0)
        ap = [((float(d), float(d)), zero) for d in a] + [(zero, zero)] * (N - n)
        bp = [((float(d), float(d)), zero) for d in b] + [(zero, zero)] * (N - n)
        A = self.fft(ap, N, False)
        B = self.fft(bp, N, False)
        P = [self.cmul(A[k], B[k]) for k in range(N)]
        c = self.fft(P, N, True)
        c = [((self.rd(F(z[0][0]) / N), self.ru(F(z[0][1]) / N)),
              (self.rd(F(z[1][0]) / N), self.ru(F(z[1][1]) / N))) for z in c]
        iv = np.array([[z[0][0], z[0][1], z[1][0], z[1][1]] for z in c], np.float64)
        used = iv[:2 * n - 1]
        rad_re = max(ru64(F(hi) - F(lo)) / 2 + 0.0 for lo, hi in used[:, 0:2])
        rad_im = max(ru64(F(hi) - F(lo)) / 2 + 0.0 for lo, hi in used[:, 2:4])
        return {"N": N, "intervals": iv, "max_radius": max(rad_re, rad_im),
                "radius_re": rad_re, "radius_im": rad_im}
