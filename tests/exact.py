"""Exact-rational helpers for the pins (tests only; independent of oracle/).

Directed rounding of an exact rational to binary64 / binary32, written from
the IEEE 754 definition (largest float <= q, smallest float >= q) with
``math.nextafter`` / ``numpy.nextafter`` and exact ``Fraction`` comparisons.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np


def rd64(q: Fraction) -> float:
    f = float(q)
    while Fraction(f) > q:
        f = math.nextafter(f, -math.inf)
    while Fraction(math.nextafter(f, math.inf)) <= q:
        f = math.nextafter(f, math.inf)
    return f


def ru64(q: Fraction) -> float:
    return -rd64(-q)


def rd32(q: Fraction) -> float:
    f = np.float32(float(q))
    while Fraction(float(f)) > q:
        f = np.nextafter(f, np.float32(-np.inf))
    while Fraction(float(np.nextafter(f, np.float32(np.inf)))) <= q:
        f = np.nextafter(f, np.float32(np.inf))
    return float(f)


def ru32(q: Fraction) -> float:
    return -rd32(-q)


def F(x) -> Fraction:
    return Fraction(float(x))
