"""Pins of the oracle's twiddle enclosures (§2.2).

Pinned against: the paper's base roots, the paper's own recurrence
omega_{2n} = (1 + omega_n)/|1 + omega_n| evaluated independently at high
precision, the Lemma's geometric sums, the unit circle, and
direct evaluation of every octant without symmetry.
"""
import json
import os
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import oracle
from oracle.twiddles import direct_enclosure, twiddle_table
from tests.exact import F

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def test_paper_base_roots():
    for ex in GOLD["roots"]:
        t = twiddle_table(ex["N"], "f64")
        assert list(t[ex["j"]]) == ex["w"], ex


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("N", [8, 64, 2048, 8192])
def test_exact_quadrant_points(N, prec):
    t = twiddle_table(N, prec)
    assert list(t[0]) == [1, 1, 0, 0]
    assert list(t[N // 4]) == [0, 0, 1, 1]
    assert list(t[N // 2]) == [-1, -1, 0, 0]
    assert list(t[3 * N // 4]) == [0, 0, -1, -1]


def _recurrence_roots(kmax):
    """omega_1 = 1, omega_2 = -1, omega_4 = i, omega_{2n} = (1+omega_n)/|1+omega_n|."""
    out = {}
    with mpmath.workprec(400):
        w = mpmath.mpc(0, 1)
        out[4] = w
        n = 4
        while n < 2 ** kmax:
            s = 1 + w
            w = s / abs(s)
            n *= 2
            out[n] = w
    return out


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_first_root_contains_paper_recurrence(prec):
    rec = _recurrence_roots(18)
    for N, w in rec.items():
        t = twiddle_table(N, prec) if N <= 8192 else None
        e = t[1] if t is not None else direct_enclosure(N, 1, prec)
        with mpmath.workprec(400):
            wr, wi = w.real, w.imag
            assert mpmath.mpf(float(e[0])) <= wr <= mpmath.mpf(float(e[1])), (N, e, wr)
            assert mpmath.mpf(float(e[2])) <= wi <= mpmath.mpf(float(e[3])), (N, e, wi)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_entries_are_one_ulp_or_exact(prec):
    N = 4096
    t = twiddle_table(N, prec)
    dt = np.float64 if prec == "f64" else np.float32
    for col in (0, 2):
        lo, hi = t[:, col].astype(dt), t[:, col + 1].astype(dt)
        exact = lo == hi
        nxt = np.nextafter(lo, dt(np.inf))
        assert np.all(exact | (hi == nxt))
        # exact only where the value is 0 or +-1
        ex_vals = np.unique(np.abs(lo[exact]))
        assert set(ex_vals.tolist()) <= {0.0, 1.0}


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_every_octant_matches_direct_evaluation(prec):
    rng = np.random.default_rng(5)
    for N in (16, 1024, 32768):
        t = twiddle_table(N, prec)
        js = set(rng.integers(0, N, 60).tolist()) | {1, N // 8, N // 8 + 1, N - 1, N // 2 + 3}
        for j in js:
            d = direct_enclosure(N, j, prec)
            assert tuple(float(x) for x in t[j]) == tuple(float(x) for x in d), (N, j)


def test_contains_true_value_high_precision():
    N = 2048
    t = twiddle_table(N, "f64")
    with mpmath.workprec(500):
        for j in range(0, N, 37):
            th = 2 * mpmath.pi * j / N
            c, s = mpmath.cos(th), mpmath.sin(th)
            assert mpmath.mpf(t[j, 0]) <= c <= mpmath.mpf(t[j, 1])
            assert mpmath.mpf(t[j, 2]) <= s <= mpmath.mpf(t[j, 3])


@pytest.mark.parametrize("N", [8, 16, 64, 256])
def test_lemma_geometric_sums_contain_zero(N):
    """sum_{i<n} omega^{ik} = 0 for 0 < k < n (interval sum contains 0)."""
    t = twiddle_table(N, "f64")
    for k in range(1, N):
        acc = np.array([[0.0, 0.0, 0.0, 0.0]])
        for i in range(N):
            acc = oracle.cinterval_op("add", acc, t[(i * k) % N][None])
        assert acc[0, 0] <= 0 <= acc[0, 1] and acc[0, 2] <= 0 <= acc[0, 3], (N, k, acc)


def test_unit_modulus():
    """|omega^j|^2 = 1: the interval cos^2 + sin^2 contains 1."""
    t = twiddle_table(1024, "f64")
    for j in range(0, 1024, 7):
        c = oracle.interval_op("mul", t[j:j + 1, 0:2], t[j:j + 1, 0:2])
        s = oracle.interval_op("mul", t[j:j + 1, 2:4], t[j:j + 1, 2:4])
        r = oracle.interval_op("add", c, s)
        assert r[0, 0] <= 1.0 <= r[0, 1]
