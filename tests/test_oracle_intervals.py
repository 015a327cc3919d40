"""Pins of the oracle's interval arithmetic (§2.5).

Pinned against exact rational arithmetic (fractions.Fraction) rounded by the
IEEE definition in tests/exact.py, and against worked examples in
tests/golden/worked_examples.json.  A swapped rounding direction, a dropped
endpoint product, or a wrong endpoint pairing fails these tests.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests.exact import F, rd32, rd64, ru32, ru64

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def test_rounding_self_check():
    assert oracle.self_check()


def _rand_intervals(rng, m, dtype, straddle=True):
    a = rng.standard_normal((m, 2)) * np.exp(rng.uniform(-20, 20, (m, 1)))
    if not straddle:
        a = np.abs(a)
    a = a.astype(dtype)
    a.sort(axis=1)
    return a


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("op", ["add", "sub", "mul"])
def test_interval_ops_are_optimal(prec, op):
    """Each endpoint equals RD / RU of the exact real result."""
    rng = np.random.default_rng(1234 + hash(op) % 100)
    dt = np.float64 if prec == "f64" else np.float32
    rd, ru = (rd64, ru64) if prec == "f64" else (rd32, ru32)
    a = _rand_intervals(rng, 400, dt)
    b = _rand_intervals(rng, 400, dt)
    # include sign classes explicitly: positive, negative, straddling, zero
    a[:50] = np.abs(a[:50]); a[50:100] = -np.abs(a[50:100])[:, ::-1]
    b[100:150] = 0
    r = oracle.interval_op(op, a, b, prec)
    for i in range(a.shape[0]):
        al, ah, bl, bh = map(F, (a[i, 0], a[i, 1], b[i, 0], b[i, 1]))
        if op == "add":
            lo, hi = al + bl, ah + bh
        elif op == "sub":
            lo, hi = al - bh, ah - bl
        else:
            ps = [al * bl, al * bh, ah * bl, ah * bh]
            lo, hi = min(ps), max(ps)
        assert r[i, 0] == rd(lo) and r[i, 1] == ru(hi), (op, i, a[i], b[i], r[i])


def test_interval_worked_examples():
    for ex in GOLD["interval_ops_f64"]:
        r = oracle.interval_op(ex["op"], np.array([ex["a"]]), np.array([ex["b"]]))
        assert list(r[0]) == ex["r"], ex


def test_cinterval_worked_examples():
    for ex in GOLD["cinterval_mul_f64"]:
        r = oracle.cinterval_op("mul", np.array([ex["a"]], float), np.array([ex["b"]], float))
        assert list(r[0]) == ex["r"], ex


def test_cmul_contains_sampled_products():
    """the rectangular product contains z*w for every z, w in the boxes."""
    rng = np.random.default_rng(7)
    m = 300
    z = np.concatenate([_rand_intervals(rng, m, np.float64), _rand_intervals(rng, m, np.float64)], 1)
    w = np.concatenate([_rand_intervals(rng, m, np.float64), _rand_intervals(rng, m, np.float64)], 1)
    r = oracle.cinterval_op("mul", z, w)
    for i in range(m):
        for _ in range(6):
            t = rng.uniform(0, 1, 4)
            zr = F(z[i, 0]) + (F(z[i, 1]) - F(z[i, 0])) * Fraction(float(t[0]))
            zi = F(z[i, 2]) + (F(z[i, 3]) - F(z[i, 2])) * Fraction(float(t[1]))
            wr = F(w[i, 0]) + (F(w[i, 1]) - F(w[i, 0])) * Fraction(float(t[2]))
            wi = F(w[i, 2]) + (F(w[i, 3]) - F(w[i, 2])) * Fraction(float(t[3]))
            pr, pi = zr * wr - zi * wi, zr * wi + zi * wr
            assert F(r[i, 0]) <= pr <= F(r[i, 1])
            assert F(r[i, 2]) <= pi <= F(r[i, 3])
    # and it is the exact textbook enclosure (rounded outward once per op)
    for i in range(20):
        zr = (F(z[i, 0]), F(z[i, 1])); zi = (F(z[i, 2]), F(z[i, 3]))
        wr = (F(w[i, 0]), F(w[i, 1])); wi = (F(w[i, 2]), F(w[i, 3]))

        def imul(x, y):
            ps = [x[0] * y[0], x[0] * y[1], x[1] * y[0], x[1] * y[1]]
            return (F(rd64(min(ps))), F(ru64(max(ps))))
        a1, a2 = imul(zr, wr), imul(zi, wi)
        b1, b2 = imul(zr, wi), imul(zi, wr)
        assert r[i, 0] == rd64(a1[0] - a2[1]) and r[i, 1] == ru64(a1[1] - a2[0])
        assert r[i, 2] == rd64(b1[0] + b2[0]) and r[i, 3] == ru64(b1[1] + b2[1])


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_certify_worked_examples(prec):
    for ex in GOLD["certify"]:
        c, f = oracle.certify(np.array(ex["iv"], float), prec)
        assert bool(f[0]) == ex["unique"], ex
        if ex["unique"]:
            assert c[0] == ex["value"]


def test_certify_nan_never_certifies():
    c, f = oracle.certify(np.array([np.nan, 3.0, 0.0, 0.0]))
    assert not f[0]
