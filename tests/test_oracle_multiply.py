"""Pins of the oracle's multiplication paths (§2.1, §2.3, §2.4).

Long multiplication, coefficient sums and carry
are pinned to worked examples and to Python's exact int multiplication.  The
interval Schoenhage-Strassen multiply is pinned to: the same Python ints
(whenever it certifies it must equal the exact product: soundness), the
closed form of (256^n - 1)^2, shifts by unit vectors, brute force over all
single-digit and a grid of two-digit pairs, containment of the exact
coefficients in every output interval, and the paper's 75,000-digit
statement (P:5) on a sample.
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_1006_0405_b200 import inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def to_int(d):
    return int.from_bytes(bytes(np.asarray(d, np.uint8)), "little")


def from_int(v, length):
    return np.frombuffer(v.to_bytes(length, "little"), np.uint8)


def test_long_multiply_worked_examples():
    for ex in GOLD["long_multiply"]:
        z = oracle.long_multiply(np.array([ex["x"]]), np.array([ex["y"]]))
        assert z[0].tolist() == ex["z"], ex


def test_coefficients_worked_examples():
    for ex in GOLD["coefficients"]:
        c = oracle.coefficients(np.array([ex["x"]]), np.array([ex["y"]]))
        assert c[0].tolist() == ex["c"], ex


def test_carry_worked_examples():
    for ex in GOLD["carry"]:
        v = ex["v"] if len(ex["v"]) % 2 == 1 else ex["v"] + [0]
        z = oracle.carry(np.array(v))
        assert z.tolist()[:len(ex["z"])] == ex["z"], ex


@pytest.mark.parametrize("n", [1, 2, 3, 17, 100, 1000])
def test_long_multiply_matches_python_int(n):
    a, b = inputs.pair_digits(99, np.arange(6), n, "uniform")
    z = oracle.long_multiply(a, b)
    c = oracle.coefficients(a, b)
    for p in range(a.shape[0]):
        want = to_int(a[p]) * to_int(b[p])
        assert to_int(z[p]) == want
        assert sum(int(v) << (8 * i) for i, v in enumerate(c[p])) == want
        assert np.array_equal(oracle.carry(c[p]), z[p])


def test_ivmul_single_digit_brute_force():
    """All 65,536 single-digit pairs (N = 1: the FFT is the identity)."""
    g = np.arange(256, dtype=np.uint8)
    a = np.repeat(g, 256)[:, None]
    b = np.tile(g, 256)[:, None]
    r = oracle.ivmul(a, b)
    assert r["cert"].all()
    want = (a[:, 0].astype(np.int64) * b[:, 0].astype(np.int64))
    got = r["prod"][:, 0].astype(np.int64) + 256 * r["prod"][:, 1].astype(np.int64)
    assert np.array_equal(got, want)


def test_ivmul_two_digit_grid_brute_force():
    vals = [0, 1, 2, 127, 128, 254, 255]
    pairs = [(a0, a1, b0, b1) for a0 in vals for a1 in vals for b0 in vals for b1 in vals]
    a = np.array([[p[0], p[1]] for p in pairs], np.uint8)
    b = np.array([[p[2], p[3]] for p in pairs], np.uint8)
    r = oracle.ivmul(a, b, want_coeffs=True)
    assert r["cert"].all()
    for p in range(len(pairs)):
        assert to_int(r["prod"][p]) == to_int(a[p]) * to_int(b[p])


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n", [3, 16, 33, 128, 1000])
def test_ivmul_sound_and_exact(n, prec):
    """Certified => equals Python's exact product; intervals contain c_i and 0."""
    if prec == "f64":
        kinds = np.array([0, 0, 1, 2, 3, 0, 1, 2])  # uniform / all255 / sparse / msd
        a, b = inputs.pair_digits(inputs.config_seed(2), np.arange(8), n, kinds)
    else:
        a, b, kinds = inputs.config_inputs("C4", n=n, pairs=np.array([0, 1, 2, 3, 600, 601]))
    r = oracle.ivmul(a, b, prec=prec, want_coeffs=True, want_intervals=True)
    exact = oracle.coefficients(a, b)
    for p in range(a.shape[0]):
        iv = r["intervals"][p].astype(np.float64)
        c = exact[p].astype(np.float64)
        assert np.all(iv[:2 * n - 1, 0] <= c) and np.all(c <= iv[:2 * n - 1, 1])
        assert np.all(iv[:, 2] <= 0) and np.all(0 <= iv[:, 3])
        # padding region (indices >= 2n-1) holds exact zeros of the convolution
        assert np.all(iv[2 * n - 1:, 0] <= 0) and np.all(0 <= iv[2 * n - 1:, 1])
        if r["cert"][p]:
            assert to_int(r["prod"][p]) == to_int(a[p]) * to_int(b[p])
            assert np.array_equal(r["coeffs"][p], exact[p])
        else:
            assert not r["prod"][p].any()
    if prec == "f64":
        assert r["cert"].all()


@pytest.mark.parametrize("n", [1, 2, 5, 64, 1000, 4096])
def test_all255_closed_form(n):
    """(256^n - 1)^2 = 256^{2n} - 2*256^n + 1 -> digits [1, 0*(n-1), 254, 255*(n-1)]."""
    a = np.full((1, n), 255, np.uint8)
    r = oracle.ivmul(a, a, want_coeffs=True)
    assert r["cert"][0]
    want = [1] + [0] * (n - 1) + [254] + [255] * (n - 1)
    assert r["prod"][0].tolist() == want
    i = np.arange(2 * n - 1)
    assert np.array_equal(r["coeffs"][0], 65025 * np.minimum(i + 1, 2 * n - 1 - i))


def test_unit_vector_shift_identity_and_commutativity():
    n = 300
    a, b = inputs.pair_digits(17, np.arange(3), n, "uniform")
    for k in (0, 1, 150, n - 1):
        e = np.zeros((1, n), np.uint8); e[0, k] = 1
        r = oracle.ivmul(e, a[:1])
        want = np.zeros(2 * n, np.uint8); want[k:k + n] = a[0]
        assert r["cert"][0] and np.array_equal(r["prod"][0], want)
    z = np.zeros((1, n), np.uint8)
    r0 = oracle.ivmul(z, a[:1])
    assert r0["cert"][0] and not r0["prod"].any()
    rab, rba = oracle.ivmul(a, b), oracle.ivmul(b, a)
    assert np.array_equal(rab["prod"], rba["prod"])


def test_fp32_anecdote_shape():
    """binary32 'usually' right near 120 digits for a naive multiply; with
    containment sets the flag is false there, never a wrong product."""
    a, b, kinds = inputs.config_inputs("C4", n=120, pairs=np.arange(0, 1024, 64))
    r = oracle.ivmul(a, b, prec="f32")
    exact = oracle.long_multiply(a, b)
    assert np.array_equal(r["prod"][r["cert"]], exact[r["cert"]])


@pytest.mark.slow
def test_paper_limit_75000_digits_certifies_sample():
    """P:5/P:271/P:282: 75,000-digit base-256 operands with double containment
    sets are 'usually' certified.  Checked on one uniform and one all-255 pair
    of config C3 (full config runs in the GPU parity tests)."""
    a, b, kinds = inputs.config_inputs("C3", pairs=np.array([0, 32]))
    r = oracle.ivmul(a, b, want_coeffs=False)
    assert r["cert"].all()
    assert r["max_radius"].max() < 0.25
    for p in range(2):
        assert to_int(r["prod"][p]) == to_int(a[p]) * to_int(b[p])


def test_residue_check_pins():
    """S:432 residue check: agrees with Python int arithmetic, accepts every
    true product and rejects products with one wrong digit."""
    primes = oracle.random_primes(2, seed=7)
    for p in primes:
        assert p.bit_length() == 61 and oracle._is_prime(p)
    assert oracle._is_prime(2 ** 61 - 1) and not oracle._is_prime((2 ** 61 - 1) * 3)
    for n in (1, 2, 7, 100, 1000):
        a, b = inputs.pair_digits(0x7E5 + n, np.arange(8), n, np.array([0, 1, 2, 3, 0, 1, 2, 3]))
        z = oracle.long_multiply(a, b)
        assert oracle.residue_check(a, b, z, primes).all()
        for q in range(8):
            want = to_int(a[q]) * to_int(b[q])
            for p in primes:  # the residues the C code compares, by Python ints
                assert (to_int(a[q]) % p) * (to_int(b[q]) % p) % p == want % p == to_int(z[q]) % p
        bad = z.copy()
        rng = np.random.default_rng(n)
        for q in range(8):
            i = rng.integers(0, 2 * n)
            bad[q, i] ^= 1 << int(rng.integers(0, 8))
        assert not oracle.residue_check(a, b, bad, primes).any()
    # the paper's limit: a 75,000-digit all-255 pair by its closed form
    n = 75000
    a = np.full((1, n), 255, np.uint8)
    z = np.array([[1] + [0] * (n - 1) + [254] + [255] * (n - 1)], np.uint8)
    assert oracle.residue_check(a, a, z, primes).all()
    z[0, n] = 253
    assert not oracle.residue_check(a, a, z, primes).any()
