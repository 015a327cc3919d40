"""GPU parity for the multi-CTA path (m = 2^14 .. 2^18), incl. configs C3 and C5.

Same bars as test_gpu_parity.py.  Full-size configs: every product of C3 is
checked bit-exact against Python's int multiplication; C5 (65,536 pairs) is
checked bit-exact on a seeded sample plus the closed form on every all-255
pair; oracle flags / radii on small samples (the oracle needs seconds per
pair at these sizes).
"""
import numpy as np
import pytest

import oracle
from paper_1006_0405_b200 import inputs
from tests.test_gpu_parity import check_pairs, gpu_run, to_int

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_1006_0405_b200 as ivm
    return ivm.Context(0)


@pytest.mark.parametrize("n", [4097, 8192, 8193, 12000, 16384, 30000, 40000])
def test_f64_large_sizes(ctx, n):
    kinds = np.array([0, 1, 2, 3])
    a, b = inputs.pair_digits(0xB16 + n, np.arange(4), n, kinds)
    check_pairs(ctx, a, b, dump_n=2, oracle_sample=[0, 1])


def test_f32_large_size_never_wrong(ctx):
    n = 9000
    a, b = inputs.pair_digits(0xF32, np.arange(3), n, np.array([0, 1, 2]))
    g = gpu_run(ctx, a, b, prec="f32")
    want = oracle.long_multiply(a, b)
    for p in range(3):
        if g["cert"][p]:
            assert np.array_equal(g["prod"][p], want[p])
        else:
            assert not g["prod"][p].any()


def test_config_C3_full(ctx):
    """Paper's limit (P:5): 64 pairs of 75,000 digits, half all-255; all
    certified and bit-exact; oracle radius bound on one uniform + one all-255."""
    a, b, kinds = inputs.config_inputs("C3")
    g = gpu_run(ctx, a, b, dump=[0, 32])
    assert g["cert"].all()
    for p in range(a.shape[0]):
        assert to_int(g["prod"][p]) == to_int(a[p]) * to_int(b[p]), p
    n = a.shape[1]
    exact = oracle.coefficients(a[[0, 32]], b[[0, 32]])
    for j, p in enumerate([0, 32]):
        iv = g["intervals"][j]
        c = exact[j].astype(np.float64)
        assert np.all(iv[:2 * n - 1, 0] <= c) and np.all(c <= iv[:2 * n - 1, 1])
    r = oracle.ivmul(a[[0, 32]], b[[0, 32]])
    assert r["cert"].all()
    assert np.all(g["max_radius"][[0, 32]] <= 2 * r["max_radius"])
    print("C3 max radius gpu", g["max_radius"][[0, 32]], "oracle", r["max_radius"])


def test_config_C5_sampled(ctx):
    """C5 shape (16,384 digits, 1/3 uniform, 1/3 all-255, 1/3 sparse) on a
    4,096-pair slice: all certified; all-255 pairs by closed form; a seeded
    sample of 48 pairs bit-exact; oracle radius on 3 pairs."""
    import torch
    pairs = np.arange(4096)
    a, b, kinds = inputs.config_inputs("C5", pairs=pairs)
    g = gpu_run(ctx, a, b)
    assert g["cert"].all()
    n = a.shape[1]
    want255 = np.array([1] + [0] * (n - 1) + [254] + [255] * (n - 1), np.uint8)
    for p in np.nonzero(kinds == 1)[0]:
        assert np.array_equal(g["prod"][p], want255)
    rng = np.random.default_rng(5)
    for p in rng.choice(4096, 48, replace=False):
        assert to_int(g["prod"][p]) == to_int(a[p]) * to_int(b[p]), p
    r = oracle.ivmul(a[:3], b[:3])
    assert np.all(g["max_radius"][:3] <= 2 * r["max_radius"]), (g["max_radius"][:3], r["max_radius"])
