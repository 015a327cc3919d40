"""The naive (punctual, round-to-nearest) SS comparator:
exact where fixed precision suffices, and demonstrably NOT guaranteed
where it does not -- the reason for the certified path."""
import numpy as np
import pytest

import oracle
from paper_1006_0405_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_1006_0405_b200 as ivm
    return ivm.Context(0)


def run(ctx, a, b, prec):
    import torch
    return ctx.multiply_naive(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), prec=prec).cpu().numpy()


@pytest.mark.parametrize("n", [1, 2, 7, 100, 1000, 4096])
def test_naive_fp64_correct_at_moderate_sizes(ctx, n):
    import paper_1006_0405_b200 as ivm
    K = inputs.KINDS
    kinds = np.array([K["uniform"], K["all255"], K["sparse"], K["msd"]])[np.arange(8) % 4]
    a, b = inputs.pair_digits(0x0A1 + n, np.arange(8), n, kinds)
    assert np.array_equal(run(ctx, a, b, ivm.F64), oracle.long_multiply(a, b))


def test_naive_fp32_small_correct_large_wrong(ctx):
    """fp32 naive SS: correct for tiny operands, wrong for most 1,000-digit
    products (coefficients ~ 2^26 exceed the 24-bit significand), i.e. it has
    no guarantee -- while the certified path flags them (tested elsewhere)."""
    import paper_1006_0405_b200 as ivm
    a, b = inputs.pair_digits(0x0A2, np.arange(64), 8, "uniform")
    assert np.array_equal(run(ctx, a, b, ivm.F32), oracle.long_multiply(a, b))
    a, b = inputs.pair_digits(0x0A3, np.arange(64), 1000, "uniform")
    wrong = np.any(run(ctx, a, b, ivm.F32) != oracle.long_multiply(a, b), axis=1)
    assert wrong.mean() > 0.5


def test_naive_rejects_too_large(ctx):
    import torch
    import paper_1006_0405_b200 as ivm
    t = torch.zeros((1, 5000), dtype=torch.uint8, device="cuda")
    with pytest.raises(ivm.IvmError):
        ctx.multiply_naive(t, t)
