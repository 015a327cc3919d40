"""GPU exact long multiplication and the precision escalation
fp32 -> fp64 -> long multiplication, through the C ABI.

Bars: every product bit-exact against the oracle's long multiplication (or
Python's int product at large n); the method recorded per pair is the first
tier that certifies, so it must agree with the fp32 / fp64 flags of the plain
certified calls on the same inputs.
"""
import numpy as np
import pytest

import oracle
from paper_1006_0405_b200 import inputs

pytestmark = pytest.mark.gpu

K = inputs.KINDS


@pytest.fixture(scope="module")
def ctx():
    import paper_1006_0405_b200 as ivm
    return ivm.Context(0)


def to_int(d):
    return int.from_bytes(bytes(np.asarray(d, np.uint8)), "little")


def kinds_mix(B):
    return np.array([K["uniform"], K["all255"], K["sparse"], K["msd"]])[np.arange(B) % 4]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 31, 64, 255, 256, 257, 1000, 4095, 4097, 8200])
def test_long_multiply_bit_exact(ctx, n):
    import torch
    B = 6
    a, b = inputs.pair_digits(0x10A6 + n, np.arange(B), n, kinds_mix(B))
    out = ctx.long_multiply(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.long_multiply(a, b))


def test_long_multiply_large_and_closed_form(ctx):
    """75,000 digits (the paper's limit) and 150,000 (past fp64's limit):
    Python int products; all-255 by the closed form (256^n - 1)^2."""
    import torch
    for n in (75000, 150000):
        a, b = inputs.pair_digits(0x10A7 + n, np.arange(2), n, np.array([K["uniform"], K["all255"]]))
        out = ctx.long_multiply(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
        assert to_int(out[0]) == to_int(a[0]) * to_int(b[0])
        assert to_int(out[1]) == (256 ** n - 1) ** 2


def test_long_multiply_many_pairs_chunked(ctx):
    """Enough pairs that the int64 sums are processed in several chunks."""
    import torch
    n, B = 20000, 900  # 900 x 39,999 x 8 B > 256 MiB
    a, b = inputs.pair_digits(0x10A8, np.arange(B), n, kinds_mix(B))
    out = ctx.long_multiply(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    for p in (0, 1, 2, 3, 447, 448, 449, B - 1):
        assert to_int(out[p]) == to_int(a[p]) * to_int(b[p]), p


@pytest.mark.parametrize("n", [8, 20, 32, 33, 120, 1000])
def test_multiply_exact_escalation(ctx, n):
    """Always exact; method = first tier that certifies: fp32 (n <= 32) then fp64
    then long multiplication; consistent with the plain certified calls."""
    import torch
    import paper_1006_0405_b200 as ivm
    B = 64
    a, b = inputs.pair_digits(0xE5C + n, np.arange(B), n, kinds_mix(B))
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    out, method = ctx.multiply_exact(ta, tb)
    torch.cuda.synchronize()
    out, method = out.cpu().numpy(), method.cpu().numpy()
    assert np.array_equal(out, oracle.long_multiply(a, b))
    _, c64 = ctx.multiply(ta, tb, prec=ivm.F64)
    c64 = c64.cpu().numpy().astype(bool)
    if n <= 32:
        _, c32 = ctx.multiply(ta, tb, prec=ivm.F32)
        c32 = c32.cpu().numpy().astype(bool)
        want = np.where(c32, 1, np.where(c64, 2, 3))
    else:
        want = np.where(c64, 2, 3)
    assert np.array_equal(method, want)
    print("n", n, "methods", np.bincount(method, minlength=4)[1:])


@pytest.mark.parametrize("n", [8, 16, 17, 100, 600])
def test_multiply_exact_fastest_policy(ctx, n):
    """policy 1: long multiplication below m = 64, fp64 first above; exact."""
    import torch
    import paper_1006_0405_b200 as ivm
    B = 40
    a, b = inputs.pair_digits(0xE5E + n, np.arange(B), n, kinds_mix(B))
    out, method = ctx.multiply_exact(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), policy=1)
    assert np.array_equal(out.cpu().numpy(), oracle.long_multiply(a, b))
    want = 3 if ivm.fft_length(n) < 64 else 2
    assert (method.cpu().numpy() == want).all()


def test_multiply_exact_rejects_bad_policy(ctx):
    import torch
    import paper_1006_0405_b200 as ivm
    t = torch.zeros((1, 4), dtype=torch.uint8, device="cuda")
    L = ivm.lib()
    assert L.ivm_multiply_exact(ctx._h, t.data_ptr(), t.data_ptr(), 4, 1, t.data_ptr(), None, 7, None) == -1


def test_multiply_exact_past_fp64_limit(ctx):
    """n > max_digits(F64): long multiplication for every pair."""
    import torch
    import paper_1006_0405_b200 as ivm
    n = ivm.max_digits(ivm.F64) + 5
    a, b = inputs.pair_digits(0xE5D, np.arange(2), n, np.array([K["uniform"], K["sparse"]]))
    out, method = ctx.multiply_exact(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    out, method = out.cpu().numpy(), method.cpu().numpy()
    assert (method == 3).all()
    for p in range(2):
        assert to_int(out[p]) == to_int(a[p]) * to_int(b[p])
