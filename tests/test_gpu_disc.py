"""GPU circular-containment-set multiply (ivm_multiply_disc, DESIGN.md
R15) against the disc oracle (oracle/ivm_oracle_disc.c) on the same seeded
inputs: products bit-exact with the schoolbook oracle, the certified flag equal
wherever the oracle certifies with margin, the GPU disc radius within 2x of the
oracle's (both directions reported), uncertified products zero."""
import numpy as np
import pytest

import oracle
from paper_1006_0405_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_1006_0405_b200 as ivm
    return ivm.Context(0)


def run(ctx, a, b):
    import torch
    p, c, r = ctx.multiply_disc(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    return p.cpu().numpy(), c.cpu().numpy().astype(bool), r.cpu().numpy()


@pytest.mark.parametrize("n", [1, 2, 3, 31, 100, 257, 300, 512, 513, 1000, 2048, 2049, 3000, 4096])
def test_disc_parity_with_oracle(ctx, n):
    K = inputs.KINDS
    B = 12
    kinds = np.array([K["uniform"], K["all255"], K["sparse"], K["msd"]])[np.arange(B) % 4]
    a, b = inputs.pair_digits(0xD15C + n, np.arange(B), n, kinds)
    prod, cert, rad = run(ctx, a, b)
    ref = oracle.disc_mul(a, b)
    exact = oracle.long_multiply(a, b)
    margin = ref["max_radius"] < 0.25
    assert np.array_equal(cert[margin], ref["cert"][margin])
    assert np.array_equal(prod[cert], exact[cert])
    assert not prod[~cert].any()
    # R15: the GPU keeps radii as binary32 rounded up, so a radius that is only
    # the 2^-1000 subnormal guards (zero products) becomes the smallest binary32
    # subnormal; radii are compared above a 1e-30 floor (certification needs r < 0.5)
    floor = 1e-30
    ratio = np.maximum(rad, floor) / np.maximum(ref["max_radius"], floor)
    assert (ratio <= 2.0).all(), (n, ratio.max())
    assert (ratio >= 0.25).all(), (n, ratio.min())  # not suspiciously tight either


def test_disc_all_255_closed_form(ctx):
    n = 4096
    a = np.full((2, n), 255, np.uint8)
    prod, cert, _ = run(ctx, a, a)
    want = np.concatenate([[1], np.zeros(n - 1), [254], np.full(n - 1, 255)]).astype(np.uint8)
    assert cert.all() and (prod == want).all()


def test_disc_batch_ragged_and_deterministic(ctx):
    """A batch larger than the grid (several pairs per CTA), odd n; two runs
    bitwise identical (products, flags and radii)."""
    n = 777
    a, b = inputs.pair_digits(0xD15D, np.arange(600), n, "uniform")
    p1, c1, r1 = run(ctx, a, b)
    p2, c2, r2 = run(ctx, a, b)
    assert np.array_equal(p1, p2) and np.array_equal(c1, c2) and np.array_equal(r1, r2)
    assert c1.all()
    sel = np.arange(0, 600, 37)
    assert np.array_equal(p1[sel], oracle.long_multiply(a[sel], b[sel]))


def test_disc_rejects_too_large(ctx):
    import torch
    import paper_1006_0405_b200 as ivm
    t = torch.zeros((1, ivm.max_digits() + 1), dtype=torch.uint8, device="cuda")
    with pytest.raises(ivm.IvmError):
        ctx.multiply_disc(t, t)


@pytest.mark.parametrize("n", [4097, 4112, 5000, 6000, 8192, 8193, 8208, 12000, 16384, 20000, 40000])
def test_disc_group_parity_with_oracle(ctx, n):
    """m = 2^14 .. 2^17: the cluster kernel in disc arithmetic (m = 2^14 .. 2^16:
    ivm_d4.cuh) and the pipelined group kernel (m = 2^17: ivm_d7.cuh), aligned and
    unaligned digit rows (8192 x m/8192
    DIT factorization; the other sizes) against the disc oracle: products bit-exact, flags where the oracle
    certifies with margin, radius within 2x (and not below 1/4)."""
    K = inputs.KINDS
    kinds = np.array([K["uniform"], K["all255"], K["sparse"], K["msd"]])
    a, b = inputs.pair_digits(0xD15E + n, np.arange(4), n, kinds)
    prod, cert, rad = run(ctx, a, b)
    ref = oracle.disc_mul(a, b)
    assert ref["cert"].all() and cert.all()
    assert np.array_equal(prod, oracle.long_multiply(a, b))
    floor = 1e-30
    ratio = np.maximum(rad, floor) / np.maximum(ref["max_radius"], floor)
    assert (ratio <= 2.0).all() and (ratio >= 0.25).all(), (n, ratio)


def test_disc_group_C3_size(ctx):
    """The paper's limit (C3 shape, n = 75,000, m = 2^18, 32 CTAs per
    multiplication): a uniform and an all-255 pair certified and exact, the
    radius within 2x of the disc oracle's, and (P:290's question) far below the
    rectangular oracle's."""
    n = 75000
    a, b = inputs.pair_digits(inputs.config_seed(3), np.arange(2), n, np.array([0, 1]))
    a[1] = 255
    b[1] = 255
    prod, cert, rad = run(ctx, a, b)
    assert cert.all()
    to_int = lambda d: int.from_bytes(bytes(d), "little")
    for p in range(2):
        assert to_int(prod[p]) == to_int(a[p]) * to_int(b[p])
    ref = oracle.disc_mul(a, b)
    assert (rad <= 2 * ref["max_radius"]).all() and (rad >= 0.25 * ref["max_radius"]).all()
    rect = oracle.ivmul(a, b)
    assert (rad < rect["max_radius"]).all(), (rad, rect["max_radius"])


def test_disc_group_batch_deterministic(ctx):
    """More pairs than groups (persistent loop), two runs bitwise identical."""
    n = 9000
    B = 40
    a, b = inputs.pair_digits(0xD160, np.arange(B), n, np.arange(B) % 3)
    p1, c1, r1 = run(ctx, a, b)
    p2, c2, r2 = run(ctx, a, b)
    assert np.array_equal(p1, p2) and np.array_equal(c1, c2) and np.array_equal(r1, r2)
    assert c1.all() and oracle.residue_check(a, b, p1).all()


@pytest.mark.parametrize("n", [300, 512, 777, 1024, 1500, 2048, 2049, 4096])
def test_disc_radix8_kernel_against_radix2_kernel(n, monkeypatch):
    """m = 2^10 .. 2^13 run the one-CTA odd-frequency radix-8 schedule in disc
    arithmetic (csrc/ivm_d3.cuh); IVM_DISC3=0 keeps the paper's radix-2 DIT
    (csrc/ivm_disc.cu).  Different FFT schedules, same products and flags on
    certifiable inputs, radii within 2x of each other; a batch larger than the
    grid, all digit kinds."""
    import torch
    import paper_1006_0405_b200 as ivm
    B = 700
    kinds = np.arange(B) % 4
    a, b = inputs.pair_digits(0xD3 + n, np.arange(B), n, kinds)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    res = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("IVM_DISC3", flag)
        c = ivm.Context(0)
        p, ce, r = c.multiply_disc(ta, tb)
        torch.cuda.synchronize()
        res[flag] = (p.cpu().numpy(), ce.cpu().numpy().astype(bool), r.cpu().numpy())
        c.close()
    assert res["1"][1].all() and res["0"][1].all()
    assert np.array_equal(res["1"][0], res["0"][0])
    sel = np.arange(0, B, 53)
    assert np.array_equal(res["1"][0][sel], oracle.long_multiply(a[sel], b[sel]))
    ratio = np.maximum(res["1"][2], 1e-30) / np.maximum(res["0"][2], 1e-30)
    assert (ratio <= 2.0).all() and (ratio >= 0.25).all(), (ratio.min(), ratio.max())
    print("radix-8 / radix-2 disc radius", n, ratio.min(), ratio.max())


@pytest.mark.parametrize("n,B", [(8192, 230), (9001, 90), (16384, 120), (20000, 70), (32768, 50), (40000, 40), (50001, 30), (65536, 24), (75000, 20), (131072, 10)])
def test_disc_cluster_kernel_against_group_kernel(n, B, monkeypatch):
    """m = 2^14 .. 2^16 run the cluster schedule in disc arithmetic (csrc/ivm_d4.cuh;
    staged digits for 16-byte aligned rows, else through L2: n = 9,001), m = 2^17, 2^18
    the pipelined group schedule (csrc/ivm_d7.cuh; word or byte digit loads: n = 50,001);
    IVM_DISC3=0 keeps the radix-2 group kernel.  A
    batch of several pairs per cluster / several tasks per CTA, all digit kinds: same products and flags,
    radii within 2x of each other, a sample bit-exact against Python ints."""
    import torch
    import paper_1006_0405_b200 as ivm
    kinds = np.arange(B) % 4
    a, b = inputs.pair_digits(0xD4 + n, np.arange(B), n, kinds)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    res = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("IVM_DISC3", flag)
        c = ivm.Context(0)
        p, ce, r = c.multiply_disc(ta, tb)
        p2, ce2, r2 = c.multiply_disc(ta, tb)  # (a second call on the same context: deterministic)
        torch.cuda.synchronize()
        assert torch.equal(p, p2) and torch.equal(ce, ce2) and torch.equal(r, r2)
        res[flag] = (p.cpu().numpy(), ce.cpu().numpy().astype(bool), r.cpu().numpy())
        c.close()
    assert res["1"][1].all() and res["0"][1].all()
    assert np.array_equal(res["1"][0], res["0"][0])
    big = lambda d: int.from_bytes(bytes(d), "little")
    for i in range(0, B, 29):
        assert big(res["1"][0][i]) == big(a[i]) * big(b[i]), i
    ratio = np.maximum(res["1"][2], 1e-30) / np.maximum(res["0"][2], 1e-30)
    assert (ratio <= 2.0).all() and (ratio >= 0.25).all(), (ratio.min(), ratio.max())
    print("cluster / group disc radius", n, ratio.min(), ratio.max())
