"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star):
  * every certified GPU product is bit-exact against long multiplication
     / Python int, and its snapped coefficients equal the exact
    coefficient sums -- containment, since the snapped integer lies in
    the interval by construction;
  * the GPU flag is 1 wherever the oracle certifies with margin (oracle max
    radius < 0.25, i.e. width < 0.5; R11);
  * dumped GPU intervals contain the exact coefficients, imag parts contain 0;
  * max GPU radius <= 2 x the oracle's, per pair (R12);
  * runs are bitwise deterministic.
Inputs come from paper_1006_0405_b200.inputs only.
"""
import numpy as np
import pytest

import oracle
from paper_1006_0405_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_1006_0405_b200 as ivm
    return ivm.Context(0)


def to_int(d):
    return int.from_bytes(bytes(np.asarray(d, np.uint8)), "little")


def gpu_run(ctx, a, b, prec="f64", dump=None):
    import torch
    import paper_1006_0405_b200 as ivm
    ta = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    tb = torch.from_numpy(np.ascontiguousarray(b)).cuda()
    r = ctx.multiply_diag(ta, tb, prec=ivm.F64 if prec == "f64" else ivm.F32, dump_pairs=dump)
    torch.cuda.synchronize()
    out = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in r.items()}
    out["cert"] = out["cert"].astype(bool)
    return out


def real_interval_kernel(m, prec):
    """The odd-frequency (R13) kernels compute real coefficient intervals:
    binary64 m >= 64 (v6, v3, v4, v5), binary32 m >= 1024 (v3, v4, v5)."""
    return m >= 1024 or (prec == "f64" and m >= 64)


def check_pairs(ctx, a, b, prec="f64", dump_n=4, oracle_sample=None, expect_all_cert=True):
    B, n = a.shape
    dump = list(range(min(dump_n, B)))
    g = gpu_run(ctx, a, b, prec, dump=dump)
    exact = oracle.coefficients(a, b)
    want = oracle.long_multiply(a, b)
    # (1) certified products bit-exact, coefficients exact; uncertified zero
    for p in range(B):
        if g["cert"][p]:
            assert np.array_equal(g["prod"][p], want[p]), p
            assert np.array_equal(g["coeffs"][p], exact[p]), p
            assert g["first_bad"][p] == -1
        else:
            assert not g["prod"][p].any()
            assert 0 <= g["first_bad"][p] < 2 * n - 1
    # (2) containment of the dumped intervals
    m = g["m"]
    for j, p in enumerate(dump):
        iv = g["intervals"][j]
        c = exact[p].astype(np.float64)
        assert np.all(iv[:2 * n - 1, 0] <= c) and np.all(c <= iv[:2 * n - 1, 1]), p
        if real_interval_kernel(m, prec):  # imag not computed (R13): NaN
            assert np.isnan(iv[:, 2:]).all(), p
        else:
            assert np.all(iv[:, 2] <= 0) and np.all(0 <= iv[:, 3]), p
        assert np.all(iv[2 * n - 1:, 0] <= 0) and np.all(0 <= iv[2 * n - 1:, 1]), p
        assert iv.shape == (m, 4)
    # (3) oracle flag agreement with margin, radius within 2x
    sample = np.arange(B) if oracle_sample is None else np.asarray(oracle_sample)
    r = oracle.ivmul(a[sample], b[sample], prec=prec)
    for i, p in enumerate(sample):
        if r["cert"][i] and r["max_radius"][i] < 0.25:
            assert g["cert"][p], (p, r["max_radius"][i], g["max_radius"][p])
        if r["cert"][i]:
            assert g["max_radius"][p] <= 2.0 * r["max_radius"][i] + 1e-300, (
                p, g["max_radius"][p], r["max_radius"][i])
    if expect_all_cert:
        assert g["cert"].all()
    return g, r


SIZES = [2, 3, 4, 5, 8, 9, 16, 17, 31, 33, 64, 100, 128, 255, 256, 257, 500, 513, 1000, 1024,
         1025, 2000, 2048, 2049, 3000, 4095, 4096]


@pytest.mark.parametrize("n", SIZES)
def test_f64_sizes_mixed_kinds(ctx, n):
    """Every FFT length 4..8192, ragged n, all digit kinds."""
    kinds = np.array([0, 1, 2, 3, 0, 1, 2, 0])
    a, b = inputs.pair_digits(0x5EED + n, np.arange(8), n, kinds)
    check_pairs(ctx, a, b)


def test_n1_brute_force(ctx):
    """n = 1: all 65,536 single-digit pairs (m = 1)."""
    g = np.arange(256, dtype=np.uint8)
    a = np.repeat(g, 256)[:, None]
    b = np.tile(g, 256)[:, None]
    r = gpu_run(ctx, a, b)
    assert r["cert"].all()
    got = r["prod"][:, 0].astype(np.int64) + 256 * r["prod"][:, 1].astype(np.int64)
    assert np.array_equal(got, a[:, 0].astype(np.int64) * b[:, 0])


def test_two_digit_grid_brute_force(ctx):
    vals = [0, 1, 2, 127, 128, 254, 255]
    pairs = [(a0, a1, b0, b1) for a0 in vals for a1 in vals for b0 in vals for b1 in vals]
    a = np.array([[p[0], p[1]] for p in pairs], np.uint8)
    b = np.array([[p[2], p[3]] for p in pairs], np.uint8)
    check_pairs(ctx, a, b, dump_n=8)


@pytest.mark.parametrize("n", [1, 2, 7, 64, 1000, 4096])
def test_all255_closed_form(ctx, n):
    a = np.full((2, n), 255, np.uint8)
    r = gpu_run(ctx, a, a)
    want = [1] + [0] * (n - 1) + [254] + [255] * (n - 1)
    assert r["cert"].all()
    assert r["prod"][0].tolist() == want and r["prod"][1].tolist() == want


def test_unit_vectors_and_zero(ctx):
    n = 777
    x, _ = inputs.pair_digits(3, np.arange(1), n, "uniform")
    a = np.zeros((5, n), np.uint8)
    for j, k in enumerate([0, 1, 400, n - 1]):
        a[j, k] = 1
    b = np.repeat(x, 5, axis=0)
    r = gpu_run(ctx, a, b)
    assert r["cert"].all()
    for j, k in enumerate([0, 1, 400, n - 1]):
        want = np.zeros(2 * n, np.uint8); want[k:k + n] = x[0]
        assert np.array_equal(r["prod"][j], want)
    assert not r["prod"][4].any()


def test_config_C1(ctx):
    a, b, _ = inputs.config_inputs("C1")
    g, r = check_pairs(ctx, a, b, dump_n=1)
    assert to_int(g["prod"][0]) == to_int(a[0]) * to_int(b[0])


def test_config_C2_full(ctx):
    """All 4,096 pairs bit-exact; oracle flags / radii on a seeded sample."""
    a, b, _ = inputs.config_inputs("C2")
    sample = np.random.default_rng(2).choice(a.shape[0], 48, replace=False)
    g, r = check_pairs(ctx, a, b, dump_n=6, oracle_sample=sample)


def test_config_C4_fp32_sweep(ctx):
    """fp32 precision sweep: certified => exact; flags where the oracle has margin."""
    report = {}
    for n in inputs.CONFIGS["C4"][0] + [8, 12, 16, 20, 24]:
        a, b, kinds = inputs.config_inputs("C4", n=n)
        sample = np.concatenate([np.arange(0, 512, 16), [512, 1023]])
        g, r = check_pairs(ctx, a, b, prec="f32", dump_n=4, oracle_sample=sample,
                           expect_all_cert=False)
        report[n] = (g["cert"][:512].mean(), bool(g["cert"][512]), r["cert"][:32].mean())
    print("C4 certified fraction (gpu uniform, gpu all255, oracle uniform sample):", report)


def test_deterministic(ctx):
    a, b = inputs.pair_digits(11, np.arange(64), 3000, "uniform")
    g1 = gpu_run(ctx, a, b, dump=[0, 5])
    g2 = gpu_run(ctx, a, b, dump=[0, 5])
    for k in ("prod", "cert", "max_radius", "first_bad", "coeffs", "intervals"):
        assert np.array_equal(g1[k], g2[k], equal_nan=(k == "intervals")), k


def test_host_entry_point_matches_device(ctx):
    import torch
    a, b = inputs.pair_digits(12, np.arange(32), 1500, "uniform")
    pa = torch.from_numpy(a).pin_memory()
    pb = torch.from_numpy(b).pin_memory()
    out, cert = ctx.multiply_host(pa, pb)
    assert cert.numpy().all()
    assert np.array_equal(out.numpy(), oracle.long_multiply(a, b))


@pytest.mark.parametrize("n,batch", [(200, 1000), (2048, 700), (1000, 2 * 148 + 3)])
def test_host_entry_point_chunked_pipeline(ctx, n, batch):
    """Batches of >= 2 waves go through the chunked copy/compute pipeline: the
    result must equal the device-pointer path pair by pair, with the unequal
    last chunk included; a sample of pairs is checked against the oracle."""
    import torch
    K = inputs.KINDS
    kinds = np.array([K["uniform"], K["all255"], K["sparse"]])[np.arange(batch) % 3]
    a, b = inputs.pair_digits(13, np.arange(batch), n, kinds)
    pa = torch.from_numpy(a).pin_memory()
    pb = torch.from_numpy(b).pin_memory()
    out, cert = ctx.multiply_host(pa, pb)
    dout, dcert = ctx.multiply(pa.cuda(), pb.cuda())
    assert np.array_equal(out.numpy(), dout.cpu().numpy())
    assert np.array_equal(cert.numpy(), dcert.cpu().numpy())
    assert cert.numpy().all()
    idx = np.array([0, batch // 2, batch - 1])
    assert np.array_equal(out.numpy()[idx], oracle.long_multiply(a[idx], b[idx]))


@pytest.mark.parametrize("n", [513, 1000, 1500, 2048, 3000, 4096])
def test_f32_cta_sizes_never_wrong(ctx, n):
    """fp32 through the one-CTA kernel (m = 2^10 .. 2^13): far past the fp32
    limit, so pairs are mostly uncertified -- but a certified product must be
    exact and an uncertified one all zeros, and the dumped intervals must still
    contain the exact coefficients."""
    a, b = inputs.pair_digits(0xF3 + n, np.arange(4), n, np.array([0, 1, 2, 3]))
    g = gpu_run(ctx, a, b, prec="f32", dump=[0, 1])
    want = oracle.long_multiply(a, b)
    exact = oracle.coefficients(a[:2], b[:2])
    for p in range(4):
        if g["cert"][p]:
            assert np.array_equal(g["prod"][p], want[p])
        else:
            assert not g["prod"][p].any()
    for j in range(2):
        iv = g["intervals"][j]
        c = exact[j].astype(np.float64)
        assert np.all(iv[:2 * n - 1, 0] <= c) and np.all(c <= iv[:2 * n - 1, 1])


def test_argument_errors(ctx):
    import torch
    import paper_1006_0405_b200 as ivm
    L = ivm.lib()
    t = torch.zeros(8, dtype=torch.uint8, device="cuda")
    p = t.data_ptr()
    assert L.ivm_multiply_batched(ctx._h, p, p, 0, 1, p, p, 0, None) == -1   # n = 0
    assert L.ivm_multiply_batched(ctx._h, p, p, 4, 0, p, p, 0, None) == -1   # batch = 0
    assert L.ivm_multiply_batched(ctx._h, None, p, 4, 1, p, p, 0, None) == -1
    assert L.ivm_multiply_batched(ctx._h, p, p, 4, 1, p, p, 5, None) == -1   # precision
    big = ivm.max_digits(ivm.F64) + 1
    assert L.ivm_multiply_batched(ctx._h, p, p, big, 1, p, p, 0, None) == -4


@pytest.mark.parametrize("n", [1024, 4096, 16384])
def test_misaligned_operands_and_products(ctx, n):
    """Operand / product pointers at odd byte offsets: the digit staging (TMA,
    16-B aligned rows only) and the 4-byte digit stores take their fallbacks;
    results identical to the aligned call."""
    import torch
    B = 6
    a, b = inputs.pair_digits(0x0DD + n, np.arange(B), n, np.array([0, 1, 2, 3, 0, 1]))
    ta = torch.zeros(B * n + 3, dtype=torch.uint8, device="cuda")
    tb = torch.zeros(B * n + 5, dtype=torch.uint8, device="cuda")
    ta[3:] = torch.from_numpy(a.reshape(-1)).cuda()
    tb[5:] = torch.from_numpy(b.reshape(-1)).cuda()
    va, vb = ta[3:].view(B, n), tb[5:].view(B, n)
    po = torch.zeros(B * 2 * n + 7, dtype=torch.uint8, device="cuda")
    pc = torch.zeros(B + 1, dtype=torch.uint8, device="cuda")
    out, cert = ctx.multiply(va, vb, out=po[7:].view(B, 2 * n), cert=pc[1:])
    torch.cuda.synchronize()
    assert cert.cpu().numpy().all()
    big = lambda d: int.from_bytes(bytes(d), "little")
    o = out.cpu().numpy()
    for p in range(B):
        assert big(o[p]) == big(a[p]) * big(b[p]), p


@pytest.mark.parametrize("n", [4096, 16384])
def test_two_streams_one_context(ctx, n):
    """Calls on one context from two streams (include/ivm.h "streams"): the
    context's scratch is shared, so the second call must wait for the first;
    both batches must come back exact."""
    import torch
    B = 300
    a1, b1 = inputs.pair_digits(0xA1 + n, np.arange(B), n, "uniform")
    a2, b2 = inputs.pair_digits(0xA2 + n, np.arange(B), n, "uniform")
    t = [torch.from_numpy(x).cuda() for x in (a1, b1, a2, b2)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    outs = []
    for rep in range(3):
        p1, c1 = ctx.multiply(t[0], t[1], stream=s1)
        p2, c2 = ctx.multiply(t[2], t[3], stream=s2)
        outs.append((p1, c1, p2, c2))
    torch.cuda.synchronize()
    w1 = oracle.long_multiply(a1[:16], b1[:16])
    w2 = oracle.long_multiply(a2[:16], b2[:16])
    r1 = oracle.residue_check(a1, b1, outs[0][0].cpu().numpy())
    r2 = oracle.residue_check(a2, b2, outs[0][2].cpu().numpy())
    assert r1.all() and r2.all()
    for p1, c1, p2, c2 in outs:
        assert c1.cpu().numpy().all() and c2.cpu().numpy().all()
        assert np.array_equal(p1.cpu().numpy()[:16], w1) and np.array_equal(p2.cpu().numpy()[:16], w2)
        assert torch.equal(p1, outs[0][0]) and torch.equal(p2, outs[0][2])
