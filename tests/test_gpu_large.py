"""GPU parity for the multi-CTA path (m = 2^14 .. 2^18), incl. configs C3 and C5.

Same bars as test_gpu_parity.py.  Full-size configs: every product of C3 is
checked bit-exact against Python's int multiplication; every one of C5's 65,536
products against the exact product modulo two random 61-bit primes,
the all-255 ones by closed form, a sample by Python ints; oracle flags / radii
on small samples here (tools/radius_ratios.py records the full distributions).
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


def c5_chunks(ctx, chunk=8192):
    """All 65,536 C5 pairs in chunks, digits generated on the device by the
    seeded generator (bit-equal to inputs.py, tests/test_inputs.py)."""
    import torch
    n, B = 16384, 65536
    kinds_all = inputs.class_of_pairs("C5", B).astype(np.uint8)
    seed = inputs.config_seed(5)
    for p0 in range(0, B, chunk):
        kt = torch.from_numpy(kinds_all[p0:p0 + chunk]).cuda()
        a = ctx.generate_digits(n, chunk, seed, 0, kind=kt, pair0=p0)
        b = ctx.generate_digits(n, chunk, seed, 1, kind=kt, pair0=p0)
        yield p0, a, b, kinds_all[p0:p0 + chunk]


def test_config_C5_full(ctx):
    """C5 (16,384 digits, 1/3 uniform, 1/3 all-255, 1/3 sparse): EVERY one of
    the 65,536 products is certified and checked -- against the exact product
    modulo two fresh random 61-bit primes (oracle.residue_check), the
    all-255 pairs also against the closed form (256^n - 1)^2 -- and 16 pairs per
    chunk bit-exact against Python ints; the inputs of the first chunk are
    checked against inputs.py."""
    import torch
    primes = oracle.random_primes(2)
    n = 16384
    want255 = np.array([1] + [0] * (n - 1) + [254] + [255] * (n - 1), np.uint8)
    rng = np.random.default_rng(55)
    checked = 0
    for p0, a, b, kinds in c5_chunks(ctx):
        prod, cert = ctx.multiply(a, b)
        torch.cuda.synchronize()
        prod, cert = prod.cpu().numpy(), cert.cpu().numpy().astype(bool)
        ah, bh = a.cpu().numpy(), b.cpu().numpy()
        if p0 == 0:
            ra, rb, _ = inputs.config_inputs("C5", pairs=np.arange(64))
            assert np.array_equal(ah[:64], ra) and np.array_equal(bh[:64], rb)
        assert cert.all(), np.nonzero(~cert)[0][:8] + p0
        ok = oracle.residue_check(ah, bh, prod, primes)
        assert ok.all(), np.nonzero(~ok)[0][:8] + p0
        assert (prod[kinds == 1] == want255).all()
        for q in rng.choice(len(ah), 16, replace=False):
            assert to_int(prod[q]) == to_int(ah[q]) * to_int(bh[q]), p0 + q
        checked += len(ah)
    assert checked == 65536


def test_config_C5_radius_vs_oracle(ctx):
    """C5 radius bound (R10) on 6 pairs, two of each kind."""
    pairs = np.array([0, 1, 2, 3, 4, 5])
    a, b, kinds = inputs.config_inputs("C5", pairs=pairs)
    g = gpu_run(ctx, a, b)
    assert g["cert"].all()
    r = oracle.ivmul(a, b)
    assert np.all(g["max_radius"] <= 2 * r["max_radius"]), (g["max_radius"], r["max_radius"])


@pytest.mark.parametrize("n", [5000, 12000, 30000])
def test_group_kernel_forced_at_cluster_sizes(n, monkeypatch):
    """IVM_KERNEL=v5: the group kernel at m = 2^14 .. 2^16 (normally the cluster
    kernel's sizes; the variant the host can pick to fill SMs clusters leave idle)."""
    import paper_1006_0405_b200 as ivm
    monkeypatch.setenv("IVM_KERNEL", "v5")
    c5 = ivm.Context(0)
    kinds = np.array([0, 1, 2, 3])
    a, b = inputs.pair_digits(0x55 + n, np.arange(4), n, kinds)
    check_pairs(c5, a, b, dump_n=2, oracle_sample=[0, 1])
    c5.close()


@pytest.mark.parametrize("n", [12000, 30000])
def test_cluster_and_group_corun(n, monkeypatch):
    """A batch large enough for the co-run (the group kernel on the SMs whole
    clusters leave free): the same products and flags as the
    cluster kernel alone (IVM_CORUN=0); certified products exact; diagnostics
    (radius, first-bad, dumps) land on the right pairs in both portions."""
    import torch
    import paper_1006_0405_b200 as ivm
    B = 400
    kinds = np.arange(B) % 3
    a, b = inputs.pair_digits(0xC0 + n, np.arange(B), n, kinds)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("IVM_CORUN", mode)
        cx = ivm.Context(0)
        r = cx.multiply_diag(ta, tb, dump_pairs=[0, B - 1], coeffs=False)
        torch.cuda.synchronize()
        res[mode] = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in r.items()}
        cx.close()
    for mode in ("0", "1"):
        g = res[mode]
        assert g["cert"].all()
        assert oracle.residue_check(a, b, g["prod"]).all()
        assert (g["first_bad"] == -1).all() and (g["max_radius"] > 0).all()
        exact = oracle.coefficients(a[[0, B - 1]], b[[0, B - 1]])
        for j in range(2):
            iv = g["intervals"][j]
            c = exact[j].astype(np.float64)
            assert np.all(iv[:2 * n - 1, 0] <= c) and np.all(c <= iv[:2 * n - 1, 1])
    assert np.array_equal(res["0"]["prod"], res["1"]["prod"])
    assert np.array_equal(res["0"]["cert"], res["1"]["cert"])
    o = oracle.ivmul(a[[B - 1]], b[[B - 1]])
    assert res["1"]["max_radius"][B - 1] <= 2 * o["max_radius"][0]


@pytest.mark.parametrize("n", [40001, 65537])
def test_group_kernel_odd_n_byte_loads(ctx, n):
    """n % 4 != 0 at m = 2^17 / 2^18: the tensor-core cross pass (DESIGN R16)
    assembles its digit words from byte loads instead of word loads; products,
    coefficients, containment, flags and radii against the oracle."""
    kinds = np.array([0, 1, 2])
    a, b = inputs.pair_digits(0x0DD1 + n, np.arange(3), n, kinds)
    check_pairs(ctx, a, b, dump_n=2, oracle_sample=[0, 1])


@pytest.mark.parametrize("n", [40000, 75000])
def test_group_kernel_misaligned_operands(ctx, n):
    """Operands at odd byte offsets at m = 2^17 / 2^18 (the cross pass's word
    loads need 4-byte aligned rows; it falls back to byte loads): identical,
    exact products."""
    import torch
    B = 3
    a, b = inputs.pair_digits(0x0DD2 + n, np.arange(B), n, np.array([0, 1, 3]))
    ta = torch.zeros(B * n + 1, dtype=torch.uint8, device="cuda")
    tb = torch.zeros(B * n + 2, dtype=torch.uint8, device="cuda")
    ta[1:] = torch.from_numpy(a.reshape(-1)).cuda()
    tb[2:] = torch.from_numpy(b.reshape(-1)).cuda()
    out, cert = ctx.multiply(ta[1:].view(B, n), tb[2:].view(B, n))
    torch.cuda.synchronize()
    assert cert.cpu().numpy().all()
    o = out.cpu().numpy()
    for p in range(B):
        assert to_int(o[p]) == to_int(a[p]) * to_int(b[p]), p


def test_config_C3_radius_tightness(ctx):
    """The exact tensor-core cross pass (DESIGN R16) keeps C3's enclosures well
    inside the north-star bar: GPU max radius <= 0.75 x the oracle's on a
    uniform and an all-255 pair (round 1, FP64 direct sums: up to 0.56)."""
    a, b, kinds = inputs.config_inputs("C3")
    sel = [0, 32]
    g = gpu_run(ctx, a[sel], b[sel])
    r = oracle.ivmul(a[sel], b[sel])
    assert g["cert"].all() and r["cert"].all()
    assert np.all(g["max_radius"] <= 0.75 * r["max_radius"]), (g["max_radius"], r["max_radius"])


@pytest.mark.parametrize("n,B", [(40000, 1), (40000, 70), (75000, 3), (75000, 64), (120000, 5)])
def test_pipelined_group_kernel_matches_lockstep(n, B, monkeypatch):
    """The pipelined group kernel (v7, fp64 m = 2^17 / 2^18: one CTA per SM
    dealing batch x C stage-split tasks, per-pair scratch in a ring) against the
    lockstep group kernel (IVM_V7=0): bit-identical products, flags, radii,
    first failing indices, snapped coefficients and interval dumps.  B = 70 and
    64 reuse ring slots (ring 48 and 25 pairs on 148 SMs); B = 1 runs C CTAs;
    n = 120,000 is beyond the paper's 75,000-digit limit."""
    import torch
    import paper_1006_0405_b200 as ivm
    kinds = np.arange(B) % 3
    kinds[-1] = 1
    a, b = inputs.pair_digits(0x7707 + n + B, np.arange(B), n, kinds)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("IVM_V7", mode)
        cx = ivm.Context(0)
        r = cx.multiply_diag(ta, tb, dump_pairs=sorted({0, B - 1}), coeffs=True)
        torch.cuda.synchronize()
        res[mode] = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in r.items()}
        cx.close()
    for k in res["0"]:
        assert np.array_equal(res["0"][k], res["1"][k], equal_nan=True), k
    g = res["1"]
    if n <= 75000:
        assert g["cert"].all()
    assert (g["first_bad"][~g["cert"].astype(bool)] >= 0).all()
    okp = g["cert"].astype(bool)
    assert not g["prod"][~okp].any()
    assert oracle.residue_check(a[okp], b[okp], g["prod"][okp]).all()


@pytest.mark.parametrize("n", [40000, 75000])
def test_large_m_carry_patterns(ctx, n):
    """Products whose digits run through long stretches of 0xFF and 0x00 across
    chunk boundaries (the chunk carry: generate / propagate / a carry arriving
    only through the value passed up from the chunk below): a = 256^n - 1 times
    b in {1, 256^j + 1, 256^j - 1 (j = n / 3), 2, 255, 256^(n-1) + 1,
    random digits in [0, 1]}, bit-exact against Python integers."""
    import torch
    B = 8
    a = np.full((B, n), 255, np.uint8)
    b = np.zeros((B, n), np.uint8)
    j = n // 3
    b[0, 0] = 1
    b[1, 0] = 1
    b[1, j] = 1
    b[2, :j] = 255
    b[3, 0] = 2
    b[4, 0] = 255
    b[5, 0] = 1
    b[5, n - 1] = 1
    rng = np.random.default_rng(n)
    b[6] = rng.integers(0, 2, n, dtype=np.uint8)
    a[7] = rng.integers(254, 256, n, dtype=np.uint8)
    b[7] = 255
    out, cert = ctx.multiply(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    torch.cuda.synchronize()
    cert, out = cert.cpu().numpy(), out.cpu().numpy()
    assert cert.all()
    for p in range(B):
        assert to_int(out[p]) == to_int(a[p]) * to_int(b[p]), p


@pytest.mark.parametrize("n", [40, 100, 256, 500, 1000, 1024, 2048, 4088, 4096, 8192, 16384, 32768, 65536, 75000, 131072])
def test_throughput_variants_match_diagnostic_kernels(ctx, n):
    """The one-CTA, cluster and pipelined group kernels each have a throughput
    variant compiled without the interval-dump / coefficient / unaligned-digit
    paths (picked when no diagnostics are asked for; the one-CTA kernel has one for
    16-byte aligned rows, with staged digits, and one for the rest: n = 500, 1000, 4088).
    Same arithmetic: products, flags, max radii and first failing indices must be
    bit-identical to the diagnostic build's, and every certified product exact
    (n = 131,072 is the largest size the library takes; its enclosures are tighter
    than the paper's, so even past P:5's 75,000 digits pairs may certify: whatever
    the flag, both builds must agree and an uncertified product must be zero)."""
    import torch
    kinds = np.array([0, 1, 2, 3])
    a, b = inputs.pair_digits(0xFA57 + n, np.arange(4), n, kinds)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    assert ta.data_ptr() % 16 == 0 and tb.data_ptr() % 16 == 0
    diag = ctx.multiply_diag(ta, tb, dump_pairs=[0])      # dump + coefficients: diagnostic kernel
    fast = ctx.multiply_diag(ta, tb, coeffs=False)        # no dump, no coefficients: throughput kernel
    p, c = ctx.multiply(ta, tb)
    torch.cuda.synchronize()
    for k in ("prod", "cert", "first_bad"):
        assert torch.equal(diag[k], fast[k]), k
    assert torch.equal(diag["max_radius"].view(torch.int64), fast["max_radius"].view(torch.int64))
    assert torch.equal(p, fast["prod"]) and torch.equal(c, fast["cert"])
    cert = c.cpu().numpy().astype(bool)
    prod = p.cpu().numpy()
    if n <= 75000:
        assert cert.all()
    for i in range(4):
        if cert[i]:
            assert to_int(prod[i]) == to_int(a[i]) * to_int(b[i]), i
        else:
            assert not prod[i].any()


@pytest.mark.parametrize("n,bound", [(1000, 1.55), (4096, 1.35), (16384, 1.25), (75000, 0.75)])
def test_radius_tightness_per_size(ctx, n, bound):
    """Tightness regression (SURVEY hard part 1): per pair, GPU max radius / oracle max
    radius stays at the measured level (profiles/r02/radius_ratios.json: C1 1.45, C2
    <= 1.27, C5 <= 1.14, C3 <= 0.56), well inside the north-star's 2x.  The excess over 1
    at small m is the output-side untwist of the half-spectrum transform (R13)."""
    B = 4 if n <= 16384 else 2
    kinds = np.array([0, 0, 3, 3])[:B]  # uniform digits (all-255 ratios are lower)
    a, b = inputs.pair_digits(0x71D + n, np.arange(B), n, kinds)
    g = gpu_run(ctx, a, b)
    r = oracle.ivmul(a, b)
    assert g["cert"].all() and r["cert"].all()
    ratio = g["max_radius"] / r["max_radius"]
    assert np.all(ratio <= bound), (n, ratio)
