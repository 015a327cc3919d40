"""The C-ABI library loads, exports every symbol include/ivm.h declares, and
its host-side pieces (twiddle planner, argument checks) behave; no GPU needed.

The twiddle cross-check compares the library's __float128 planner with the
oracle's independent mpmath tables bit for bit (reading R2).
"""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_1006_0405_b200 as ivm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "ivm.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ivm_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = ivm.lib()
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(ivm.EXPORTS) == syms


def test_version_and_strerror():
    L = ivm.lib()
    assert b"sm_100a" in L.ivm_version()
    assert L.ivm_strerror(0) == b"ok"
    assert L.ivm_strerror(-1) == b"invalid argument"


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 1000, 4096, 4097, 75000])
def test_fft_length_matches_paper_rule(n):
    """m = 2^ceil(log2(2n-1)); same rule as the oracle's."""
    assert ivm.fft_length(n) == oracle.fft_length(n)


@pytest.mark.parametrize("prec", [ivm.F64, ivm.F32])
@pytest.mark.parametrize("log2m", [0, 1, 2, 3, 5, 8, 11, 13, 15])
def test_planner_twiddles_bit_equal_to_oracle(log2m, prec):
    lib_tw = ivm.twiddle_table(log2m, prec)
    ora_tw = oracle.twiddle_table(1 << log2m, "f64" if prec == ivm.F64 else "f32")
    assert lib_tw.dtype == ora_tw.dtype
    assert np.array_equal(lib_tw.view(np.uint8), ora_tw.view(np.uint8)) or np.array_equal(lib_tw, ora_tw)
    # same values (+0 vs -0 aside, the planner canonicalises zeros to +0)
    assert np.array_equal(lib_tw, ora_tw)


def test_create_without_device_reports_enodev_or_ok():
    h = ctypes.c_void_p()
    st = ivm.lib().ivm_create(ctypes.byref(h), 0)
    try:
        import torch
        if torch.cuda.is_available():
            assert st == 0
        else:
            assert st in (-6, -3)
    finally:
        if st == 0:
            ivm.lib().ivm_destroy(h)


def test_argument_errors_before_launch():
    L = ivm.lib()
    # NULL context
    assert L.ivm_multiply_batched(None, None, None, 4, 1, None, None, 0, None) == -1
    assert L.ivm_reserve(None, 1, 1, 0) == -1
    assert L.ivm_twiddle_table(3, 7, None) == -1


def test_max_digits():
    assert ivm.max_digits(ivm.F64) >= 4096
    assert ivm.max_digits(ivm.F32) >= 256
    assert ivm.lib().ivm_max_digits(9) == 0


def test_binding_operand_checks():
    """Every wrapper validates operands before the C call: a
    shorter b, a strided view or a CUDA tensor on the host path would make the
    library multiply (and certify) the wrong digits."""
    import torch
    from paper_1006_0405_b200 import _check_operands, _check_out
    a = torch.zeros((4, 8), dtype=torch.uint8)
    _check_operands(a, a.clone(), False)
    with pytest.raises(ValueError):
        _check_operands(a, torch.zeros((4, 7), dtype=torch.uint8), False)
    with pytest.raises(ValueError):
        _check_operands(torch.zeros((4, 16), dtype=torch.uint8)[:, :8], a, False)
    with pytest.raises(TypeError):
        _check_operands(a.to(torch.int16), a, False)
    with pytest.raises(ValueError):
        _check_operands(a, a, True, 0)  # host tensors on a device entry point
    with pytest.raises(ValueError):
        _check_operands(torch.zeros((0, 8), dtype=torch.uint8), torch.zeros((0, 8), dtype=torch.uint8), False)
    _check_out(torch.zeros((4, 16), dtype=torch.uint8), (4, 16), torch.uint8, False, "out")
    with pytest.raises(ValueError):
        _check_out(torch.zeros((4, 15), dtype=torch.uint8), (4, 16), torch.uint8, False, "out")


@pytest.mark.parametrize("prec", [ivm.F64, ivm.F32])
@pytest.mark.parametrize("log2m", [16, 17, 18, 19])
def test_planner_twiddles_large_m_sampled(log2m, prec):
    """The tables the large-m kernels plan (up to 2^(m+1) = 2^19 for C3):
    sampled entries, every octant and the quarter-turn points, equal to the
    oracle's direct mpmath enclosure of omega_N^j (no symmetry used)."""
    N = 1 << log2m
    lib_tw = ivm.twiddle_table(log2m, prec)
    p = "f64" if prec == ivm.F64 else "f32"
    rng = np.random.default_rng(log2m)
    js = set(rng.integers(0, N, 48).tolist()) | {0, 1, N // 8, N // 8 + 1, N // 4 - 1, N // 4, N // 2 + 3, N - 1}
    for j in sorted(js):
        want = np.array(oracle.direct_enclosure(N, j, p), dtype=lib_tw.dtype)
        assert np.array_equal(lib_tw[j], want), (N, j, lib_tw[j], want)
