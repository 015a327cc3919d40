"""CPU oracle for the certified interval-FFT multiplication (arxiv 1006.0405).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  It shares no
code with the CUDA path (paper_1006_0405_b200/); the product never imports it.

- ``ivm_oracle.c``  (built to ``liboracle.so``): long multiplication P:44-56,
  coefficient sums P:37, carry P:229-235, and the paper's interval
  Schoenhage-Strassen multiply (P:143-155 FFT, P:203-211 fast convolution,
  P:250-265 interval arithmetic) with fesetround directed rounding.
- ``ivm_oracle_disc.c`` (same library): the circular-containment-set variant the
  paper proposes as future work, disc arithmetic per DESIGN.md reading R15.
- ``twiddles.py``: optimal enclosures of omega_N^j from mpmath.

Parity status: every function here is pinned by ``tests/test_oracle_*.py``
against values that do not come from this package (paper values, exact
rationals, closed forms, Python int, brute force, mpmath DFTs).  The interval
radii, which the paper does not print, are pinned by an independent
exact-rational recomputation of whole small multiplications
(tests/test_oracle_exact_ss.py: every output interval and the max radius,
bit for bit).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .twiddles import twiddle_table, direct_enclosure  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "ivm_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "ivm_oracle_disc.c")]

CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-frounding-math", "-ffp-contract=off",
          "-fno-fast-math", "-std=c11", "-Wall", "-Wno-unknown-pragmas",
          "-Wno-unused-function"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc) if missing or stale."""
    if force or not os.path.exists(_SO) or any(os.path.getmtime(_SO) < os.path.getmtime(f) for f in _SRCS):
        subprocess.check_call(["gcc", *CFLAGS, *_SRCS, "-o", _SO, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        S = ctypes.c_size_t
        I = ctypes.c_int
        L.oracle_ivmul_batch.argtypes = [P, P, S, S, I, P, P, P, P, P, P, P, I]
        L.oracle_ivmul_batch.restype = I
        L.oracle_long_multiply_batch.argtypes = [P, P, S, S, P, I]
        L.oracle_coefficients_batch.argtypes = [P, P, S, S, P, I]
        L.oracle_carry.argtypes = [P, S, P]
        L.oracle_interval_op_f64.argtypes = [I, P, P, P, S]
        L.oracle_interval_op_f32.argtypes = [I, P, P, P, S]
        L.oracle_cinterval_op_f64.argtypes = [I, P, P, P, S]
        L.oracle_fft_f64.argtypes = [P, P, P, S, I]
        L.oracle_fft_f32.argtypes = [P, P, P, S, I]
        L.oracle_fft_length.argtypes = [S]
        L.oracle_fft_length.restype = S
        L.oracle_certify_f64.argtypes = [P, S, P, P]
        L.oracle_certify_f32.argtypes = [P, S, P, P]
        L.oracle_max_radius_f64.argtypes = [P, S]
        L.oracle_max_radius_f64.restype = ctypes.c_double
        L.oracle_max_radius_f32.argtypes = [P, S]
        L.oracle_max_radius_f32.restype = ctypes.c_double
        L.oracle_self_check.restype = I
        L.oracle_disc_batch.argtypes = [P, P, S, S, P, P, P, P, P, P, P, I]
        L.oracle_disc_batch.restype = I
        L.oracle_disc_op.argtypes = [I, P, P, P, S]
        L.oracle_disc_fft.argtypes = [P, P, P, S, I]
        L.oracle_max_threads.restype = I
        L.oracle_residue_check_batch.argtypes = [P, P, P, S, S, P, I, P, I]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def fft_length(n: int) -> int:
    """m = 2^k, k = ceil(log2(2n - 1))."""
    return int(lib().oracle_fft_length(n))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def ivmul(a: np.ndarray, b: np.ndarray, prec: str = "f64", want_coeffs: bool = False,
          want_intervals: bool = False, nthreads: int = 0) -> dict:
    """The paper's interval multiply on a batch [B][n] of digit pairs."""
    a = np.ascontiguousarray(a, dtype=np.uint8)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    if a.ndim == 1:
        a, b = a[None], b[None]
    B, n = a.shape
    N = fft_length(n)
    tw = np.ascontiguousarray(twiddle_table(N, prec))
    prod = np.zeros((B, 2 * n), np.uint8)
    cert = np.zeros(B, np.uint8)
    rad = np.zeros(B, np.float64)
    bad = np.zeros(B, np.int32)
    coeffs = np.zeros((B, 2 * n - 1), np.int64) if want_coeffs else None
    ivs = None
    if want_intervals:
        ivs = np.zeros((B, N, 4), np.float64 if prec == "f64" else np.float32)
    rc = lib().oracle_ivmul_batch(_p(a), _p(b), n, B, 0 if prec == "f64" else 1, _p(tw),
                                  _p(prod), _p(cert), _p(rad), _p(bad), _p(coeffs), _p(ivs),
                                  nthreads)
    assert rc == 0
    return {"prod": prod, "cert": cert.astype(bool), "max_radius": rad, "first_bad": bad,
            "coeffs": coeffs, "intervals": ivs, "N": N}


def disc_mul(a: np.ndarray, b: np.ndarray, want_coeffs: bool = False, want_discs: bool = False,
             nthreads: int = 0) -> dict:
    """The multiply with circular containment sets (R15), fp64,
    on a batch [B][n] of digit pairs.  max_radius = the largest disc radius over
    the used coefficients; discs [B][N][3] = (center re, center im, radius)."""
    a = np.ascontiguousarray(a, dtype=np.uint8)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    if a.ndim == 1:
        a, b = a[None], b[None]
    B, n = a.shape
    N = fft_length(n)
    tw = np.ascontiguousarray(twiddle_table(N, "f64"))
    prod = np.zeros((B, 2 * n), np.uint8)
    cert = np.zeros(B, np.uint8)
    rad = np.zeros(B, np.float64)
    bad = np.zeros(B, np.int32)
    coeffs = np.zeros((B, 2 * n - 1), np.int64) if want_coeffs else None
    discs = np.zeros((B, N, 3), np.float64) if want_discs else None
    rc = lib().oracle_disc_batch(_p(a), _p(b), n, B, _p(tw), _p(prod), _p(cert), _p(rad), _p(bad),
                                 _p(coeffs), _p(discs), nthreads)
    assert rc == 0
    return {"prod": prod, "cert": cert.astype(bool), "max_radius": rad, "first_bad": bad,
            "coeffs": coeffs, "discs": discs, "N": N}


def disc_op(op: str, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Disc primitive (R15) on [len][3] arrays: add, sub, mul, conj."""
    code = {"add": 0, "sub": 1, "mul": 2, "conj": 3}[op]
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    r = np.zeros_like(a)
    lib().oracle_disc_op(code, _p(a), _p(b), _p(r), a.shape[0])
    return r


def disc_fft(x: np.ndarray, inverse: int = 0) -> np.ndarray:
    """The paper's recursive FFT on discs [N][3], unscaled."""
    x = np.ascontiguousarray(x, np.float64)
    N = x.shape[0]
    tw = np.ascontiguousarray(twiddle_table(N, "f64"))
    out = np.zeros_like(x)
    lib().oracle_disc_fft(_p(x), _p(out), _p(tw), N, inverse)
    return out


def long_multiply(a: np.ndarray, b: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """P:44-56 for a batch of equal-length pairs -> [B][2n] digits."""
    a = np.ascontiguousarray(a, dtype=np.uint8)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    if a.ndim == 1:
        a, b = a[None], b[None]
    B, n = a.shape
    z = np.zeros((B, 2 * n), np.uint8)
    lib().oracle_long_multiply_batch(_p(a), _p(b), n, B, _p(z), nthreads)
    return z


def coefficients(a: np.ndarray, b: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """P:37 exact coefficient sums -> [B][2n-1] int64."""
    a = np.ascontiguousarray(a, dtype=np.uint8)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    if a.ndim == 1:
        a, b = a[None], b[None]
    B, n = a.shape
    z = np.zeros((B, 2 * n - 1), np.int64)
    lib().oracle_coefficients_batch(_p(a), _p(b), n, B, _p(z), nthreads)
    return z


def _is_prime(p: int) -> bool:
    """Deterministic Miller-Rabin for p < 3.3e24 (bases: the first 12 primes)."""
    if p < 2:
        return False
    small = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37]
    for q in small:
        if p % q == 0:
            return p == q
    d, s = p - 1, 0
    while d % 2 == 0:
        d, s = d // 2, s + 1
    for a in small:
        x = pow(a, d, p)
        if x in (1, p - 1):
            continue
        for _ in range(s - 1):
            x = x * x % p
            if x == p - 1:
                break
        else:
            return False
    return True


def random_primes(k: int = 2, bits: int = 61, seed: int | None = None) -> list[int]:
    """k distinct random primes of `bits` bits (the residue check's moduli)."""
    import random
    rng = random.Random(seed)
    out = []
    while len(out) < k:
        p = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
        if p not in out and _is_prime(p):
            out.append(p)
    return out


def residue_check(a: np.ndarray, b: np.ndarray, z: np.ndarray, primes=None, nthreads: int = 0) -> np.ndarray:
    """per pair, True iff z == a*b modulo every prime in `primes`
    (default: two fresh random 61-bit primes).  [B][n], [B][n], [B][2n]."""
    a = np.ascontiguousarray(a, dtype=np.uint8)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    z = np.ascontiguousarray(z, dtype=np.uint8)
    if a.ndim == 1:
        a, b, z = a[None], b[None], z[None]
    B, n = a.shape
    assert b.shape == (B, n) and z.shape == (B, 2 * n)
    pr = np.array(primes if primes is not None else random_primes(2), np.uint64)
    assert all(0 < int(p) < 2 ** 62 for p in pr)
    ok = np.zeros(B, np.uint8)
    lib().oracle_residue_check_batch(_p(a), _p(b), _p(z), n, B, _p(pr), len(pr), _p(ok), nthreads)
    return ok.astype(bool)


def carry(coeffs: np.ndarray) -> np.ndarray:
    """2n-1 non-negative coefficients -> 2n digits."""
    c = np.ascontiguousarray(coeffs, dtype=np.int64)
    n = (c.shape[0] + 1) // 2
    z = np.zeros(2 * n, np.uint8)
    lib().oracle_carry(_p(c), n, _p(z))
    return z


def interval_op(op: str, a: np.ndarray, b: np.ndarray, prec: str = "f64") -> np.ndarray:
    """Real interval op of P:251-253 on [len][2] endpoint arrays."""
    dt = np.float64 if prec == "f64" else np.float32
    a = np.ascontiguousarray(a, dtype=dt)
    b = np.ascontiguousarray(b, dtype=dt)
    r = np.zeros_like(a)
    code = {"add": 0, "sub": 1, "mul": 2}[op]
    f = lib().oracle_interval_op_f64 if prec == "f64" else lib().oracle_interval_op_f32
    f(code, _p(a), _p(b), _p(r), a.shape[0])
    return r


def cinterval_op(op: str, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Complex interval op of P:264-265 on [len][4] arrays (binary64)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    r = np.zeros_like(a)
    code = {"add": 0, "sub": 1, "mul": 2}[op]
    lib().oracle_cinterval_op_f64(code, _p(a), _p(b), _p(r), a.shape[0])
    return r


def fft(x: np.ndarray, inverse: int = 0, prec: str = "f64") -> np.ndarray:
    """Interval FFT of [N][4]; inverse=1 unscaled, 2 scaled by 1/N."""
    dt = np.float64 if prec == "f64" else np.float32
    x = np.ascontiguousarray(x, dtype=dt)
    N = x.shape[0]
    tw = np.ascontiguousarray(twiddle_table(N, prec))
    out = np.zeros_like(x)
    f = lib().oracle_fft_f64 if prec == "f64" else lib().oracle_fft_f32
    f(_p(x), _p(out), _p(tw), N, inverse)
    return out


def certify(iv: np.ndarray, prec: str = "f64"):
    """P:24 rule on [len][4] intervals -> (coeff int64, flag bool).  The same C
    function ss_multiply_* applies to its output (R8)."""
    dt = np.float64 if prec == "f64" else np.float32
    iv = np.ascontiguousarray(iv, dtype=dt).reshape(-1, 4)
    c = np.zeros(iv.shape[0], np.int64)
    f = np.zeros(iv.shape[0], np.uint8)
    fn = lib().oracle_certify_f64 if prec == "f64" else lib().oracle_certify_f32
    fn(_p(iv), iv.shape[0], _p(c), _p(f))
    return c, f.astype(bool)


def max_radius(iv: np.ndarray, prec: str = "f64") -> float:
    """DESIGN.md R10 radius over [len][4] intervals: max over both parts of
    RU(hi - lo)/2 (NaN -> inf).  The same C function ss_multiply_* applies."""
    dt = np.float64 if prec == "f64" else np.float32
    iv = np.ascontiguousarray(iv, dtype=dt).reshape(-1, 4)
    fn = lib().oracle_max_radius_f64 if prec == "f64" else lib().oracle_max_radius_f32
    return float(fn(_p(iv), iv.shape[0]))


def self_check() -> bool:
    return lib().oracle_self_check() == 0
