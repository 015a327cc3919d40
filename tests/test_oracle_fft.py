"""Pins of the oracle's interval FFT (§2.2).

Pinned against exact special cases (impulse, constant), the DFT definition
P:68 evaluated independently in mpmath (O(N^2) direct sums), the inverse
Proposition P:97 (round trip), and the closed form of the all-255 spectrum.
"""
import mpmath
import numpy as np
import pytest

import oracle
from tests.exact import F


def _punctual(x):
    x = np.asarray(x, dtype=np.complex128)
    out = np.zeros((x.shape[0], 4))
    out[:, 0] = out[:, 1] = x.real
    out[:, 2] = out[:, 3] = x.imag
    return out


def _contains(iv, re, im):
    return (mpmath.mpf(float(iv[0])) <= re <= mpmath.mpf(float(iv[1])) and
            mpmath.mpf(float(iv[2])) <= im <= mpmath.mpf(float(iv[3])))


@pytest.mark.parametrize("N", [1, 2, 4, 16, 256, 2048])
def test_fft_impulse_is_exact_ones(N):
    x = np.zeros(N); x[0] = 1
    X = oracle.fft(_punctual(x))
    assert np.all(X[:, 0] == 1) and np.all(X[:, 1] == 1)
    assert np.all(X[:, 2] == 0) and np.all(X[:, 3] == 0)


@pytest.mark.parametrize("N", [2, 8, 64, 1024])
def test_fft_constant_is_exact_delta(N):
    X = oracle.fft(_punctual(np.ones(N)))
    assert X[0, 0] == N and X[0, 1] == N and X[0, 2] == 0 and X[0, 3] == 0
    assert np.all(X[1:] == 0)


def test_fft_n1_is_identity():
    """for n = 1 the DFT is the identity."""
    x = _punctual([3.5 + 2j])
    assert np.array_equal(oracle.fft(x), x)


@pytest.mark.parametrize("N", [8, 32, 64])
def test_fft_contains_mpmath_dft(N):
    """P:68 DFT_i = sum_j x_j omega^{ij}, omega = e^{2 pi i/N}."""
    rng = np.random.default_rng(N)
    x = rng.integers(0, 256, N) + 1j * rng.integers(-50, 50, N)
    X = oracle.fft(_punctual(x))
    Xi = oracle.fft(_punctual(x), inverse=1)
    with mpmath.workprec(200):
        for i in range(N):
            s = mpmath.mpc(0)
            si = mpmath.mpc(0)
            for j in range(N):
                w = mpmath.expjpi(mpmath.mpf(2 * i * j) / N)
                s += mpmath.mpc(x[j].real, x[j].imag) * w
                si += mpmath.mpc(x[j].real, x[j].imag) / w
            assert _contains(X[i], s.real, s.imag), (N, i)
            assert _contains(Xi[i], si.real, si.imag), (N, i)


def test_fft_impulse_e1_contains_roots():
    N = 64
    x = np.zeros(N); x[1] = 1
    X = oracle.fft(_punctual(x))
    with mpmath.workprec(200):
        for k in range(N):
            w = mpmath.expjpi(mpmath.mpf(2 * k) / N)
            assert _contains(X[k], w.real, w.imag)


@pytest.mark.parametrize("N", [16, 512])
def test_round_trip_contains_input(N):
    """P:97 Proposition: IDFT(DFT(x)) = x; the interval round trip contains x."""
    rng = np.random.default_rng(3)
    x = rng.integers(0, 256, N).astype(float)
    y = oracle.fft(oracle.fft(_punctual(x)), inverse=2)
    assert np.all(y[:, 0] <= x) and np.all(x <= y[:, 1])
    assert np.all(y[:, 2] <= 0) and np.all(0 <= y[:, 3])
    assert np.max(y[:, 1] - y[:, 0]) < 1e-9


def test_all255_spectrum_closed_form():
    """A_k = 255 (omega^{nk} - 1)/(omega^k - 1) for k != 0, A_0 = 255 n."""
    n, N = 100, 256
    x = np.zeros(N); x[:n] = 255
    X = oracle.fft(_punctual(x))
    assert X[0, 0] <= 255 * n <= X[0, 1]
    with mpmath.workprec(200):
        for k in range(1, N, 5):
            w = mpmath.expjpi(mpmath.mpf(2 * k) / N)
            A = 255 * (w ** n - 1) / (w - 1)
            assert _contains(X[k], A.real, A.imag), k


def test_f32_fft_contains_dft():
    N = 32
    rng = np.random.default_rng(11)
    x = rng.integers(0, 256, N).astype(float)
    X = oracle.fft(_punctual(x).astype(np.float32), prec="f32")
    with mpmath.workprec(200):
        for i in range(N):
            s = sum(mpmath.mpf(x[j]) * mpmath.expjpi(mpmath.mpf(2 * i * j) / N) for j in range(N))
            assert _contains(X[i], s.real, s.imag), i
