"""Index-logic prototype of the v2 schedule (point arithmetic, complex128).

Dev tool only.  Forward: half-spectrum Stockham DIT, rows kappa in [0, L/2),
row 0 packs the two real rows (kappa = 0 in .re, kappa = L/2 in .im);
boundary task = rdft (real DFT) + odft (odd real DFT).  Inverse: the m/2-point
complex IFFT of Z_k = U_k + i V_k, U_k = P_k + P_{k+m/2},
V_k = wbar_m^k (P_k - P_{k+m/2}); IFFT(Z)_j = m (c_{2j} + i c_{2j+1}).
"""
import numpy as np


def w(M, j):
    return np.exp(2j * np.pi * j / M)


def dft(v, inv=False):
    R = len(v)
    s = -1 if inv else 1
    return np.array([sum(v[q] * w(R, s * q * r) for q in range(R)) for r in range(R)])


def rdft(a):
    """X_s, s in [0, M/2] by the DIT recursion of the kernel."""
    M = len(a)
    if M == 1:
        return np.array([a[0] + 0j])
    if M == 2:
        return np.array([a[0] + a[1], a[0] - a[1]], complex)
    E, O = rdft(a[0::2]), rdft(a[1::2])
    X = np.zeros(M // 2 + 1, complex)
    X[0] = E[0].real + O[0].real
    X[M // 2] = E[0].real - O[0].real
    X[M // 4] = E[M // 4].real + 1j * O[M // 4].real
    for s in range(1, M // 4):
        t = w(M, s) * O[s]
        X[s] = E[s] + t
        X[M // 2 - s] = np.conj(E[s] - t)
    return X


def odft(b):
    """Y_r = sum_i b_i w_{2M}^{i(2r+1)}, r in [0, M/2)."""
    M = len(b)
    if M == 1:
        return np.array([b[0] + 0j])
    if M == 2:
        return np.array([b[0] + 1j * b[1]])
    E, O = odft(b[0::2]), odft(b[1::2])
    Y = np.zeros(M // 2, complex)
    for r in range(M // 4):
        t = w(2 * M, 2 * r + 1) * O[r]
        Y[r] = E[r] + t
        Y[M // 2 - 1 - r] = np.conj(E[r] - t)
    return Y


def forward(x, plan):
    """Returns per-thread register contents of the last pass:
    list of (k0, class1_vals[R], class2, vals2[R]) plus the full half spectrum."""
    N = len(x)
    R0 = plan[0]
    S1 = N // R0
    L = R0
    F = np.full((L // 2, S1), np.nan + 0j)
    for v in range(S1):
        xs = np.array([x[v + S1 * q] for q in range(R0 // 2)])  # upper half zero (n <= N/2)
        assert all(x[v + S1 * q] == 0 for q in range(R0 // 2, R0))
        Xe = rdft(xs)   # X_{2s}
        Yo = odft(xs)   # X_{2s+1}
        full = np.zeros(R0, complex)
        for s in range(R0 // 4 + 1):
            full[2 * s] = Xe[s]
        for s in range(R0 // 4):
            full[2 * s + 1] = Yo[s]
        assert np.allclose(full[:R0 // 2 + 1], dft(np.concatenate([xs, np.zeros(R0 // 2)]))[:R0 // 2 + 1])
        F[0, v] = full[0].real + 1j * full[R0 // 2].real
        for r in range(1, R0 // 2):
            F[r, v] = full[r]
    S = S1
    regs = None
    for p, R in enumerate(plan[1:], 1):
        Sp = S // R
        last = p == len(plan) - 1
        Fn = np.full((L * R // 2, Sp), np.nan + 0j)
        regs = []
        for k0 in range(L // 2):
            for v in range(Sp):
                if k0 == 0:
                    a = np.array([F[0, v + Sp * q].real for q in range(R)])
                    b = np.array([F[0, v + Sp * q].imag for q in range(R)])
                    X = rdft(a)
                    Y = odft(b)
                    Fn[0, v] = X[0].real + 1j * X[R // 2].real
                    for s in range(1, R // 2):
                        Fn[L * s, v] = X[s]
                    for r in range(R // 2):
                        Fn[L // 2 + L * r, v] = Y[r]
                    c1 = np.array([X[s] if s <= R // 2 else np.conj(X[R - s]) for s in range(R)])
                    c2 = np.array([Y[r] if r < R // 2 else np.conj(Y[R - 1 - r]) for r in range(R)])
                    regs.append((0, c1, L // 2, c2))
                else:
                    vals = [w(L * R, q * k0) * F[k0, v + Sp * q] for q in range(R)]
                    O = dft(vals)
                    for r in range(R):
                        kap = k0 + L * r
                        if 2 * kap < L * R:
                            Fn[kap, v] = O[r]
                        else:
                            Fn[L * R - kap, v] = np.conj(O[r])
                    c2 = np.array([np.conj(O[R - 1 - r]) for r in range(R)])
                    regs.append((k0, O, L - k0, c2))
        if not last:
            assert not np.isnan(Fn).any(), p
        F, L, S = Fn, L * R, Sp
    return regs, N // plan[-1]


def check(N, fplan, iplan, n=None):
    rng = np.random.default_rng(N)
    n = n or N // 2
    a = np.zeros(N); b = np.zeros(N)
    a[:n] = rng.integers(0, 256, n); b[:n] = rng.integers(0, 256, n)
    XA = np.fft.ifft(a) * N  # DFT with e^{+2 pi i/N}
    XB = np.fft.ifft(b) * N
    regsA, L = forward(a, fplan)
    regsB, _ = forward(b, fplan)
    R = fplan[-1]
    assert L == N // R
    # class values: X[cls + L r] for r < R
    for (c1, v1, c2, v2) in regsA:
        for r in range(R):
            assert np.isclose(v1[r], XA[c1 + L * r]), (c1, r)
            assert np.isclose(v2[r], XA[c2 + L * r]), (c2, r)
    # fused: pointwise, pre-step, inverse pass 0 (Q0 = R/2, M = N/2, S1 = L)
    M = N // 2
    Q0 = R // 2
    assert iplan[0] == Q0
    E = np.full((Q0, L), np.nan + 0j)
    for (ra, rb) in zip(regsA, regsB):
        for cls, va, vb in ((ra[0], ra[1], rb[1]), (ra[2], ra[3], rb[3])):
            P = va * vb
            Z = []
            for r in range(Q0):
                k = cls + L * r
                U = P[r] + P[r + R // 2]
                V = w(N, -k) * (P[r] - P[r + R // 2])
                Z.append(U + 1j * V)
            O = dft(np.array(Z), inv=True)
            for rp in range(Q0):
                E[rp, cls] = O[rp]
    assert not np.isnan(E).any()
    Lc, S = Q0, L
    for p, Q in enumerate(iplan[1:], 1):
        Sp = S // Q
        En = np.full((Lc * Q, Sp), np.nan + 0j)
        for k0 in range(Lc):
            for v in range(Sp):
                vals = [w(Lc * Q, -q * k0) * E[k0, v + Sp * q] for q in range(Q)]
                O = dft(vals, inv=True)
                for r in range(Q):
                    En[k0 + Lc * r, v] = O[r]
        E, Lc, S = En, Lc * Q, Sp
    wv = E[:, 0] / N
    c = np.zeros(N)
    c[0::2] = wv.real
    c[1::2] = wv.imag
    exact = np.convolve(a[:n], b[:n])
    assert np.allclose(c[:2 * n - 1], exact, atol=1e-6), np.abs(c[:2 * n - 1] - exact).max()
    assert np.allclose(c[2 * n - 1:], 0, atol=1e-6)
    print("ok", N, fplan, iplan)


if __name__ == "__main__":
    for M in (2, 4, 8, 16, 32):
        x = np.random.default_rng(M).standard_normal(M)
        assert np.allclose(rdft(x), dft(x)[:M // 2 + 1])
        y = np.random.default_rng(M + 1).standard_normal(M)
        ref = np.array([sum(y[i] * w(2 * M, i * (2 * r + 1)) for i in range(M)) for r in range(M // 2)])
        assert np.allclose(odft(y), ref)
    check(32, [4, 8], [4, 4])
    check(64, [4, 16], [8, 4])
    check(128, [8, 16], [8, 8])
    check(256, [16, 16], [8, 16])
    check(512, [32, 16], [8, 16, 2])
    check(1024, [4, 16, 16], [8, 16, 4], n=300)
    check(2048, [8, 16, 16], [8, 16, 8])
    check(4096, [16, 16, 16], [8, 16, 16])
    check(8192, [32, 16, 16], [8, 16, 16, 2])
