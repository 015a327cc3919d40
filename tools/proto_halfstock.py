"""Index-logic prototype of the CUDA kernel's FFT schedule (point arithmetic).

Dev tool only (not product, not oracle): validates in complex128 the task /
storage rules of the half-storage Stockham DIT used by csrc/ivm_kernels.cu,
before they are written in CUDA.  Run: python tools/proto_halfstock.py

Forward (real input x, length N):   F_p[k][v], k in [0, L_p/2], v in [0, S_p)
  pass p:  F_{p+1}[k0 + L r][v] = sum_q w_R^{qr} (w_{LR}^{q k0} F_p[k0][v + S' q])
Inverse (Hermitian input P):        E_p[k][v], k in [0, L_p), v in [0, S_p/2]
  mirror:  E_p[k][S - v] = w_L^{k} conj(E_p[k][v])
  pass p:  E_{p+1}[k0 + L r][v] = sum_q wbar_Q^{qr} (wbar_{LQ}^{q k0} E_p[k0][v + S' q])
"""
import numpy as np


def w(M, j):
    return np.exp(2j * np.pi * j / M)


def dft(v, inverse=False):
    R = len(v)
    s = -1 if inverse else 1
    return np.array([sum(v[q] * w(R, s * q * r) for q in range(R)) for r in range(R)])


def forward_half(x, plan):
    N = len(x)
    # pass 0 (real input)
    R = plan[0]
    L, S1 = 1, N // R
    F = np.zeros(((R // 2 + 1), S1), complex)
    for v in range(S1):
        O = dft([x[v + S1 * q] for q in range(R)])
        for r in range(R // 2 + 1):
            F[r, v] = O[r]
    L = R
    S = S1
    outs = []
    for p, R in enumerate(plan[1:], 1):
        Sn = S // R
        Fn = np.full((L * R // 2 + 1, Sn), np.nan + 0j)
        last = (p == len(plan) - 1)
        for k0 in range(L // 2 + 1):
            for v in range(Sn):
                vals = [w(L * R, q * k0) * F[k0, v + Sn * q] for q in range(R)]
                O = dft(vals)
                if last:
                    outs.append((k0, O))
                for r in range(R):
                    k = k0 + L * r
                    if k0 == 0:
                        if r <= R // 2:
                            Fn[k, v] = O[r]
                    elif 2 * k0 == L:
                        if r < R // 2:
                            Fn[k, v] = O[r]
                    else:
                        if 2 * k <= L * R:
                            Fn[k, v] = O[r]
                        else:
                            Fn[L * R - k, v] = np.conj(O[r])
        assert not np.isnan(Fn).any(), p
        F, L, S = Fn, L * R, Sn
    return F[:, 0], outs


def inverse_half_fused(outsA, X_A_half, outsB, plan_inv, N):
    """B's last forward pass registers * A -> inverse pass 0 -> ... -> real c."""
    Q0 = plan_inv[0]
    L1, S1 = Q0, N // Q0
    E = np.full((L1, S1 // 2 + 1), np.nan + 0j)
    for k0, OB in outsB:  # task holds X_B[k0 + S1 r], r < Q0 (L_last = S1)
        v = k0
        P = []
        for q in range(Q0):
            idx = v + S1 * q
            a = X_A_half[idx] if idx <= N // 2 else np.conj(X_A_half[N - idx])
            P.append(a * OB[q])
        O = dft(P, inverse=True)
        for r in range(Q0):
            E[r, v] = O[r]
    assert not np.isnan(E).any()
    L, S = L1, S1
    for p, Q in enumerate(plan_inv[1:], 1):
        Sn = S // Q
        last = (p == len(plan_inv) - 1)
        if last:
            c = np.zeros(N, complex)
        else:
            En = np.full((L * Q, Sn // 2 + 1), np.nan + 0j)
        for k0 in range(L):
            for v in range(Sn // 2 + 1):
                vals = []
                for q in range(Q):
                    mu = v + Sn * q
                    if 2 * mu <= S:
                        vals.append(w(L * Q, -q * k0) * E[k0, mu])
                    else:
                        vals.append(w(L * Q, (Q - q) * k0) * np.conj(E[k0, S - mu]))
                O = dft(vals, inverse=True)
                for r in range(Q):
                    if last:
                        c[k0 + L * r] = O[r] / N
                    else:
                        En[k0 + L * r, v] = O[r]
        if last:
            return c
        assert not np.isnan(En).any(), p
        E, L, S = En, L * Q, Sn
    raise AssertionError


def check(N, plan_f, plan_i, n=None):
    rng = np.random.default_rng(N)
    n = n or N // 2
    a = np.zeros(N); b = np.zeros(N)
    a[:n] = rng.integers(0, 256, n); b[:n] = rng.integers(0, 256, n)
    XA, _ = forward_half(a, plan_f)
    XB, outsB = forward_half(b, plan_f)
    ref = np.fft.ifft(a)  # numpy: ifft has e^{+}; our DFT uses e^{+2 pi i/N}
    assert np.allclose(XA, (np.fft.ifft(a) * N)[:N // 2 + 1]), "forward"
    c = inverse_half_fused(None, XA, outsB, plan_i, N)
    exact = np.convolve(a[:n], b[:n])
    assert np.allclose(c.real[:2 * n - 1], exact, atol=1e-6), "conv"
    assert np.allclose(c.imag, 0, atol=1e-6)
    print("ok", N, plan_f, plan_i)


if __name__ == "__main__":
    check(16, [4, 4], [4, 4])
    check(64, [4, 16], [16, 4])
    check(512, [2, 16, 16], [16, 2, 16])
    check(256, [16, 16], [16, 16])
    check(2048, [8, 16, 16], [16, 8, 16])
    check(8192, [32, 16, 16], [16, 4, 8, 16])
    check(4096, [16, 16, 16], [16, 16, 16], n=1000)
