"""Index-logic prototype of the odd-frequency ("twisted") schedule, point arithmetic.

Dev tool only.  T(x)_k = sum_j x_j z^{j(2k+1)}, z = e^{2 pi i/(2m)}.  For real x,
T_{m-1-k} = conj(T_k) (no self-conjugate bin) and T(a) T(b) = T(a*b) when
a*b has < m terms (negacyclic = linear under zero padding).

Forward (Stockham DIT, half storage G_p[k][v], k < L/2, v < S):
  G_{p+1}[k0 + L r][v] = sum_q w_R^{qr} (w_{2LR}^{q(2k0+1)} G_p[k0][v + S'q])
  r < R/2 stored at row k0 + L r; r >= R/2 stored conj at row LR-1-k0-Lr.
Inverse (half storage in v: E_p[k][v], v < S/2; mirror E[k][S-1-v] = w_L^k conj E[k][v]):
  E_{p+1}[k0 + L r][v] = sum_q wbar_Q^{qr} (wbar_{LQ}^{q k0} E_p[k0][v + S'q])
  final radix-2 step (S = 2): v = z^{-k} E[k][0], c_k = 2 Re(v)/m, c_{k+m/2} = 2 Im(v)/m.
"""
import numpy as np


def w(M, j):
    return np.exp(2j * np.pi * j / M)


def dft(v, inv=False):
    R = len(v)
    s = -1 if inv else 1
    return np.array([sum(v[q] * w(R, s * q * r) for q in range(R)) for r in range(R)])


def check(N, fplan, iplan, n=None):
    assert np.prod(fplan) == N and np.prod(iplan) * 2 == N and fplan[-1] == iplan[0]
    rng = np.random.default_rng(N)
    n = n or N // 2
    a = np.zeros(N); b = np.zeros(N)
    a[:n] = rng.integers(0, 256, n); b[:n] = rng.integers(0, 256, n)
    z2N = lambda j: w(2 * N, j)
    TA = np.array([sum(a[j] * z2N(j * (2 * k + 1)) for j in range(N)) for k in range(N)]) if N <= 512 else None

    def forward(x):
        # pass 0, R0 = 2 (trivial, x[v + N/2] = 0): G_1[0][v] = x[v]
        assert fplan[0] == 2
        L, S = 2, N // 2
        G = np.array([x[:N // 2].astype(complex)])  # [1][N/2]
        regs = None
        for p, R in enumerate(fplan[1:], 1):
            Sp = S // R
            last = p == len(fplan) - 1
            Gn = np.full((L * R // 2, Sp), np.nan + 0j)
            regs = []
            for k0 in range(L // 2):
                for v in range(Sp):
                    vals = [w(2 * L * R, q * (2 * k0 + 1)) * G[k0, v + Sp * q] for q in range(R)]
                    O = dft(vals)
                    for r in range(R):
                        kap = k0 + L * r
                        if r < R // 2:
                            Gn[kap, v] = O[r]
                        else:
                            Gn[L * R - 1 - kap, v] = np.conj(O[r])
                    if last:
                        regs.append((k0, O))
            if not last:
                assert not np.isnan(Gn).any(), p
            G, L, S = Gn, L * R, Sp
        return G[:, 0], regs, N // fplan[-1]

    XA, regsA, Llast = forward(a)
    XB, regsB, _ = forward(b)
    if TA is not None:
        assert np.allclose(XA, TA[:N // 2])
        for k0, O in regsA:
            for r in range(len(O)):
                assert np.isclose(O[r], TA[k0 + Llast * r])
    # fused: pointwise + inverse pass 0 (Q0 = R, S1 = Llast, v = k0 < S1/2)
    Q0 = iplan[0]
    E = np.full((Q0, Llast // 2), np.nan + 0j)
    for (k0, OA), (_, OB) in zip(regsA, regsB):
        P = OA * OB
        O = dft(P, inv=True)
        for rp in range(Q0):
            E[rp, k0] = O[rp]
    L, S = Q0, Llast
    for p, Q in enumerate(iplan[1:], 1):
        Sp = S // Q
        H = S // 2
        En = np.full((L * Q, Sp // 2), np.nan + 0j)
        for k0 in range(L):
            for v in range(Sp // 2):
                vals = []
                for q in range(Q):
                    mu = v + Sp * q
                    if mu < H:
                        vals.append(w(L * Q, -q * k0) * E[k0, mu])
                    else:
                        vals.append(w(L * Q, (Q - q) * k0) * np.conj(E[k0, S - 1 - mu]))
                O = dft(vals, inv=True)
                for r in range(Q):
                    En[k0 + L * r, v] = O[r]
        assert not np.isnan(En).any(), p
        E, L, S = En, L * Q, Sp
    assert S == 2 and L == N // 2
    c = np.zeros(N)
    for k in range(N // 2):
        v = w(2 * N, -k) * E[k, 0]
        c[k] = 2 * v.real / N
        c[k + N // 2] = 2 * v.imag / N
    exact = np.convolve(a[:n], b[:n])
    assert np.allclose(c[:2 * n - 1], exact, atol=1e-6), np.abs(c[:2 * n - 1] - exact).max()
    assert np.allclose(c[2 * n - 1:], 0, atol=1e-6)
    print("ok", N, fplan, iplan)


if __name__ == "__main__":
    check(16, [2, 8], [8])
    check(32, [2, 16], [16])
    check(64, [2, 2, 16], [16, 2])
    check(128, [2, 4, 16], [16, 4])
    check(256, [2, 8, 16], [16, 8])
    check(512, [2, 16, 16], [16, 16])
    check(1024, [2, 2, 16, 16], [16, 16, 2], n=300)
    check(2048, [2, 4, 16, 16], [16, 16, 4])
    check(4096, [2, 8, 16, 16], [16, 16, 8])
    check(8192, [2, 16, 16, 16], [16, 16, 16])


def check_r8():
    check(8192, [2, 8, 8, 8, 8], [8, 8, 8, 8])
    check(4096, [2, 4, 8, 8, 8], [8, 8, 8, 4])
    check(2048, [2, 2, 8, 8, 8], [8, 8, 8, 2])
    check(1024, [2, 8, 8, 8], [8, 8, 8])
