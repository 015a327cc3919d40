// ivm_v3g.cuh -- large transforms (m = 2^14 .. 2^18): the v3 odd-frequency
// schedule with the state in global memory (L2-resident: only a few
// multiplications are in flight), executed by a GROUP of C co-resident CTAs per
// multiplication (cooperative launch), passes separated by group barriers,
// ping-pong state buffers.  Same pass arithmetic as ivm_v3.cuh (P:143-155 DIT,
// P:210 pointwise, P:97 inverse, P:24 certify), carry P:229-235 across the group.
#pragma once

namespace ivm {
namespace v3 {

struct GroupCtx {
  unsigned *ctr;         // [groups] barrier counters (zeroed by the host)
  int C;                 // CTAs per group
  void *state;           // per group: A | S0 | S1 : 3 x (2 x m/2) V2 elements
  long long *coef;       // per group: [m]
  int *cert;             // per group: [4] ok, first_bad, maxrad(lo), maxrad(hi)
  unsigned *agg;         // per group: [C] carry aggregates
};

__device__ __forceinline__ void group_sync(unsigned *ctr, int C, unsigned &gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned target = (gen + 1) * (unsigned)C;
    atomicAdd(ctr, 1u);
    while (*(volatile unsigned *)ctr < target) {
    }
    __threadfence();
  }
  gen++;
  __syncthreads();
}

template <typename T, int M> struct GG {
  static constexpr Plan P = plan(M);
  static constexpr int N = 1 << M;
  static constexpr int C = N / 8192 < 1 ? 1 : N / 8192;  // CTAs per group
  static constexpr int TH = 256;
};

// ---- one task of forward pass 1 (digits -> dst) ----
template <typename T, int M>
__device__ __forceinline__ void g_fwd_first(int nu, const uint8_t *__restrict__ dig, int n, Buf<T> dst) {
  constexpr Plan PL = plan(M);
  constexpr int N = 1 << M, R = PL.f[1], L = 2, S = N / 2, Sp = S / R;
  CI<T> v[R];
#pragma unroll
  for (int q = 0; q < R; q++) {
    const int idx = nu + Sp * q;
    const T x = idx < n ? T(dig[idx]) : T(0);
    if (q == 0) {
      v[q] = punctual(x);
    } else {
      const TwC<T> w = cw64<T>(q * (16 / R));
      v[q] = CI<T>{DR<T>::mul_rd(w.c, x), DR<T>::mul_ru(TB<T>::sel(w.c, 1u), x), DR<T>::mul_rd(w.s, x),
                   DR<T>::mul_ru(TB<T>::sel(w.s, 1u), x)};
    }
  }
  cdft<T, R, false>(v);
#pragma unroll
  for (int r = 0; r < R; r++) {
    if (r < R / 2) dst.st((L * r) * Sp + nu, v[r]);
    else dst.st((L * R - 1 - L * r) * Sp + nu, cconj(v[r]));
  }
}

// ---- forward pass p >= 2: load + twiddle + DFT of task t ----
template <typename T, int M, int p>
__device__ __forceinline__ void g_fwd_load(int t, Buf<T> src, const TwC<T> *__restrict__ tw,
                                           CI<T> (&v)[plan(M).f[p]], int &k0) {
  constexpr Plan PL = plan(M);
  constexpr int N = 1 << M, R = PL.f[p], L = fL(PL, p), S = N / L, Sp = S / R;
  constexpr int TW = G3<M>::tw_fwd(p);
  k0 = t / Sp;
  const int nu = t % Sp;
#pragma unroll
  for (int q = 0; q < R; q++) {
    CI<T> z = src.ld(k0 * S + nu + Sp * q);
    if (q > 0) z = rtmul<T, false>(ldg_twc(tw, TW + (q - 1) * (L / 2) + k0), z);
    v[q] = z;
  }
  cdft<T, R, false>(v);
}

template <typename T, int M, int p>
__device__ __forceinline__ void g_fwd_pass(int t, Buf<T> src, Buf<T> dst, const TwC<T> *__restrict__ tw) {
  constexpr Plan PL = plan(M);
  constexpr int N = 1 << M, R = PL.f[p], L = fL(PL, p), Sp = N / L / R;
  CI<T> v[R];
  int k0;
  g_fwd_load<T, M, p>(t, src, tw, v, k0);
  const int nu = t % Sp;
#pragma unroll
  for (int r = 0; r < R; r++) {
    if (r < R / 2) dst.st((k0 + L * r) * Sp + nu, v[r]);
    else dst.st((L * R - 1 - k0 - L * r) * Sp + nu, cconj(v[r]));
  }
}

template <typename T, int M>
__device__ __forceinline__ void g_fwd_last_a(int t, Buf<T> src, Buf<T> A, const TwC<T> *__restrict__ tw) {
  constexpr Plan PL = plan(M);
  constexpr int p = PL.nf - 1, R = PL.f[p], L = fL(PL, p);
  CI<T> v[R];
  int k0;
  g_fwd_load<T, M, p>(t, src, tw, v, k0);
#pragma unroll
  for (int r = 0; r < R; r++) A.st(r * (L / 2) + k0, v[r]);
}

template <typename T, int M>
__device__ __forceinline__ void g_fused(int t, Buf<T> src, Buf<T> A, Buf<T> dst, const TwC<T> *__restrict__ tw) {
  constexpr Plan PL = plan(M);
  constexpr int p = PL.nf - 1, R = PL.f[p], L = fL(PL, p);
  static_assert(PL.q[0] == R, "fused radix");
  constexpr int H1 = L / 2;  // inverse state E_1: rows R, cols (N/R)/2
  CI<T> v[R];
  int k0;
  g_fwd_load<T, M, p>(t, src, tw, v, k0);
#pragma unroll
  for (int r = 0; r < R; r++) v[r] = cmul(A.ld(r * (L / 2) + k0), v[r]);
  cdft<T, R, true>(v);
#pragma unroll
  for (int r = 0; r < R; r++) dst.st(r * H1 + k0, v[r]);
}

template <typename T, int M, int p>
__device__ __forceinline__ void g_inv_load(int t, Buf<T> src, const TwC<T> *__restrict__ tw,
                                           CI<T> (&v)[plan(M).q[p]], int &k0, int &nu) {
  constexpr Plan PL = plan(M);
  constexpr int N = 1 << M, Q = PL.q[p], L = iL(PL, p), S = N / L, Sp = S / Q, H = Sp / 2;
  constexpr int TW = G3<M>::tw_inv(p);
  k0 = t / H;
  nu = t % H;
#pragma unroll
  for (int q = 0; q < Q; q++) {
    CI<T> z;
    if (2 * q < Q) z = src.ld(k0 * (S / 2) + nu + Sp * q);
    else z = cconj(src.ld(k0 * (S / 2) + (S - 1 - nu - Sp * q)));
    if (q > 0) {
      const TwC<T> w = ldg_twc(tw, TW + (q - 1) * L + k0);
      z = (2 * q < Q) ? rtmul<T, true>(w, z) : rtmul<T, false>(w, z);
    }
    v[q] = z;
  }
  cdft<T, Q, true>(v);
}

template <typename T, int M, int p>
__device__ __forceinline__ void g_inv_pass(int t, Buf<T> src, Buf<T> dst, const TwC<T> *__restrict__ tw) {
  constexpr Plan PL = plan(M);
  constexpr int N = 1 << M, Q = PL.q[p], L = iL(PL, p), Sp = N / L / Q;
  CI<T> v[Q];
  int k0, nu;
  g_inv_load<T, M, p>(t, src, tw, v, k0, nu);
#pragma unroll
  for (int r = 0; r < Q; r++) dst.st((k0 + L * r) * (Sp / 2) + nu, v[r]);
}

// certification into the group's global record
template <typename T>
__device__ __forceinline__ void g_certify(T lo, T hi, int i, int n, long long *coef, int *cert, double *dump) {
  if (dump) reinterpret_cast<double4 *>(dump)[i] = make_double4((double)lo, (double)hi, 0.0, 0.0);
  if (i >= 2 * n - 1) return;
  const double l = (double)lo, h = (double)hi;
  const double cl = ceil(l);
  const bool ok = cl == floor(h);
  double rad = __dmul_ru(__dadd_ru(h, -l), 0.5);
  if (!(rad <= 1e300)) rad = __longlong_as_double(0x7ff0000000000000ll);
  atomicMax(reinterpret_cast<unsigned long long *>(cert + 2), (unsigned long long)__double_as_longlong(rad));
  if (ok) {
    coef[i] = (long long)cl;
  } else {
    coef[i] = 0;
    cert[0] = 0;
    atomicMin(cert + 1, i);
  }
}

template <typename T, int M>
__device__ __forceinline__ void g_inv_last(int t, Buf<T> src, const TwC<T> *__restrict__ tw, int n,
                                           long long *coef, int *cert, double *dump) {
  constexpr Plan PL = plan(M);
  constexpr int N = 1 << M, p = PL.ni - 1, Q = PL.q[p], L = iL(PL, p);
  constexpr int TWF = G3<M>::tw_fin();
  CI<T> v[Q];
  int k0, nu;
  g_inv_load<T, M, p>(t, src, tw, v, k0, nu);
  const T s = T(2) / T(N);
#pragma unroll
  for (int r = 0; r < Q; r++) {
    const int k = k0 + L * r;
    const CI<T> w = rtmul<T, true>(ldg_twc(tw, TWF + k), v[r]);
    g_certify(DR<T>::mul_rd(w.rl, s), DR<T>::mul_ru(w.rh, s), k, n, coef, cert, dump);
    g_certify(DR<T>::mul_rd(w.il, s), DR<T>::mul_ru(w.ih, s), k + N / 2, n, coef, cert, dump);
  }
}

// ---- group carry: c_i < 2^40 in 5 bytes; t_i <= 1275, u_i <= 259 ----
__device__ __forceinline__ long long gcoef(const long long *c, long long i, long long nc) {
  return (i >= 0 && i < nc) ? c[i] : 0;
}
__device__ __forceinline__ int gt(const long long *c, long long i, long long nc) {
  int t = 0;
#pragma unroll
  for (int b = 0; b < 5; b++) t += (int)((gcoef(c, i - b, nc) >> (8 * b)) & 255);
  return t;
}
__device__ __forceinline__ int gu(const long long *c, long long i, long long nc) {
  return (gt(c, i, nc) & 255) + (gt(c, i - 1, nc) >> 8);
}

__device__ void g_carry(const long long *coef, int n, uint8_t *__restrict__ out, bool certified, int rank,
                        int C, unsigned *agg, unsigned *ctr, unsigned &gen) {
  const long long nout = 2LL * n, nc = 2LL * n - 1, npos = 2LL * n + 5;
  const int T = blockDim.x;
  const long long total = (long long)C * T;
  const long long me = (long long)rank * T + threadIdx.x;
  if (!certified) {
    for (long long i = me; i < nout; i += total) out[i] = 0;
    return;
  }
  const long long K = (npos + total - 1) / total;
  const long long p0 = me * K, p1 = (p0 + K < npos) ? p0 + K : npos;
  int c = 0;
  bool allp = true;
  for (long long i = p0; i < p1; i++) {
    const int u = gu(coef, i, nc);
    allp = allp && (u == 255);
    c = (u + c) >> 8;
  }
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (T + 31) >> 5;
  const unsigned g = __ballot_sync(0xffffffffu, c != 0), pp = __ballot_sync(0xffffffffu, allp);
  __shared__ unsigned wg[32], wp[32], wc[32];
  __shared__ unsigned blk_cin;
  if (lane == 0) {
    const unsigned long long s = (unsigned long long)(g | pp) + g;
    wg[warp] = (unsigned)(s >> 32);
    wp[warp] = (pp == 0xffffffffu);
  }
  __syncthreads();
  if (warp == 0) {
    const bool gg = lane < nw ? wg[lane] != 0 : false;
    const bool pq = lane < nw ? wp[lane] != 0 : true;
    const unsigned G2 = __ballot_sync(0xffffffffu, gg), P2 = __ballot_sync(0xffffffffu, pq);
    const unsigned long long s2 = (unsigned long long)(G2 | P2) + G2;
    if (lane == 0) agg[rank] = ((unsigned)(s2 >> 32) & 1u) | ((P2 == 0xffffffffu) ? 2u : 0u);
    if (lane < nw) wc[lane] = 0;  // placeholder until the block carry-in is known
  }
  group_sync(ctr, C, gen);
  if (threadIdx.x == 0) {
    unsigned cin = 0;
    for (int r = 0; r < rank; r++) {
      const unsigned a = *(volatile unsigned *)(agg + r);
      cin = (a & 1u) | ((a >> 1) & cin);
    }
    blk_cin = cin;
  }
  __syncthreads();
  if (warp == 0) {
    const bool gg = lane < nw ? wg[lane] != 0 : false;
    const bool pq = lane < nw ? wp[lane] != 0 : true;
    const unsigned G2 = __ballot_sync(0xffffffffu, gg), P2 = __ballot_sync(0xffffffffu, pq);
    const unsigned cinv = (unsigned)(((unsigned long long)(G2 | P2) + G2 + blk_cin) ^ P2);
    if (lane < nw) wc[lane] = (cinv >> lane) & 1u;
  }
  __syncthreads();
  const unsigned long long s = (unsigned long long)(g | pp) + g + wc[warp];
  int cc = (int)(((unsigned)s ^ pp) >> lane) & 1;
  for (long long i = p0; i < p1; i++) {
    const int u = gu(coef, i, nc) + cc;
    if (i < nout) out[i] = (uint8_t)(u & 255);
    cc = u >> 8;
  }
}

template <typename T, int M>
__global__ void __launch_bounds__(256, 1) ivm_v3g_kernel(KParams kp, GroupCtx gc) {
  using V = typename V2t<T>::t;
  constexpr Plan PL = plan(M);
  constexpr int N = 1 << M, H = N / 2;
  const int C = gc.C;
  const int group = blockIdx.x / C, rank = blockIdx.x % C, groups = gridDim.x / C;
  if (group >= groups) return;
  unsigned *ctr = gc.ctr + group;
  unsigned gen = 0;
  V *base = reinterpret_cast<V *>(gc.state) + (size_t)group * 6 * H;
  Buf<T> A{base, base + H}, S0{base + 2 * H, base + 3 * H}, S1{base + 4 * H, base + 5 * H};
  long long *coef = gc.coef + (size_t)group * N;
  int *cert = gc.cert + 4 * group;
  unsigned *agg = gc.agg + (size_t)group * C;
  const TwC<T> *tw = reinterpret_cast<const TwC<T> *>(kp.tw);
  const int n = kp.n;
  const int tid = rank * 256 + threadIdx.x, nth = C * 256;

  for (int pair = group; pair < kp.batch; pair += groups) {
    for (int op = 0; op < 2; op++) {
      const uint8_t *dig = (op == 0 ? kp.a : kp.b) + (size_t)pair * n;
      constexpr int T1 = (N / 2) / PL.f[1];
      for (int t = tid; t < T1; t += nth) g_fwd_first<T, M>(t, dig, n, S0);
      group_sync(ctr, C, gen);
      // forward passes 2 .. nf-2 ping-pong S0 -> S1 -> S0 ...
      Buf<T> cur = S0, nxt = S1;
#define IVM_G_FWD(P_)                                                            \
      if constexpr ((P_) < PL.nf - 1) {                                           \
        constexpr int TP = (N / 2) / PL.f[(P_)];                                   \
        for (int t = tid; t < TP; t += nth) g_fwd_pass<T, M, (P_)>(t, cur, nxt, tw); \
        group_sync(ctr, C, gen);                                                  \
        Buf<T> tmp = cur; cur = nxt; nxt = tmp;                                   \
      }
      IVM_G_FWD(2) IVM_G_FWD(3) IVM_G_FWD(4)
#undef IVM_G_FWD
      constexpr int TL = (N / 2) / PL.f[PL.nf - 1];
      if (op == 0) {
        for (int t = tid; t < TL; t += nth) g_fwd_last_a<T, M>(t, cur, A, tw);
        group_sync(ctr, C, gen);
      } else {
        if (rank == 0 && threadIdx.x == 0) {
          cert[0] = 1;
          cert[1] = 0x7fffffff;
          reinterpret_cast<unsigned long long *>(cert + 2)[0] = 0ull;
        }
        for (int t = tid; t < TL; t += nth) g_fused<T, M>(t, cur, A, nxt, tw);
        group_sync(ctr, C, gen);
        Buf<T> tmp = cur; cur = nxt; nxt = tmp;
#define IVM_G_INV(P_)                                                            \
        if constexpr ((P_) < PL.ni - 1) {                                         \
          constexpr int TP = (N / 2) / PL.q[(P_)];                                 \
          for (int t = tid; t < TP; t += nth) g_inv_pass<T, M, (P_)>(t, cur, nxt, tw); \
          group_sync(ctr, C, gen);                                                \
          Buf<T> tmp2 = cur; cur = nxt; nxt = tmp2;                               \
        }
        IVM_G_INV(1) IVM_G_INV(2) IVM_G_INV(3) IVM_G_INV(4)
#undef IVM_G_INV
        double *dump = nullptr;
        if (kp.dump_slot) {
          const int s = kp.dump_slot[pair];
          if (s >= 0) dump = kp.intervals + (size_t)s * N * 4;
        }
        constexpr int TF = (N / 2) / PL.q[PL.ni - 1];
        for (int t = tid; t < TF; t += nth) g_inv_last<T, M>(t, cur, tw, n, coef, cert, dump);
        group_sync(ctr, C, gen);
        const bool certified = *(volatile int *)cert != 0;
        g_carry(coef, n, kp.prod + (size_t)pair * 2 * n, certified, rank, C, agg, ctr, gen);
        if (kp.coeffs) {
          int64_t *co = kp.coeffs + (size_t)pair * (2 * n - 1);
          for (int i = tid; i < 2 * n - 1; i += nth) co[i] = certified ? coef[i] : 0;
        }
        if (rank == 0 && threadIdx.x == 0) {
          kp.cert[pair] = certified ? 1 : 0;
          if (kp.max_radius)
            kp.max_radius[pair] = __longlong_as_double(*(volatile long long *)(cert + 2));
          if (kp.first_bad) kp.first_bad[pair] = certified ? -1 : *(volatile int *)(cert + 1);
        }
        group_sync(ctr, C, gen);
      }
    }
  }
}

}  // namespace v3
}  // namespace ivm
