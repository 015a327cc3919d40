// ivm_v3.cuh -- balanced odd-frequency ("twisted") schedule (included by ivm_kernels.cu).
//
// Transform: T(x)_k = sum_j x_j z^{j(2k+1)}, z = e^{2 pi i/(2m)}, i.e. the DFT of
// PAPER.md P:68 evaluated at the half-integer frequencies k + 1/2.  For real
// digits T_{m-1-k} = conj(T_k) with no self-conjugate bin, so exactly m/2 values
// carry the spectrum, and T(a) T(b) = T(a*b) because the product a*b has
// 2n-1 <= m-1 terms (the zero padding of P:206-208 makes the negacyclic
// wrap empty).  The coefficients come back as c_s = (1/m) sum_k P_k z^{-s(2k+1)}
// (P:97 with the same half-integer frequencies).
//
// Every pass is a radix-R decimation-in-time step: the inputs of a
// task are the sub-transforms of decimated subsequences, each multiplied by
// ONE twiddle, then an R-point DFT of DIT-form butterflies.  All tasks
// of a pass are identical (m/(2R) tasks, no boundary cases), so one CTA of m/32
// threads holds a whole half-spectrum in registers while a pass runs in place.
// Index rules are prototyped in tools/proto_v3.py.
#pragma once

namespace ivm {
namespace v3 {

// ---------------------------------------------------------------------------
// plans: forward radices f[0] = 2 (trivial: G_1 = the digits), inverse q[0] = f[nf-1]
// (fused with fwd(b)'s last pass); product(f) = m, product(q) * 2 = m.
// ---------------------------------------------------------------------------
struct Plan {
  int nf, f[6];
  int ni, q[6];
};

__host__ __device__ constexpr Plan plan(int m) {
  switch (m) {
    case 4: return Plan{2, {2, 8, 0, 0, 0, 0}, 1, {8, 0, 0, 0, 0, 0}};
    case 5: return Plan{2, {2, 16, 0, 0, 0, 0}, 1, {16, 0, 0, 0, 0, 0}};
    case 6: return Plan{3, {2, 2, 16, 0, 0, 0}, 2, {16, 2, 0, 0, 0, 0}};
    case 7: return Plan{3, {2, 4, 16, 0, 0, 0}, 2, {16, 4, 0, 0, 0, 0}};
    case 8: return Plan{3, {2, 8, 16, 0, 0, 0}, 2, {16, 8, 0, 0, 0, 0}};
    case 9: return Plan{3, {2, 16, 16, 0, 0, 0}, 2, {16, 16, 0, 0, 0, 0}};
    case 10: return Plan{4, {2, 2, 16, 16, 0, 0}, 3, {16, 16, 2, 0, 0, 0}};
    case 11: return Plan{4, {2, 4, 16, 16, 0, 0}, 3, {16, 16, 4, 0, 0, 0}};
    case 12: return Plan{4, {2, 8, 16, 16, 0, 0}, 3, {16, 16, 8, 0, 0, 0}};
    case 13: return Plan{4, {2, 16, 16, 16, 0, 0}, 3, {16, 16, 16, 0, 0, 0}};
    // global-memory (multi-CTA) path
    case 14: return Plan{5, {2, 2, 16, 16, 16, 0}, 4, {16, 16, 16, 2, 0, 0}};
    case 15: return Plan{5, {2, 4, 16, 16, 16, 0}, 4, {16, 16, 16, 4, 0, 0}};
    case 16: return Plan{5, {2, 8, 16, 16, 16, 0}, 4, {16, 16, 16, 8, 0, 0}};
    case 17: return Plan{5, {2, 16, 16, 16, 16, 0}, 4, {16, 16, 16, 16, 0, 0}};
    case 18: return Plan{6, {2, 2, 16, 16, 16, 16}, 5, {16, 16, 16, 16, 2, 0}};
    default: return Plan{0, {0, 0, 0, 0, 0, 0}, 0, {0, 0, 0, 0, 0, 0}};
  }
}

__host__ __device__ constexpr int cmax3(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int fL(const Plan &P, int p) { return p == 0 ? 1 : fL(P, p - 1) * P.f[p - 1]; }
__host__ __device__ constexpr int iL(const Plan &P, int p) { return p == 0 ? 1 : iL(P, p - 1) * P.q[p - 1]; }

// row stride with padding so that the lanes of a quarter warp (8 x 16 B) hit
// distinct 16-byte bank groups when the reading pass has S' < 8 columns per task
__host__ __device__ constexpr int rstride(int S, int Sread) {
  return Sread >= 8 ? S : S + (((Sread - S) % 8) + 8) % 8;
}

template <int M> struct G3 {
  static constexpr Plan P = plan(M);  // (host-side use; device code calls plan(M))
  static constexpr int N = 1 << M;
  static constexpr int THREADS = N / 32 < 32 ? 32 : N / 32;
  static constexpr int TASKS = N / 32;  // tasks x radix = N/2 per pass
  // forward state after pass p (p >= 1): rows L_p/2, cols S_p
  __host__ __device__ static constexpr int fS(int p) { return N / fL(plan(M), p); }
  __host__ __device__ static constexpr int fRS(int p) {  // read by forward pass p (radix f[p])
    return rstride(fS(p), p < plan(M).nf ? fS(p) / plan(M).f[p] : 1);
  }
  // inverse state after pass p: rows L_p, cols S_p/2 (S_p = N / L_p)
  __host__ __device__ static constexpr int iS(int p) { return N / iL(plan(M), p); }
  __host__ __device__ static constexpr int iRS(int p) { return rstride(iS(p) / 2, p < plan(M).ni ? iS(p) / plan(M).q[p] / 2 : 1); }
  __host__ __device__ static constexpr int cap() {
    int c = 0;
    for (int p = 2; p < plan(M).nf; p++) c = cmax3(c, (fL(plan(M), p) / 2) * fRS(p));
    for (int p = 1; p < plan(M).ni; p++) c = cmax3(c, iL(plan(M), p) * iRS(p));
    return c;
  }
  static constexpr int CAP = cap();
  // twiddle table segment offsets (entries of CI<T>)
  __host__ __device__ static constexpr int tw_fwd(int p) {  // p >= 1: [R-1][L/2]
    int o = 0;
    for (int k = 1; k < p; k++) o += (plan(M).f[k] - 1) * (fL(plan(M), k) / 2);
    return o;
  }
  __host__ __device__ static constexpr int tw_inv(int p) {  // p >= 1: [Q-1][L]
    int o = tw_fwd(plan(M).nf);
    for (int k = 1; k < p; k++) o += (plan(M).q[k] - 1) * iL(plan(M), k);
    return o;
  }
  __host__ __device__ static constexpr int tw_fin() { return tw_inv(plan(M).ni); }  // [Q_last][L_last]
  __host__ __device__ static constexpr int tw_total() { return tw_fin() + N / 2; }
};

// ---------------------------------------------------------------------------
// compact twiddles.  A first-quadrant enclosure [cl, ch] + i[sl, sh] is held as
// its lower endpoints (cl, sl): every upper endpoint is the next representable
// number and (checked by the planner for every table) shares the lower
// endpoint's high 32-bit word, so "choose lo or hi" is an integer add of 0/1 on
// the low word.  Exact entries (0, 1) are widened by that one ulp (sound).
// Runtime table entries w = i^k (c + i s) keep k in the sign bit of s.
// ---------------------------------------------------------------------------
template <typename T> struct TB;
template <> struct TB<double> {
  static __device__ __forceinline__ double sel(double lo, unsigned add) {
    return __hiloint2double(__double2hiint(lo), (int)((unsigned)__double2loint(lo) + add));
  }
  static __device__ __forceinline__ unsigned sgn(double x) { return (unsigned)__double2hiint(x) >> 31; }
  static __device__ __forceinline__ double neg(double x) {
    return __hiloint2double(__double2hiint(x) ^ (int)0x80000000, __double2loint(x));
  }
  static __device__ __forceinline__ double absb(double x) {
    return __hiloint2double(__double2hiint(x) & 0x7fffffff, __double2loint(x));
  }
};
template <> struct TB<float> {
  static __device__ __forceinline__ float sel(float lo, unsigned add) {
    return __int_as_float((int)((unsigned)__float_as_int(lo) + add));
  }
  static __device__ __forceinline__ unsigned sgn(float x) { return (unsigned)__float_as_int(x) >> 31; }
  static __device__ __forceinline__ float neg(float x) { return __int_as_float(__float_as_int(x) ^ (int)0x80000000); }
  static __device__ __forceinline__ float absb(float x) { return __int_as_float(__float_as_int(x) & 0x7fffffff); }
};

template <typename T> struct TwC { T c, s; };  // lower endpoints (+ flag in sign of s)

// w = c + i s (first quadrant, compact) times any interval d: 8 directed ops.
//   lo(w*y) = y.lo * (y.lo < 0 ? w.hi : w.lo),  hi(w*y) = y.hi * (y.hi < 0 ? w.lo : w.hi)
template <typename T>
__device__ __forceinline__ CI<T> q1mul(T c, T s, const CI<T> &d) {
  using B = TB<T>;
  const unsigned nxl = B::sgn(d.rl), nxh = B::sgn(d.rh), nyl = B::sgn(d.il), nyh = B::sgn(d.ih);
  CI<T> t;
  t.rl = DR<T>::fma_rd(-B::sel(s, 1u - nyh), d.ih, DR<T>::mul_rd(B::sel(c, nxl), d.rl));
  t.rh = DR<T>::fma_ru(-B::sel(s, nyl), d.il, DR<T>::mul_ru(B::sel(c, 1u - nxh), d.rh));
  t.il = DR<T>::fma_rd(B::sel(s, nxl), d.rl, DR<T>::mul_rd(B::sel(c, nyl), d.il));
  t.ih = DR<T>::fma_ru(B::sel(s, 1u - nxh), d.rh, DR<T>::mul_ru(B::sel(c, 1u - nyh), d.ih));
  return t;
}

// k ? i*t : t  (exact; i*t = (-t.im, t.re))
template <typename T>
__device__ __forceinline__ CI<T> rot_if(const CI<T> &t, unsigned k) {
  using B = TB<T>;
  const T nih = B::neg(t.ih), nil = B::neg(t.il);
  return CI<T>{k ? nih : t.rl, k ? nil : t.rh, k ? t.rl : t.il, k ? t.rh : t.ih};
}

// runtime table twiddle (upper half plane, compact + rotation flag) times d;
// CONJ: conj(w) * d = conj(w * conj(d))
template <typename T, bool CONJ>
__device__ __forceinline__ CI<T> rtmul(const TwC<T> &w, const CI<T> &d) {
  using B = TB<T>;
  const unsigned k = B::sgn(w.s);
  const T s = B::absb(w.s);
  if (CONJ) return cconj(rot_if(q1mul(w.c, s, cconj(d)), k));
  return rot_if(q1mul(w.c, s, d), k);
}

template <typename T>
__device__ __forceinline__ TwC<T> ldg_twc(const TwC<T> *__restrict__ tw, int i) {
  if constexpr (sizeof(T) == 8) {
    const double2 v = __ldg(reinterpret_cast<const double2 *>(tw) + i);
    return TwC<T>{(T)v.x, (T)v.y};
  } else {
    const float2 v = __ldg(reinterpret_cast<const float2 *>(tw) + i);
    return TwC<T>{(T)v.x, (T)v.y};
  }
}

// ---------------------------------------------------------------------------
// register DFT, complex interval inputs, DIT radix 2 with first-quadrant
// constant twiddles (w_64^j) and compile-time rotations / conjugations
// ---------------------------------------------------------------------------
__constant__ TwC<double> c_w64_f64[17];  // w_64^j, j = 0..16 (first quadrant, compact)
__constant__ TwC<float> c_w64_f32[17];

template <typename T> __device__ __forceinline__ const TwC<T> &cw64(int j);
template <> __device__ __forceinline__ const TwC<double> &cw64<double>(int j) { return c_w64_f64[j]; }
template <> __device__ __forceinline__ const TwC<float> &cw64<float>(int j) { return c_w64_f32[j]; }

// t = w_M^j * o (INV: conj(w_M^j) * o), M <= 64 a power of two, 0 <= j < M/2
template <typename T, bool INV>
__device__ __forceinline__ CI<T> ctw(const CI<T> &o, int j, int M) {
  if (j == 0) return o;
  if (4 * j == M) return INV ? mul_mi(o) : mul_i(o);
  if (4 * j < M) {  // first quadrant
    const TwC<T> w = cw64<T>(j * (64 / M));
    return INV ? cconj(q1mul(w.c, w.s, cconj(o))) : q1mul(w.c, w.s, o);
  }
  // second quadrant: w = i * w', w' = w_M^{j - M/4}
  const TwC<T> w = cw64<T>((j - M / 4) * (64 / M));
  return INV ? mul_mi(cconj(q1mul(w.c, w.s, cconj(o)))) : mul_i(q1mul(w.c, w.s, o));
}

__host__ __device__ constexpr int brev3(int i, int bits) {  // non-recursive: folds after unrolling
  int r = 0;
  for (int b = 0; b < bits; b++) r |= ((i >> b) & 1) << (bits - 1 - b);
  return r;
}
__host__ __device__ constexpr int ilog2_3(int x) { return x <= 1 ? 0 : 1 + ilog2_3(x / 2); }

template <typename T, int R, bool INV>
__device__ __forceinline__ void cdft(CI<T> (&v)[R]) {
  constexpr int B = ilog2_3(R);
  CI<T> a[R];
#pragma unroll
  for (int i = 0; i < R; i++) a[i] = v[brev3(i, B)];
#pragma unroll
  for (int h = 1; h < R; h *= 2) {
#pragma unroll
    for (int blk = 0; blk < R; blk += 2 * h) {
#pragma unroll
      for (int j = 0; j < h; j++) {
        CI<T> t = ctw<T, INV>(a[blk + j + h], j, 2 * h);
        bfly(a[blk + j], a[blk + j + h], t);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < R; i++) v[i] = a[i];
}

// ---------------------------------------------------------------------------
// state access
// ---------------------------------------------------------------------------
template <typename T> struct V2t;
template <> struct V2t<double> { using t = double2; };
template <> struct V2t<float> { using t = float2; };

template <typename T> struct Buf {
  typename V2t<T>::t *re, *im;
  __device__ __forceinline__ CI<T> ld(int i) const {
    auto r = re[i], m = im[i];
    return CI<T>{r.x, r.y, m.x, m.y};
  }
  __device__ __forceinline__ void st(int i, const CI<T> &z) const {
    re[i] = typename V2t<T>::t{z.rl, z.rh};
    im[i] = typename V2t<T>::t{z.il, z.ih};
  }
};


// ---------------------------------------------------------------------------
// forward passes
// ---------------------------------------------------------------------------
// pass 1: G_1[0][v] = x[v] (the trivial radix-2 pass 0), read from HBM;
// G_2[2r][v] = sum_q w_R^{qr} (w_{4R}^q x[v + S'q]), stored with the mirror.
template <typename T, int M>
__device__ __forceinline__ void fwd_first(const uint8_t *__restrict__ dig, int n, Buf<T> st,
                                          const TwC<T> *__restrict__ tw) {
  using Gm = G3<M>;
  constexpr int N = Gm::N, R = Gm::P.f[1], L = 2, S = N / 2, Sp = S / R, G = 16 / R;
  constexpr int RSo = Gm::fRS(2);
  CI<T> v[G][R];
#pragma unroll
  for (int g = 0; g < G; g++) {
    const int nu = threadIdx.x + g * Gm::THREADS;
    if (Gm::THREADS * G == Sp || nu < Sp) {
#pragma unroll
      for (int q = 0; q < R; q++) {
        const int idx = nu + Sp * q;
        const T x = idx < n ? T(dig[idx]) : T(0);
        if (q == 0) {
          v[g][q] = punctual(x);
        } else {
          // x >= 0 and w_{4R}^q in the first quadrant: lo * x rounded down, hi * x up
          const TwC<T> w = cw64<T>(q * (16 / R));
          v[g][q] = CI<T>{DR<T>::mul_rd(w.c, x), DR<T>::mul_ru(TB<T>::sel(w.c, 1u), x),
                          DR<T>::mul_rd(w.s, x), DR<T>::mul_ru(TB<T>::sel(w.s, 1u), x)};
        }
      }
      cdft<T, R, false>(v[g]);
#pragma unroll
      for (int r = 0; r < R; r++) {
        if (r < R / 2) st.st((L * r) * RSo + nu, v[g][r]);
        else st.st((L * R - 1 - L * r) * RSo + nu, cconj(v[g][r]));
      }
    }
  }
}

// forward pass p >= 2 (in place when DST aliases the state)
template <typename T, int M, int p>
__device__ __forceinline__ void fwd_load_compute(Buf<T> st, const TwC<T> *__restrict__ tw,
                                                 CI<T> (&v)[16 / G3<M>::P.f[p]][G3<M>::P.f[p]],
                                                 int (&k0s)[16 / G3<M>::P.f[p]],
                                                 int (&nus)[16 / G3<M>::P.f[p]]) {
  using Gm = G3<M>;
  constexpr int N = Gm::N, R = Gm::P.f[p], L = fL(Gm::P, p), S = N / L, Sp = S / R, G = 16 / R;
  constexpr int RSi = Gm::fRS(p);
  constexpr int TW = Gm::tw_fwd(p);
  constexpr int COUNT = (L / 2) * Sp;
#pragma unroll
  for (int g = 0; g < G; g++) {
    const int t = threadIdx.x + g * Gm::THREADS;
    const int k0 = t / Sp, nu = t % Sp;
    k0s[g] = (Gm::THREADS * G == COUNT || t < COUNT) ? k0 : -1;
    nus[g] = nu;
    if (!(Gm::THREADS * G == COUNT || t < COUNT)) continue;
#pragma unroll
    for (int q = 0; q < R; q++) {
      CI<T> z = st.ld(k0 * RSi + nu + Sp * q);
      if (q > 0) z = rtmul<T, false>(ldg_twc(tw, TW + (q - 1) * (L / 2) + k0), z);
      v[g][q] = z;
    }
    cdft<T, R, false>(v[g]);
  }
}

template <typename T, int M, int p>
__device__ __forceinline__ void fwd_mid(Buf<T> st, const TwC<T> *__restrict__ tw) {
  using Gm = G3<M>;
  constexpr int R = Gm::P.f[p], L = fL(Gm::P, p), G = 16 / R;
  constexpr int RSo = Gm::fRS(p + 1);
  CI<T> v[G][R];
  int k0s[G], nus[G];
  fwd_load_compute<T, M, p>(st, tw, v, k0s, nus);
  __syncthreads();
#pragma unroll
  for (int g = 0; g < G; g++) {
    if (k0s[g] < 0) continue;
#pragma unroll
    for (int r = 0; r < R; r++) {
      if (r < R / 2) st.st((k0s[g] + L * r) * RSo + nus[g], v[g][r]);
      else st.st((L * R - 1 - k0s[g] - L * r) * RSo + nus[g], cconj(v[g][r]));
    }
  }
}

// last forward pass of a: spectrum class k0 (all R values) -> A store [r][k0]
template <typename T, int M>
__device__ __forceinline__ void fwd_last_a(Buf<T> st, Buf<T> A, const TwC<T> *__restrict__ tw) {
  using Gm = G3<M>;
  constexpr int p = Gm::P.nf - 1, R = Gm::P.f[p], L = fL(Gm::P, p), G = 16 / R;
  CI<T> v[G][R];
  int k0s[G], nus[G];
  fwd_load_compute<T, M, p>(st, tw, v, k0s, nus);
#pragma unroll
  for (int g = 0; g < G; g++) {
    if (k0s[g] < 0) continue;
#pragma unroll
    for (int r = 0; r < R; r++) A.st(r * (L / 2) + k0s[g], v[g][r]);
  }
}

// inverse pass: loads of E_p[k0][v + S'q] with the mirror (q >= Q/2)
template <typename T, int M, int p>
__device__ __forceinline__ void inv_load_compute(Buf<T> st, const TwC<T> *__restrict__ tw,
                                                 CI<T> (&v)[16 / G3<M>::P.q[p]][G3<M>::P.q[p]],
                                                 int (&k0s)[16 / G3<M>::P.q[p]],
                                                 int (&nus)[16 / G3<M>::P.q[p]]) {
  using Gm = G3<M>;
  constexpr int N = Gm::N, Q = Gm::P.q[p], L = iL(Gm::P, p), S = N / L, Sp = S / Q, G = 16 / Q;
  constexpr int H = Sp / 2, RSi = Gm::iRS(p);
  constexpr int TW = Gm::tw_inv(p);
  constexpr int COUNT = L * H;
#pragma unroll
  for (int g = 0; g < G; g++) {
    const int t = threadIdx.x + g * Gm::THREADS;
    const int k0 = t / H, nu = t % H;
    k0s[g] = (Gm::THREADS * G == COUNT || t < COUNT) ? k0 : -1;
    nus[g] = nu;
    if (!(Gm::THREADS * G == COUNT || t < COUNT)) continue;
#pragma unroll
    for (int q = 0; q < Q; q++) {
      CI<T> z;
      if (2 * q < Q) z = st.ld(k0 * RSi + nu + Sp * q);
      else z = cconj(st.ld(k0 * RSi + (S - 1 - nu - Sp * q)));
      if (q > 0) {
        const TwC<T> w = ldg_twc(tw, TW + (q - 1) * L + k0);
        z = (2 * q < Q) ? rtmul<T, true>(w, z) : rtmul<T, false>(w, z);
      }
      v[g][q] = z;
    }
    cdft<T, Q, true>(v[g]);
  }
}

template <typename T, int M, int p>
__device__ __forceinline__ void inv_mid(Buf<T> st, const TwC<T> *__restrict__ tw) {
  using Gm = G3<M>;
  constexpr int N = Gm::N, Q = Gm::P.q[p], L = iL(Gm::P, p), G = 16 / Q;
  constexpr int RSo = Gm::iRS(p + 1);
  CI<T> v[G][Q];
  int k0s[G], nus[G];
  inv_load_compute<T, M, p>(st, tw, v, k0s, nus);
  __syncthreads();
#pragma unroll
  for (int g = 0; g < G; g++) {
    if (k0s[g] < 0) continue;
#pragma unroll
    for (int r = 0; r < Q; r++) st.st((k0s[g] + L * r) * RSo + nus[g], v[g][r]);
  }
  (void)N;
}

// ---------------------------------------------------------------------------
// round-and-certify of the real coefficients c_k, c_{k + m/2}
// ---------------------------------------------------------------------------
struct Cert3 {
  int ok;
  int first_bad;
  unsigned long long maxrad;
};

struct CertAcc {  // per-thread; reduced once per multiplication
  int ok = 1;
  int bad = 0x7fffffff;
  double rad = 0.0;
};

template <typename T>
__device__ __forceinline__ void certify_real(T lo, T hi, int i, int n, int32_t *coef, CertAcc &acc,
                                             double *dump) {
  if (dump) reinterpret_cast<double4 *>(dump)[i] = make_double4((double)lo, (double)hi, 0.0, 0.0);
  if (i >= 2 * n - 1) return;
  const double l = (double)lo, h = (double)hi;
  const double cl = ceil(l);
  const bool ok = cl == floor(h);
  const double rad = __dmul_ru(__dadd_ru(h, -l), 0.5);
  acc.rad = (rad <= acc.rad) ? acc.rad : rad;  // NaN propagates (comparison false)
  coef[i] = ok ? (int32_t)cl : 0;
  if (!ok) {
    acc.ok = 0;
    acc.bad = min(acc.bad, i);
  }
}

__device__ __forceinline__ void cert_flush(const CertAcc &acc, Cert3 &cs) {
  const int ok = __reduce_and_sync(0xffffffffu, (unsigned)acc.ok);
  const int bad = (int)__reduce_min_sync(0xffffffffu, (unsigned)acc.bad);
  double rad = acc.rad;
  for (int o = 16; o; o >>= 1) {
    const double r2 = __shfl_xor_sync(0xffffffffu, rad, o);
    rad = (r2 <= rad) ? rad : r2;
  }
  if ((threadIdx.x & 31) == 0) {
    if (!ok) {
      cs.ok = 0;
      atomicMin(&cs.first_bad, bad);
    }
    unsigned long long rb = (rad == rad) ? (unsigned long long)__double_as_longlong(rad) : 0x7ff0000000000000ull;
    atomicMax(&cs.maxrad, rb);
  }
}

// final output of the last inverse pass: v = z^{-k} O, c_k = 2 Re v / m,
// c_{k+m/2} = 2 Im v / m  (the folded radix-2 step)
template <typename T, int M>
__device__ __forceinline__ void emit_coeffs(const CI<T> &o, int k, const TwC<T> *__restrict__ tw, int twi,
                                            int n, int32_t *coef, CertAcc &acc, double *dump) {
  constexpr int N = 1 << M;
  const CI<T> v = rtmul<T, true>(ldg_twc(tw, twi), o);  // z^{-k} = conj(z^k)
  const T s = T(2) / T(N);  // exact power of two
  certify_real(DR<T>::mul_rd(v.rl, s), DR<T>::mul_ru(v.rh, s), k, n, coef, acc, dump);
  certify_real(DR<T>::mul_rd(v.il, s), DR<T>::mul_ru(v.ih, s), k + N / 2, n, coef, acc, dump);
}

template <typename T, int M>
__device__ __forceinline__ void inv_last(Buf<T> st, const TwC<T> *__restrict__ tw, int n, int32_t *coef,
                                         CertAcc &acc, double *dump) {
  using Gm = G3<M>;
  constexpr int p = Gm::P.ni - 1, Q = Gm::P.q[p], L = iL(Gm::P, p), G = 16 / Q;
  constexpr int TWF = Gm::tw_fin();
  CI<T> v[G][Q];
  int k0s[G], nus[G];
  inv_load_compute<T, M, p>(st, tw, v, k0s, nus);
#pragma unroll
  for (int g = 0; g < G; g++) {
    if (k0s[g] < 0) continue;
#pragma unroll
    for (int r = 0; r < Q; r++) {
      const int k = k0s[g] + L * r;
      emit_coeffs<T, M>(v[g][r], k, tw, TWF + k, n, coef, acc, dump);
    }
  }
}

template <typename T, int M, int p>
__device__ __forceinline__ void run_fwd(Buf<T> st, const TwC<T> *tw) {
  if constexpr (p < G3<M>::P.nf - 1) {
    fwd_mid<T, M, p>(st, tw);
    __syncthreads();
    run_fwd<T, M, p + 1>(st, tw);
  }
}

template <typename T, int M, int p>
__device__ __forceinline__ void run_inv(Buf<T> st, const TwC<T> *tw) {
  if constexpr (p < G3<M>::P.ni - 1) {
    inv_mid<T, M, p>(st, tw);
    __syncthreads();
    run_inv<T, M, p + 1>(st, tw);
  }
}

// ---------------------------------------------------------------------------
// runtime-parameterised radix-16 pass bodies: ONE code copy serves every
// forward pass p >= 2 (and the last / fused one) and every inverse pass, so the
// straight-line kernel stays small enough for the instruction cache.
// ---------------------------------------------------------------------------
struct PassRT {
  int lgSp, L, RSi, RSo, tw;
};

__host__ __device__ constexpr int ilog2r(int x) { return x <= 1 ? 0 : 1 + ilog2r(x / 2); }

template <int M> struct RT3 {
  static constexpr int nf = plan(M).nf, ni = plan(M).ni;
  static constexpr int NFWD = nf - 2;  // forward passes 2 .. nf-1 (all radix 16)
  static constexpr bool LAST16 = plan(M).q[ni - 1] == 16;
  static constexpr int NINV = LAST16 ? ni - 1 : ni - 2;  // inverse passes 1 .. via the shared body
  __host__ __device__ static constexpr PassRT fwd(int i) {
    return PassRT{ilog2r((1 << M) / fL(plan(M), i + 2) / 16), fL(plan(M), i + 2), G3<M>::fRS(i + 2),
                  (i + 3 < nf) ? G3<M>::fRS(i + 3) : G3<M>::iRS(1), G3<M>::tw_fwd(i + 2)};
  }
  __host__ __device__ static constexpr PassRT inv(int i) {
    return PassRT{ilog2r((1 << M) / iL(plan(M), i + 1) / 16), iL(plan(M), i + 1), G3<M>::iRS(i + 1),
                  (i + 2 < ni) ? G3<M>::iRS(i + 2) : 0, G3<M>::tw_inv(i + 1)};
  }
};

template <int M>
__device__ __forceinline__ PassRT pick_fwd(int i) {
  static_assert(RT3<M>::NFWD >= 1 && RT3<M>::NFWD <= 3, "forward passes");
  constexpr PassRT p0 = RT3<M>::fwd(0);
  constexpr PassRT p1 = RT3<M>::fwd(RT3<M>::NFWD > 1 ? 1 : 0);
  constexpr PassRT p2 = RT3<M>::fwd(RT3<M>::NFWD > 2 ? 2 : 0);
  return i == 0 ? p0 : (i == 1 ? p1 : p2);
}
template <int M>
__device__ __forceinline__ PassRT pick_inv(int i) {
  static_assert(RT3<M>::NINV >= 1 && RT3<M>::NINV <= 3, "inverse passes");
  constexpr PassRT p0 = RT3<M>::inv(0);
  constexpr PassRT p1 = RT3<M>::inv(RT3<M>::NINV > 1 ? 1 : 0);
  constexpr PassRT p2 = RT3<M>::inv(RT3<M>::NINV > 2 ? 2 : 0);
  return i == 0 ? p0 : (i == 1 ? p1 : p2);
}

// L1 prefetch of the twiddles a thread will read in a later pass
template <typename T>
__device__ __forceinline__ void prefetch_tw(const TwC<T> *tw, const PassRT &pp, bool inverse) {
  const int t = threadIdx.x;
  const int k0 = inverse ? (t >> (pp.lgSp - 1)) : (t >> pp.lgSp);
  const int stride = inverse ? pp.L : (pp.L >> 1);
  const TwC<T> *b = tw + pp.tw + k0;
#pragma unroll
  for (int q = 1; q < 16; q++) asm volatile("prefetch.global.L1 [%0];" ::"l"(b + (q - 1) * stride));
}

// forward: F_p[k0][nu + Sp q] * w_{32L}^{q(2k0+1)} -> 16-point DFT
template <typename T>
__device__ __forceinline__ void fwd16(Buf<T> st, const TwC<T> *__restrict__ tw, const PassRT &pp,
                                      CI<T> (&v)[16], int &k0, int &nu) {
  const int t = threadIdx.x, Sp = 1 << pp.lgSp;
  k0 = t >> pp.lgSp;
  nu = t & (Sp - 1);
  const int base = k0 * pp.RSi + nu, tb = pp.tw + k0, tstride = pp.L >> 1;
#pragma unroll
  for (int q = 0; q < 16; q++) {
    CI<T> z = st.ld(base + Sp * q);
    if (q > 0) z = rtmul<T, false>(ldg_twc(tw, tb + (q - 1) * tstride), z);
    v[q] = z;
  }
  cdft<T, 16, false>(v);
}

// inverse: E_p[k0][mu] (mirror for q >= 8) * twiddle -> 16-point inverse DFT
template <typename T>
__device__ __forceinline__ void inv16(Buf<T> st, const TwC<T> *__restrict__ tw, const PassRT &pp,
                                      CI<T> (&v)[16], int &k0, int &nu) {
  const int t = threadIdx.x, Sp = 1 << pp.lgSp, lgH = pp.lgSp - 1, S = 16 * Sp;
  k0 = t >> lgH;
  nu = t & ((Sp >> 1) - 1);
  const int base = k0 * pp.RSi, tb = pp.tw + k0;
#pragma unroll
  for (int q = 0; q < 16; q++) {
    CI<T> z;
    if (q < 8) z = st.ld(base + nu + Sp * q);
    else z = cconj(st.ld(base + (S - 1 - nu - Sp * q)));
    if (q > 0) {
      const TwC<T> w = ldg_twc(tw, tb + (q - 1) * pp.L);
      z = (q < 8) ? rtmul<T, true>(w, z) : rtmul<T, false>(w, z);
    }
    v[q] = z;
  }
  cdft<T, 16, true>(v);
}

template <typename T, int M> struct Cfg3 {
  using Gm = G3<M>;
  static constexpr int N = Gm::N, THREADS = Gm::THREADS, CAP = Gm::CAP;
  static constexpr size_t E = sizeof(typename V2t<T>::t);
  static constexpr size_t STATE_BYTES = 2 * E * (size_t)CAP;
  static constexpr size_t COEF_BYTES = 4 * (size_t)N;
  static constexpr size_t A_BYTES = 2 * E * (size_t)(N / 2);  // [R][L/2] x (re, im)
  static constexpr size_t SMEM = STATE_BYTES + COEF_BYTES;
};

template <typename T, int M>
__global__ void __launch_bounds__(Cfg3<T, M>::THREADS, 1) ivm_v3_kernel(KParams kp) {
  using C = Cfg3<T, M>;
  using Gm = G3<M>;
  using V = typename V2t<T>::t;
  constexpr int N = C::N;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Cert3 cs;
  Buf<T> st{reinterpret_cast<V *>(smem), reinterpret_cast<V *>(smem) + C::CAP};
  int32_t *coef = reinterpret_cast<int32_t *>(smem + C::STATE_BYTES);
  Buf<T> A{reinterpret_cast<V *>(kp.ascratch) + (size_t)blockIdx.x * N, nullptr};
  A.im = A.re + N / 2;
  const TwC<T> *tw = reinterpret_cast<const TwC<T> *>(kp.tw);
  const int n = kp.n;

  constexpr int NFWD = RT3<M>::NFWD, NINV = RT3<M>::NINV;
  constexpr bool LAST16 = RT3<M>::LAST16;
  constexpr int RSI1 = Gm::iRS(1), TWF = Gm::tw_fin();

  for (int pair = blockIdx.x; pair < kp.batch; pair += gridDim.x) {
    double *dump = nullptr;
    if (kp.dump_slot) {
      const int s = kp.dump_slot[pair];
      if (s >= 0) dump = kp.intervals + (size_t)s * N * 4;
    }
#pragma unroll 1
    for (int op = 0; op < 2; op++) {
      fwd_first<T, M>((op == 0 ? kp.a : kp.b) + (size_t)pair * n, n, st, tw);
      if (op == 1 && threadIdx.x == 0) {
        cs.ok = 1;
        cs.first_bad = 0x7fffffff;
        cs.maxrad = 0ull;
      }
      __syncthreads();
#pragma unroll 1
      for (int i = 0; i < NFWD; i++) {
        const PassRT pp = pick_fwd<M>(i);
        CI<T> v[16];
        int k0, nu;
        if (i + 1 < NFWD) prefetch_tw<T>(tw, pick_fwd<M>(i + 1), false);
        else if (op == 1) prefetch_tw<T>(tw, pick_inv<M>(0), true);
        fwd16<T>(st, tw, pp, v, k0, nu);
        if (i < NFWD - 1) {  // mid pass: store both halves (mirror conjugated)
          __syncthreads();
#pragma unroll
          for (int r = 0; r < 16; r++) {
            if (r < 8) st.st((k0 + pp.L * r) * pp.RSo + nu, v[r]);
            else st.st((16 * pp.L - 1 - k0 - pp.L * r) * pp.RSo + nu, cconj(v[r]));
          }
        } else if (op == 0) {  // last pass of a: spectrum class k0 -> A
#pragma unroll
          for (int r = 0; r < 16; r++) A.st(r * (pp.L >> 1) + k0, v[r]);
        } else {  // last pass of b + pointwise + inverse pass 0
#pragma unroll
          for (int r = 0; r < 16; r++) v[r] = cmul(A.ld(r * (pp.L >> 1) + k0), v[r]);
          cdft<T, 16, true>(v);
          __syncthreads();
#pragma unroll
          for (int r = 0; r < 16; r++) st.st(r * RSI1 + k0, v[r]);
        }
        __syncthreads();
      }
    }
    CertAcc acc;
#pragma unroll 1
    for (int i = 0; i < NINV; i++) {
      const PassRT pp = pick_inv<M>(i);
      CI<T> v[16];
      int k0, nu;
      if (i + 1 < NINV) prefetch_tw<T>(tw, pick_inv<M>(i + 1), true);
      inv16<T>(st, tw, pp, v, k0, nu);
      if (!LAST16 || i < NINV - 1) {
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 16; r++) st.st((k0 + pp.L * r) * pp.RSo + nu, v[r]);
      } else {
#pragma unroll
        for (int r = 0; r < 16; r++) {
          const int k = k0 + pp.L * r;
          emit_coeffs<T, M>(v[r], k, tw, TWF + k, n, coef, acc, dump);
        }
      }
      __syncthreads();
    }
    if constexpr (!LAST16) inv_last<T, M>(st, tw, n, coef, acc, dump);
    cert_flush(acc, cs);
    __syncthreads();
    const bool certified = cs.ok != 0;
    carry_store(coef, n, kp.prod + (size_t)pair * 2 * n, certified, reinterpret_cast<uint16_t *>(smem));
    if (kp.coeffs) {
      int64_t *co = kp.coeffs + (size_t)pair * (2 * n - 1);
      for (int i = threadIdx.x; i < 2 * n - 1; i += blockDim.x) co[i] = certified ? coef[i] : 0;
    }
    if (threadIdx.x == 0) {
      kp.cert[pair] = certified ? 1 : 0;
      if (kp.max_radius) kp.max_radius[pair] = __longlong_as_double((long long)cs.maxrad);
      if (kp.first_bad) kp.first_bad[pair] = certified ? -1 : cs.first_bad;
    }
    __syncthreads();
  }
}

}  // namespace v3
}  // namespace ivm
