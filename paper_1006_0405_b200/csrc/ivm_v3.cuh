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
#include "ivm_phase.cuh"

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

// plans of the one-CTA kernel by radix (R = 16: plan(m); R = 8: more passes,
// half the registers per task, twice the warps per SM)
__host__ __device__ constexpr Plan plan_cta(int m, int R) {
  if (R != 8) return plan(m);
  switch (m) {
    // warp-per-multiplication kernel (ivm_v6.cuh)
    case 6: return Plan{3, {2, 4, 8, 0, 0, 0}, 2, {8, 4, 0, 0, 0, 0}};
    case 7: return Plan{3, {2, 8, 8, 0, 0, 0}, 2, {8, 8, 0, 0, 0, 0}};
    case 8: return Plan{4, {2, 2, 8, 8, 0, 0}, 3, {8, 8, 2, 0, 0, 0}};
    case 9: return Plan{4, {2, 4, 8, 8, 0, 0}, 3, {8, 8, 4, 0, 0, 0}};
    // one-CTA kernel
    case 10: return Plan{4, {2, 8, 8, 8, 0, 0}, 3, {8, 8, 8, 0, 0, 0}};
    case 11: return Plan{5, {2, 2, 8, 8, 8, 0}, 4, {8, 8, 8, 2, 0, 0}};
    case 12: return Plan{5, {2, 4, 8, 8, 8, 0}, 4, {8, 8, 8, 4, 0, 0}};
    case 13: return Plan{5, {2, 8, 8, 8, 8, 0}, 4, {8, 8, 8, 8, 0, 0}};
    default: return plan(m);
  }
}

__host__ __device__ constexpr int cmax3(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int fL(const Plan &P, int p) { return p == 0 ? 1 : fL(P, p - 1) * P.f[p - 1]; }
__host__ __device__ constexpr int iL(const Plan &P, int p) { return p == 0 ? 1 : iL(P, p - 1) * P.q[p - 1]; }

// row stride with padding so that the lanes of a quarter warp (8 x 16 B) hit
// distinct 16-byte bank groups when the reading pass has S' < 8 columns per task
__host__ __device__ constexpr int rstride(int S, int Sread) { return S; }
// XOR swizzle of the column within groups of 8 (no padding): element (row, col)
// lives at row * S + (col ^ (row & SW)); used when the reading pass takes fewer
// than 8 consecutive columns per task, so that a quarter warp's 16-B accesses
// spread over distinct bank groups
__host__ __device__ constexpr int swzmask(int S, int Sread) { return Sread >= 8 ? 0 : (S >= 8 ? 7 : S - 1); }
__host__ __device__ __forceinline__ int sidx(int row, int col, int RS, int SW) { return row * RS + (col ^ (row & SW)); }

template <int M, int R = 16> struct G3 {
  static constexpr Plan P = plan_cta(M, R);  // (host-side use; device code calls plan_cta(M, R))
  static constexpr int N = 1 << M;
  static constexpr int THREADS = N / (2 * R) < 32 ? 32 : N / (2 * R);
  static constexpr int TASKS = N / (2 * R);  // tasks x radix = N/2 per pass
  // forward state after pass p (p >= 1): rows L_p/2, cols S_p
  __host__ __device__ static constexpr int fS(int p) { return N / fL(plan_cta(M, R), p); }
  __host__ __device__ static constexpr int fRS(int p) {  // read by forward pass p (radix f[p])
    return rstride(fS(p), p < plan_cta(M, R).nf ? fS(p) / plan_cta(M, R).f[p] : 1);
  }
  __host__ __device__ static constexpr int fSW(int p) {
    return swzmask(fS(p), p < plan_cta(M, R).nf ? fS(p) / plan_cta(M, R).f[p] : 1);
  }
  // inverse state after pass p: rows L_p, cols S_p/2 (S_p = N / L_p)
  __host__ __device__ static constexpr int iS(int p) { return N / iL(plan_cta(M, R), p); }
  __host__ __device__ static constexpr int iRS(int p) { return rstride(iS(p) / 2, p < plan_cta(M, R).ni ? iS(p) / plan_cta(M, R).q[p] / 2 : 1); }
  __host__ __device__ static constexpr int iSW(int p) { return swzmask(iS(p) / 2, p < plan_cta(M, R).ni ? iS(p) / plan_cta(M, R).q[p] / 2 : 1); }
  __host__ __device__ static constexpr int cap() {
    int c = 0;
    for (int p = 2; p < plan_cta(M, R).nf; p++) c = cmax3(c, (fL(plan_cta(M, R), p) / 2) * fRS(p));
    for (int p = 1; p < plan_cta(M, R).ni; p++) c = cmax3(c, iL(plan_cta(M, R), p) * iRS(p));
    return c;
  }
  static constexpr int CAP = cap();
  // twiddle table segment offsets (compact entries); every segment starts at an
  // even entry so that bulk copies of segments are 16-byte aligned in fp32 too
  __host__ __device__ static constexpr int even(int x) { return (x + 1) & ~1; }
  __host__ __device__ static constexpr int tw_fwd(int p) {  // p >= 1: [R-1][L/2]
    int o = 0;
    for (int k = 1; k < p; k++) o += even((plan_cta(M, R).f[k] - 1) * (fL(plan_cta(M, R), k) / 2));
    return o;
  }
  __host__ __device__ static constexpr int tw_inv(int p) {  // p >= 1: [Q-1][L]
    int o = tw_fwd(plan_cta(M, R).nf);
    for (int k = 1; k < p; k++) o += even((plan_cta(M, R).q[k] - 1) * iL(plan_cta(M, R), k));
    return o;
  }
  __host__ __device__ static constexpr int tw_fin() { return tw_inv(plan_cta(M, R).ni); }  // [Q_last][L_last]
  // last inverse pass of radix 16 with the final twist z^{-k0} folded into its
  // input twiddles: [16][L_last] (q = 0 included)
  static constexpr bool LAST16 = plan_cta(M, R).q[plan_cta(M, R).ni - 1] == R;  // last inverse radix = R
  __host__ __device__ static constexpr int tw_l16() { return tw_fin() + N / 2; }
  __host__ __device__ static constexpr int LASTL() { return iL(plan_cta(M, R), plan_cta(M, R).ni - 1); }
  __host__ __device__ static constexpr int tw_total() { return tw_l16() + (LAST16 ? R * LASTL() : 0); }
  // shared-memory twiddle buffer: the forward last pass table or the folded one
  __host__ __device__ static constexpr int FLAST_ENT() { return (R - 1) * (fL(plan_cta(M, R), plan_cta(M, R).nf - 1) / 2); }
  __host__ __device__ static constexpr int TWB_ENT() {
    return cmax3(FLAST_ENT(), LAST16 ? R * LASTL() : 0);
  }
  // resident small tables (shared memory, loaded once per CTA): the forward
  // mid passes 2 .. nf-2 and the inverse mid passes 1 .. ni-2
  __host__ __device__ static constexpr int SMF_BEGIN() { return tw_fwd(2); }
  __host__ __device__ static constexpr int SMF_ENT() { return tw_fwd(plan_cta(M, R).nf - 1) - tw_fwd(2); }
  __host__ __device__ static constexpr int SMI_BEGIN() { return tw_inv(1); }
  __host__ __device__ static constexpr int SMI_ENT() { return tw_inv(plan_cta(M, R).ni - 1) - tw_inv(1); }
  __host__ __device__ static constexpr int SM_ENT() { return TWB_ENT() + SMF_ENT() + SMI_ENT(); }
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

// w * conj(d) for a compact first-quadrant w = c + i s, without materialising
// conj(d): q1mul's formulas with d.il -> -d.ih, d.ih -> -d.il (the sign bits
// flip, the negations become free FMA operand modifiers)
template <typename T>
__device__ __forceinline__ CI<T> q1mul_cd(T c, T s, const CI<T> &d) {
  using B = TB<T>;
  const unsigned nxl = B::sgn(d.rl), nxh = B::sgn(d.rh), nyl = B::sgn(d.il), nyh = B::sgn(d.ih);
  CI<T> t;
  t.rl = DR<T>::fma_rd(B::sel(s, nyl), d.il, DR<T>::mul_rd(B::sel(c, nxl), d.rl));
  t.rh = DR<T>::fma_ru(B::sel(s, 1u - nyh), d.ih, DR<T>::mul_ru(B::sel(c, 1u - nxh), d.rh));
  t.il = DR<T>::fma_rd(B::sel(s, nxl), d.rl, DR<T>::mul_rd(B::sel(c, 1u - nyh), -d.ih));
  t.ih = DR<T>::fma_ru(B::sel(s, 1u - nxh), d.rh, DR<T>::mul_ru(B::sel(c, nyl), -d.il));
  return t;
}

// w = c (1 + i) (c == s, i.e. w_8): the c- and s-selects coincide (4 instead of 8)
template <typename T>
__device__ __forceinline__ CI<T> q1mul_eq(T c, const CI<T> &d) {
  using B = TB<T>;
  const unsigned nxl = B::sgn(d.rl), nxh = B::sgn(d.rh), nyl = B::sgn(d.il), nyh = B::sgn(d.ih);
  const T cxl = B::sel(c, nxl), cxh = B::sel(c, 1u - nxh), cyl = B::sel(c, nyl), cyh = B::sel(c, 1u - nyh);
  CI<T> t;
  t.rl = DR<T>::fma_rd(-cyh, d.ih, DR<T>::mul_rd(cxl, d.rl));
  t.rh = DR<T>::fma_ru(-cyl, d.il, DR<T>::mul_ru(cxh, d.rh));
  t.il = DR<T>::fma_rd(cxl, d.rl, DR<T>::mul_rd(cyl, d.il));
  t.ih = DR<T>::fma_ru(cxh, d.rh, DR<T>::mul_ru(cyh, d.ih));
  return t;
}

// conj(d) variant of q1mul_eq (see q1mul_cd)
template <typename T>
__device__ __forceinline__ CI<T> q1mul_eq_cd(T c, const CI<T> &d) {
  using B = TB<T>;
  const unsigned nxl = B::sgn(d.rl), nxh = B::sgn(d.rh), nyl = B::sgn(d.il), nyh = B::sgn(d.ih);
  const T cxl = B::sel(c, nxl), cxh = B::sel(c, 1u - nxh), cya = B::sel(c, nyl), cyb = B::sel(c, 1u - nyh);
  CI<T> t;
  t.rl = DR<T>::fma_rd(cya, d.il, DR<T>::mul_rd(cxl, d.rl));
  t.rh = DR<T>::fma_ru(cyb, d.ih, DR<T>::mul_ru(cxh, d.rh));
  t.il = DR<T>::fma_rd(cxl, d.rl, DR<T>::mul_rd(cyb, -d.ih));
  t.ih = DR<T>::fma_ru(cxh, d.rh, DR<T>::mul_ru(cya, -d.il));
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
template <typename T, bool CONJ, bool MAYROT = true>
__device__ __forceinline__ CI<T> rtmul(const TwC<T> &w, const CI<T> &d) {
  using B = TB<T>;
  if constexpr (!MAYROT) {  // the table guarantees k = 0 (angle < pi/2) and s >= 0
    CI<T> t = CONJ ? q1mul_cd(w.c, w.s, d) : q1mul(w.c, w.s, d);
    return CONJ ? cconj(t) : t;
  } else {
    const unsigned k = B::sgn(w.s);
    const T s = B::absb(w.s);
    CI<T> t = CONJ ? q1mul_cd(w.c, s, d) : q1mul(w.c, s, d);
    t = rot_if(t, k);
    return CONJ ? cconj(t) : t;
  }
}

// (CONJ ? conj(w) : w) * conj(d) for a runtime table twiddle (a mirrored input
// read without materialising its conjugate): conj(w) conj(d) = conj(w d)
template <typename T, bool CONJ, bool MAYROT = true>
__device__ __forceinline__ CI<T> rtmul_cd(const TwC<T> &w, const CI<T> &d) {
  using B = TB<T>;
  const unsigned k = MAYROT ? B::sgn(w.s) : 0u;
  const T s = MAYROT ? B::absb(w.s) : w.s;
  CI<T> t = CONJ ? q1mul(w.c, s, d) : q1mul_cd(w.c, s, d);
  if constexpr (MAYROT) t = rot_if(t, k);
  return CONJ ? cconj(t) : t;
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
    const int e = j * (64 / M);
    const TwC<T> w = cw64<T>(e);
    if (e == 8) return INV ? cconj(q1mul_eq_cd(w.c, o)) : q1mul_eq(w.c, o);  // w_8
    return INV ? cconj(q1mul_cd(w.c, w.s, o)) : q1mul(w.c, w.s, o);
  }
  // second quadrant: w = i * w', w' = w_M^{j - M/4}
  const int e = (j - M / 4) * (64 / M);
  const TwC<T> w = cw64<T>(e);
  if (e == 8) return INV ? mul_mi(cconj(q1mul_eq_cd(w.c, o))) : mul_i(q1mul_eq(w.c, o));
  return INV ? mul_mi(cconj(q1mul_cd(w.c, w.s, o))) : mul_i(q1mul(w.c, w.s, o));
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
  // stores conj(z): the imaginary endpoints negated and swapped by flipping
  // sign bits in the integer pipe (the compiler would otherwise negate with
  // FP64 DADDs, ~6 % of the FP64 instructions of the one-CTA kernel)
  __device__ __forceinline__ void st_conj(int i, const CI<T> &z) const {
    re[i] = typename V2t<T>::t{z.rl, z.rh};
    im[i] = typename V2t<T>::t{TB<T>::neg(z.ih), TB<T>::neg(z.il)};
  }
};


// ---------------------------------------------------------------------------
// forward passes
// ---------------------------------------------------------------------------
// pass 1: G_1[0][v] = x[v] (the trivial radix-2 pass 0), read from HBM;
// G_2[2r][v] = sum_q w_R^{qr} (w_{4R}^q x[v + S'q]), stored with the mirror.
// SMEMDIG: the digits are in shared memory (staged; the compiler emits LDS for
// them), else global
// a digit (< 256) as T without an I2F: (2^52 + x) - 2^52 (fp32: 2^23), exact
template <typename T> __device__ __forceinline__ T digit_val(unsigned x);
template <> __device__ __forceinline__ double digit_val<double>(unsigned x) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)x), 4503599627370496.0);
}
template <> __device__ __forceinline__ float digit_val<float>(unsigned x) {
  return __fsub_rn(__int_as_float(0x4B000000 | (int)x), 8388608.0f);
}

template <typename T, int M, int RK, bool SMEMDIG = false>
__device__ __forceinline__ void fwd_first(const uint8_t *__restrict__ dig, int n, Buf<T> st,
                                          const TwC<T> *__restrict__ tw, int tid = threadIdx.x) {
  using Gm = G3<M, RK>;
  constexpr int N = Gm::N, R = Gm::P.f[1], L = 2, S = N / 2, Sp = S / R, G = RK / R;
  constexpr int RSo = Gm::fRS(2), SWo = Gm::fSW(2);
  CI<T> v[G][R];
#pragma unroll
  for (int g = 0; g < G; g++) {
    const int nu = tid + g * Gm::TASKS;  // TASKS threads per multiplication
    if (Gm::TASKS * G == Sp || nu < Sp) {
#pragma unroll
      for (int q = 0; q < R; q++) {
        const int idx = nu + Sp * q;
        const unsigned dv = idx < n ? (unsigned)dig[idx] : 0u;
        const T x = digit_val<T>(dv);
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
        if (r < R / 2) st.st(sidx(L * r, nu, RSo, SWo), v[g][r]);
        else st.st_conj(sidx(L * R - 1 - L * r, nu, RSo, SWo), v[g][r]);
      }
    }
  }
}

// inverse pass: loads of E_p[k0][v + S'q] with the mirror (q >= Q/2)
template <typename T, int M, int RK, int p>
__device__ __forceinline__ void inv_load_compute(Buf<T> st, const TwC<T> *__restrict__ tw,
                                                 CI<T> (&v)[RK / G3<M, RK>::P.q[p]][G3<M, RK>::P.q[p]],
                                                 int (&k0s)[RK / G3<M, RK>::P.q[p]],
                                                 int (&nus)[RK / G3<M, RK>::P.q[p]], int tid = threadIdx.x) {
  using Gm = G3<M, RK>;
  constexpr int N = Gm::N, Q = Gm::P.q[p], L = iL(Gm::P, p), S = N / L, Sp = S / Q, G = RK / Q;
  constexpr int H = Sp / 2, RSi = Gm::iRS(p), SWi = Gm::iSW(p);
  constexpr int TW = Gm::tw_inv(p);
  constexpr int COUNT = L * H;
#pragma unroll
  for (int g = 0; g < G; g++) {
    const int t = tid + g * Gm::TASKS;
    const int k0 = t / H, nu = t % H;
    k0s[g] = (Gm::TASKS * G == COUNT || t < COUNT) ? k0 : -1;
    nus[g] = nu;
    if (!(Gm::TASKS * G == COUNT || t < COUNT)) continue;
#pragma unroll
    for (int q = 0; q < Q; q++) {
      CI<T> z;
      if (2 * q < Q) {
        z = st.ld(sidx(k0, nu + Sp * q, RSi, SWi));
        if (q > 0) z = rtmul<T, true>(ldg_twc(tw, TW + (q - 1) * L + k0), z);
      } else {  // the mirror's conjugate, times the twiddle (q >= Q/2 > 0)
        z = rtmul_cd<T, false>(ldg_twc(tw, TW + (q - 1) * L + k0), st.ld(sidx(k0, S - 1 - nu - Sp * q, RSi, SWi)));
      }
      v[g][q] = z;
    }
    cdft<T, Q, true>(v[g]);
  }
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
  bool radius = true;  // track the max radius (diagnostic output only)
};

// coefficient i (global index) -> *dst (the snapped integer, or 0).  int32
// destinations are used only for n <= 32768 (m <= 2^16), where every certified
// coefficient is an exact convolution value <= 255^2 n < 2^31; m = 2^17, 2^18
// use int64 destinations (v5)
// (DUMP = false: the caller has no interval dump; callers branch once on the dump
// pointer around a whole emit loop, so the common path carries no dump code)
template <typename T, typename D, bool DUMP = true>
__device__ __forceinline__ void certify_real(T lo, T hi, int i, int n, D *dst, CertAcc &acc, double *dump) {
  // the odd-frequency kernels compute each coefficient as a REAL containment
  // interval (R13): the imaginary slots of the dump are NaN ("not
  // computed"), never a synthetic [0, 0]
  if (DUMP && dump) {
    const double qnan = __longlong_as_double(0x7ff8000000000000LL);
    reinterpret_cast<double4 *>(dump)[i] = make_double4((double)lo, (double)hi, qnan, qnan);
  }
  if (i >= 2 * n - 1) return;
  const double l = (double)lo, h = (double)hi;
  const double cl = ceil(l);
  const bool ok = cl == floor(h);
  if (acc.radius) {  // the width RU(h - l); halved (exactly) once, in cert_flush
    const double wd = __dadd_ru(h, -l);
    acc.rad = (wd <= acc.rad) ? acc.rad : wd;  // NaN propagates (comparison false)
  }
  *dst = ok ? (D)cl : (D)0;
  if (!ok) {
    acc.ok = 0;
    acc.bad = min(acc.bad, i);
  }
}

// experiment build only (-DIVM_DUMP_PREROT, tools/untwist_cost.py): the dump's
// otherwise-NaN imaginary slots of coefficients k and k + m/2 carry the real and
// imaginary part of the packed value before the final untwist rotation (scaled
// by 2/m), so the rotation's share of the coefficient widths can be measured
template <typename T>
__device__ __forceinline__ void dump_prerot(double *dump, int k, int N, const CI<T> &o, T s) {
#ifdef IVM_DUMP_PREROT
  if (dump) {
    reinterpret_cast<double2 *>(dump)[2 * k + 1] =
        make_double2((double)DR<T>::mul_rd(o.rl, s), (double)DR<T>::mul_ru(o.rh, s));
    reinterpret_cast<double2 *>(dump)[2 * (k + N / 2) + 1] =
        make_double2((double)DR<T>::mul_rd(o.il, s), (double)DR<T>::mul_ru(o.ih, s));
  }
#endif
}

__device__ __forceinline__ void cert_flush(const CertAcc &acc, Cert3 &cs) {
  const int ok = __reduce_and_sync(0xffffffffu, (unsigned)acc.ok);
  const int bad = (int)__reduce_min_sync(0xffffffffu, (unsigned)acc.bad);
  double rad = acc.rad * 0.5;  // radius = width / 2 (exact)
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
template <typename T, int M, int QS = 0>
__device__ __forceinline__ void emit_coeffs(const CI<T> &o, int k, const TwC<T> *__restrict__ tw, int twi,
                                            int n, int32_t *coef, CertAcc &acc, double *dump) {
  constexpr int N = 1 << M;
  // (2/m) z^{-k} = conj of the table entry: the scale of P:97 is in the table
  const CI<T> v = rtmul<T, true>(ldg_twc(tw, twi), o);
  certify_real(v.rl, v.rh, k, n, coef + cpos<QS>(k), acc, dump);
  certify_real(v.il, v.ih, k + N / 2, n, coef + cpos<QS>(k + N / 2), acc, dump);
  dump_prerot(dump, k, N, o, T(1));
}

// folded variant: the input twiddles already carried z^{-k0}; the remaining
// factor z^{-L r} = conj(w_RATIO^r) (RATIO = 2m/L) is a compile-time constant
// (c_k -> *d0, c_{k+m/2} -> *d1)
template <typename T, int M, int RATIO, bool DUMP = true>
__device__ __forceinline__ void emit_fold(const CI<T> &o, int r, int k, int n, int32_t *d0, int32_t *d1,
                                          CertAcc &acc, double *dump) {
  constexpr int N = 1 << M;
  const CI<T> v = ctw<T, true>(o, r, RATIO);  // (the input twiddles carried the scale 2/m)
  certify_real<T, int32_t, DUMP>(v.rl, v.rh, k, n, d0, acc, dump);
  certify_real<T, int32_t, DUMP>(v.il, v.ih, k + N / 2, n, d1, acc, dump);
  if (DUMP) dump_prerot(dump, k, N, o, T(1));
}

template <typename T, int M, int RK, bool WARP = false, int QS = 0>
__device__ __forceinline__ void inv_last(Buf<T> st, const TwC<T> *__restrict__ tw, int n, int32_t *coef,
                                         CertAcc &acc, double *dump, int tid = threadIdx.x) {
  using Gm = G3<M, RK>;
  constexpr int p = Gm::P.ni - 1, Q = Gm::P.q[p], L = iL(Gm::P, p), G = RK / Q;
  constexpr int TWF = Gm::tw_fin();
  CI<T> v[G][Q];
  int k0s[G], nus[G];
  inv_load_compute<T, M, RK, p>(st, tw, v, k0s, nus, tid);
  // every input loaded: the coefficients may overwrite the state
  if constexpr (WARP) __syncwarp();
  else __syncthreads();
#pragma unroll
  for (int g = 0; g < G; g++) {
    if (k0s[g] < 0) continue;
#pragma unroll
    for (int r = 0; r < Q; r++) {
      const int k = k0s[g] + L * r;
      emit_coeffs<T, M, QS>(v[g][r], k, tw, TWF + k, n, coef, acc, dump);
    }
  }
}

// ---------------------------------------------------------------------------
// runtime-parameterised radix-16 pass bodies: ONE code copy serves every
// forward pass p >= 2 (and the last / fused one) and every inverse pass, so the
// straight-line kernel stays small enough for the instruction cache.
// ---------------------------------------------------------------------------
struct PassRT {
  int lgSp, L, RSi, RSo, SWi, SWo;
  int tw;    // offset of the pass table in the shared-memory twiddle area
  int big;   // table lives in the swapped big buffer (forward-last / folded)
  int fold;  // last inverse pass with the final twist folded in (q = 0 twiddled too)
};

__host__ __device__ constexpr int ilog2r(int x) { return x <= 1 ? 0 : 1 + ilog2r(x / 2); }

// shared-memory twiddle area: [TWB_ENT big buffer][forward mid tables][inverse mid tables]
template <int M, int R> struct RT3 {
  using Gm = G3<M, R>;
  static constexpr int nf = plan_cta(M, R).nf, ni = plan_cta(M, R).ni;
  static constexpr int NFWD = nf - 2;  // forward passes 2 .. nf-1
  static constexpr bool LAST16 = plan_cta(M, R).q[ni - 1] == R;
  static constexpr int NINV = LAST16 ? ni - 1 : ni - 2;  // inverse passes 1 .. via the shared body
  __host__ __device__ static constexpr PassRT fwd(int i) {
    return PassRT{ilog2r((1 << M) / fL(plan_cta(M, R), i + 2) / R), fL(plan_cta(M, R), i + 2), Gm::fRS(i + 2),
                  (i + 3 < nf) ? Gm::fRS(i + 3) : Gm::iRS(1), Gm::fSW(i + 2),
                  (i + 3 < nf) ? Gm::fSW(i + 3) : Gm::iSW(1),
                  (i == NFWD - 1) ? 0 : Gm::TWB_ENT() + Gm::tw_fwd(i + 2) - Gm::SMF_BEGIN(), (i == NFWD - 1) ? 1 : 0,
                  0};
  }
  __host__ __device__ static constexpr PassRT inv(int i) {
    return PassRT{ilog2r((1 << M) / iL(plan_cta(M, R), i + 1) / R), iL(plan_cta(M, R), i + 1), Gm::iRS(i + 1),
                  (i + 2 < ni) ? Gm::iRS(i + 2) : 0, Gm::iSW(i + 1), (i + 2 < ni) ? Gm::iSW(i + 2) : 0,
                  (LAST16 && i == NINV - 1) ? 0
                                            : Gm::TWB_ENT() + Gm::SMF_ENT() + Gm::tw_inv(i + 1) - Gm::SMI_BEGIN(),
                  (LAST16 && i == NINV - 1) ? 1 : 0, (LAST16 && i == NINV - 1) ? 1 : 0};
  }
};

template <int M, int R>
__device__ __forceinline__ PassRT pick_fwd(int i) {
  using X = RT3<M, R>;
  static_assert(X::NFWD >= 1 && X::NFWD <= 3, "forward passes");
  constexpr PassRT p0 = X::fwd(0);
  constexpr PassRT p1 = X::fwd(X::NFWD > 1 ? 1 : 0);
  constexpr PassRT p2 = X::fwd(X::NFWD > 2 ? 2 : 0);
  return i == 0 ? p0 : (i == 1 ? p1 : p2);
}
template <int M, int R>
__device__ __forceinline__ PassRT pick_inv(int i) {
  using X = RT3<M, R>;
  static_assert(X::NINV >= 1 && X::NINV <= 3, "inverse passes");
  constexpr PassRT p0 = X::inv(0);
  constexpr PassRT p1 = X::inv(X::NINV > 1 ? 1 : 0);
  constexpr PassRT p2 = X::inv(X::NINV > 2 ? 2 : 0);
  return i == 0 ? p0 : (i == 1 ? p1 : p2);
}

// split write-after-read barrier of an in-place pass:
// each warp's lane 0 arrives on `bar` (count = warps) once the warp's state loads
// are done (__syncwarp orders the lanes' loads before lane 0's release-arrive)
__device__ __forceinline__ void pb_arrive_warp(unsigned long long *bar) {
  __syncwarp();
  if ((threadIdx.x & 31u) == 0u) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
  }
}

// radix-8 DIT of twiddled inputs, written so that the input twiddle products
// (integer-heavy endpoint selects) of one half sit next to the butterflies
// (FP64-dense) of the other in program order: in(q) gives input q times its
// twiddle; operations and operands are exactly cdft<T, 8, INV>'s, so the result
// is bit-identical -- only the instruction order the scheduler starts from changes
template <typename T, bool INV, typename IN, typename AL>
__device__ __forceinline__ void dit8(CI<T> (&v)[8], IN &&in, AL &&loaded) {
  CI<T> a0 = in(0), a1 = in(4);
  bfly(a0, a1, CI<T>(a1));
  CI<T> a2 = in(2), a3 = in(6);
  bfly(a2, a3, CI<T>(a3));
  bfly(a0, a2, CI<T>(a2));
  bfly(a1, a3, ctw<T, INV>(a3, 1, 4));
  CI<T> a4 = in(1), a5 = in(5);
  bfly(a4, a5, CI<T>(a5));
  CI<T> a6 = in(3), a7 = in(7);
  loaded();  // every input has been read
  bfly(a6, a7, CI<T>(a7));
  bfly(a4, a6, CI<T>(a6));
  bfly(a5, a7, ctw<T, INV>(a7, 1, 4));
  bfly(a0, a4, CI<T>(a4));
  bfly(a1, a5, ctw<T, INV>(a5, 1, 8));
  bfly(a2, a6, ctw<T, INV>(a6, 2, 8));
  bfly(a3, a7, ctw<T, INV>(a7, 3, 8));
  v[0] = a0, v[1] = a1, v[2] = a2, v[3] = a3, v[4] = a4, v[5] = a5, v[6] = a6, v[7] = a7;
}

// the input after q in dit8's order 0, 4, 2, 6, 1, 5, 3, 7 (-1: q was the last)
__host__ __device__ constexpr int dit8_next(int q) {
  return q == 0 ? 4 : q == 4 ? 2 : q == 2 ? 6 : q == 6 ? 1 : q == 1 ? 5 : q == 5 ? 3 : q == 3 ? 7 : -1;
}

// pointwise product with a's spectrum from L2 (one load in flight ahead of the
// product), fused with the 8-point inverse DFT of inverse pass 0 in dit8's order
template <typename T, bool COLD, typename AB>
__device__ __forceinline__ void pointwise_dit8(CI<T> (&v)[8], const AB &A, int k0, int stride) {
#ifndef IVM_NO_DIT8
  CI<T> an = A.ld(k0);
  dit8<T, true>(
      v,
      [&](int q) {
        const CI<T> a = an;
        const int nq = dit8_next(q);
        if (nq >= 0) an = A.ld(nq * stride + k0);
        return cmul_ss<T, COLD>(a, v[q]);
      },
      [] {});
#else
  CI<T> an = A.ld(k0);
#pragma unroll
  for (int r = 0; r < 8; r++) {
    const CI<T> a = an;
    if (r + 1 < 8) an = A.ld((r + 1) * stride + k0);
    v[r] = cmul_ss<T, COLD>(a, v[r]);
  }
  cdft<T, 8, true>(v);
#endif
}

// forward: F_p[k0][nu + Sp q] * w_{2LR}^{q(2k0+1)} -> R-point DFT
template <typename T, int R>
__device__ __forceinline__ void fwdR(Buf<T> st, const TwC<T> *twb, const PassRT &pp, CI<T> (&v)[R], int &k0,
                                     int &nu, int t = threadIdx.x, unsigned long long *wbar = nullptr) {
  const int Sp = 1 << pp.lgSp;
  k0 = t >> pp.lgSp;
  nu = t & (Sp - 1);
  const int base = k0 * pp.RSi, sw = k0 & pp.SWi, tstride = pp.L >> 1;
  const TwC<T> *tp = twb + pp.tw + k0;
#ifndef IVM_NO_DIT8
  if constexpr (R == 8) {
    dit8<T, false>(
        v,
        [&](int q) {
          const CI<T> z = st.ld(base + ((nu + Sp * q) ^ sw));
          if (q == 0) return z;
          const TwC<T> w = tp[(q - 1) * tstride];
          return (2 * q <= R) ? rtmul<T, false, false>(w, z) : rtmul<T, false, true>(w, z);
        },
        [&]() {
          if (wbar) pb_arrive_warp(wbar);
        });
    return;
  }
#endif
#pragma unroll
  for (int q = 0; q < R; q++) {
    CI<T> z = st.ld(base + ((nu + Sp * q) ^ sw));
    // angle of w_{2LR}^{q(2k0+1)} < q pi / R: no quadrant rotation for q <= R/2
    if (q > 0) {
      const TwC<T> w = tp[(q - 1) * tstride];
      z = (2 * q <= R) ? rtmul<T, false, false>(w, z) : rtmul<T, false, true>(w, z);
    }
    v[q] = z;
  }
  if (wbar) pb_arrive_warp(wbar);
  cdft<T, R, false>(v);
}

// inverse: E_p[k0][mu] (mirror for q >= R/2) * twiddle -> R-point inverse DFT
template <typename T, int R, bool FOLD>
__device__ __forceinline__ void invR(Buf<T> st, const TwC<T> *twb, const PassRT &pp, CI<T> (&v)[R], int &k0,
                                     int &nu, int t = threadIdx.x, unsigned long long *wbar = nullptr) {
  const int Sp = 1 << pp.lgSp, lgH = pp.lgSp - 1, S = R * Sp;
  k0 = t >> lgH;
  nu = t & ((Sp >> 1) - 1);
  const int base = k0 * pp.RSi, sw = k0 & pp.SWi;
  // folded last pass: entries [q][k0] for q = 0..15, else [q-1][k0]
  const TwC<T> *tp = twb + pp.tw + k0 + (FOLD ? 0 : -pp.L);
#ifndef IVM_NO_DIT8
  if constexpr (R == 8) {
    dit8<T, true>(
        v,
        [&](int q) {
          const int qq = (2 * q < R) ? q : R - q;
          if (2 * q < R) {
            const CI<T> z = st.ld(base + ((nu + Sp * q) ^ sw));
            if (q == 0 && !FOLD) return z;
            const TwC<T> w = tp[q * pp.L];
            return (FOLD || 4 * qq > R) ? rtmul<T, true, true>(w, z) : rtmul<T, true, false>(w, z);
          }
          const CI<T> d = st.ld(base + ((S - 1 - nu - Sp * q) ^ sw));
          const TwC<T> w = tp[q * pp.L];
          return (FOLD || 4 * qq > R) ? rtmul_cd<T, false, true>(w, d) : rtmul_cd<T, false, false>(w, d);
        },
        [&]() {
          if (wbar) pb_arrive_warp(wbar);
        });
    return;
  }
#endif
#pragma unroll
  for (int q = 0; q < R; q++) {
    CI<T> z;
    // unfolded: angle of w_{LQ}^{q' k0} < q' 2pi / Q (q' = min(q, Q-q) <= Q/2): no
    // rotation unless q' > Q/4
    const int qq = (2 * q < R) ? q : R - q;
    if (2 * q < R) {
      z = st.ld(base + ((nu + Sp * q) ^ sw));
      if (q > 0 || FOLD) {
        const TwC<T> w = tp[q * pp.L];
        z = (FOLD || 4 * qq > R) ? rtmul<T, true, true>(w, z) : rtmul<T, true, false>(w, z);
      }
    } else {  // the mirror's conjugate times the twiddle, the conjugate never materialised
      const CI<T> d = st.ld(base + ((S - 1 - nu - Sp * q) ^ sw));
      const TwC<T> w = tp[q * pp.L];
      z = (FOLD || 4 * qq > R) ? rtmul_cd<T, false, true>(w, d) : rtmul_cd<T, false, false>(w, d);
    }
    v[q] = z;
  }
  if (wbar) pb_arrive_warp(wbar);
  cdft<T, R, true>(v);
}

// ---- 1-D bulk async copies (TMA engine) into shared memory, mbarrier-tracked ----
__device__ __forceinline__ void mbar_init(unsigned long long *bar) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one arrival announcing `bytes` of transactions; precedes the copies it covers
__device__ __forceinline__ void mbar_expect(unsigned long long *bar, unsigned bytes) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  // generic-proxy accesses of the destination (ordered before this by a CTA
  // barrier) complete before the async proxy overwrites it
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst), b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
               "l"(src), "r"(bytes), "r"(b)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned phase) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(b), "r"(phase)
        : "memory");
  }
}

// shared memory of the one-CTA kernel (bytes):
//   [state: 2 planes x CAP]  (the int32 coefficients alias it once the last
//                             inverse pass has loaded its inputs)
//   [twiddles: big buffer (forward-last table <-> folded inverse table) + the
//              resident mid-pass tables]
//   [digits: a | b of the current pair, staged by a bulk copy one pair ahead]
template <typename T, int M, int R> struct Cfg3 {
  using Gm = G3<M, R>;
  static_assert(R == 8, "one-CTA kernel: radix 8 (<= 128 registers, 16 warps per SM)");
  static constexpr int N = Gm::N, THREADS = Gm::THREADS, CAP = Gm::CAP;
  static constexpr int MINB = 512 / THREADS < 1 ? 1 : 512 / THREADS;
  static constexpr size_t E = sizeof(typename V2t<T>::t);
  static constexpr size_t STATE_BYTES = 2 * E * (size_t)CAP;
  static constexpr size_t COEF_BYTES = 4 * (size_t)N;
  static constexpr size_t A_BYTES = 2 * E * (size_t)(N / 2);  // [R][L/2] x (re, im)
  static constexpr size_t TW_BYTES = sizeof(TwC<T>) * (size_t)Gm::SM_ENT();
  static constexpr size_t DIG_BYTES = (size_t)N;  // 2n <= N
  static constexpr size_t SMEM = STATE_BYTES + TW_BYTES + DIG_BYTES;
  static_assert(STATE_BYTES >= COEF_BYTES, "the coefficients alias the state");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

// diagnostic interval dump of this pair (ivm_multiply_batched_diag), else null
__device__ __forceinline__ double *diag_dump(const KParams &kp, int pair, int N) {
  if (!kp.dump_slot) return nullptr;
  const int s = kp.dump_slot[pair];
  return s >= 0 ? kp.intervals + (size_t)s * N * 4 : nullptr;
}

// MODE 1, 2: the throughput kernels.  The host guarantees no diagnostic outputs
// (interval dump, snapped coefficients) and picks 1 when every digit row is 16-byte
// aligned (digits staged by bulk copies) and 2 when not (digits read through L2), so
// the other paths and the values they keep live across the pair loop are compiled
// out.  MODE 0 has every path (runtime choices).
template <typename T, int M, int R, int MODE = 0>
__global__ void __launch_bounds__(Cfg3<T, M, R>::THREADS, Cfg3<T, M, R>::MINB) ivm_v3_kernel(KParams kp) {
  using C = Cfg3<T, M, R>;
  using Gm = G3<M, R>;
  using V = typename V2t<T>::t;
  constexpr int N = C::N;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Cert3 cs;
  __shared__ __align__(8) unsigned long long tbar, dbar, pbar;
  Buf<T> st{reinterpret_cast<V *>(smem), reinterpret_cast<V *>(smem) + C::CAP};
  int32_t *coef = reinterpret_cast<int32_t *>(smem);  // aliases the state (see Cfg3)
#ifdef IVM_NO_SPLITBAR
  unsigned long long *wbar = nullptr;
#else
  unsigned long long *wbar = &pbar;  // split write-after-read barrier of the mid passes
#endif
  unsigned pph = 0u;
  TwC<T> *twb = reinterpret_cast<TwC<T> *>(smem + C::STATE_BYTES);
  uint8_t *sdig = smem + C::STATE_BYTES + C::TW_BYTES;
  Buf<T> A{reinterpret_cast<V *>(kp.ascratch) + (size_t)blockIdx.x * N, nullptr};
  A.im = A.re + N / 2;
  const TwC<T> *tw = reinterpret_cast<const TwC<T> *>(kp.tw);
  const int n = kp.n;

  constexpr int NFWD = RT3<M, R>::NFWD, NINV = RT3<M, R>::NINV;
  constexpr bool LAST16 = RT3<M, R>::LAST16;
  constexpr int RSI1 = Gm::iRS(1), SWI1 = Gm::iSW(1);
  constexpr unsigned FL_BYTES = sizeof(TwC<T>) * Gm::FLAST_ENT();
  constexpr unsigned L16_BYTES = LAST16 ? sizeof(TwC<T>) * R * Gm::LASTL() : 0;
  constexpr unsigned SMF_BYTES = sizeof(TwC<T>) * Gm::SMF_ENT(), SMI_BYTES = sizeof(TwC<T>) * Gm::SMI_ENT();
  constexpr int RATIO = 2 * N / Gm::LASTL();
  constexpr int QS = C::THREADS;  // coefficient layout of the 4-words-per-thread carry (cpos)
  // digits staged by bulk copies when every row is 16-byte aligned
  constexpr bool FAST = MODE != 0;
  const bool staged =
      MODE == 1 ||
      (MODE == 0 && (n % 16 == 0) && ((reinterpret_cast<uintptr_t>(kp.a) | reinterpret_cast<uintptr_t>(kp.b)) % 16 == 0));
  if (threadIdx.x == 0) {
    mbar_init(&tbar);
    mbar_init(&dbar);
    const unsigned a = (unsigned)__cvta_generic_to_shared(&pbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"((unsigned)(C::THREADS / 32)));
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x < kp.batch) {
    mbar_expect(&tbar, FL_BYTES + SMF_BYTES + SMI_BYTES);
    bulk_copy(twb, tw + Gm::tw_fwd(Gm::P.nf - 1), FL_BYTES, &tbar);
    if (SMF_BYTES) bulk_copy(twb + Gm::TWB_ENT(), tw + Gm::SMF_BEGIN(), SMF_BYTES, &tbar);
    if (SMI_BYTES) bulk_copy(twb + Gm::TWB_ENT() + Gm::SMF_ENT(), tw + Gm::SMI_BEGIN(), SMI_BYTES, &tbar);
    if (staged) {
      mbar_expect(&dbar, 2u * n);
      bulk_copy(sdig, kp.a + (size_t)blockIdx.x * n, n, &dbar);
      bulk_copy(sdig + n, kp.b + (size_t)blockIdx.x * n, n, &dbar);
    }
  }
  // tbar phases: 0 = initial tables; per pair (LAST16) the folded table and
  // then the forward-last restore, so the folded-table wait has parity 1 and the
  // forward-last wait parity 0 (trivially complete in the first pair).  dbar:
  // one phase per pair.
  if (blockIdx.x < kp.batch) mbar_wait(&tbar, 0);
  IVM_PH_DECL
  for (int pair = blockIdx.x; pair < kp.batch; pair += gridDim.x) {
    const int nxt = pair + (int)gridDim.x;
    if (!staged && nxt < kp.batch) {  // L2 prefetch of the next pair's digits
      for (int off = threadIdx.x * 128; off < n; off += blockDim.x * 128) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.a + (size_t)nxt * n + off));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.b + (size_t)nxt * n + off));
      }
    }
    if (staged) mbar_wait(&dbar, (unsigned)((pair - (int)blockIdx.x) / (int)gridDim.x) & 1u);
#pragma unroll 1
    for (int op = 0; op < 2; op++) {
      if (staged) fwd_first<T, M, R, true>(sdig + op * n, n, st, tw);
      else fwd_first<T, M, R>((op == 0 ? kp.a : kp.b) + (size_t)pair * n, n, st, tw);
      if (op == 1 && threadIdx.x == 0) {
        cs.ok = 1;
        cs.first_bad = 0x7fffffff;
        cs.maxrad = 0ull;
      }
      __syncthreads();
      if (op == 1 && staged && threadIdx.x == 0 && nxt < kp.batch) {  // digits of the next pair
        mbar_expect(&dbar, 2u * n);
        bulk_copy(sdig, kp.a + (size_t)nxt * n, n, &dbar);
        bulk_copy(sdig + n, kp.b + (size_t)nxt * n, n, &dbar);
      }
      IVM_PH(2 * op);
#pragma unroll  // (specialised per pass: addresses fold into immediates)
      for (int i = 0; i < NFWD; i++) {
        const PassRT pp = pick_fwd<M, R>(i);
        CI<T> v[R];
        int k0, nu;
        if (LAST16 && op == 0 && pp.big) mbar_wait(&tbar, 0);  // forward-last table restored
        fwdR<T, R>(st, twb, pp, v, k0, nu, threadIdx.x, i < NFWD - 1 ? wbar : nullptr);
        if (i < NFWD - 1) {  // mid pass: store both halves (mirror conjugated)
          if (wbar) {
            mbar_wait(wbar, pph);
            pph ^= 1u;
          } else {
            __syncthreads();
          }
#pragma unroll
          for (int r = 0; r < R; r++) {
            if (2 * r < R) st.st(sidx(k0 + pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
            else st.st_conj(sidx(R * pp.L - 1 - k0 - pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
          }
        } else if (op == 0) {  // last pass of a: spectrum class k0 -> A
#pragma unroll
          for (int r = 0; r < R; r++) A.st(r * (pp.L >> 1) + k0, v[r]);
        } else {  // last pass of b + pointwise + inverse pass 0
          pointwise_dit8<T, false>(v, A, k0, pp.L >> 1);
          __syncthreads();
          if (LAST16 && threadIdx.x == 0) {  // the folded inverse table replaces the forward-last one
            mbar_expect(&tbar, L16_BYTES);
            bulk_copy(twb, tw + Gm::tw_l16(), L16_BYTES, &tbar);
          }
#pragma unroll
          for (int r = 0; r < R; r++) st.st(sidx(r, k0, RSI1, SWI1), v[r]);
        }
        __syncthreads();
      }
      IVM_PH(2 * op + 1);
    }
    CertAcc acc;
    acc.radius = kp.max_radius != nullptr;
#pragma unroll  // (specialised per pass: addresses fold into immediates)
    for (int i = 0; i < NINV; i++) {
      const PassRT pp = pick_inv<M, R>(i);
      CI<T> v[R];
      int k0, nu;
      if (LAST16 && i == NINV - 1) {
        mbar_wait(&tbar, 1);  // folded table
        invR<T, R, true>(st, twb, pp, v, k0, nu);
        __syncthreads();  // every input loaded: the coefficients may overwrite the state
        double *dump = FAST ? nullptr : diag_dump(kp, pair, N);
        if (!FAST && dump) {
#pragma unroll
          for (int r = 0; r < R; r++) {
            const int k = k0 + pp.L * r;
            emit_fold<T, M, RATIO, true>(v[r], r, k, n, coef + cpos<QS>(k), coef + cpos<QS>(k + N / 2), acc, dump);
          }
        } else {
#pragma unroll
          for (int r = 0; r < R; r++) {
            const int k = k0 + pp.L * r;
            emit_fold<T, M, RATIO, false>(v[r], r, k, n, coef + cpos<QS>(k), coef + cpos<QS>(k + N / 2), acc,
                                          nullptr);
          }
        }
      } else {
        invR<T, R, false>(st, twb, pp, v, k0, nu, threadIdx.x, wbar);
        if (wbar) {
          mbar_wait(wbar, pph);
          pph ^= 1u;
        } else {
          __syncthreads();
        }
#pragma unroll
        for (int r = 0; r < R; r++) st.st(sidx(k0 + pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
      }
      __syncthreads();
    }
    if constexpr (!LAST16) inv_last<T, M, R, false, QS>(st, tw, n, coef, acc, FAST ? nullptr : diag_dump(kp, pair, N));
    IVM_PH(4);
    cert_flush(acc, cs);
    __syncthreads();
    IVM_PH(5);
    if (LAST16 && threadIdx.x == 0 && nxt < kp.batch) {  // restore the forward-last table
      mbar_expect(&tbar, FL_BYTES);
      bulk_copy(twb, tw + Gm::tw_fwd(Gm::P.nf - 1), FL_BYTES, &tbar);
    }
    const bool certified = cs.ok != 0;
    carry_store4<QS>(coef, n, kp.prod + (size_t)pair * 2 * n, certified);
    if (!FAST && kp.coeffs) {
      int64_t *co = kp.coeffs + (size_t)pair * (2 * n - 1);
      for (int i = threadIdx.x; i < 2 * n - 1; i += blockDim.x) co[i] = certified ? coef[cpos<QS>(i)] : 0;
    }
    if (threadIdx.x == 0) {
      kp.cert[pair] = certified ? 1 : 0;
      if (kp.max_radius) kp.max_radius[pair] = __longlong_as_double((long long)cs.maxrad);
      if (kp.first_bad) kp.first_bad[pair] = certified ? -1 : cs.first_bad;
    }
    __syncthreads();
    IVM_PH(6);
  }
}

}  // namespace v3
}  // namespace ivm
