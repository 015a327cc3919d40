// ivm_disc.cu -- the multiplication with CIRCULAR containment sets, the variant
// the paper proposes as future work ("use circular containment sets
// rather than rectangular containment sets ... they easily deal with complex
// rotations"); SURVEY §8(f) rank 4.  fp64, m <= 8192 (n <= 4096).
//
// A disc <c, r> = { z : |z - c| <= r }.  Arithmetic (reading R15):
// centers are round-to-nearest binary64 operations; radii are upper bounds in
// round-up arithmetic, U = 2^-52 bounds one rounding relative to its result,
// ETA = 2^-1000 guards subnormals (radii are kept as binary32 rounded up, and
// every twiddle disc uses the largest twiddle radius):
//   sum        <a.c +- b.c, a.r + b.r + U (|s.re| + |s.im|) + 2 ETA>
//   product    t1..t4 = the four center products, p = (t1 - t2, t3 + t4),
//              r = |a.c| b.r + |b.c| a.r + a.r b.r + U (sum of |t_i| and |p|) + 6 ETA
//              with |c| <= |re| + |im| (data) or 1 + w.r (a twiddle: |w.c - omega| <= w.r)
//   conjugate  <conj c, r>;  1/m = 2^-L exact.
// The FFT is the paper's radix-2 DIT in iterative form: digits
// loaded bit-reversed, log2 m butterfly stages (E + w O, E - w O) in shared
// memory, one CTA per multiplication; the pointwise product, the
// inverse with conjugated twiddles, then certify (the real
// part [c.re - r, c.re + r] holds one integer, the imaginary part only 0) and
// the word carry (ivm_carry.cuh).  Shares no code with oracle/ivm_oracle_disc.c.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ivm_internal.h"
#include "ivm_carry.cuh"

namespace ivm {
namespace dk {

constexpr int TH = 512;
constexpr double U = 0x1p-52, ETA = 0x1p-1000;

struct Disc { double cr, ci, r; };

__device__ __forceinline__ double ru_add(double a, double b) { return __dadd_ru(a, b); }
__device__ __forceinline__ double ru_mul(double a, double b) { return __dmul_ru(a, b); }

__device__ __forceinline__ Disc dsum(const Disc &a, const Disc &b, bool sub) {
  Disc s;
  s.cr = sub ? __dsub_rn(a.cr, b.cr) : __dadd_rn(a.cr, b.cr);
  s.ci = sub ? __dsub_rn(a.ci, b.ci) : __dadd_rn(a.ci, b.ci);
  const double e = __fma_ru(U, ru_add(fabs(s.cr), fabs(s.ci)), 2 * ETA);
  s.r = ru_add(ru_add(a.r, b.r), e);
  return s;
}

// a * b; na, nb: upper bounds of |a.c|, |b.c|
__device__ __forceinline__ Disc dmul(const Disc &a, const Disc &b, double na, double nb) {
  const double t1 = __dmul_rn(a.cr, b.cr), t2 = __dmul_rn(a.ci, b.ci);
  const double t3 = __dmul_rn(a.cr, b.ci), t4 = __dmul_rn(a.ci, b.cr);
  Disc p;
  p.cr = __dsub_rn(t1, t2);
  p.ci = __dadd_rn(t3, t4);
  const double s = ru_add(ru_add(ru_add(fabs(t1), fabs(t2)), ru_add(fabs(t3), fabs(t4))),
                          ru_add(fabs(p.cr), fabs(p.ci)));
  const double e = __fma_ru(U, s, 6 * ETA);
  p.r = ru_add(__fma_ru(na, b.r, __fma_ru(nb, a.r, ru_mul(a.r, b.r))), e);
  return p;
}
__device__ __forceinline__ double l1(const Disc &a) { return ru_add(fabs(a.cr), fabs(a.ci)); }

// disc planes: centers (double2) and radii stored as binary32 rounded up (an
// upper bound again: sound), 20 bytes per disc, so that the m = 8192 state and
// the twiddle centers fit in shared memory together
struct SDisc {
  double2 *c;
  float *r;
  __device__ __forceinline__ Disc ld(int i) const {
    const double2 v = c[i];
    return Disc{v.x, v.y, (double)r[i]};
  }
  __device__ __forceinline__ void st(int i, const Disc &d) const {
    c[i] = make_double2(d.cr, d.ci);
    r[i] = __double2float_ru(d.r);
  }
};

__device__ __forceinline__ int brev(int j, int lg) { return lg ? (int)(__brev((unsigned)j) >> (32 - lg)) : 0; }

// P:143-155 iteratively: stage s combines half-length-2^s transforms; the
// twiddle of butterfly j is omega_{2^{s+1}}^j = omega_m^{j m / 2^{s+1}}
// tw: twiddle centers omega_m^j (j < m/2) in shared memory; rw: one radius
// bound for all of them (the host's max over j)
__device__ __forceinline__ void bfly(Disc &e, Disc &o, const double2 t, bool inv, double rw, double nw) {
  const Disc w{t.x, inv ? -t.y : t.y, rw};
  const Disc wo = dmul(w, o, nw, l1(o));
  o = dsum(e, wo, true);
  e = dsum(e, wo, false);
}
// K stages per shared-memory round trip: a group of 2^K elements
// i0 + q half (q < 2^K, half = 2^s) runs, for t = 0 .. K-1, the stage-(s + t)
// butterflies (q, q + 2^t) with twiddle index (j + (q mod 2^t) half) m / 2^(s+t+1)
// -- the same butterflies, in the same order per element, as one stage at a
// time (the radii between them stay binary64 instead of being stored as
// binary32: slightly tighter).  K = 3 while three stages remain, then 2 or 1.
template <bool INV, int K>
__device__ __forceinline__ void dstages(SDisc x, int m, int s, const double2 *tw, double rw, double nw) {
  constexpr int E = 1 << K;
  const int half = 1 << s;
  for (int g = threadIdx.x; g < m / E; g += blockDim.x) {
    const int j = g & (half - 1), i0 = ((g >> s) << (s + K)) + j;
    Disc v[E];
#pragma unroll
    for (int q = 0; q < E; q++) v[q] = x.ld(i0 + q * half);
#pragma unroll
    for (int t = 0; t < K; t++) {
      const int h = 1 << t, stride = m >> (s + t + 1);
#pragma unroll
      for (int q = 0; q < E; q++)
        if ((q & h) == 0) bfly(v[q], v[q + h], tw[(j + (q & (h - 1)) * half) * stride], INV, rw, nw);
    }
#pragma unroll
    for (int q = 0; q < E; q++) x.st(i0 + q * half, v[q]);
  }
  __syncthreads();
}
template <bool INV>
__device__ __forceinline__ void dfft(SDisc x, int lg, const double2 *tw, double rw) {
  const int m = 1 << lg;
  const double nw = ru_add(1.0, rw);
  int s = 0;
  for (; s + 3 <= lg; s += 3) dstages<INV, 3>(x, m, s, tw, rw, nw);
  if (lg - s == 2) dstages<INV, 2>(x, m, s, tw, rw, nw);
  if (lg - s == 1) dstages<INV, 1>(x, m, s, tw, rw, nw);
}

__global__ void __launch_bounds__(TH, 1)
    disc_kernel(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b, int n, int batch, int lg,
                const double2 *__restrict__ twg, double rw, double *__restrict__ scratch,
                uint8_t *__restrict__ prod, uint8_t *__restrict__ cert, double *__restrict__ max_radius) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int m = 1 << lg, nc = 2 * n - 1;
  SDisc x{reinterpret_cast<double2 *>(smem), reinterpret_cast<float *>(smem + 16 * (size_t)m)};
  double2 *tw = reinterpret_cast<double2 *>(smem + ((20 * (size_t)m + 15) & ~(size_t)15));  // m/2 centers
  for (int j = threadIdx.x; j < m / 2; j += blockDim.x) tw[j] = twg[j];
  SDisc A{reinterpret_cast<double2 *>(scratch) + (size_t)blockIdx.x * 2 * m, nullptr};
  A.r = reinterpret_cast<float *>(A.c + m);
  __shared__ int s_ok;
  __shared__ unsigned long long s_rad;
  for (int pair = blockIdx.x; pair < batch; pair += gridDim.x) {
    for (int op = 0; op < 2; op++) {  // a', b' as points (radius 0), bit-reversed
      const uint8_t *d = (op == 0 ? a : b) + (size_t)pair * n;
      __syncthreads();
      for (int j = threadIdx.x; j < m; j += blockDim.x) {
        const int s = brev(j, lg);
        x.st(j, Disc{s < n ? (double)d[s] : 0.0, 0.0, 0.0});
      }
      __syncthreads();
      dfft<false>(x, lg, tw, rw);
      if (op == 0) {
        for (int j = threadIdx.x; j < m; j += blockDim.x) A.st(j, x.ld(j));
      } else {  // P:210 pointwise, written bit-reversed for the inverse DIT
        for (int j = threadIdx.x; j < m; j += blockDim.x) {
          const Disc p = A.ld(j), q = x.ld(j);
          A.st(j, dmul(p, q, l1(p), l1(q)));
        }
      }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += blockDim.x) x.st(brev(j, lg), A.ld(j));
    if (threadIdx.x == 0) {
      s_ok = 1;
      s_rad = 0ull;
    }
    __syncthreads();
    dfft<true>(x, lg, tw, rw);  // P:211 with omega^-1 = conj
    // 1/m exact; certify c_i, i < 2n-1, snap into int32 coefficients
    const double sc = 1.0 / (double)m;
    int32_t cv[16];  // m / TH <= 16
    int cnt = 0, ok = 1;
    double rad = 0.0;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
      const Disc z = x.ld(i);
      const double cr = z.cr * sc, ci = z.ci * sc, r = z.r * sc;
      const double lo = __dsub_rd(cr, r), hi = __dadd_ru(cr, r), il = __dsub_rd(ci, r), ih = __dadd_ru(ci, r);
      const double cl = ceil(lo);
      const bool good = cl == floor(hi) && ceil(il) == 0.0 && floor(ih) == 0.0;
      ok &= good ? 1 : 0;
      rad = r > rad ? r : (r != r ? __longlong_as_double(0x7ff0000000000000ll) : rad);
      cv[cnt++] = good ? (int32_t)cl : 0;
    }
    if (!ok) atomicAnd(&s_ok, 0);
    atomicMax(&s_rad, (unsigned long long)__double_as_longlong(rad));  // radii >= 0: bit order = value order
    __syncthreads();
    int32_t *coef = reinterpret_cast<int32_t *>(smem);
    cnt = 0;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) coef[i] = cv[cnt++];
    __syncthreads();
    const bool certified = s_ok != 0;
    carry_store(coef, n, prod + (size_t)pair * 2 * n, certified);
    if (threadIdx.x == 0) {
      cert[pair] = certified ? 1 : 0;
      if (max_radius) max_radius[pair] = __longlong_as_double((long long)s_rad);
    }
  }
}


// ---------------------------------------------------------------------------
// m = 2^14 .. 2^18: one group of C = m / 8192 co-resident CTAs per
// multiplication (cooperative launch), exchanging through L2-resident global
// scratch with group barriers.  The paper's DIT is factored as
// m = 8192 C (a valid DIT-form factorization: every twiddle multiplies the
// input of the butterflies that follow it):
//   forward  X_{k1 + 8192 k2} = sum_{j2<C} w_C^{j2 k2} [ w_m^{j2 k1} Y_{j2}(k1) ],
//            Y_{j2} = DFT_8192 of x_{C j1 + j2}          (CTA j2, shared memory)
//            then C-point DFTs over j2 for the CTA's B = 8192/C values of k1
//   pointwise in that layout (the same for both operands)
//   inverse  c_{s1 + C s2} = sum_{k1} w_8192^{-s2 k1} [ w_m^{-s1 k1}
//                            sum_{k2<C} w_C^{-s1 k2} P_{k1 + 8192 k2} ]
//            C-point inverse DFTs over k2 for the CTA's k1, then CTA s1 the
//            8192-point inverse over k1
// then 1/m, certify into a group-global int64 coefficient array, and a
// group carry over contiguous word chunks (ivm_carry.cuh, one CTA per chunk,
// chunk carries from the published generate / propagate bits).
// ---------------------------------------------------------------------------
struct DiscGroup {
  unsigned *ctr;        // [groups] barrier counters (zeroed before the launch)
  double2 *xc;          // [groups][3][C][8192] disc centers: forward a, forward b, inverse exchange
  float *xr;            // [groups][3][C][8192] disc radii (binary32 rounded up)
  double2 *ac;          // [groups][C][8192] the CTA's spectrum of a (centers)
  float *ar;            // [groups][C][8192] (radii)
  long long *coef;      // [groups][m] snapped coefficients
  unsigned *link;       // [groups][C][4] ok, max radius bits
  unsigned *bits;       // [groups][C] chunk generate | all-propagate << 1
};

__device__ __forceinline__ void gbar(unsigned *ctr, unsigned C, unsigned &gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = (gen + 1u) * C;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  gen++;
  __syncthreads();
}

// twiddle disc w_m^e (any integer e), from the centers of w_m^j, j < m/2:
// w^{j + m/2} = -w^j (exact), radius rw for all
__device__ __forceinline__ Disc twm(const double2 *__restrict__ tw, int lgm, long long e, bool conj, double rw) {
  const long long mm = 1ll << lgm;
  e &= mm - 1;
  double2 t = __ldg(tw + (e & (mm / 2 - 1)));
  if (e >= mm / 2) t = make_double2(-t.x, -t.y);
  return Disc{t.x, conj ? -t.y : t.y, rw};
}

// rows of C-point DFTs (B rows, row-major, inputs bit-reversed within a row),
// radix-2 DIT one stage per shared-memory round trip; twiddle of butterfly j
// at stage s: w_{2^{s+1}}^j = w_m^{j m / 2^{s+1}}
template <bool INV>
__device__ __forceinline__ void row_dfts(SDisc x, int lgC, int rows, const double2 *__restrict__ tw, int lgm,
                                         double rw, double nw) {
  const int C = 1 << lgC, nb = rows * (C / 2);
  for (int st = 0; st < lgC; st++) {
    const int half = 1 << st;
    for (int g = threadIdx.x; g < nb; g += blockDim.x) {
      const int row = g >> (lgC - 1), jj = g & (C / 2 - 1), j = jj & (half - 1);
      const int e = row * C + ((jj >> st) << (st + 1)) + j;
      Disc ve = x.ld(e), vo = x.ld(e + half);
      const Disc w = twm(tw, lgm, (long long)j << (lgm - st - 1), INV, rw);
      const Disc wo = dmul(w, vo, nw, l1(vo));
      vo = dsum(ve, wo, true);
      ve = dsum(ve, wo, false);
      x.st(e, ve);
      x.st(e + half, vo);
    }
    __syncthreads();
  }
}

struct CoefG {  // a group-global int64 coefficient array written by other CTAs (read through L2)
  const long long *c;
  __device__ __forceinline__ void quad(int k, unsigned long long (&o)[4]) const {
    const longlong2 x = __ldcg(reinterpret_cast<const longlong2 *>(c) + 2 * k);
    const longlong2 y = __ldcg(reinterpret_cast<const longlong2 *>(c) + 2 * k + 1);
    o[0] = (unsigned long long)x.x, o[1] = (unsigned long long)x.y;
    o[2] = (unsigned long long)y.x, o[3] = (unsigned long long)y.y;
  }
  __device__ __forceinline__ unsigned long long one(int i) const { return (unsigned long long)__ldcg(c + i); }
};

__global__ void __launch_bounds__(TH, 1)
    disc_group_kernel(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b, int n, int batch, int lgm,
                      const double2 *__restrict__ twg, double rw, DiscGroup g, uint8_t *__restrict__ prod,
                      uint8_t *__restrict__ cert, double *__restrict__ max_radius) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int ML = 8192, LGL = 13;
  const int lgC = lgm - LGL, C = 1 << lgC, B = ML / C, nc = 2 * n - 1, nout = 2 * n;
  const unsigned crank = blockIdx.x % C;
  const int gi = (int)(blockIdx.x / C), ngr = (int)(gridDim.x / C);
  SDisc x{reinterpret_cast<double2 *>(smem), reinterpret_cast<float *>(smem + 16 * (size_t)ML)};
  double2 *tw = reinterpret_cast<double2 *>(smem + 20 * (size_t)ML);  // w_8192^j = w_m^{j C}, j < 4096
  for (int j = threadIdx.x; j < ML / 2; j += blockDim.x) tw[j] = twg[(size_t)j << lgC];
  const double nw = ru_add(1.0, rw);
  unsigned *ctr = g.ctr + gi;
  const size_t plane = (size_t)C * ML;
  double2 *xc = g.xc + (size_t)gi * 3 * plane;
  float *xr = g.xr + (size_t)gi * 3 * plane;
  SDisc A{g.ac + ((size_t)gi * C + crank) * ML, g.ar + ((size_t)gi * C + crank) * ML};
  long long *coefG = g.coef + ((size_t)gi << lgm);
  unsigned *link = g.link + (size_t)gi * C * 4;
  unsigned *bits = g.bits + (size_t)gi * C;
  __shared__ int s_ok;
  __shared__ unsigned long long s_rad;
  __shared__ unsigned s_cin;
  __shared__ CarrySeg seg;
  unsigned gen = 0;
  __syncthreads();
  for (int pair = gi; pair < batch; pair += ngr) {
    // ---- step 1: Y_c = DFT_8192(x_{C j1 + c}), both operands -> exchange planes 0, 1
    for (int op = 0; op < 2; op++) {
      const uint8_t *d = (op == 0 ? a : b) + (size_t)pair * n;
      for (int j = threadIdx.x; j < ML; j += blockDim.x) {
        const int idx = (brev(j, LGL) << lgC) + (int)crank;  // points, zero padding
        x.st(j, Disc{idx < n ? (double)d[idx] : 0.0, 0.0, 0.0});
      }
      __syncthreads();
      dfft<false>(x, LGL, tw, rw);
      for (int j = threadIdx.x; j < ML; j += blockDim.x) {
        const size_t o = (size_t)op * plane + (size_t)crank * ML + j;
        xc[o] = x.c[j];
        xr[o] = x.r[j];
      }
    }
    gbar(ctr, C, gen);  // (1) every Y_{j2} written
    // ---- step 2/3: rows k1 = crank B + kl: twiddle w_m^{j2 k1}, C-point DFT over j2
    for (int op = 0; op < 2; op++) {
      for (int e = threadIdx.x; e < ML; e += blockDim.x) {
        const int kl = e >> lgC, j2 = e & (C - 1), k1 = (int)crank * B + kl;
        const size_t o = (size_t)op * plane + (size_t)j2 * ML + k1;
        const double2 cc = __ldcg(xc + o);
        const Disc z{cc.x, cc.y, (double)__ldcg(xr + o)};
        const Disc w = twm(twg, lgm, (long long)j2 * k1, false, rw);
        x.st(kl * C + brev(j2, lgC), dmul(w, z, nw, l1(z)));
      }
      __syncthreads();
      row_dfts<false>(x, lgC, B, twg, lgm, rw, nw);  // X[k1 + 8192 k2] at kl C + k2
      if (op == 0) {
        for (int e = threadIdx.x; e < ML; e += blockDim.x) A.st(e, x.ld(e));
      } else {  // P:210, stored bit-reversed along k2 for the inverse DIT over k2
        Disc pv[ML / TH];
#pragma unroll
        for (int q = 0; q < ML / TH; q++) {
          const int e = (int)threadIdx.x + q * TH;
          const Disc p = A.ld(e), v = x.ld(e);
          pv[q] = dmul(p, v, l1(p), l1(v));
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < ML / TH; q++) {
          const int e = (int)threadIdx.x + q * TH;
          x.st((e & ~(C - 1)) | brev(e & (C - 1), lgC), pv[q]);
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      s_ok = 1;
      s_rad = 0ull;
    }
    __syncthreads();
    // ---- inverse step 1: C-point inverse DFTs over k2, twiddle w_m^{-s1 k1} -> plane 2 [s1][k1]
    row_dfts<true>(x, lgC, B, twg, lgm, rw, nw);
    for (int e = threadIdx.x; e < ML; e += blockDim.x) {
      const int kl = e >> lgC, s1 = e & (C - 1), k1 = (int)crank * B + kl;
      const Disc z = x.ld(e);
      const Disc w = twm(twg, lgm, (long long)s1 * k1, true, rw);
      const Disc t = dmul(w, z, nw, l1(z));
      const size_t o = 2 * plane + (size_t)s1 * ML + k1;
      xc[o] = make_double2(t.cr, t.ci);
      xr[o] = __double2float_ru(t.r);
    }
    gbar(ctr, C, gen);  // (2) the inverse exchange written
    // ---- inverse step 2: CTA s1 = crank, 8192-point inverse over k1 (bit-reversed in)
    for (int j = threadIdx.x; j < ML; j += blockDim.x) {
      const size_t o = 2 * plane + (size_t)crank * ML + brev(j, LGL);
      const double2 cc = __ldcg(xc + o);
      x.st(j, Disc{cc.x, cc.y, (double)__ldcg(xr + o)});
    }
    __syncthreads();
    dfft<true>(x, LGL, tw, rw);
    // 1/m exact; c_s, s = crank + C s2 < 2n - 1; snapped into the group array
    {
      const double sc = 1.0 / (double)(1 << lgm);
      int ok = 1;
      double rad = 0.0;
      for (int s2 = threadIdx.x; s2 < ML; s2 += blockDim.x) {
        const int sidx = (int)crank + (s2 << lgC);
        if (sidx >= nc) continue;
        const Disc z = x.ld(s2);
        const double cr = z.cr * sc, ci = z.ci * sc, r = z.r * sc;
        const double lo = __dsub_rd(cr, r), hi = __dadd_ru(cr, r), il = __dsub_rd(ci, r), ih = __dadd_ru(ci, r);
        const double cl = ceil(lo);
        const bool good = cl == floor(hi) && ceil(il) == 0.0 && floor(ih) == 0.0;
        ok &= good ? 1 : 0;
        rad = r > rad ? r : (r != r ? __longlong_as_double(0x7ff0000000000000ll) : rad);
        coefG[sidx] = good ? (long long)cl : 0ll;
      }
      if (!ok) atomicAnd(&s_ok, 0);
      atomicMax(&s_rad, (unsigned long long)__double_as_longlong(rad));
      __syncthreads();
      if (threadIdx.x == 0) {
        link[crank * 4 + 0] = (unsigned)s_ok;
        link[crank * 4 + 1] = (unsigned)(s_rad & 0xffffffffu);
        link[crank * 4 + 2] = (unsigned)(s_rad >> 32);
      }
    }
    gbar(ctr, C, gen);  // (3) coefficients and certificates of every CTA
    if (threadIdx.x < 32) {  // the group's certificate
      const unsigned l = threadIdx.x;
      int okl = 1;
      unsigned long long radl = 0ull;
      if ((int)l < C) {
        okl = (int)__ldcg(link + l * 4);
        radl = (unsigned long long)__ldcg(link + l * 4 + 1) | ((unsigned long long)__ldcg(link + l * 4 + 2) << 32);
      }
      okl = __reduce_and_sync(0xffffffffu, (unsigned)okl);
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long r2 = __shfl_xor_sync(0xffffffffu, radl, o);
        radl = r2 > radl ? r2 : radl;
      }
      if (l == 0) {
        s_ok = okl;
        s_rad = radl;
      }
    }
    __syncthreads();
    const bool certified = s_ok != 0;
    uint8_t *out = prod + (size_t)pair * nout;
    const int words = (nout + 3) / 4, wc = (words + C - 1) / C;
    const int kb = min((int)crank * wc, words), ke = min(kb + wc, words);
    const CoefG src{coefG};
    if (certified) {  // chunk carry: scan, publish, carry-in from the chunks below, emit
      unsigned gn = 0u, ap = 1u;
      carry_seg_scan(src, nc, kb, ke, seg, gn, ap);
      if (threadIdx.x == 0) bits[crank] = gn | (ap << 1);
    }
    gbar(ctr, C, gen);  // (4) chunk generate / propagate bits
    if (certified) {
      if (threadIdx.x == 0) {
        unsigned cin = 0u;
        for (int j = 0; j < (int)crank; j++) {
          const unsigned bb = __ldcg(bits + j);
          cin = (bb & 1u) | ((bb >> 1) & cin);
        }
        s_cin = cin;
      }
      __syncthreads();
      carry_seg_emit(src, nc, nout, kb, ke, seg, s_cin, out);
    } else {
      for (int i = 4 * kb + (int)threadIdx.x; i < min(4 * ke, nout); i += blockDim.x) out[i] = 0;
    }
    if (crank == 0 && threadIdx.x == 0) {
      cert[pair] = certified ? 1 : 0;
      if (max_radius) max_radius[pair] = __longlong_as_double((long long)s_rad);
    }
    __syncthreads();
  }
}
}  // namespace dk

int disc_smem(int lg) {  // state + m/2 twiddle centers (the group kernel: its 8192-point share)
  if (lg > 13) lg = 13;
  return (((20 << lg) + 15) & ~15) + (8 << lg) + 16;
}

int disc_launch(const uint8_t *a, const uint8_t *b, int n, int batch, int lg, const void *tw, double rw,
                void *scratch, uint8_t *prod, uint8_t *cert, double *max_radius, int grid, cudaStream_t s) {
  const int smem = disc_smem(lg);
  if (cudaFuncSetAttribute(dk::disc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return -1;
  dk::disc_kernel<<<grid, dk::TH, smem, s>>>(a, b, n, batch, lg, (const double2 *)tw, rw, (double *)scratch, prod,
                                             cert, max_radius);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace ivm

namespace ivm {
int disc_group_blocks_per_sm() {
  if (cudaFuncSetAttribute(dk::disc_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, disc_smem(13)) !=
      cudaSuccess)
    return -1;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dk::disc_group_kernel, dk::TH, disc_smem(13)) != cudaSuccess)
    return -1;
  return nb;
}
size_t disc_group_scratch(int lg, size_t groups) {  // bytes (DiscGroupArgs layout, 256-B aligned pieces)
  const size_t C = (size_t)1 << (lg - 13), pl = C * 8192, al = 256;
  auto up = [&](size_t x) { return (x + al - 1) / al * al; };
  return up(groups * 4) + up(groups * 3 * pl * 16) + up(groups * 3 * pl * 4) + up(groups * pl * 16) +
         up(groups * pl * 4) + up(groups * ((size_t)8 << lg)) + up(groups * C * 16) + up(groups * C * 4);
}
int disc_group_launch(const uint8_t *a, const uint8_t *b, int n, int batch, int lg, const void *tw, double rw,
                      void *scratch, size_t groups, uint8_t *prod, uint8_t *cert, double *max_radius, cudaStream_t s) {
  const size_t C = (size_t)1 << (lg - 13), pl = C * 8192, al = 256;
  auto up = [&](size_t x) { return (x + al - 1) / al * al; };
  char *p = (char *)scratch;
  dk::DiscGroup g;
  g.ctr = (unsigned *)p;
  p += up(groups * 4);
  g.xc = (double2 *)p;
  p += up(groups * 3 * pl * 16);
  g.xr = (float *)p;
  p += up(groups * 3 * pl * 4);
  g.ac = (double2 *)p;
  p += up(groups * pl * 16);
  g.ar = (float *)p;
  p += up(groups * pl * 4);
  g.coef = (long long *)p;
  p += up(groups * ((size_t)8 << lg));
  g.link = (unsigned *)p;
  p += up(groups * C * 16);
  g.bits = (unsigned *)p;
  if (cudaMemsetAsync(g.ctr, 0, groups * 4, s) != cudaSuccess) return -1;
  const double2 *twp = (const double2 *)tw;
  void *args[] = {(void *)&a, (void *)&b, (void *)&n, (void *)&batch, (void *)&lg, (void *)&twp, (void *)&rw,
                  (void *)&g, (void *)&prod, (void *)&cert, (void *)&max_radius};
  return cudaLaunchCooperativeKernel((const void *)dk::disc_group_kernel, dim3((unsigned)(groups * C)), dim3(dk::TH),
                                     args, disc_smem(13), s) == cudaSuccess
             ? 0
             : -1;
}
}  // namespace ivm
