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

}  // namespace dk

int disc_smem(int lg) { return (((20 << lg) + 15) & ~15) + (8 << lg) + 16; }  // state + m/2 twiddle centers

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
