// ivm_d3.cuh -- circular containment sets (R15) on the one-CTA
// odd-frequency radix-8 schedule of ivm_v3.cuh (included by ivm_v3.cu): fp64,
// m = 2^10 .. 2^13 (the other sizes keep the radix-2 kernels of ivm_disc.cu).
//
// Same transform, plans, index rules, tables and carry as ivm_v3_kernel; what
// changes is the element: a disc <c, r> = { z : |z - c| <= r } instead of a
// rectangle.  Centers are round-to-nearest binary64 operations, radii upper
// bounds in round-up arithmetic (U = 2^-52 bounds one rounding relative to its
// result, ETA = 2^-1000 guards subnormal products), kept in shared memory and
// in the L2 scratch as binary32 rounded up (still upper bounds):
//   e +- t      <e.c +- t.c,  e.r + t.r + U |c'|_1 + 2 ETA>     (|x|_1 = |re| + |im|)
//   w d         w = c + i s a table twiddle: the lower corner of the optimal
//               enclosure of omega, so |w - omega| <= RW = 2^-52 |omega| (each
//               component is within 2^-53 |omega| of the true value);
//               p = (c d.re - s d.im, c d.im + s d.re) by one product and one
//               FMA per part; |omega z - p| <= |omega| d.r + RW |omega| |d.c|_1
//               + U (|t2| + |t4| + |p|_1) + 4 ETA for every z in d
//   a b         general product (pointwise step): |a.c|_1 b.r + |b.c|_1 a.r + a.r b.r
//               + U (|t2| + |t4| + |p|_1) + 4 ETA
//   i d, conj d exact.  Scaling by 2/m (a power of two) is carried by the last
//   pass's tables, as in ivm_v3.cuh (|omega| = 2/m there).
// A disc needs no endpoint selects (the rectangles' twiddle product is 8 FP64
// and 17 integer instructions, the disc's 11 FP64), and 20 bytes of shared
// memory instead of 32.  Certification: the coefficient 2 Re / m lies in
// [c.re - r, c.re + r] (endpoints rounded outwards), likewise 2 Im / m; each
// must hold exactly one integer.  Shares no code with oracle/ivm_oracle_disc.c.
#pragma once

namespace ivm {
namespace d3 {

using namespace v3;

struct DI { double cr, ci, r; };

constexpr double DU = 0x1p-52, DETA = 0x1p-1000, DRW = 0x1p-52;

__device__ __forceinline__ double l1(const DI &a) { return __dadd_ru(fabs(a.cr), fabs(a.ci)); }
__device__ __forceinline__ DI dconj(const DI &a) { return DI{a.cr, -a.ci, a.r}; }
__device__ __forceinline__ DI dmul_i(const DI &a) { return DI{-a.ci, a.cr, a.r}; }
__device__ __forceinline__ DI dmul_mi(const DI &a) { return DI{a.ci, -a.cr, a.r}; }

// butterfly (e + t, e - t)
__device__ __forceinline__ void dbfly(DI &e, DI &o, const DI &t) {
  const double base = __dadd_ru(__dadd_ru(e.r, t.r), 2 * DETA);
  DI s{__dadd_rn(e.cr, t.cr), __dadd_rn(e.ci, t.ci), 0.0};
  DI d{__dsub_rn(e.cr, t.cr), __dsub_rn(e.ci, t.ci), 0.0};
  s.r = __fma_ru(DU, l1(s), base);
  d.r = __fma_ru(DU, l1(d), base);
  e = s;
  o = d;
}

// (c + i s) d for a twiddle center (c, s) of a true twiddle of modulus sc
__device__ __forceinline__ DI dtw(double c, double s, const DI &d, double sc) {
  const double t2 = __dmul_rn(s, d.ci), t4 = __dmul_rn(s, d.cr);
  DI p;
  p.cr = __fma_rn(c, d.cr, -t2);
  p.ci = __fma_rn(c, d.ci, t4);
  const double e = __dadd_ru(__dadd_ru(fabs(t2), fabs(t4)), __dadd_ru(fabs(p.cr), fabs(p.ci)));
  const double lin = __fma_ru(__dmul_ru(DRW, sc), l1(d), __fma_ru(sc, d.r, 4 * DETA));
  p.r = __fma_ru(DU, e, lin);
  return p;
}
// the same with |omega| = 1 (one multiplication less)
__device__ __forceinline__ DI dtw1(double c, double s, const DI &d) {
  const double t2 = __dmul_rn(s, d.ci), t4 = __dmul_rn(s, d.cr);
  DI p;
  p.cr = __fma_rn(c, d.cr, -t2);
  p.ci = __fma_rn(c, d.ci, t4);
  const double e = __dadd_ru(__dadd_ru(fabs(t2), fabs(t4)), __dadd_ru(fabs(p.cr), fabs(p.ci)));
  const double lin = __fma_ru(DRW, l1(d), __dadd_ru(d.r, 4 * DETA));
  p.r = __fma_ru(DU, e, lin);
  return p;
}

// general product
__device__ __forceinline__ DI dmul(const DI &a, const DI &b) {
  const double t2 = __dmul_rn(a.ci, b.ci), t4 = __dmul_rn(a.ci, b.cr);
  DI p;
  p.cr = __fma_rn(a.cr, b.cr, -t2);
  p.ci = __fma_rn(a.cr, b.ci, t4);
  const double e = __dadd_ru(__dadd_ru(fabs(t2), fabs(t4)), __dadd_ru(fabs(p.cr), fabs(p.ci)));
  const double lin = __fma_ru(l1(a), b.r, __fma_ru(l1(b), a.r, __fma_ru(a.r, b.r, 4 * DETA)));
  p.r = __fma_ru(DU, e, lin);
  return p;
}

// runtime table twiddle w = i^k (c + i s) (k in the sign bit of s, ivm_v3.cuh),
// CONJ: conj(w) d; SC: the table carries the scale 2/m (modulus sc)
template <bool CONJ, bool MAYROT, bool SC = false>
__device__ __forceinline__ DI drt(const TwC<double> &w, const DI &d, double sc = 1.0) {
  using B = TB<double>;
  const unsigned k = MAYROT ? B::sgn(w.s) : 0u;
  const double s = MAYROT ? B::absb(w.s) : w.s;
  DI t = SC ? dtw(w.c, CONJ ? -s : s, d, sc) : dtw1(w.c, CONJ ? -s : s, d);
  if (MAYROT) {  // conj(i w') = -i conj(w')
    const DI u = CONJ ? dmul_mi(t) : dmul_i(t);
    t = k ? u : t;
  }
  return t;
}

// constant twiddle w_M^j (INV: its conjugate), M <= 64, 0 <= j < M/2 (ctw of ivm_v3.cuh)
template <bool INV>
__device__ __forceinline__ DI dctw(const DI &o, int j, int M) {
  if (j == 0) return o;
  if (4 * j == M) return INV ? dmul_mi(o) : dmul_i(o);
  if (4 * j < M) {
    const TwC<double> w = cw64<double>(j * (64 / M));
    return dtw1(w.c, INV ? -w.s : w.s, o);
  }
  const TwC<double> w = cw64<double>((j - M / 4) * (64 / M));
  const DI t = dtw1(w.c, INV ? -w.s : w.s, o);
  return INV ? dmul_mi(t) : dmul_i(t);
}

// radix-8 DIT in dit8's order (ivm_v3.cuh)
struct NoOp { __device__ __forceinline__ void operator()() const {} };
template <bool INV, typename IN, typename AL = NoOp>
__device__ __forceinline__ void ddit8(DI (&v)[8], IN &&in, AL &&loaded = AL()) {
  DI a0 = in(0), a1 = in(4);
  dbfly(a0, a1, DI(a1));
  DI a2 = in(2), a3 = in(6);
  dbfly(a2, a3, DI(a3));
  dbfly(a0, a2, DI(a2));
  dbfly(a1, a3, dctw<INV>(a3, 1, 4));
  DI a4 = in(1), a5 = in(5);
  dbfly(a4, a5, DI(a5));
  DI a6 = in(3), a7 = in(7);
  loaded();  // every input has been read
  dbfly(a6, a7, DI(a7));
  dbfly(a4, a6, DI(a6));
  dbfly(a5, a7, dctw<INV>(a7, 1, 4));
  dbfly(a0, a4, DI(a4));
  dbfly(a1, a5, dctw<INV>(a5, 1, 8));
  dbfly(a2, a6, dctw<INV>(a6, 2, 8));
  dbfly(a3, a7, dctw<INV>(a7, 3, 8));
  v[0] = a0, v[1] = a1, v[2] = a2, v[3] = a3, v[4] = a4, v[5] = a5, v[6] = a6, v[7] = a7;
}

// R-point DFT of DIT butterflies, R = 2, 4, 8 (cdft of ivm_v3.cuh)
template <int R, bool INV>
__device__ __forceinline__ void dcdft(DI (&v)[R]) {
  static_assert(R == 2 || R == 4 || R == 8, "radices");
  if constexpr (R == 8) {
    ddit8<INV>(v, [&](int q) { return v[q]; });
  } else if constexpr (R == 2) {
    dbfly(v[0], v[1], DI(v[1]));
  } else {
    DI a0 = v[0], a1 = v[2], a2 = v[1], a3 = v[3];
    dbfly(a0, a1, DI(a1));
    dbfly(a2, a3, DI(a3));
    dbfly(a0, a2, DI(a2));
    dbfly(a1, a3, dctw<INV>(a3, 1, 4));
    v[0] = a0, v[1] = a1, v[2] = a2, v[3] = a3;
  }
}

// state planes: centers (16 B) and radii (binary32, rounded up)
struct BufD {
  double2 *c;
  float *r;
  __device__ __forceinline__ DI ld(int i) const {
    const double2 v = c[i];
    return DI{v.x, v.y, (double)r[i]};
  }
  __device__ __forceinline__ void st(int i, const DI &z) const {
    c[i] = make_double2(z.cr, z.ci);
    r[i] = __double2float_ru(z.r);
  }
  __device__ __forceinline__ void st_conj(int i, const DI &z) const {
    c[i] = make_double2(z.cr, -z.ci);
    r[i] = __double2float_ru(z.r);
  }
};

template <int M> struct CfgD {
  using Gm = G3<M, 8>;
  static constexpr int N = Gm::N, THREADS = Gm::THREADS, CAP = Gm::CAP;
  static constexpr int MINB = 512 / THREADS < 1 ? 1 : 512 / THREADS;
  static constexpr size_t STATE_BYTES = (size_t)CAP * 16 + (size_t)CAP * 4;
  static constexpr size_t COEF_BYTES = 4 * (size_t)N;
  static constexpr size_t A_BYTES = (size_t)(N / 2) * 16 + (size_t)(N / 2) * 4;  // <= the rectangles' scratch
  static constexpr size_t TW_BYTES = sizeof(TwC<double>) * (size_t)Gm::SM_ENT();
  static constexpr size_t SMEM = STATE_BYTES + TW_BYTES;
  static_assert((size_t)CAP * 16 >= COEF_BYTES, "the coefficients alias the center plane");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

template <int M>
__global__ void __launch_bounds__(CfgD<M>::THREADS, CfgD<M>::MINB) ivm_d3_kernel(KParams kp) {
  using C = CfgD<M>;
  using Gm = G3<M, 8>;
  constexpr int N = C::N, R = 8;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Cert3 cs;
  __shared__ __align__(8) unsigned long long tbar, pbar;
#ifndef IVM_D3_NOSPLIT
  unsigned long long *wbar = &pbar;  // split write-after-read barrier of the mid passes (ivm_v3.cuh)
#else
  unsigned long long *wbar = nullptr;
#endif
  unsigned pph = 0u;
  BufD st{reinterpret_cast<double2 *>(smem), reinterpret_cast<float *>(smem + (size_t)C::CAP * 16)};
  int32_t *coef = reinterpret_cast<int32_t *>(smem);
  TwC<double> *twb = reinterpret_cast<TwC<double> *>(smem + C::STATE_BYTES);
  unsigned char *ab = reinterpret_cast<unsigned char *>(kp.ascratch) + (size_t)blockIdx.x * C::A_BYTES;
  BufD A{reinterpret_cast<double2 *>(ab), reinterpret_cast<float *>(ab + (size_t)(N / 2) * 16)};
  const TwC<double> *tw = reinterpret_cast<const TwC<double> *>(kp.tw);
  const int n = kp.n;
  constexpr int NFWD = RT3<M, R>::NFWD, NINV = RT3<M, R>::NINV;
  constexpr int RSI1 = Gm::iRS(1), SWI1 = Gm::iSW(1);
  constexpr unsigned FL_BYTES = sizeof(TwC<double>) * Gm::FLAST_ENT();
  constexpr bool LAST16 = RT3<M, R>::LAST16;
  constexpr unsigned L16_BYTES = LAST16 ? sizeof(TwC<double>) * R * Gm::LASTL() : 0;
  constexpr unsigned SMF_BYTES = sizeof(TwC<double>) * Gm::SMF_ENT(), SMI_BYTES = sizeof(TwC<double>) * Gm::SMI_ENT();
  constexpr int RATIO = 2 * N / Gm::LASTL();
  constexpr int QS = C::THREADS;
  constexpr double SCALE = 2.0 / (double)N;  // |omega| of the last pass's tables

  if (threadIdx.x == 0) {
    mbar_init(&tbar);
    const unsigned pa = (unsigned)__cvta_generic_to_shared(&pbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(pa), "r"((unsigned)(C::THREADS / 32)));
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x < kp.batch) {
    mbar_expect(&tbar, FL_BYTES + SMF_BYTES + SMI_BYTES);
    bulk_copy(twb, tw + Gm::tw_fwd(Gm::P.nf - 1), FL_BYTES, &tbar);
    if (SMF_BYTES) bulk_copy(twb + Gm::TWB_ENT(), tw + Gm::SMF_BEGIN(), SMF_BYTES, &tbar);
    if (SMI_BYTES) bulk_copy(twb + Gm::TWB_ENT() + Gm::SMF_ENT(), tw + Gm::SMI_BEGIN(), SMI_BYTES, &tbar);
  }
  if (blockIdx.x < kp.batch) mbar_wait(&tbar, 0);
  for (int pair = blockIdx.x; pair < kp.batch; pair += gridDim.x) {
    const int nxt = pair + (int)gridDim.x;
    if (nxt < kp.batch) {  // L2 prefetch of the next pair's digits
      for (int off = threadIdx.x * 128; off < n; off += blockDim.x * 128) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.a + (size_t)nxt * n + off));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.b + (size_t)nxt * n + off));
      }
    }
#pragma unroll 1
    for (int op = 0; op < 2; op++) {
      {  // pass 1 (ivm_v3.cuh fwd_first): x[nu + S' q] w_{4 R1}^q, R1-point DFT, mirror stores
        constexpr int R1 = Gm::P.f[1], G1 = R / R1, S = N / 2, Sp = S / R1, L = 2;
        constexpr int RSo = Gm::fRS(2), SWo = Gm::fSW(2);
        const uint8_t *dig = (op == 0 ? kp.a : kp.b) + (size_t)pair * n;
        auto in1 = [&](int nu, int q) {
          const int idx = nu + Sp * q;
          const double x = digit_val<double>(idx < n ? (unsigned)dig[idx] : 0u);
          if (q == 0) return DI{x, 0.0, 0.0};
          const TwC<double> w = cw64<double>(q * (16 / R1));
          DI p{__dmul_rn(w.c, x), __dmul_rn(w.s, x), 0.0};
          p.r = __fma_ru(x, DRW, __fma_ru(DU, l1(p), 2 * DETA));
          return p;
        };
#pragma unroll
        for (int g = 0; g < G1; g++) {
          const int nu = (int)threadIdx.x + g * Gm::TASKS;
          DI v[R1];
          if constexpr (R1 == 8) {
            ddit8<false>(v, [&](int q) { return in1(nu, q); });
          } else {
#pragma unroll
            for (int q = 0; q < R1; q++) v[q] = in1(nu, q);
            dcdft<R1, false>(v);
          }
#pragma unroll
          for (int r = 0; r < R1; r++) {
            if (r < R1 / 2) st.st(sidx(L * r, nu, RSo, SWo), v[r]);
            else st.st_conj(sidx(L * R1 - 1 - L * r, nu, RSo, SWo), v[r]);
          }
        }
      }
      if (op == 1 && threadIdx.x == 0) {
        cs.ok = 1;
        cs.first_bad = 0x7fffffff;
        cs.maxrad = 0ull;
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < NFWD; i++) {
        const PassRT pp = pick_fwd<M, R>(i);
        if (LAST16 && op == 0 && pp.big) mbar_wait(&tbar, 0);  // forward-last table restored
        const int Sp = 1 << pp.lgSp, t = (int)threadIdx.x;
        const int k0 = t >> pp.lgSp, nu = t & (Sp - 1);
        const int base = k0 * pp.RSi, sw = k0 & pp.SWi, tstride = pp.L >> 1;
        const TwC<double> *tp = twb + pp.tw + k0;
        DI v[R];
        ddit8<false>(v, [&](int q) {
          const DI z = st.ld(base + ((nu + Sp * q) ^ sw));
          if (q == 0) return z;
          const TwC<double> w = tp[(q - 1) * tstride];
          return (2 * q <= R) ? drt<false, false>(w, z) : drt<false, true>(w, z);
        }, [&]() {
          if (wbar && i < NFWD - 1) pb_arrive_warp(wbar);
        });
        if (i < NFWD - 1) {
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
        } else if (op == 0) {
#pragma unroll
          for (int r = 0; r < R; r++) A.st(r * (pp.L >> 1) + k0, v[r]);
        } else {  // pointwise product + inverse pass 0
          DI an = A.ld(k0);
          DI u[R];
          ddit8<true>(u, [&](int q) {
            const DI a = an;
            const int nq = dit8_next(q);
            if (nq >= 0) an = A.ld(nq * (pp.L >> 1) + k0);
            return dmul(a, v[q]);
          });
          __syncthreads();
          if (LAST16 && threadIdx.x == 0) {  // the folded inverse table replaces the forward-last one
            mbar_expect(&tbar, L16_BYTES);
            bulk_copy(twb, tw + Gm::tw_l16(), L16_BYTES, &tbar);
          }
#pragma unroll
          for (int r = 0; r < R; r++) st.st(sidx(r, k0, RSI1, SWI1), u[r]);
        }
        __syncthreads();
      }
    }
    CertAcc acc;
    acc.radius = kp.max_radius != nullptr;
#pragma unroll
    for (int i = 0; i < NINV; i++) {
      const PassRT pp = pick_inv<M, R>(i);
      const bool last = LAST16 && i == NINV - 1;
      if (last) mbar_wait(&tbar, 1);  // folded table
      const int Sp = 1 << pp.lgSp, lgH = pp.lgSp - 1, S = R * Sp, t = (int)threadIdx.x;
      const int k0 = t >> lgH, nu = t & ((Sp >> 1) - 1);
      const int base = k0 * pp.RSi, sw = k0 & pp.SWi;
      const TwC<double> *tp = twb + pp.tw + k0 + (last ? 0 : -pp.L);
      DI v[R];
      ddit8<true>(v, [&](int q) {
        const int qq = (2 * q < R) ? q : R - q;
        if (2 * q < R) {
          const DI z = st.ld(base + ((nu + Sp * q) ^ sw));
          if (q == 0 && !last) return z;
          const TwC<double> w = tp[q * pp.L];
          if (last) return drt<true, true, true>(w, z, SCALE);
          return (4 * qq > R) ? drt<true, true>(w, z) : drt<true, false>(w, z);
        }
        // the mirror's conjugate times the twiddle (rtmul_cd of ivm_v3.cuh)
        const DI d = dconj(st.ld(base + ((S - 1 - nu - Sp * q) ^ sw)));
        const TwC<double> w = tp[q * pp.L];
        if (last) return drt<false, true, true>(w, d, SCALE);
        return (4 * qq > R) ? drt<false, true>(w, d) : drt<false, false>(w, d);
      }, [&]() {
        if (wbar && !last) pb_arrive_warp(wbar);
      });
      // every input loaded (last pass: the coefficients may overwrite the state)
      if (wbar && !last) {
        mbar_wait(wbar, pph);
        pph ^= 1u;
      } else {
        __syncthreads();
      }
      if (last) {
#pragma unroll
        for (int r = 0; r < R; r++) {
          const int k = k0 + pp.L * r;
          const DI w = dctw<true>(v[r], r, RATIO);  // the remaining untwist z^{-L r} (emit_fold)
          certify_real<double, int32_t, false>(__dadd_rd(w.cr, -w.r), __dadd_ru(w.cr, w.r), k, n, coef + cpos<QS>(k), acc,
                                               nullptr);
          certify_real<double, int32_t, false>(__dadd_rd(w.ci, -w.r), __dadd_ru(w.ci, w.r), k + N / 2, n,
                                               coef + cpos<QS>(k + N / 2), acc, nullptr);
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; r++) st.st(sidx(k0 + pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
      }
      __syncthreads();
    }
    if constexpr (!LAST16) {  // last inverse pass of radix 2 or 4 (ivm_v3.cuh inv_last), tables from L2
      constexpr int p = Gm::P.ni - 1, Q = Gm::P.q[p], L = iL(Gm::P, p), S = N / L, Sp = S / Q, G = R / Q;
      constexpr int H = Sp / 2, RSi = Gm::iRS(p), SWi = Gm::iSW(p), TW = Gm::tw_inv(p), TWF = Gm::tw_fin();
      static_assert(Gm::TASKS * G == L * H, "every thread has G tasks");
      DI v[G][Q];
      int k0s[G];
#pragma unroll
      for (int g = 0; g < G; g++) {
        const int t = (int)threadIdx.x + g * Gm::TASKS;
        const int k0 = t / H, nu = t % H;
        k0s[g] = k0;
#pragma unroll
        for (int q = 0; q < Q; q++) {
          if (2 * q < Q) {
            const DI z = st.ld(sidx(k0, nu + Sp * q, RSi, SWi));
            v[g][q] = q > 0 ? drt<true, true>(ldg_twc(tw, TW + (q - 1) * L + k0), z) : z;
          } else {
            const DI d = dconj(st.ld(sidx(k0, S - 1 - nu - Sp * q, RSi, SWi)));
            v[g][q] = drt<false, true>(ldg_twc(tw, TW + (q - 1) * L + k0), d);
          }
        }
        dcdft<Q, true>(v[g]);
      }
      __syncthreads();  // every input loaded: the coefficients may overwrite the state
#pragma unroll
      for (int g = 0; g < G; g++) {
#pragma unroll
        for (int r = 0; r < Q; r++) {
          const int k = k0s[g] + L * r;
          // (2/m) z^{-k}: the conjugate of the (scaled) table entry (emit_coeffs)
          const DI w = drt<true, true, true>(ldg_twc(tw, TWF + k), v[g][r], SCALE);
          certify_real<double, int32_t, false>(__dadd_rd(w.cr, -w.r), __dadd_ru(w.cr, w.r), k, n, coef + cpos<QS>(k), acc,
                                               nullptr);
          certify_real<double, int32_t, false>(__dadd_rd(w.ci, -w.r), __dadd_ru(w.ci, w.r), k + N / 2, n,
                                               coef + cpos<QS>(k + N / 2), acc, nullptr);
        }
      }
      __syncthreads();
    }
    cert_flush(acc, cs);
    __syncthreads();
    if (LAST16 && threadIdx.x == 0 && nxt < kp.batch) {  // restore the forward-last table
      mbar_expect(&tbar, FL_BYTES);
      bulk_copy(twb, tw + Gm::tw_fwd(Gm::P.nf - 1), FL_BYTES, &tbar);
    }
    const bool certified = cs.ok != 0;
    carry_store4<QS>(coef, n, kp.prod + (size_t)pair * 2 * n, certified);
    if (threadIdx.x == 0) {
      kp.cert[pair] = certified ? 1 : 0;
      if (kp.max_radius) kp.max_radius[pair] = __longlong_as_double((long long)cs.maxrad);
    }
    __syncthreads();
  }
}

}  // namespace d3
}  // namespace ivm
