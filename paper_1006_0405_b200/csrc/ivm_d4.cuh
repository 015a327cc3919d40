// ivm_d4.cuh -- circular containment sets (R15) on the cluster
// schedule of ivm_v4.cuh: fp64, m = 2^14 .. 2^16, one thread-block cluster of
// C = m/8192 CTAs per multiplication, digits staged by bulk copies when every row
// is 16-byte aligned, else read through L2.
// Included by ivm_v4.cu after ivm_v4.cuh and ivm_d3.cuh.
//
// Same row split, role tables, passes, exchanges, certificate and carry as
// ivm_v4_kernel; the element is a disc (arithmetic: ivm_d3.cuh).  The cross pass
// fused with local pass 1 (cross_pass1) sums x_q Theta[j][q] over the C digit
// terms of input j: the center by a chain of round-to-nearest FMAs (partial sum k
// has |re|, |im| <= S1_k = sum_{q<=k} x_q, so the roundings cost at most
// U sum_k S1_k in modulus), the table centers are within RW of the true roots of
// unity (another RW S1): r = RW S1 + U sum_k S1_k, rounded up.
#pragma once

namespace ivm {
namespace d4 {

using namespace v3;
using namespace v4;
using namespace d3;

__device__ __forceinline__ float dsm_ld_f32(unsigned a) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}

template <int M> struct CfgD4 {
  using GL = G3<13, 8>;
  static_assert(M >= 14 && M <= 16, "C = 2, 4, 8; the digits of one operand staged (they fit beside the 80 KB disc state)");
  static constexpr int THREADS = 512;
  static constexpr size_t STATE_BYTES = (size_t)GL::CAP * 16 + (size_t)GL::CAP * 4;
  static constexpr size_t TW_BYTES = sizeof(TwC<double>) * (size_t)G4<M>::S_ENT;
  static constexpr size_t DIG_BYTES = (size_t)(1 << M) / 2;
  static constexpr size_t SMEM = STATE_BYTES + TW_BYTES + DIG_BYTES;
  static constexpr size_t A_BYTES = (size_t)4096 * 16 + (size_t)4096 * 4;
  static_assert(sizeof(TwC<double>) * 4096 >= 4 * 8192, "local coefficients fit the twiddle swap buffer");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

template <int M>
__global__ void __launch_bounds__(512, 1) ivm_d4_kernel(KParams kp) {
  using X = G4<M>;
  using GL = G3<13, 8>;
  using CF = CfgD4<M>;
  constexpr int C = X::C, B = X::B, R = 8, N = 1 << M;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Cert3 cs;
  __shared__ unsigned s_chunk[2 * (1 << (M - 13))][2];
  __shared__ unsigned s_cin[4];
  __shared__ __align__(8) unsigned long long tbar, dbar;
  BufD st{reinterpret_cast<double2 *>(smem), reinterpret_cast<float *>(smem + (size_t)GL::CAP * 16)};
  TwC<double> *twb = reinterpret_cast<TwC<double> *>(smem + CF::STATE_BYTES);
  int32_t *coefL = reinterpret_cast<int32_t *>(twb + X::S_SWAP);
  uint8_t *sdig = smem + CF::STATE_BYTES + CF::TW_BYTES;
  const unsigned crank = cluster_rank();
  const int cid = (int)(blockIdx.x / C), ncl = (int)(gridDim.x / C);
  const TwC<double> *tw = reinterpret_cast<const TwC<double> *>(kp.tw);
  unsigned char *ab = reinterpret_cast<unsigned char *>(kp.ascratch) + (size_t)blockIdx.x * CF::A_BYTES;
  BufD A{reinterpret_cast<double2 *>(ab), reinterpret_cast<float *>(ab + (size_t)4096 * 16)};
  const int n = kp.n, nc = 2 * n - 1, nout = 2 * n;
  constexpr int RSI1 = GL::iRS(1), SWI1 = GL::iSW(1);
  constexpr unsigned EB = sizeof(TwC<double>);
  constexpr double SCALE = 2.0 / (double)N;

  if (threadIdx.x == 0) {
    mbar_init(&tbar);
    mbar_init(&dbar);
  }
  __syncthreads();
  const bool staged = n % 16 == 0 && ((reinterpret_cast<uintptr_t>(kp.a) | reinterpret_cast<uintptr_t>(kp.b)) % 16) == 0;
  if (threadIdx.x == 0 && cid < kp.batch) {
    mbar_expect(&tbar, EB * (X::FLAST + X::MF_ENT + X::MI_ENT + 2 * C + 16 * C));
    bulk_copy(twb + X::S_SWAP, tw + X::FWD(crank) + X::FP(4), EB * X::FLAST, &tbar);
    bulk_copy(twb + X::S_MF, tw + X::FWD(crank), EB * X::MF_ENT, &tbar);
    bulk_copy(twb + X::S_MI, tw + X::INV, EB * X::MI_ENT, &tbar);
    bulk_copy(twb + X::S_TH, tw + X::TH(crank), EB * 2 * C, &tbar);
    bulk_copy(twb + X::S_TH1, tw + X::TH1(crank), EB * 16 * C, &tbar);
    if (staged) {
      mbar_expect(&dbar, (unsigned)n);  // operand a of the first pair (dbar phases: a = even, b = odd)
      bulk_copy(sdig, kp.a + (size_t)cid * n, (unsigned)n, &dbar);
    }
  }
  if (cid < kp.batch) mbar_wait(&tbar, 0);
  // tbar phases per pair it: 3 it (forward-last), 3 it + 1 (inverse pass 3), 3 it + 2 (last inverse pass)

  int it = 0;
  for (int pair = cid; pair < kp.batch; pair += ncl, it++) {
    const unsigned par = (unsigned)it & 1u;
    if (!staged && pair + ncl < kp.batch) {  // L2 prefetch of the next pair's digits
      const int nxt = pair + ncl;
      for (int off = (int)threadIdx.x * 128; off < n; off += (int)blockDim.x * 128) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.a + (size_t)nxt * n + off));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.b + (size_t)nxt * n + off));
      }
    }
#pragma unroll 1
    for (int op = 0; op < 2; op++) {
      if (staged) mbar_wait(&dbar, (unsigned)op);
      const uint8_t *dsrc = staged ? sdig : (op == 0 ? kp.a : kp.b) + (size_t)pair * n;
      {  // the cross pass fused with local pass 1 (cross_pass1), stored in the pass-2 layout
        const PassRT pp = pick_fwd4<M>(0);
        // TH1: [8 j][C q] full intervals (rl, rh, il, ih); the lower corner is the center
        const double4 *th1 = reinterpret_cast<const double4 *>(twb + X::S_TH1);
        const int t = (int)threadIdx.x;
        DI v[R];
        ddit8<false>(v, [&](int j) {
          double cr = 0.0, ci = 0.0;
          unsigned s1 = 0u, ss = 0u;  // S1 and the sum of its partial sums S1_k
#pragma unroll
          for (int q = 0; q < C; q++) {
            const double4 th = th1[j * C + q];
            const int idx = t + 512 * j + 4096 * q;
            const unsigned d = idx < n ? (unsigned)dsrc[idx] : 0u;
            const double x = digit_val<double>(d);
            s1 += d;
            ss += s1;
            cr = __fma_rn(x, th.x, cr);
            ci = __fma_rn(x, th.z, ci);
          }
          // RW S1 + U sum_k S1_k (partial sum k is bounded by S1_k per part), rounded up
          return DI{cr, ci, __dmul_ru(__fma_ru((double)ss, DU, __dmul_ru((double)s1, DRW)), 1.0 + 0x1p-40)};
        });
        if (op == 0 && it > 0) cluster_wait();  // the previous pair's remote reads of this state are done
        const int nu = t;
#pragma unroll
        for (int r = 0; r < R; r++) {
          if (2 * r < R) st.st(sidx(pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
          else st.st_conj(sidx(R * pp.L - 1 - pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
        }
      }
      if (op == 0 && it > 0 && threadIdx.x == 0) {
        mbar_expect(&tbar, EB * X::FLAST);
        bulk_copy(twb + X::S_SWAP, tw + X::FWD(crank) + X::FP(4), EB * X::FLAST, &tbar);
      }
      if (op == 1 && threadIdx.x == 0) {
        cs.ok = 1;
        cs.first_bad = 0x7fffffff;
        cs.maxrad = 0ull;
      }
      __syncthreads();
      if (staged && threadIdx.x == 0) {  // the next operand: b of this pair, or a of the next
        const uint8_t *nx = op == 0 ? kp.b + (size_t)pair * n : kp.a + (size_t)(pair + ncl) * n;
        if (op == 0 || pair + ncl < kp.batch) {
          mbar_expect(&dbar, (unsigned)n);
          bulk_copy(sdig, nx, (unsigned)n, &dbar);
        }
      }
#pragma unroll
      for (int i = 1; i < 4; i++) {
        const PassRT pp = pick_fwd4<M>(i);
        if (op == 0 && i == 3) mbar_wait(&tbar, par);  // forward-last table of this role
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
        });
        if (i < 3) {
          __syncthreads();
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
          if (threadIdx.x == 0) {  // inverse pass 3 table replaces the forward-last one
            mbar_expect(&tbar, EB * X::FLAST);
            bulk_copy(twb + X::S_SWAP, tw + X::INV + X::INV3, EB * X::FLAST, &tbar);
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
    for (int i = 0; i < 3; i++) {
      const PassRT pp = pick_inv4<M>(i);
      if (i == 2) mbar_wait(&tbar, par ^ 1u);
      const int Sp = 1 << pp.lgSp, lgH = pp.lgSp - 1, S = R * Sp, t = (int)threadIdx.x;
      const int k0 = t >> lgH, nu = t & ((Sp >> 1) - 1);
      const int base = k0 * pp.RSi, sw = k0 & pp.SWi;
      const TwC<double> *tp = twb + pp.tw + k0 - pp.L;
      DI v[R];
      ddit8<true>(v, [&](int q) {
        const int qq = (2 * q < R) ? q : R - q;
        if (2 * q < R) {
          const DI z = st.ld(base + ((nu + Sp * q) ^ sw));
          if (q == 0) return z;
          const TwC<double> w = tp[q * pp.L];
          return (4 * qq > R) ? drt<true, true>(w, z) : drt<true, false>(w, z);
        }
        const DI d = dconj(st.ld(base + ((S - 1 - nu - Sp * q) ^ sw)));
        const TwC<double> w = tp[q * pp.L];
        return (4 * qq > R) ? drt<false, true>(w, d) : drt<false, false>(w, d);
      });
      __syncthreads();
      if (i == 2 && threadIdx.x == 0) {  // the last inverse pass table (this role's rows) streams in
        mbar_expect(&tbar, EB * 4096);
        bulk_copy(twb + X::S_SWAP, tw + X::XINV(crank), EB * 4096, &tbar);
      }
#pragma unroll
      for (int r = 0; r < R; r++) st.st(sidx(k0 + pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
      __syncthreads();
    }
    cluster_sync();  // (1) every CTA's column of the 4096 rows is in its shared memory
    {
      constexpr int G = 8 / C;  // rows (tasks) per thread
      DI v[G][C];
      const unsigned c0 = (unsigned)__cvta_generic_to_shared(st.c), r0 = (unsigned)__cvta_generic_to_shared(st.r);
#pragma unroll
      for (int g = 0; g < G; g++) {
        const int k0 = (int)crank * B + (int)threadIdx.x + 512 * g;
#pragma unroll
        for (int q = 0; q < C; q++) {
          const unsigned src = (2 * q < C) ? (unsigned)(2 * q) : (unsigned)(2 * C - 1 - 2 * q);
          const double2 cc = dsm_ld(dsm_map_addr(c0 + 16u * (unsigned)k0, src), (double2 *)nullptr);
          const float rr = dsm_ld_f32(dsm_map_addr(r0 + 4u * (unsigned)k0, src));
          v[g][q] = DI{cc.x, cc.y, (double)rr};
        }
      }
      mbar_wait(&tbar, par);
#pragma unroll
      for (int g = 0; g < G; g++) {
        const int kl = (int)threadIdx.x + 512 * g;
#pragma unroll
        for (int q = 0; q < C; q++) {
          const TwC<double> w = twb[X::S_SWAP + q * B + kl];
          v[g][q] = (2 * q < C) ? drt<true, true, true>(w, v[g][q], SCALE) : drt<false, true, true>(w, dconj(v[g][q]), SCALE);
        }
        dcdft<C, true>(v[g]);
      }
      __syncthreads();  // every twiddle read: the swap buffer takes the coefficients
#pragma unroll
      for (int g = 0; g < G; g++) {
        const int kl = (int)threadIdx.x + 512 * g, k0 = (int)crank * B + kl;
#pragma unroll
        for (int r = 0; r < C; r++) {
          const int k = k0 + 4096 * r;
          const DI w = dctw<true>(v[g][r], r, 4 * C);  // the remaining untwist z^{-4096 r} (emit_fold)
          certify_real<double, int32_t, false>(__dadd_rd(w.cr, -w.r), __dadd_ru(w.cr, w.r), k, n,
                                               coefL + r * B + cpos<B / 16>(kl), acc, nullptr);
          certify_real<double, int32_t, false>(__dadd_rd(w.ci, -w.r), __dadd_ru(w.ci, w.r), k + N / 2, n,
                                               coefL + (C + r) * B + cpos<B / 16>(kl), acc, nullptr);
        }
      }
    }
    cert_flush(acc, cs);
    __syncthreads();
    cluster_sync();  // (3) coefficients and per-CTA certificates complete
    __shared__ int s_ok, s_bad;
    __shared__ unsigned long long s_rad;
    if (threadIdx.x < 32) {
      int okl = 1, badl = 0x7fffffff;
      unsigned long long radl = 0ull;
      if ((int)threadIdx.x < C) {
        okl = dsm_ld_i32(dsm_map(&cs.ok, threadIdx.x));
        badl = dsm_ld_i32(dsm_map(&cs.first_bad, threadIdx.x));
        radl = dsm_ld_u64(dsm_map(&cs.maxrad, threadIdx.x));
      }
      okl = (int)__reduce_and_sync(0xffffffffu, (unsigned)okl);
      badl = __reduce_min_sync(0xffffffffu, badl);
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long r2 = __shfl_xor_sync(0xffffffffu, radl, o);
        radl = r2 > radl ? r2 : radl;
      }
      if (threadIdx.x == 0) {
        s_ok = okl;
        s_bad = badl;
        s_rad = radl;
      }
    }
    __syncthreads();
    const int ok = s_ok;
    const unsigned long long rad = s_rad;
    // the carry of ivm_v4_kernel (chunks of B coefficients, Carry4, cluster adder)
    constexpr int NCH = 2 * C, WB = B / 4, TPC = WB / 4, NCHT = 2 * C * C;
    static_assert(NCH * TPC == 512, "one thread per four words");
    const int lc = (int)threadIdx.x / TPC, tc = (int)threadIdx.x % TPC, ch = lc * C + (int)crank;
    const int words = (nout + 3) / 4;
    uint8_t *out = kp.prod + (size_t)pair * nout;
    __shared__ unsigned s_w[16];
    Carry4<TPC> cy;
    if (ok) {
      const unsigned cbase = (unsigned)__cvta_generic_to_shared(coefL);
      unsigned long long V[6];
#pragma unroll
      for (int j = 0; j < 6; j++) {
        const int wj = 4 * tc - 2 + j;
        const int gi = ch * B + 4 * wj;
        V[j] = 0ull;
        if (wj >= 0) {
          const int4 q = *reinterpret_cast<const int4 *>(coefL + lc * B + cpos<TPC>(4 * wj));
          V[j] = word_of((unsigned)q.x, (unsigned)q.y, (unsigned)q.z, (unsigned)q.w, gi, nc);
        } else if (ch > 0) {
          const int pc = ch - 1;
          const int4 q = dsm_ld_i4(dsm_map_addr(cbase + 4u * (unsigned)((pc / C) * B + cpos<TPC>(4 * (WB + wj))),
                                                (unsigned)(pc % C)));
          V[j] = word_of((unsigned)q.x, (unsigned)q.y, (unsigned)q.z, (unsigned)q.w, gi, nc);
        }
      }
      cy.words(V);
      unsigned cb;
      if constexpr (TPC > 32) {
        if ((threadIdx.x & 31u) == 0u) s_w[threadIdx.x >> 5] = cy.seg_bits();
        __syncthreads();
        cb = Carry4<TPC>::chunk_bits(s_w);
      } else {
        cb = cy.seg_bits();
      }
      if (tc == 0) {
        s_chunk[lc][0] = cb & 1u;
        s_chunk[lc][1] = cb >> 1;
      }
    }
    cluster_sync();  // (4) every chunk's generate / all-propagate published
    if (ok) {
      if (threadIdx.x < 32) {
        unsigned G[4], P[4];
#pragma unroll
        for (int w = 0; w < 4; w++) {
          const int q = 32 * w + (int)threadIdx.x;
          bool g = false, pq = true;
          if (q < NCHT) {
            g = dsm_ld_i32(dsm_map(&s_chunk[q / C][0], (unsigned)(q % C))) != 0;
            pq = dsm_ld_i32(dsm_map(&s_chunk[q / C][1], (unsigned)(q % C))) != 0;
          }
          G[w] = __ballot_sync(0xffffffffu, g);
          P[w] = __ballot_sync(0xffffffffu, pq);
        }
        if (threadIdx.x == 0) {
          unsigned long long cyc = 0ull;
#pragma unroll
          for (int w = 0; w < 4; w++) {
            const unsigned long long S = (unsigned long long)(G[w] | P[w]) + G[w] + cyc;
            s_cin[w] = (unsigned)S ^ P[w];
            cyc = S >> 32;
          }
        }
      }
      __syncthreads();
      const unsigned cin = (s_cin[ch >> 5] >> (ch & 31)) & 1u;
      unsigned d[4];
      cy.digits(cy.lane_cin(cin, s_w), d);
      const int k0 = ch * WB + 4 * tc;
      if (k0 < words) store_words4(out, k0, nout, d);
    } else {
      for (int i = ch * B + 4 * tc; i < min(ch * B + B, nout); i += 4 * TPC)
        for (int b = 0; b < 4 && i + b < nout; b++) out[i + b] = 0;
    }
    if (crank == 0 && threadIdx.x == 0) {
      kp.cert[pair] = ok ? 1 : 0;
      if (kp.max_radius) kp.max_radius[pair] = __longlong_as_double((long long)rad);
    }
    cluster_arrive_release();  // (5) remote reads done before the next pair overwrites them
  }
  if (it > 0) cluster_wait();
}

}  // namespace d4
}  // namespace ivm
