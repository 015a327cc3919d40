// ivm_d7.cuh -- circular containment sets (R15) on the pipelined
// group schedule of ivm_v7.cuh: fp64, m = 2^17, 2^18 (C = 16, 32 tasks per
// multiplication).  Included by ivm_v5.cu after ivm_v7.cuh and ivm_d3.cuh.
//
// Same task split, stages (L / A / Cs), counters, ring, tables, certificate and
// carry as ivm_v7_kernel; the element is a disc (arithmetic: ivm_d3.cuh).  The
// exchange keeps 32-byte slots (center, radius, pad), so the scratch layout is
// ivm_v7.cuh's.  The tensor-core cross pass gives the exact integer sums S of
// digits times round(theta 2^54); the center is S 2^-54 rounded once per part
// (error <= 2^-53 S1 each, S1 = sum_q x_q bounding both parts) and theta is within
// 3 2^-55 of its integer form per part, so r = S1 (2^-52 + 3 2^-54), rounded up.
#pragma once

namespace ivm {
namespace d7 {

using namespace v3;
using namespace v4;
using namespace v5;
using namespace v7;
using namespace d3;

template <int M> struct CfgD7 {
  using GL = G3<13, 8>;
  static constexpr int THREADS = 512;
  static constexpr size_t STATE_BYTES = (size_t)GL::CAP * 16 + (size_t)GL::CAP * 4;
  static constexpr int S_ENT = G4<M>::S_FO + 2 * G4<M>::C;
  static constexpr size_t TW_BYTES = sizeof(TwC<double>) * (size_t)S_ENT;
  static constexpr size_t SMEM = STATE_BYTES + TW_BYTES;
  static constexpr size_t A_BYTES = (size_t)4096 * 16 + (size_t)4096 * 4;
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

struct XD { double2 c, r; };  // exchange slot: center, (radius, pad)
__device__ __forceinline__ void st_xd(XD *p, const DI &z) {
  p->c = make_double2(z.cr, z.ci);
  p->r = make_double2(z.r, 0.0);
}
__device__ __forceinline__ DI ldcg_xd(const XD *p) {
  const double2 c = __ldcg(&p->c), r = __ldcg(&p->r);
  return DI{c.x, c.y, r.x};
}

// the tensor-core cross pass (cross_tc of ivm_v5.cuh, word loads) with disc outputs
template <int M, bool WORDS>
__device__ __forceinline__ void cross_tc_d(const uint8_t *__restrict__ dig, int n, BufD st, const void *limbs,
                                           unsigned crank) {
  constexpr int C = G4<M>::C;
  unsigned bf[8];
  tc_limbs(limbs, crank, bf);
  const bool odd = (crank & 1u) != 0u;
  const int lane = (int)(threadIdx.x & 31u), warp = (int)(threadIdx.x >> 5), g = lane >> 2, t = lane & 3;
  const bool rowhi = t >= 2, im = (t & 1) != 0;
  double *cpl = reinterpret_cast<double *>(st.c);
  unsigned nx[4][4];
  tc_load_group<C, WORDS>(dig, n, warp * 256, g, t, nx);
#pragma unroll 1
  for (int grp = 0; grp < 4; grp++) {
    const int vb = warp * 256 + grp * 64;
    unsigned a[4][4];
#pragma unroll
    for (int r = 0; r < 4; r++) tr4x4(nx[r][0], nx[r][1], nx[r][2], nx[r][3], a[r]);
    if (grp < 3) tc_load_group<C, WORDS>(dig, n, vb + 64, g, t, nx);
#pragma unroll
    for (int j = 0; j < 4; j++) {
      int x[4][2];
#pragma unroll
      for (int s = 0; s < 4; s++) {
        int d[4];
        mma_u8s8(d, a[0][j], a[1][j], a[2][j], a[3][j], bf[2 * s], bf[2 * s + 1]);
        x[s][0] = rowhi ? d[2] : d[0];
        x[s][1] = rowhi ? d[3] : d[1];
      }
      const long long Lo = (long long)(x[0][0] + 256 * x[0][1]) + 65536ll * (long long)(x[1][0] + 256 * x[1][1]);
      const long long H = (long long)(x[2][0] + 256 * x[2][1]) + 65536ll * (long long)x[3][0];
      // S 2^-54 = H 2^-22 + Lo 2^-54 (both exact), one rounding
      const double cv = __fma_rn((double)H, 2.384185791015625e-07, (double)Lo * 5.551115123125783e-17);
      const int v = vb + (rowhi ? 32 : 0) + 4 * g + j;
      cpl[2 * v + (im ? 1 : 0)] = (im && odd) ? -cv : cv;
      if (!im) st.r[v] = __double2float_ru(__dmul_ru((double)x[3][1], (0x1p-52 + 3 * 0x1p-54) * (1.0 + 0x1p-40)));
    }
  }
}

template <int M>
__global__ void __launch_bounds__(512, 1) ivm_d7_kernel(KParams kp, Pipe7 g) {
  using T = double;
  using X = G4<M>;
  using GL = G3<13, 8>;
  using CF = CfgD7<M>;
  using V = double2;
  constexpr int C = X::C, B = X::B, R = 8, NL = 8192, N = 1 << M;
  static_assert(C == 16 || C == 32, "two-stage last pass, tensor-core cross pass");
  constexpr int C2 = C / 8;
  constexpr int NCH = 2 * C, NCHT = 2 * C * C, WB = B / 4;
  constexpr int TPC = WB / 4;  // threads per chunk, four words each (Carry4)
  static_assert(NCH * TPC == 512 && TPC < 32, "one thread per four words, chunks inside a warp");
  static_assert(sizeof(TwC<T>) * 4096 >= 8 * (size_t)(NCH * B), "the coefficients fit the swap buffer");
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Cert3 cs;
  __shared__ __align__(8) unsigned long long tbar;
  __shared__ int s_ok, s_bad;
  __shared__ unsigned long long s_rad;
  __shared__ uint8_t s_cin[64];
  __shared__ unsigned s_din[64], s_wgp[4];
  BufD st{reinterpret_cast<double2 *>(smem), reinterpret_cast<float *>(smem + (size_t)GL::CAP * 16)};
  TwC<T> *twb = reinterpret_cast<TwC<T> *>(smem + CF::STATE_BYTES);
  const TwC<T> *s2tw = twb + X::S_S2;  // w_C^{-j}: s2tw[2 j], upper-half form
  const TwC<T> *fold = twb + X::S_FO;  // fold[2 r] = z^{4096 r}
  long long *coefL = reinterpret_cast<long long *>(twb + X::S_SWAP);
  const TwC<T> *tw = reinterpret_cast<const TwC<T> *>(kp.tw);
  unsigned char *ab = reinterpret_cast<unsigned char *>(kp.ascratch) + (size_t)blockIdx.x * CF::A_BYTES;
  BufD A{reinterpret_cast<double2 *>(ab), reinterpret_cast<float *>(ab + (size_t)4096 * 16)};
  constexpr double SCALE = 2.0 / (double)N;
  const int n = kp.n, nc = 2 * n - 1, nout = 2 * n;
  const int P = (int)gridDim.x, NT = kp.batch * C;
  const int K = (int)blockIdx.x < NT ? (NT - 1 - (int)blockIdx.x) / P + 1 : 0;
  constexpr int RSI1 = GL::iRS(1), SWI1 = GL::iSW(1);
  constexpr unsigned EB = sizeof(TwC<T>);
  unsigned tph = 0;  // phases of tbar waited so far (issue and wait strictly alternate)

  if (threadIdx.x == 0) mbar_init(&tbar);
  __syncthreads();
  if (K == 0) return;
  if (threadIdx.x == 0) {  // resident tables and the first task's role tables
    const unsigned role = blockIdx.x % C;
    mbar_expect(&tbar, EB * (X::FLAST + X::MF_ENT + X::MI_ENT + 4 * C));
    bulk_copy(twb + X::S_SWAP, tw + X::FWD(role) + X::FP(4), EB * X::FLAST, &tbar);
    bulk_copy(twb + X::S_MF, tw + X::FWD(role), EB * X::MF_ENT, &tbar);
    bulk_copy(twb + X::S_MI, tw + X::INV, EB * X::MI_ENT, &tbar);
    bulk_copy(twb + X::S_S2, tw + X::S2, EB * 4 * C, &tbar);  // S2 and FO are adjacent
  }
  IVM_PH_DECL
#pragma unroll 1
  for (int k = 0; k < K + 2; k++) {
    // ================= L stage: task t_k =================
    if (k < K) {
      const int t = (int)blockIdx.x + P * k, pair = t / C;
      const unsigned role = (unsigned)(t % C);
      const int slot = pair % g.rp;
      if (pair >= g.rp) await7(g.cnt + 4 * (pair - g.rp) + 2, C);  // the ring slot is free
      IVM_PH(12);
      XD *xch = reinterpret_cast<XD *>(g.xch) + (size_t)slot * C * 4096;
      if (t + P < NT) {  // L2 prefetch of this role's slice of the next task's digits
        const int nxt = (t + P) / C, nrole = (t + P) % C, sl = (n + C - 1) / C;
        for (int off = nrole * sl + (int)threadIdx.x * 128; off < min(n, (nrole + 1) * sl); off += (int)blockDim.x * 128) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.a + (size_t)nxt * n + off));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.b + (size_t)nxt * n + off));
        }
      }
#pragma unroll 1
      for (int op = 0; op < 2; op++) {
        {  // word loads when every row is word-aligned, else byte loads
          const uint8_t *dg = (op == 0 ? kp.a : kp.b) + (size_t)pair * n;
          if (((reinterpret_cast<uintptr_t>(dg) | (uintptr_t)n) & 3) == 0) cross_tc_d<M, true>(dg, n, st, tw + X::LIMB, role);
          else cross_tc_d<M, false>(dg, n, st, tw + X::LIMB, role);
        }
        __syncthreads();
        IVM_PH(2 * op);
#pragma unroll  // (specialised per pass: addresses fold into immediates)
        for (int i = 0; i < 4; i++) {
          const PassRT pp = pick_fwd4<M>(i);
          if (op == 0 && i == 0) mbar_wait(&tbar, (tph++) & 1u);  // this role's tables
          const int Sp = 1 << pp.lgSp, t_ = (int)threadIdx.x;
          const int k0 = t_ >> pp.lgSp, nu = t_ & (Sp - 1);
          const int base = k0 * pp.RSi, sw = k0 & pp.SWi, tstride = pp.L >> 1;
          const TwC<T> *tp = twb + pp.tw + k0;
          DI v[R];
          ddit8<false>(v, [&](int q) {
            const DI z = st.ld(base + ((nu + Sp * q) ^ sw));
            if (q == 0) return z;
            const TwC<T> w = tp[(q - 1) * tstride];
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
          } else {
            DI an = A.ld(k0);
            DI u[R];
            ddit8<true>(u, [&](int q) {
              const DI a = an;
              const int nq = dit8_next(q);
              if (nq >= 0) an = A.ld(nq * (pp.L >> 1) + k0);
              return dmul(a, v[q]);
            });
#pragma unroll
            for (int r = 0; r < R; r++) v[r] = u[r];
            __syncthreads();
            if (threadIdx.x == 0) {
              mbar_expect(&tbar, EB * X::FLAST);
              bulk_copy(twb + X::S_SWAP, tw + X::INV + X::INV3, EB * X::FLAST, &tbar);
            }
#pragma unroll
            for (int r = 0; r < R; r++) st.st(sidx(r, k0, RSI1, SWI1), v[r]);
          }
          __syncthreads();
        }
        IVM_PH(2 * op + 1);
      }
#pragma unroll
      for (int i = 0; i < 3; i++) {
        const PassRT pp = pick_inv4<M>(i);
        if (i == 2) mbar_wait(&tbar, (tph++) & 1u);
        const int Sp = 1 << pp.lgSp, lgH = pp.lgSp - 1, S = R * Sp, t_ = (int)threadIdx.x;
        const int k0 = t_ >> lgH, nu = t_ & ((Sp >> 1) - 1);
        const int base = k0 * pp.RSi, sw = k0 & pp.SWi;
        const TwC<T> *tp = twb + pp.tw + k0 - pp.L;
        DI v[R];
        ddit8<true>(v, [&](int q) {
          const int qq = (2 * q < R) ? q : R - q;
          if (2 * q < R) {
            const DI z = st.ld(base + ((nu + Sp * q) ^ sw));
            if (q == 0) return z;
            const TwC<T> w = tp[q * pp.L];
            return (4 * qq > R) ? drt<true, true>(w, z) : drt<true, false>(w, z);
          }
          const DI d = dconj(st.ld(base + ((S - 1 - nu - Sp * q) ^ sw)));
          const TwC<T> w = tp[q * pp.L];
          return (4 * qq > R) ? drt<false, true>(w, d) : drt<false, false>(w, d);
        });
        if (i < 2) {
          __syncthreads();
#pragma unroll
          for (int r = 0; r < R; r++) st.st(sidx(k0 + pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
          __syncthreads();
        } else {  // last local pass: the column goes to the pair's exchange (row k0 + L r)
#pragma unroll
          for (int r = 0; r < R; r++) st_xd(xch + (size_t)role * 4096 + k0 + pp.L * r, v[r]);
        }
      }
      __syncthreads();
      post7(g.cnt + 4 * pair + 0);
      IVM_PH(4);
    }
    // ================= A stage: task t_{k-1} =================
    if (k >= 1 && k - 1 < K) {
      const int t = (int)blockIdx.x + P * (k - 1), pair = t / C;
      const unsigned role = (unsigned)(t % C);
      const int slot = pair % g.rp;
      const XD *xch = reinterpret_cast<const XD *>(g.xch) + (size_t)slot * C * 4096;
      if (threadIdx.x == 0) {  // last inverse pass table (this role's rows); the swap buffer is free
        mbar_expect(&tbar, EB * 4096);
        bulk_copy(twb + X::S_SWAP, tw + X::XINV(role), EB * 4096, &tbar);
        cs.ok = 1;
        cs.first_bad = 0x7fffffff;
        cs.maxrad = 0ull;
      }
      await7(g.cnt + 4 * pair + 0, C);  // every column of the pair written
      IVM_PH(5);
      mbar_wait(&tbar, (tph++) & 1u);
      CertAcc acc;
      {  // stage 1: task (b, kl): y_q(kl), q = C2 a + b, from the exchange with their input
         // twiddles; DFT8 over a, times w_C^{-b r1}; into the state (free)
        const int b = (int)threadIdx.x / B, kl = (int)threadIdx.x % B;
        DI v[8];
#pragma unroll
        for (int a = 0; a < 8; a++) {  // (the L2 loads first: all eight in flight)
          const int q = C2 * a + b;
          const int src = (2 * q < C) ? 2 * q : 2 * C - 1 - 2 * q;
          v[a] = ldcg_xd(xch + (size_t)src * 4096 + (int)role * B + kl);
        }
        ddit8<true>(v, [&](int a) {
          const int q = C2 * a + b;
          const TwC<T> w = twb[X::S_SWAP + q * B + kl];
          return (2 * q < C) ? drt<true, true, true>(w, v[a], SCALE) : drt<false, true, true>(w, dconj(v[a]), SCALE);
        });
#pragma unroll
        for (int r1 = 1; r1 < 8; r1++) {  // b is warp-uniform (B >= 32)
          const int j = b * r1;
          const TwC<T> w = s2tw[2 * j];
          v[r1] = 2 * j <= C ? drt<true, true>(w, v[r1]) : drt<false, true>(w, v[r1]);
        }
#pragma unroll
        for (int r1 = 0; r1 < 8; r1++) st.st((r1 * C2 + b) * B + kl, v[r1]);
        __syncthreads();
#ifndef IVM_NO_DISCARD
        // this task was the only reader of its rows of the exchange (whole 128-byte
        // lines: 4 consecutive kl), and the next writer is another launch's or the ring's
        // next pair: drop the dirty lines from L2 instead of writing them back to HBM
        if ((kl & 3) == 0) {
#pragma unroll
          for (int a = 0; a < 8; a++) {
            const int q = C2 * a + b;
            const int src = (2 * q < C) ? 2 * q : 2 * C - 1 - 2 * q;
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(xch + (size_t)src * 4096 + (int)role * B + kl) : "memory");
          }
        }
#endif
      }
      {  // stage 2: task (r1, kl), DFT_C2 over b, untwist remainder, emit into the swap buffer
        constexpr int TASKS = 8 * B / 512;
#pragma unroll
        for (int g2 = 0; g2 < TASKS; g2++) {
          const int task = (int)threadIdx.x + 512 * g2, r1 = task / B, kl = task % B;
          const int k0 = (int)role * B + kl;
          DI v[C2];
#pragma unroll
          for (int b = 0; b < C2; b++) v[b] = st.ld((r1 * C2 + b) * B + kl);
          dcdft<C2, true>(v);
#pragma unroll
          for (int r2 = 0; r2 < C2; r2++) {
            const int r = r1 + 8 * r2, k = k0 + 4096 * r;
            const DI w = drt<true, false>(fold[2 * r], v[r2]);  // (the input twiddles carried the scale 2/m)
            certify_real<double, long long, false>(__dadd_rd(w.cr, -w.r), __dadd_ru(w.cr, w.r), k, n,
                                                   coefL + r * B + cpos<B / 16>(kl), acc, nullptr);
            certify_real<double, long long, false>(__dadd_rd(w.ci, -w.r), __dadd_ru(w.ci, w.r), k + N / 2, n,
                                                   coefL + (C + r) * B + cpos<B / 16>(kl), acc, nullptr);
          }
        }
      }
      cert_flush(acc, cs);
      __syncthreads();
      IVM_PH(6);
      {  // the chunk's carry with nothing from below (Carry4 on the words in shared memory):
         // each thread's four resolved words U to L2; per chunk the headroom hr (its carry-out
         // for an incoming value I at word 0 is [I >= hr]) and the value Dout it passes up
        const int lc = (int)threadIdx.x / TPC, tc = (int)threadIdx.x % TPC, ch = lc * C + (int)role;
        const unsigned lane = threadIdx.x & 31u, sh = lane / TPC * TPC;
        unsigned long long Vw[6];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int wj = 4 * tc + j, gi0 = ch * B + 4 * wj;
          const longlong2 *q = reinterpret_cast<const longlong2 *>(coefL + lc * B + cpos<TPC>(4 * wj));
          const longlong2 x = q[0], y = q[1];
          Vw[2 + j] = word_of((unsigned long long)x.x, (unsigned long long)x.y, (unsigned long long)y.x,
                              (unsigned long long)y.y, gi0, nc);
        }
        {
          const unsigned long long u4 = __shfl_up_sync(0xffffffffu, Vw[4], 1), u5 = __shfl_up_sync(0xffffffffu, Vw[5], 1);
          Vw[0] = tc == 0 ? 0ull : u4;
          Vw[1] = tc == 0 ? 0ull : u5;
        }
        Carry4<TPC> cy;
        cy.words(Vw);
        unsigned U[4];
        cy.digits(cy.lane_cin(0u, nullptr), U);
        const unsigned gen = cy.seg_bits() & 1u;
        // words 1 .. WB-1 all ones: then hr = 2^32 - U_0 (else the chunk cannot carry out)
        const bool ao = (tc == 0 ? (U[1] & U[2] & U[3]) : (U[0] & U[1] & U[2] & U[3])) == 0xffffffffu;
        const unsigned AO = __ballot_sync(0xffffffffu, ao);
        constexpr unsigned MASK = (1u << TPC) - 1u;
        const bool up = ((AO >> sh) & MASK) == MASK;
        // passed up: hi of the top word plus the overflow of its low half + hi of the word below
        const unsigned lo5 = (unsigned)Vw[5], hi5 = (unsigned)(Vw[5] >> 32), hi4 = (unsigned)(Vw[4] >> 32);
        const unsigned dout = __shfl_sync(0xffffffffu, hi5 + (lo5 + hi4 < lo5 ? 1u : 0u), sh + TPC - 1);
        if (tc == 0) {
          const unsigned hr = gen ? 0u : ((up && U[0] != 0u) ? 0u - U[0] : 0xffffffffu);
          g.rec[(size_t)slot * NCHT + ch] = make_uint2(hr, dout);
        }
        g.wds[((size_t)slot * C + role) * 512 + threadIdx.x] = make_uint4(U[0], U[1], U[2], U[3]);
        if (threadIdx.x == 0) {
          unsigned *link = g.link + ((size_t)slot * C + role) * 8;
          link[0] = (unsigned)cs.ok;
          link[1] = (unsigned)cs.first_bad;
          link[2] = (unsigned)(cs.maxrad & 0xffffffffu);
          link[3] = (unsigned)(cs.maxrad >> 32);
        }
      }
      __syncthreads();
      post7(g.cnt + 4 * pair + 1);
      IVM_PH(7);
    }
    if (k + 1 < K && threadIdx.x == 0) {  // next task's role tables (the swap buffer is free again)
      const unsigned role = (unsigned)(((int)blockIdx.x + P * (k + 1)) % C);
      mbar_expect(&tbar, EB * (X::FLAST + X::MF_ENT));
      bulk_copy(twb + X::S_SWAP, tw + X::FWD(role) + X::FP(4), EB * X::FLAST, &tbar);
      bulk_copy(twb + X::S_MF, tw + X::FWD(role), EB * X::MF_ENT, &tbar);
    }
    // ================= Cs stage: task t_{k-2} =================
    if (k >= 2 && k - 2 < K) {
      const int t = (int)blockIdx.x + P * (k - 2), pair = t / C;
      const unsigned role = (unsigned)(t % C);
      const int slot = pair % g.rp;
      const int lane = (int)(threadIdx.x & 31u), warp = (int)(threadIdx.x >> 5);
      const int lc = (int)threadIdx.x / TPC, tc = (int)threadIdx.x % TPC, ch = lc * C + (int)role;
      const uint4 Uw = __ldcg(g.wds + ((size_t)slot * C + role) * 512 + threadIdx.x);  // this CTA's own
      await7(g.cnt + 4 * pair + 1, C);  // every task's records and certificate
      IVM_PH(8);
      // carries into all 2C^2 chunks: lane l of warp w < RW holds chunks j0 .. j0 + 15;
      // chunk j (incoming I = Dout_{j-1} + c_j) generates iff Dout_{j-1} >= hr_j and
      // propagates iff Dout_{j-1} + 1 == hr_j; ballot adders over lanes, then warps
      constexpr int CPL = 16, RW = NCHT / (32 * CPL);
      static_assert(RW >= 1 && RW <= 4 && NCHT % (32 * CPL) == 0, "resolver shape");
      unsigned Gl = 0u, Pl = 0u, Gw = 0u, Pw = 0u;
      unsigned dp[CPL];
      const int j0 = CPL * (32 * warp + lane);
      if (warp < RW) {
        const uint2 *rec = g.rec + (size_t)slot * NCHT;
        uint4 r[CPL / 2];
#pragma unroll
        for (int i = 0; i < CPL / 2; i++) r[i] = __ldcg(reinterpret_cast<const uint4 *>(rec + j0) + i);
        unsigned d = j0 > 0 ? __ldcg(&rec[j0 - 1].y) : 0u;
#pragma unroll
        for (int i = 0; i < CPL; i++) {
          const unsigned hr = (i & 1) ? r[i / 2].z : r[i / 2].x, dn = (i & 1) ? r[i / 2].w : r[i / 2].y;
          const bool gg = d >= hr, pp = !gg && d + 1u == hr;
          Gl |= (gg ? 1u : 0u) << i;
          Pl |= (pp ? 1u : 0u) << i;
          dp[i] = d;
          d = dn;
        }
        const bool gl = ((((Gl | Pl) + Gl) >> CPL) & 1u) != 0u, pl = Pl == (1u << CPL) - 1u;
        Gw = __ballot_sync(0xffffffffu, gl);
        Pw = __ballot_sync(0xffffffffu, pl);
        if (lane == 0) {
          const unsigned gw = (unsigned)((((unsigned long long)(Gw | Pw)) + Gw) >> 32);
          s_wgp[warp] = gw | ((Pw == 0xffffffffu ? 1u : 0u) << 1);
        }
      } else if (warp == 15) {  // the pair's certificate
        const unsigned *link = g.link + (size_t)slot * C * 8;
        int okl = 1, badl = 0x7fffffff;
        unsigned long long radl = 0ull;
        if (lane < C) {
          const uint4 w = __ldcg(reinterpret_cast<const uint4 *>(link + lane * 8));
          okl = (int)w.x;
          badl = (int)w.y;
          radl = (unsigned long long)w.z | ((unsigned long long)w.w << 32);
        }
        okl = __reduce_and_sync(0xffffffffu, (unsigned)okl);
        badl = (int)__reduce_min_sync(0xffffffffu, (unsigned)badl);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const unsigned long long r2 = __shfl_xor_sync(0xffffffffu, radl, o);
          radl = r2 > radl ? r2 : radl;
        }
        if (lane == 0) {
          s_ok = okl;
          s_bad = badl;
          s_rad = radl;
        }
      }
      __syncthreads();
      if (warp < RW) {
        unsigned cw = 0u;  // carry into this warp's first chunk
        for (int j = 0; j < warp; j++) {
          const unsigned b = s_wgp[j];
          cw = (b & 1u) | (((b >> 1) & 1u) & cw);
        }
        const unsigned cl = (unsigned)((((((unsigned long long)(Gw | Pw)) + Gw + cw) ^ Pw) >> lane) & 1u);
        const unsigned cb = ((Gl | Pl) + Gl + cl) ^ Pl;  // carry into each chunk of the lane
#pragma unroll
        for (int i = 0; i < CPL; i++) {
          const int j = j0 + i;
          if (j % C == (int)role) {
            s_cin[j / C] = (cb >> i) & 1u;
            s_din[j / C] = dp[i];
          }
        }
      }
      __syncthreads();
      const int ok = s_ok;
      const int words = (nout + 3) / 4;
      uint8_t *out = kp.prod + (size_t)pair * nout;
      if (ok) {
        // (U + I) mod 2^(32 WB): the chunk's first thread adds I at word 0, the carry out of
        // its words passes through the threads above whose words are all ones
        unsigned U[4] = {Uw.x, Uw.y, Uw.z, Uw.w};
        const unsigned lanei = threadIdx.x & 31u, sh = lanei / TPC * TPC;
        unsigned c = tc == 0 ? s_din[lc] + s_cin[lc] : 0u;
        unsigned long long x = (unsigned long long)U[0] + c;
        U[0] = (unsigned)x;
        unsigned o = (unsigned)(x >> 32);
#pragma unroll
        for (int i = 1; i < 4; i++) {
          U[i] += o;
          o = (o != 0u && U[i] == 0u) ? 1u : 0u;
        }
        const bool ao = tc > 0 && (Uw.x & Uw.y & Uw.z & Uw.w) == 0xffffffffu;
        const unsigned AO = __ballot_sync(0xffffffffu, ao);
        const unsigned c0 = __shfl_sync(0xffffffffu, o, sh);
        if (tc > 0) {
          const unsigned need = (1u << (tc - 1)) - 1u;  // threads 1 .. tc-1 all ones
          const unsigned cin = (c0 != 0u && ((AO >> (sh + 1)) & need) == need) ? 1u : 0u;
          unsigned long long y = (unsigned long long)Uw.x + cin;
          U[0] = (unsigned)y;
          unsigned o2 = (unsigned)(y >> 32);
#pragma unroll
          for (int i = 1; i < 4; i++) {
            U[i] += o2;
            o2 = (o2 != 0u && U[i] == 0u) ? 1u : 0u;
          }
        }
        const int k0 = ch * WB + 4 * tc;
        if (k0 < words) store_words4(out, k0, nout, U);
      } else {
        for (int i = ch * B + 4 * tc; i < min(ch * B + B, nout); i += 4 * TPC)
          for (int b = 0; b < 4 && i + b < nout; b++) out[i + b] = 0;
      }
      if (role == 0 && threadIdx.x == 0) {
        kp.cert[pair] = ok ? 1 : 0;
        if (kp.max_radius) kp.max_radius[pair] = __longlong_as_double((long long)s_rad);
        if (kp.first_bad) kp.first_bad[pair] = ok ? -1 : s_bad;
      }
      __syncthreads();
      post7(g.cnt + 4 * pair + 2);
      IVM_PH(9);
    }
  }
}

}  // namespace d7
}  // namespace ivm
