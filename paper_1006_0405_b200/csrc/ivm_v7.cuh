// ivm_v7.cuh -- pipelined group kernel for m = 2^17, 2^18 (fp64, C = 16, 32 CTA
// tasks per multiplication; included by ivm_v5.cu).  Same transform, tables and
// arithmetic as the group kernel (ivm_v5.cuh); what changes is the schedule.
//
// The group kernel runs C co-resident CTAs in lockstep per multiplication, so on
// 148 SMs only floor(148 / C) C = 128 SMs work (C = 32) and every group waits at
// its three barriers for its slowest CTA.  Here a persistent grid of P CTAs (one
// per SM) deals the batch's batch * C tasks t = (pair t / C, role t % C) round
// robin, t_k = blockIdx.x + P k, and splits each task into three stages:
//   L  (local: cross passes, forward passes, pointwise, inverse local passes;
//       the column goes to the pair's exchange)                  -> count L[pair]
//   A  (wait L[pair] = C; last inverse pass, certify, snap; the carry of each
//       of the task's chunks with nothing coming from below: its resolved words
//       U, its headroom hr and the value Dout it passes up)      -> count A[pair]
//   Cs (wait A[pair] = C; carries into all chunks from the (hr, Dout) records:
//       chunk j, receiving I = Dout_{j-1} + c_j at word 0, carries out iff
//       I >= hr_j, so it generates iff Dout_{j-1} >= hr_j and propagates iff
//       Dout_{j-1} + 1 == hr_j -- one ballot adder; digits (U + I) mod 2^(32 WB))
// Slot k of a CTA runs L(t_k), A(t_{k-1}), Cs(t_{k-2}).  A pair's tasks lie in
// at most two consecutive slots (C < P), so every wait is for stages that
// precede it in the (slot, stage) order of every CTA: no deadlock with all CTAs
// co-resident (cooperative launch), and the waits are short (all CTAs run the
// same stages at about the same time) instead of a whole task.  The per-pair
// scratch is a ring of RP pairs (all pairs when they fit 1 GB); the L stage of
// pair p waits until pair p - RP has finished every stage (RP >= (4 P + C - 1) / C
// keeps that wait for stages at earlier slots; v7_ring() takes more).
#pragma once

namespace ivm {
namespace v7 {

using namespace v3;
using namespace v4;
using namespace v5;

struct Pipe7 {
  unsigned *cnt;    // [batch][4] stage counters L, A, Cs (zeroed by the host before the launch)
  void *xch;        // [RP][C][4096] CI<double> column exchange
  uint4 *wds;       // [RP][C][512] each thread's four words, carried with nothing from below (A -> Cs)
  uint2 *rec;       // [RP][2 C^2] per chunk: headroom hr, value passed up Dout
  unsigned *link;   // [RP][C][8] per-task certificate words
  int rp;           // ring pairs
};

// stage counters: the CTA's writes (ordered before the posting thread by the block
// barrier the caller places) are released by one thread's gpu-scope add -- the
// last warp's, so that its wait for the stores to drain overlaps thread 0's poll
// of the next stage's counter; a wait acquires the other CTAs' releases and a
// block barrier passes it on
__device__ __forceinline__ void post7(unsigned *c) {
  if (threadIdx.x == 480) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
}
__device__ __forceinline__ void await7(const unsigned *c, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// FAST: the host guarantees word-aligned digit rows and no diagnostic outputs
// (interval dump, snapped coefficients): those paths are compiled out
template <int M, bool FAST = false>
__global__ void __launch_bounds__(512, 1) ivm_v7_kernel(KParams kp, Pipe7 g) {
  using T = double;
  using X = G4<M>;
  using GL = G3<13, 8>;
  using CF = Cfg5<T, M>;
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
  Buf<T> st{reinterpret_cast<V *>(smem), reinterpret_cast<V *>(smem) + GL::CAP};
  TwC<T> *twb = reinterpret_cast<TwC<T> *>(smem + CF::STATE_BYTES);
  const TwC<T> *s2tw = twb + X::S_S2;  // w_C^{-j}: s2tw[2 j], upper-half form
  const TwC<T> *fold = twb + X::S_FO;  // fold[2 r] = z^{4096 r}
  long long *coefL = reinterpret_cast<long long *>(twb + X::S_SWAP);
  const TwC<T> *tw = reinterpret_cast<const TwC<T> *>(kp.tw);
  Buf<T> A{reinterpret_cast<V *>(kp.ascratch) + (size_t)blockIdx.x * NL, nullptr};
  A.im = A.re + NL / 2;
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
      CI<T> *xch = reinterpret_cast<CI<T> *>(g.xch) + (size_t)slot * C * 4096;
      if (t + P < NT) {  // L2 prefetch of this role's slice of the next task's digits
        const int nxt = (t + P) / C, nrole = (t + P) % C, sl = (n + C - 1) / C;
        for (int off = nrole * sl + (int)threadIdx.x * 128; off < min(n, (nrole + 1) * sl); off += (int)blockDim.x * 128) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.a + (size_t)nxt * n + off));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.b + (size_t)nxt * n + off));
        }
      }
#pragma unroll 1
      for (int op = 0; op < 2; op++) {
        cross_tc<M, FAST>((op == 0 ? kp.a : kp.b) + (size_t)pair * n, n, st, tw + X::LIMB, role);
        __syncthreads();
        IVM_PH(2 * op);
#pragma unroll  // (specialised per pass: addresses fold into immediates)
        for (int i = 0; i < 4; i++) {
          const PassRT pp = pick_fwd4<M>(i);
          CI<T> v[R];
          int k0, nu;
          if (op == 0 && i == 0) mbar_wait(&tbar, (tph++) & 1u);  // this role's tables
          fwdR<T, R>(st, twb, pp, v, k0, nu);
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
            pointwise_dit8<T, true>(v, A, k0, pp.L >> 1);
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
        CI<T> v[R];
        int k0, nu;
        if (i == 2) mbar_wait(&tbar, (tph++) & 1u);
        invR<T, R, false>(st, twb, pp, v, k0, nu);
        if (i < 2) {
          __syncthreads();
#pragma unroll
          for (int r = 0; r < R; r++) st.st(sidx(k0 + pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
          __syncthreads();
        } else {  // last local pass: the column goes to the pair's exchange (row k0 + L r)
#pragma unroll
          for (int r = 0; r < R; r++) st_ci(xch + (size_t)role * 4096 + k0 + pp.L * r, v[r]);
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
      const CI<T> *xch = reinterpret_cast<const CI<T> *>(g.xch) + (size_t)slot * C * 4096;
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
        CI<T> v[8];
#pragma unroll
        for (int a = 0; a < 8; a++) {  // (the L2 loads first: all eight in flight)
          const int q = C2 * a + b;
          const int src = (2 * q < C) ? 2 * q : 2 * C - 1 - 2 * q;
          v[a] = ldcg_ci(xch + (size_t)src * 4096 + (int)role * B + kl);
        }
        dit8<T, true>(
            v,
            [&](int a) {
              const int q = C2 * a + b;
              const TwC<T> w = twb[X::S_SWAP + q * B + kl];
              return (2 * q < C) ? rtmul<T, true, true>(w, v[a]) : rtmul_cd<T, false, true>(w, v[a]);
            },
            [] {});
#pragma unroll
        for (int r1 = 1; r1 < 8; r1++) {  // b is warp-uniform (B >= 32)
          const int j = b * r1;
          const TwC<T> w = s2tw[2 * j];
          v[r1] = 2 * j <= C ? rtmul<T, true, true>(w, v[r1]) : rtmul<T, false, true>(w, v[r1]);
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
        double *dump = FAST ? nullptr : diag_dump(kp, pair, N);
#pragma unroll
        for (int g2 = 0; g2 < TASKS; g2++) {
          const int task = (int)threadIdx.x + 512 * g2, r1 = task / B, kl = task % B;
          const int k0 = (int)role * B + kl;
          CI<T> v[C2];
#pragma unroll
          for (int b = 0; b < C2; b++) v[b] = st.ld((r1 * C2 + b) * B + kl);
          cdft<T, C2, true>(v);
#pragma unroll
          for (int r2 = 0; r2 < C2; r2++) {
            const int r = r1 + 8 * r2, k = k0 + 4096 * r;
            emit_tab<T, M>(v[r2], fold[2 * r], k, n, coefL + r * B + cpos<B / 16>(kl),
                           coefL + (C + r) * B + cpos<B / 16>(kl), acc, dump);
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
        if (!FAST && kp.coeffs) {  // snapped coefficients (zeroed in the Cs stage if the pair fails)
          int64_t *co = kp.coeffs + (size_t)pair * nc;
          for (int e = (int)threadIdx.x; e < NCH * B; e += blockDim.x) {
            const int lc2 = e / B, i = (lc2 * C + (int)role) * B + e % B;
            if (i < nc) co[i] = coefL[lc2 * B + cpos<B / 16>(e % B)];
          }
        }
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
        if (!FAST && kp.coeffs) {
          int64_t *co = kp.coeffs + (size_t)pair * nc;
          for (int e = (int)threadIdx.x; e < NCH * B; e += blockDim.x) {
            const int i = (e / B * C + (int)role) * B + e % B;
            if (i < nc) co[i] = 0;
          }
        }
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

}  // namespace v7
}  // namespace ivm
