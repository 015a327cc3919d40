// ivm_v4.cuh -- cluster kernel for m = 2^14 .. 2^16: one thread-block cluster of
// C = m/8192 CTAs per multiplication, every CTA running the m = 8192 one-CTA
// schedule of ivm_v3.cuh on its share (included by ivm_v4.cu).
//
// Row split of the odd-frequency transform (ivm_v3.cuh).  After the trivial
// radix-2 pass, a first DIT pass of radix C gives the half-stored
// rows k < C of level 2C; CTA c computes row c from the digits:
//   G[c][v] = sum_q w_{4C}^{q(1+4r)} x[v + (m/2C) q],  r = c/2 (c even), or the
//   conjugate of the r = (2C-1-c)/2 output (c odd, the mirrored row).
// Every later forward pass maps row k0 to rows k0 + L r and their mirrors, so the
// rows {k = c or 2C-1-c (mod 2C)} stay in CTA c: with local index kappa,
//   k = C kappa + (kappa even ? c : C-1-c),
// the local passes, storage and mirror rules are exactly the m = 8192 ones; only
// the twiddle values w_{2LR}^{q(2k+1)} differ per CTA ("role" tables).  The
// pointwise product and the inverse passes 0..3 are local too (the inverse rows
// are the same in every CTA, the columns are the CTA's classes); the last inverse
// pass (radix C, untwist z^{-k} folded into its input twiddles) combines one
// column from every CTA: it reads them through distributed shared memory.  The
// coefficients stay in the producing CTA's shared memory; the carry runs over
// contiguous word segments with the cluster-level ballot adder.
#pragma once

#ifndef IVM_QB_GROUP
#define IVM_QB_GROUP 4
#endif

namespace ivm {
namespace v4 {

using namespace v3;

template <int M> struct G4 {
  static_assert(M >= 14 && M <= 18, "C = 2 .. 32 CTAs");
  static constexpr int C = 1 << (M - 13);
  static constexpr int B = 4096 / C;  // rows of the last inverse pass per CTA
  static constexpr int LGB = 12 - (M - 13);
  using GL = G3<13, 8>;  // the local (m = 8192) layout
  // device table (compact entries of 2 T):
  //   FWD(c): role c, local forward passes 1..4 at FP(p) = 0, 7, 63, 512 ([R-1][L/2] each;
  //           pass 4 starts at an even entry so every bulk copy is 16-byte aligned in fp32 too)
  //   INV:    local inverse passes 1..3: [7][8], [7][64], [7][512] (shared)
  //   XINV(c): role c, last inverse pass, [C][B] (rows c B .. c B + B - 1), folded untwist
  //   TH(c):  role c, theta_q (q < C) as full intervals (2 entries each)
  //   S2:     j < C, compact at S2 + 2 j: w_C^j (2 j <= C) or w_C^{C-j}, the
  //           upper-half-plane form of w_C^{-j} (v5's two-stage last inverse pass)
  //   FO:     w_{4C}^r = z^{4096 r}, r < C (compact, first quadrant, at FO + 2 r;
  //           v5's emit multiplies by its conjugate)
  __host__ __device__ static constexpr int FWD(int c) { return c * 4096; }
  __host__ __device__ static constexpr int FP(int p) { return p == 1 ? 0 : (p == 2 ? 7 : (p == 3 ? 63 : 512)); }
  static constexpr int INV = C * 4096;
  static constexpr int INV1 = 0, INV2 = 56, INV3 = 504, INV_ENT = 4088;
  __host__ __device__ static constexpr int XINV(int c) { return INV + 4096 + c * 4096; }
  __host__ __device__ static constexpr int TH(int c) { return INV + 4096 + C * 4096 + 2 * C * c; }
  static constexpr int S2 = INV + 4096 + C * 4096 + 2 * C * C;
  static constexpr int FO = S2 + 2 * C;
  //   LIMB:   v5's tensor-core cross pass (fp64, C >= 16): role c at byte offset 1024 c,
  //           int8 [4 operands s][8 columns][32 q] (see cross_tc in ivm_v5.cuh); 64 C
  //           entries of 16 B (filled for fp64 only)
  static constexpr int LIMB = FO + 2 * C;
  //   TH1(c): role c, the cross pass fused with local pass 1 (cross_pass1): [8 j][C q]
  //           full intervals of w_j theta_q (odd roles: w_j conj(theta_q)), w_j the
  //           pass-1 twiddle of input j -- one root of unity each, optimally enclosed
  __host__ __device__ static constexpr int TH1(int c) { return LIMB + 64 * C + 16 * C * c; }
  static constexpr int TOTAL = LIMB + 64 * C + 16 * C * C;
  // shared-memory twiddle area (entries)
  static constexpr int S_SWAP = 0;          // 4096: forward-last -> inverse pass 3 -> last inverse pass
  static constexpr int S_MF = 4096;         // forward passes 1..3 (511 entries + 1 pad)
  static constexpr int S_MI = 4096 + 512;   // inverse passes 1, 2 (504 entries)
  static constexpr int S_TH = 4096 + 1016;  // theta (2C entries)
  static constexpr int S_S2 = S_TH + 2 * C;  // v5 only
  static constexpr int S_FO = S_S2 + 2 * C;  // v5 only
  static constexpr int S_TH1 = S_FO + 2 * C;  // v4: TH1 of this role (16 C entries)
  static constexpr int S_ENT = S_TH1 + 16 * C;  // v4 (v5: S_FO + 2 C)
  static constexpr int FLAST = 3584, MF_ENT = 512, MI_ENT = 504;
};

template <int M> struct RT4 {
  using GL = G3<13, 8>;
  __host__ __device__ static constexpr PassRT fwd(int i) {  // local forward pass p = i + 1
    return PassRT{ilog2r(8192 / fL(plan_cta(13, 8), i + 1) / 8), fL(plan_cta(13, 8), i + 1), GL::fRS(i + 1),
                  (i + 2 < 5) ? GL::fRS(i + 2) : GL::iRS(1), GL::fSW(i + 1), (i + 2 < 5) ? GL::fSW(i + 2) : GL::iSW(1),
                  (i < 3) ? G4<M>::S_MF + G4<M>::FP(i + 1) : G4<M>::S_SWAP, (i == 3) ? 1 : 0, 0};
  }
  __host__ __device__ static constexpr PassRT inv(int i) {  // local inverse pass p = i + 1 (unfolded)
    return PassRT{ilog2r(8192 / iL(plan_cta(13, 8), i + 1) / 8), iL(plan_cta(13, 8), i + 1), GL::iRS(i + 1),
                  GL::iRS(i + 2), GL::iSW(i + 1), GL::iSW(i + 2),
                  (i == 0) ? G4<M>::S_MI : (i == 1 ? G4<M>::S_MI + 56 : G4<M>::S_SWAP), (i == 2) ? 1 : 0, 0};
  }
};
template <int M> __device__ __forceinline__ PassRT pick_fwd4(int i) {
  constexpr PassRT p0 = RT4<M>::fwd(0), p1 = RT4<M>::fwd(1), p2 = RT4<M>::fwd(2), p3 = RT4<M>::fwd(3);
  return i == 0 ? p0 : (i == 1 ? p1 : (i == 2 ? p2 : p3));
}
template <int M> __device__ __forceinline__ PassRT pick_inv4(int i) {
  constexpr PassRT p0 = RT4<M>::inv(0), p1 = RT4<M>::inv(1), p2 = RT4<M>::inv(2);
  return i == 0 ? p0 : (i == 1 ? p1 : p2);
}

// ---- cluster primitives ----
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// split barrier: arrive now, wait later.  The arrive has release semantics:
// it orders this CTA's remote DSMEM reads before the other CTAs' writes that
// follow their wait (write-after-read across the cluster; the PTX memory model
// gives .relaxed no such ordering).
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ unsigned dsm_map(const void *p, unsigned cta) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
  return r;
}
__device__ __forceinline__ unsigned dsm_map_addr(unsigned a, unsigned cta) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
  return r;
}
__device__ __forceinline__ double2 dsm_ld(unsigned a, double2 *) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float2 dsm_ld(unsigned a, float2 *) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int4 dsm_ld_i4(unsigned a) {
  int4 v;
  asm volatile("ld.shared::cluster.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ int dsm_ld_i32(unsigned a) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long dsm_ld_u64(unsigned a) {
  unsigned long long v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}

// coefficients of the cluster: c_i lives in the CTA that owns row
// k0 = (i mod m/2) mod 4096 of the last inverse pass, at local index
// (h C + r) B + (k0 - p B), i = h m/2 + r 4096 + k0, p = k0 / B
template <int M> struct CoefCluster {
  unsigned base;  // shared::cta address of the local coefficient array
  __device__ __forceinline__ unsigned addr(int i) const {
    using X = G4<M>;
    constexpr int HALF = (1 << M) / 2;
    const int h = i >= HALF ? 1 : 0;
    const int ii = i - h * HALF;
    const int r = ii >> 12, k0 = ii & 4095, p = k0 >> X::LGB;
    const int idx = (h * X::C + r) * X::B + (k0 - (p << X::LGB));
    return dsm_map_addr(base + 4u * (unsigned)idx, (unsigned)p);
  }
  __device__ __forceinline__ void quad(int k, unsigned long long (&o)[4]) const {
    const int4 q = dsm_ld_i4(addr(4 * k));
    o[0] = (unsigned)q.x, o[1] = (unsigned)q.y, o[2] = (unsigned)q.z, o[3] = (unsigned)q.w;
  }
  __device__ __forceinline__ unsigned long long one(int i) const { return (unsigned)dsm_ld_i32(addr(i)); }
};

// first (cross-CTA) forward pass from the digits: row `crank` of level 2C,
// 4096 columns; x >= 0 is a point, so [x th.lo, x th.hi] needs no sign cases
template <typename T, int M, bool QB = false>
__device__ __forceinline__ void cross_fwd(const uint8_t *__restrict__ dig, int n, Buf<T> st, const CI<T> *theta,
                                          unsigned crank, bool wait_cluster, bool global) {
  constexpr int C = G4<M>::C;
  const int t = threadIdx.x;
  CI<T> acc[8];
#pragma unroll
  for (int j = 0; j < 8; j++) acc[j] = CI<T>{T(0), T(0), T(0), T(0)};
  auto mac = [&](CI<T> &a, T x, const CI<T> &th) {
    a.rl = DR<T>::fma_rd(x, th.rl, a.rl);
    a.rh = DR<T>::fma_ru(x, th.rh, a.rh);
    a.il = DR<T>::fma_rd(x, th.il, a.il);
    a.ih = DR<T>::fma_ru(x, th.ih, a.ih);
  };
  const bool odd = (crank & 1u) != 0u;
  if (global && ((reinterpret_cast<uintptr_t>(dig) | (uintptr_t)n) & 3) == 0) {
    // digits from L2 / HBM: word loads (the pass is bound by their latency), thread
    // t owning columns 4t + e + 2048 h (e < 4, h < 2); with n % 4 == 0 a word is
    // wholly inside or outside the digits.  (Staged digits keep the byte loads:
    // the word form's 4-apart state stores conflict in shared memory.)
    auto term = [&](int q) {
      const CI<T> th = theta[q];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int base = 4 * t + 2048 * h + 4096 * q;
        const unsigned w = base < n ? *reinterpret_cast<const unsigned *>(dig + base) : 0u;
#pragma unroll
        for (int e = 0; e < 4; e++) mac(acc[4 * h + e], T((w >> (8 * e)) & 255u), th);
      }
    };
    // QB (a separate instantiation, chosen by the host when it skips a group):
    // terms past ceil(n / 4096) multiply only zero padding and are skipped, in
    // unrolled groups of 8.  Otherwise every term, fully unrolled (all loads in
    // flight); one kernel holding both forms measured slower on both paths.
    if constexpr (QB) {
      constexpr int QG = IVM_QB_GROUP;  // terms per unrolled group
      const int qmax = (min(C, (n + 4095) >> 12) + QG - 1) / QG * QG;
#pragma unroll 1
      for (int q0 = 0; q0 < qmax; q0 += QG) {
#pragma unroll
        for (int qq = 0; qq < QG; qq++) term(q0 + qq);
      }
    } else {
#pragma unroll
      for (int q = 0; q < C; q++) term(q);
    }
    if (wait_cluster) cluster_wait();  // the previous pair's remote reads of this state are done
#pragma unroll
    for (int h = 0; h < 2; h++)
#pragma unroll
      for (int e = 0; e < 4; e++) {
        if (odd) st.st_conj(4 * t + e + 2048 * h, acc[4 * h + e]);
        else st.st(4 * t + e + 2048 * h, acc[4 * h + e]);
      }
    return;
  }
#pragma unroll
  for (int q = 0; q < C; q++) {
    const CI<T> th = theta[q];
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const int idx = t + 512 * j + 4096 * q;
      mac(acc[j], idx < n ? T(dig[idx]) : T(0), th);
    }
  }
  if (wait_cluster) cluster_wait();  // the previous pair's remote reads of this state are done
#pragma unroll
  for (int j = 0; j < 8; j++) {
    if (odd) st.st_conj(t + 512 * j, acc[j]);
    else st.st(t + 512 * j, acc[j]);
  }
}

// The cross pass fused with local pass 1 (the cluster kernel): thread t's cross
// sums are the columns t + 512 j (j < 8) of row `crank`, which are exactly the
// inputs of its local pass-1 task (k0 = 0, nu = t, Sp = 512), so they stay in
// registers: the pass-1 twiddles (one per q, the same for every thread) and the
// 8-point DFT follow at once, with no shared-memory round trip of the cross row.
// Odd roles take the conjugate (the mirrored row), as cross_fwd's st_conj does.
// The pass-1 twiddle of input j and the cross coefficients combine into one root
// of unity per (j, q) (table TH1), so the twiddle products vanish: input j of
// thread t's pass-1 task is sum_q Theta[j][q] x[t + 512 j + 4096 q], four directed
// FMAs per term (x >= 0 is a point), then the 8-point DFT.
template <typename T, int M>
__device__ __forceinline__ void cross_pass1(const uint8_t *__restrict__ dig, int n, const CI<T> *__restrict__ th1,
                                            CI<T> (&v)[8]) {
  constexpr int C = G4<M>::C;
  const int t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < 8; j++) v[j] = CI<T>{T(0), T(0), T(0), T(0)};
#pragma unroll
  for (int j = 0; j < 8; j++) {
#pragma unroll
    for (int q = 0; q < C; q++) {
      const CI<T> th = th1[j * C + q];  // shared memory, uniform: a broadcast
      const int idx = t + 512 * j + 4096 * q;
      const T x = idx < n ? digit_val<T>((unsigned)dig[idx]) : T(0);
      v[j].rl = DR<T>::fma_rd(x, th.rl, v[j].rl);
      v[j].rh = DR<T>::fma_ru(x, th.rh, v[j].rh);
      v[j].il = DR<T>::fma_rd(x, th.il, v[j].il);
      v[j].ih = DR<T>::fma_ru(x, th.ih, v[j].ih);
    }
    // (keeps the next input's loads after this one's FMAs: hoisting them all
    // would cost registers the DFT needs)
    asm volatile("" ::: "memory");
  }
  cdft<T, 8, false>(v);
}

template <typename T, int M> struct Cfg4 {
  using GL = G3<13, 8>;
  static constexpr int THREADS = 512;
  static constexpr size_t E = sizeof(typename V2t<T>::t);
  static constexpr size_t STATE_BYTES = 2 * E * (size_t)GL::CAP;
  static constexpr size_t TW_BYTES = sizeof(TwC<T>) * (size_t)G4<M>::S_ENT;
  // one operand's digits (n <= m/2 bytes), staged by a bulk copy one step ahead
  // when it fits (m <= 2^15); else read from L2/HBM with an L2 prefetch
  static constexpr size_t DIG_BYTES = STATE_BYTES + TW_BYTES + (size_t)(1 << M) / 2 <= 227 * 1024 ? (1 << M) / 2 : 0;
  static constexpr size_t SMEM = STATE_BYTES + TW_BYTES + DIG_BYTES;
  static constexpr size_t A_BYTES = 2 * E * 4096;
  static_assert(sizeof(TwC<T>) * 4096 >= 4 * 8192, "local coefficients fit the twiddle swap buffer");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

// FAST: the host guarantees no diagnostic outputs (interval dump, snapped
// coefficients) and, where the digits are staged at all (m <= 2^15), 16-byte
// aligned rows: the other paths are compiled out of the throughput kernel
template <typename T, int M, bool FAST = false>
__global__ void __launch_bounds__(512, 1) ivm_v4_kernel(KParams kp) {
  using X = G4<M>;
  using GL = G3<13, 8>;
  using CF = Cfg4<T, M>;
  using V = typename V2t<T>::t;
  constexpr int C = X::C, B = X::B, R = 8, NL = 8192, N = 1 << M;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Cert3 cs;
  __shared__ unsigned s_chunk[2 * (1 << (M - 13))][2];  // this CTA's chunks: generate, all-propagate
  __shared__ unsigned s_cin[4];                         // carry into each of the 2C^2 chunks
  __shared__ __align__(8) unsigned long long tbar, dbar;
  Buf<T> st{reinterpret_cast<V *>(smem), reinterpret_cast<V *>(smem) + GL::CAP};
  TwC<T> *twb = reinterpret_cast<TwC<T> *>(smem + CF::STATE_BYTES);
  // [2][C][B] coefficients in the twiddle swap buffer (free after the last
  // pass's twiddles are read): the state stays readable by the other CTAs
  int32_t *coefL = reinterpret_cast<int32_t *>(twb + X::S_SWAP);
  const CI<T> *theta = reinterpret_cast<const CI<T> *>(twb + X::S_TH);
  uint8_t *sdig = smem + CF::STATE_BYTES + CF::TW_BYTES;
  const unsigned crank = cluster_rank();
  const int cid = (int)(blockIdx.x / C), ncl = (int)(gridDim.x / C);
  const TwC<T> *tw = reinterpret_cast<const TwC<T> *>(kp.tw);
  Buf<T> A{reinterpret_cast<V *>(kp.ascratch) + (size_t)blockIdx.x * NL, nullptr};
  A.im = A.re + NL / 2;
  const int n = kp.n, nc = 2 * n - 1, nout = 2 * n;
  constexpr int RSI1 = GL::iRS(1), SWI1 = GL::iSW(1);
  constexpr unsigned EB = sizeof(TwC<T>);

  const bool staged = CF::DIG_BYTES > 0 &&
                      (FAST || (n % 16 == 0 &&
                                ((reinterpret_cast<uintptr_t>(kp.a) | reinterpret_cast<uintptr_t>(kp.b)) % 16) == 0));
  if (threadIdx.x == 0) {
    mbar_init(&tbar);
    mbar_init(&dbar);
  }
  __syncthreads();
  if (threadIdx.x == 0 && cid < kp.batch) {
    mbar_expect(&tbar, EB * (X::FLAST + X::MF_ENT + X::MI_ENT + 2 * C + 16 * C));
    bulk_copy(twb + X::S_SWAP, tw + X::FWD(crank) + X::FP(4), EB * X::FLAST, &tbar);
    bulk_copy(twb + X::S_MF, tw + X::FWD(crank), EB * X::MF_ENT, &tbar);
    bulk_copy(twb + X::S_MI, tw + X::INV, EB * X::MI_ENT, &tbar);
    bulk_copy(twb + X::S_TH, tw + X::TH(crank), EB * 2 * C, &tbar);
    bulk_copy(twb + X::S_TH1, tw + X::TH1(crank), EB * 16 * C, &tbar);
    if (staged) {  // operand a of the first pair (dbar phases: a = even, b = odd)
      mbar_expect(&dbar, (unsigned)n);
      bulk_copy(sdig, kp.a + (size_t)cid * n, (unsigned)n, &dbar);
    }
  }
  if (cid < kp.batch) mbar_wait(&tbar, 0);
  // tbar phases per pair it: 3 it (forward-last), 3 it + 1 (inverse pass 3),
  // 3 it + 2 (last inverse pass) -> parities it&1, (it+1)&1, it&1

  int it = 0;
  IVM_PH_DECL
  for (int pair = cid; pair < kp.batch; pair += ncl, it++) {
    const unsigned par = (unsigned)it & 1u;
    if (!staged && pair + ncl < kp.batch) {  // L2 prefetch of the next pair's digits (this CTA's slice)
      const int nxt = pair + ncl, sl = (n + C - 1) / C;
      for (int off = (int)crank * sl + (int)threadIdx.x * 128; off < min(n, ((int)crank + 1) * sl);
           off += (int)blockDim.x * 128) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.a + (size_t)nxt * n + off));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.b + (size_t)nxt * n + off));
      }
    }
#pragma unroll 1
    for (int op = 0; op < 2; op++) {
      if (staged) mbar_wait(&dbar, (unsigned)op);
      if (staged) {  // the cross pass fused with local pass 1, stored in the pass-2 layout
        const PassRT pp = pick_fwd4<M>(0);
        CI<T> v[R];
        cross_pass1<T, M>(sdig, n, reinterpret_cast<const CI<T> *>(twb + X::S_TH1), v);
        if (op == 0 && it > 0) cluster_wait();  // the previous pair's remote reads of this state are done
        const int nu = (int)threadIdx.x;
#pragma unroll
        for (int r = 0; r < R; r++) {
          if (2 * r < R) st.st(sidx(pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
          else st.st_conj(sidx(R * pp.L - 1 - pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
        }
      } else {  // digits from L2 (word loads): the cross row through shared memory, then pass 1
        cross_fwd<T, M>((op == 0 ? kp.a : kp.b) + (size_t)pair * n, n, st, theta, crank, op == 0 && it > 0, true);
        __syncthreads();
        const PassRT pp = pick_fwd4<M>(0);
        CI<T> v[R];
        int k0, nu;
        fwdR<T, R>(st, twb, pp, v, k0, nu);
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; r++) {
          if (2 * r < R) st.st(sidx(k0 + pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
          else st.st_conj(sidx(R * pp.L - 1 - k0 - pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
        }
      }
      if (op == 0 && it > 0 && threadIdx.x == 0) {
        // this pair's forward-last table into the swap buffer: the cluster wait in
        // cross_fwd ordered every remote read of the previous coefficients before it
        mbar_expect(&tbar, EB * X::FLAST);
        bulk_copy(twb + X::S_SWAP, tw + X::FWD(crank) + X::FP(4), EB * X::FLAST, &tbar);
      }
      if (op == 1 && threadIdx.x == 0) {
        cs.ok = 1;
        cs.first_bad = 0x7fffffff;
        cs.maxrad = 0ull;
      }
      __syncthreads();
      IVM_PH(2 * op);
      if (staged && threadIdx.x == 0) {  // the next operand: b of this pair, or a of the next
        const uint8_t *nx = op == 0 ? kp.b + (size_t)pair * n : kp.a + (size_t)(pair + ncl) * n;
        if (op == 0 || pair + ncl < kp.batch) {
          mbar_expect(&dbar, (unsigned)n);
          bulk_copy(sdig, nx, (unsigned)n, &dbar);
        }
      }
#pragma unroll  // (specialised per pass: addresses fold into immediates)
      for (int i = 1; i < 4; i++) {
        const PassRT pp = pick_fwd4<M>(i);
        CI<T> v[R];
        int k0, nu;
        if (op == 0 && i == 3) mbar_wait(&tbar, par);  // forward-last table of this role
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
        } else {  // last forward pass of b + pointwise + inverse pass 0
          pointwise_dit8<T, true>(v, A, k0, pp.L >> 1);
          __syncthreads();
          if (threadIdx.x == 0) {  // inverse pass 3 table replaces the forward-last one
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
    CertAcc acc;
#pragma unroll  // (specialised per pass: addresses fold into immediates)
    for (int i = 0; i < 3; i++) {
      const PassRT pp = pick_inv4<M>(i);
      CI<T> v[R];
      int k0, nu;
      if (i == 2) mbar_wait(&tbar, par ^ 1u);
      invR<T, R, false>(st, twb, pp, v, k0, nu);
      __syncthreads();
      if (i == 2 && threadIdx.x == 0) {
        // every read of the pass-3 table is done: the last inverse pass table (this
        // role's rows) streams in while pass 3 stores and the cluster synchronises
        mbar_expect(&tbar, EB * 4096);
        bulk_copy(twb + X::S_SWAP, tw + X::XINV(crank), EB * 4096, &tbar);
      }
#pragma unroll
      for (int r = 0; r < R; r++) st.st(sidx(k0 + pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
      __syncthreads();
    }
    IVM_PH(4);
    cluster_sync();  // (1) every CTA's column of the 4096 rows is in its shared memory
    IVM_PH(5);
    {
      constexpr int G = 8 / C;  // rows (tasks) per thread
      CI<T> v[G][C];
      const unsigned re0 = (unsigned)__cvta_generic_to_shared(st.re), im0 = (unsigned)__cvta_generic_to_shared(st.im);
#pragma unroll
      for (int g = 0; g < G; g++) {
        const int k0 = (int)crank * B + (int)threadIdx.x + 512 * g;
#pragma unroll
        for (int q = 0; q < C; q++) {
          const unsigned src = (2 * q < C) ? (unsigned)(2 * q) : (unsigned)(2 * C - 1 - 2 * q);
          const V r = dsm_ld(dsm_map_addr(re0 + (unsigned)(sizeof(V) * k0), src), (V *)nullptr);
          const V m = dsm_ld(dsm_map_addr(im0 + (unsigned)(sizeof(V) * k0), src), (V *)nullptr);
          const CI<T> z{r.x, r.y, m.x, m.y};
          v[g][q] = z;  // the mirrors (2 q >= C) are conjugated by the twiddle product below
        }
      }
      // (no cluster barrier here: the coefficients do not overwrite the state)
      mbar_wait(&tbar, par);
      IVM_PH(12);
#pragma unroll
      for (int g = 0; g < G; g++) {
        const int kl = (int)threadIdx.x + 512 * g;
#pragma unroll
        for (int q = 0; q < C; q++) {
          const TwC<T> w = twb[X::S_SWAP + q * B + kl];
          v[g][q] = (2 * q < C) ? rtmul<T, true, true>(w, v[g][q]) : rtmul_cd<T, false, true>(w, v[g][q]);
        }
        cdft<T, C, true>(v[g]);
      }
      __syncthreads();  // every twiddle read: the swap buffer takes the coefficients
      IVM_PH(13);
      double *dump = FAST ? nullptr : diag_dump(kp, pair, N);
      if (!FAST && dump) {
#pragma unroll
        for (int g = 0; g < G; g++) {
          const int kl = (int)threadIdx.x + 512 * g, k0 = (int)crank * B + kl;
#pragma unroll
          for (int r = 0; r < C; r++)
            emit_fold<T, M, 4 * C, true>(v[g][r], r, k0 + 4096 * r, n, coefL + r * B + cpos<B / 16>(kl),
                                         coefL + (C + r) * B + cpos<B / 16>(kl), acc, dump);
        }
      } else {
#pragma unroll
        for (int g = 0; g < G; g++) {
          const int kl = (int)threadIdx.x + 512 * g, k0 = (int)crank * B + kl;
#pragma unroll
          for (int r = 0; r < C; r++)
            emit_fold<T, M, 4 * C, false>(v[g][r], r, k0 + 4096 * r, n, coefL + r * B + cpos<B / 16>(kl),
                                          coefL + (C + r) * B + cpos<B / 16>(kl), acc, nullptr);
        }
      }
    }
    cert_flush(acc, cs);
    __syncthreads();
    IVM_PH(6);
    cluster_sync();  // (3) coefficients and per-CTA certificates complete
    IVM_PH(7);
    // the C per-CTA certificates: lane p of warp 0 reads CTA p's, the warp
    // reduces, shared memory broadcasts (one remote read per CTA, not per thread)
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
    IVM_PH(8);
    const int ok = s_ok, bad = s_bad;
    const unsigned long long rad = s_rad;
    // carry: coefficient chunk ch (B coefficients, WB = B/4 words) lives in CTA ch mod C
    // at local chunk ch / C (cpos layout inside the chunk), so each CTA carries its own
    // 2C chunks with TPC = WB/4 threads per chunk and four words per thread
    // (Carry4); only the chunks' (generate, all-propagate) bits and the two words
    // below each chunk cross the cluster
    constexpr int NCH = 2 * C, WB = B / 4, TPC = WB / 4, NCHT = 2 * C * C;
    static_assert(NCH * TPC == 512, "one thread per four words");
    const int lc = (int)threadIdx.x / TPC, tc = (int)threadIdx.x % TPC, ch = lc * C + (int)crank;
    const int words = (nout + 3) / 4;
    uint8_t *out = kp.prod + (size_t)pair * nout;
    __shared__ unsigned s_w[16];  // TPC > 32: per-warp (generate, all-propagate)
    Carry4<TPC> cy;
    if (ok) {
      const unsigned cbase = (unsigned)__cvta_generic_to_shared(coefL);
      unsigned long long V[6];
#pragma unroll
      for (int j = 0; j < 6; j++) {
        const int wj = 4 * tc - 2 + j;  // word of this chunk (< 0: the chunk below)
        const int gi = ch * B + 4 * wj;  // global index of its first coefficient
        V[j] = 0ull;
        if (wj >= 0) {
          const int4 q = *reinterpret_cast<const int4 *>(coefL + lc * B + cpos<TPC>(4 * wj));
          V[j] = word_of((unsigned)q.x, (unsigned)q.y, (unsigned)q.z, (unsigned)q.w, gi, nc);
        } else if (ch > 0) {  // the last two words of chunk ch - 1 (CTA (ch-1) mod C)
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
    IVM_PH(9);
    cluster_sync();  // (4) every chunk's generate / all-propagate published
    IVM_PH(10);
    if (ok) {
      if (threadIdx.x < 32) {  // carries into all chunks: the ballot adder over 2C^2 bits
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
    if (!FAST && kp.coeffs) {
      int64_t *co = kp.coeffs + (size_t)pair * nc;
      for (int l = tc; l < B && ch * B + l < nc; l += TPC) co[ch * B + l] = ok ? (int64_t)coefL[lc * B + cpos<TPC>(l)] : 0;
    }
    if (crank == 0 && threadIdx.x == 0) {
      kp.cert[pair] = ok ? 1 : 0;
      if (kp.max_radius) kp.max_radius[pair] = __longlong_as_double((long long)rad);
      if (kp.first_bad) kp.first_bad[pair] = ok ? -1 : bad;
    }
    // (5) remote state / coefficient / chunk-bit reads done before the next pair
    // overwrites them: arrive now, wait just before the next state write (and
    // the next forward-last table, which replaces the coefficients)
    cluster_arrive_release();
    IVM_PH(11);
  }
  if (it > 0) cluster_wait();  // no CTA leaves while its shared memory may still be read
}

}  // namespace v4
}  // namespace ivm
