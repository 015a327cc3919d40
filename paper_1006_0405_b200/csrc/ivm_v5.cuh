// ivm_v5.cuh -- group kernel for m = 2^14 .. 2^18 (C = 2 .. 32 CTAs per
// multiplication; included by ivm_v5.cu).  The default route for m = 2^17, 2^18
// (too large for a thread-block cluster); for C <= 8 it is the alternative to
// the cluster kernel that packs onto every SM (clusters of 4 and 8 CTAs must fit
// a GPC, which strands SMs).
//
// The same row split and local m = 8192 schedule as the cluster kernel
// (ivm_v4.cuh), with the C CTAs of a group co-resident (cooperative launch) and
// exchanging through L2-resident global scratch with group barriers (global
// atomics) instead of DSMEM.
//   * after the local inverse passes 0..3 every CTA writes its column of the
//     4096 inverse rows to scratch; barrier;
//   * CTA c gathers rows [c B, c B + B) of all C columns and runs the last
//     inverse pass (radix C, untwist folded into the input twiddles): for
//     C <= 8 in registers, for C = 8 C2 > 8 as two shared-memory stages
//       out_{r1 + 8 r2} = sum_b w_{C2}^{-b r2} [ w_C^{-b r1} sum_a w_8^{-a r1} y_{C2 a + b} ],
//     then scales, certifies and snaps c_k, c_{k+m/2} (k = k0 + 4096 r) into
//     its own shared memory (int64: 255^2 n > 2^31 at m >= 2^17): chunk ch of B
//     consecutive coefficients lives in CTA ch mod C; every CTA publishes its
//     chunks' last 8 coefficients; barrier;
//   * each CTA carries its own 2C chunks (a team of max(1, 8/C) warps per chunk)
//     and publishes their generate / all-propagate bits; barrier; the carries
//     into all 2 C^2 chunks follow from one ballot adder; digits out.
#pragma once

namespace ivm {
namespace v5 {

using namespace v3;
using namespace v4;

struct Group5 {
  unsigned *ctr;   // [groups] barrier counters (zeroed by the host before the launch)
  void *xch;       // [groups][C][4096] CI<T> column exchange
  unsigned *link;  // [groups][C][8] per-CTA certificate words
  long long *bnd;  // [groups][2 C^2][8] last 8 coefficients of every chunk
  uint8_t *bits;   // [groups][2 C^2] chunk generate | all-propagate << 1
};

// a complex interval written by another SM: read through L2 only (no stale L1 lines)
template <typename T> __device__ __forceinline__ CI<T> ldcg_ci(const CI<T> *p) {
  if constexpr (sizeof(T) == 8) {
    const double2 a = __ldcg(reinterpret_cast<const double2 *>(p)), b = __ldcg(reinterpret_cast<const double2 *>(p) + 1);
    return CI<T>{a.x, a.y, b.x, b.y};
  } else {
    const float4 a = __ldcg(reinterpret_cast<const float4 *>(p));
    return CI<T>{a.x, a.y, a.z, a.w};
  }
}

template <typename T> __device__ __forceinline__ void st_ci(CI<T> *p, const CI<T> &z) {  // 16-B stores
  if constexpr (sizeof(T) == 8) {
    reinterpret_cast<double2 *>(p)[0] = make_double2(z.rl, z.rh);
    reinterpret_cast<double2 *>(p)[1] = make_double2(z.il, z.ih);
  } else {
    *reinterpret_cast<float4 *>(p) = make_float4(z.rl, z.rh, z.il, z.ih);
  }
}

// coefficients of one chunk (B consecutive c_i from `first`, shared memory) and
// the last 8 coefficients of the preceding chunk (global boundary array)
struct ChunkSrc {
  const long long *local;
  const long long *prev8;  // c_{first-8} .. c_{first-1} (shared copy; zeros for the first chunk)
  int first;
  __device__ __forceinline__ unsigned long long get(int i) const {
    // (chunks past the last word prime their empty segment from far below: 0)
    return i >= first ? (unsigned long long)local[i - first]
                      : (i >= first - 8 ? (unsigned long long)prev8[i - first + 8] : 0ull);
  }
  __device__ __forceinline__ void quad(int k, unsigned long long (&o)[4]) const {
    if (4 * k >= first) {  // wholly local (first and local are 32-byte aligned): two 16-byte loads
      const longlong2 *q = reinterpret_cast<const longlong2 *>(local + (4 * k - first));
      const longlong2 x = q[0], y = q[1];
      o[0] = (unsigned long long)x.x, o[1] = (unsigned long long)x.y;
      o[2] = (unsigned long long)y.x, o[3] = (unsigned long long)y.y;
      return;
    }
#pragma unroll
    for (int e = 0; e < 4; e++) o[e] = get(4 * k + e);
  }
  __device__ __forceinline__ unsigned long long one(int i) const { return get(i); }
};

// ---------------------------------------------------------------------------
// Tensor-core cross pass (fp64, C = 16, 32).  Row c of the first radix-C pass,
//   G[c][v] = sum_{q<C} theta_q x[v + 4096 q]   (theta_q: this role's twiddles),
// is a dense contraction of exact small integers once theta_q is written as
// T_q 2^-54 + err_q with T_q an integer (|err_q| <= 3 2^-55, checked by the
// table builder): the digits (u8) times T_q's seven balanced base-256 digits
// (s8) are summed EXACTLY by int8 MMAs (int32 accumulators: |sum| < 2^20),
// 16 columns x 8 limb rows x 32 q per mma.m16n8k32; the limb sums are
// recombined exactly in int64 and the only rounding is the final one:
//   G in [RD(S 2^-54 - E), RU(S 2^-54 + E)],  S = sum_q x_q T_q,  E = 3 2^-55 sum_q x_q
// (sum_q x_q is an eighth limb row of ones).  Exactness makes the interval
// tighter than the FP64 direct sum's and no directed rounding is needed until
// the end.  A fragment (digits, 16 columns x 32 q, row-major): lane (g, t) holds
// column rows g and g+8 for q = 4t..4t+3 and 16+4t..16+4t+3, built from 32-bit
// word loads (4 consecutive columns of one q) by 4x4 byte transposes; B
// fragments (four operands s per role, loaded once per call): column n = 2u + e
// holds limb 2s + e of part u & 1, so lane (g, t) of operand s receives limbs
// 2s, 2s+1 of part t & 1 for column rows g, g+8 (C fragment) and after the four
// MMAs holds all limbs of its part: lane t finishes (part t & 1, row t >> 1) with
// no cross-lane traffic (the four lanes of a group share the A fragment).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mma_u8s8(int (&d)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3,
                                         unsigned b0, unsigned b1) {
  asm(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%10,%10,%10};"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(0));
}

// o_j = (w0[j], w1[j], w2[j], w3[j]) (bytes, low first)
__device__ __forceinline__ void tr4x4(unsigned w0, unsigned w1, unsigned w2, unsigned w3, unsigned (&o)[4]) {
  const unsigned t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w0, w1, 0x7362);
  const unsigned t2 = __byte_perm(w2, w3, 0x5140), t3 = __byte_perm(w2, w3, 0x7362);
  o[0] = __byte_perm(t0, t2, 0x5410);
  o[1] = __byte_perm(t0, t2, 0x7632);
  o[2] = __byte_perm(t1, t3, 0x5410);
  o[3] = __byte_perm(t1, t3, 0x7632);
}

// this lane's B fragments (role crank): operand s -> {bf[2 s], bf[2 s + 1]} (k = 4t.., 16+4t..; n = g)
__device__ __forceinline__ void tc_limbs(const void *tab, unsigned crank, unsigned (&bf)[8]) {
  const unsigned *lt = reinterpret_cast<const unsigned *>(reinterpret_cast<const uint8_t *>(tab) + 1024u * crank);
  const unsigned lane = threadIdx.x & 31u, g = lane >> 2, t = lane & 3u;
#pragma unroll
  for (int s = 0; s < 4; s++) {
    bf[2 * s] = __ldg(lt + 64u * s + g * 8u + t);
    bf[2 * s + 1] = __ldg(lt + 64u * s + g * 8u + 4u + t);
  }
}

// 4 consecutive digits (columns v .. v+3 of one q row) as a word, zero past n
// (rem = n - index of p: the word is wholly inside or outside when WORDS)
template <bool WORDS>
__device__ __forceinline__ unsigned tc_ld4(const uint8_t *__restrict__ p, int rem) {
  if constexpr (WORDS) {
    return rem > 0 ? __ldg(reinterpret_cast<const unsigned *>(p)) : 0u;
  } else {
    unsigned w = 0u;
#pragma unroll
    for (int e = 0; e < 4; e++)
      if (e < rem) w |= (unsigned)__ldg(p + e) << (8 * e);
    return w;
  }
}

// the 16 words of one 64-column group (columns vb ..): [fragment register r][q offset i];
// every address is the lane's base plus a compile-time offset
template <int C, bool WORDS>
__device__ __forceinline__ void tc_load_group(const uint8_t *__restrict__ dig, int n, int vb, int g, int t,
                                              unsigned (&wv)[4][4]) {
  const int b0 = vb + 4 * g + 4096 * 4 * t;  // column vb + 4g, q = 4t
  const uint8_t *p = dig + b0;
  const int rem = n - b0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    wv[0][i] = tc_ld4<WORDS>(p + 4096 * i, rem - 4096 * i);
    wv[1][i] = tc_ld4<WORDS>(p + 32 + 4096 * i, rem - 32 - 4096 * i);
    wv[2][i] = C > 16 ? tc_ld4<WORDS>(p + 65536 + 4096 * i, rem - 65536 - 4096 * i) : 0u;
    wv[3][i] = C > 16 ? tc_ld4<WORDS>(p + 65536 + 32 + 4096 * i, rem - 65536 - 32 - 4096 * i) : 0u;
  }
}

template <int M, bool WORDS>
__device__ __forceinline__ void cross_tc_impl(const uint8_t *__restrict__ dig, int n, Buf<double> st,
                                              const unsigned (&bf)[8], bool odd) {
  constexpr int C = G4<M>::C;
  static_assert(C == 16 || C == 32, "K = 32 (C = 16: the upper half of K is zero)");
  const int lane = (int)(threadIdx.x & 31u), warp = (int)(threadIdx.x >> 5), g = lane >> 2, t = lane & 3;
  const bool rowhi = t >= 2, im = (t & 1) != 0;  // this lane finishes (part t & 1, column row t >> 1)
  unsigned nx[4][4];  // the next group's words, loaded while this group computes
  tc_load_group<C, WORDS>(dig, n, warp * 256, g, t, nx);
#pragma unroll 1
  for (int grp = 0; grp < 4; grp++) {  // 64 columns per group, 4 groups per warp (16 warps x 256)
    const int vb = warp * 256 + grp * 64;
    unsigned a[4][4];  // [fragment register][tile j]
#pragma unroll
    for (int r = 0; r < 4; r++) tr4x4(nx[r][0], nx[r][1], nx[r][2], nx[r][3], a[r]);
    if (grp < 3) tc_load_group<C, WORDS>(dig, n, vb + 64, g, t, nx);
#pragma unroll
    for (int j = 0; j < 4; j++) {  // tile j: column rows g -> vb + 4g + j, g+8 -> vb + 32 + 4g + j
      // operand s gives lane t the limb sums D_2s, D_2s+1 of its part (s = 3: D_6, sum x)
      int x[4][2];
#pragma unroll
      for (int s = 0; s < 4; s++) {
        int d[4];
        mma_u8s8(d, a[0][j], a[1][j], a[2][j], a[3][j], bf[2 * s], bf[2 * s + 1]);
        x[s][0] = rowhi ? d[2] : d[0];
        x[s][1] = rowhi ? d[3] : d[1];
      }
      // S = sum_i D_i 256^i = Lo + 2^32 H (exact: |Lo|, |H| < 2^45)
      const long long Lo = (long long)(x[0][0] + 256 * x[0][1]) + 65536ll * (long long)(x[1][0] + 256 * x[1][1]);
      const long long H = (long long)(x[2][0] + 256 * x[2][1]) + 65536ll * (long long)x[3][0];
      const double E = (double)x[3][1] * 8.326672684688674e-17;  // 3 2^-55 sum_q x_q (exact)
      const double Hd = (double)H, Ld = (double)Lo;
      const double lo = __fma_rd(Hd, 2.384185791015625e-07, __fma_rd(Ld, 5.551115123125783e-17, -E));
      const double hi = __fma_ru(Hd, 2.384185791015625e-07, __fma_ru(Ld, 5.551115123125783e-17, E));
      // one store per lane into its part's plane (the conjugate of odd roles by sign flips)
      const int v = vb + (rowhi ? 32 : 0) + 4 * g + j;
      const bool cj = im && odd;
      const double l2 = cj ? TB<double>::neg(hi) : lo, h2 = cj ? TB<double>::neg(lo) : hi;
      (im ? st.im : st.re)[v] = make_double2(l2, h2);
    }
  }
}

// ALIGNED: the caller guarantees word-aligned rows (only the word-load body is compiled)
template <int M, bool ALIGNED = false>
__device__ __forceinline__ void cross_tc(const uint8_t *__restrict__ dig, int n, Buf<double> st, const void *limbs,
                                         unsigned crank) {
  unsigned bf[8];  // (reloaded per call: L1-resident, and no registers held across the passes)
  tc_limbs(limbs, crank, bf);
  if (ALIGNED || ((reinterpret_cast<uintptr_t>(dig) | (uintptr_t)n) & 3) == 0) cross_tc_impl<M, true>(dig, n, st, bf, (crank & 1u) != 0u);
  else cross_tc_impl<M, false>(dig, n, st, bf, (crank & 1u) != 0u);
}

// group barrier: the CTA's writes (ordered before thread 0 by the block barrier)
// are released by thread 0's gpu-scope release add; the poll acquires the other
// CTAs' releases
__device__ __forceinline__ void gsync(unsigned *ctr, unsigned C, unsigned &gen) {
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

template <typename T, int M> struct Cfg5 {
  using GL = G3<13, 8>;
  static constexpr int THREADS = 512;
  static constexpr size_t E = sizeof(typename V2t<T>::t);
  static constexpr size_t STATE_BYTES = 2 * E * (size_t)GL::CAP;
  static constexpr int S_ENT = G4<M>::S_FO + 2 * G4<M>::C;
  static constexpr size_t TW_BYTES = sizeof(TwC<T>) * (size_t)S_ENT;
  static constexpr size_t SMEM = STATE_BYTES + TW_BYTES;
  static constexpr size_t A_BYTES = 2 * E * 4096;
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static_assert(STATE_BYTES >= 8 * 8192, "int64 coefficients fit the state");
};

// c = 2 Re / m, 2 Im / m of t = conj(w) o (w: compact first-quadrant twiddle),
// certified into d0, d1
template <typename T, int M>
__device__ __forceinline__ void emit_tab(const CI<T> &o, const TwC<T> &w, int k, int n, long long *d0,
                                         long long *d1, CertAcc &acc, double *dump) {
  constexpr int N = 1 << M;
  const CI<T> v = rtmul<T, true, false>(w, o);  // (the input twiddles carried the scale 2/m)
  certify_real(v.rl, v.rh, k, n, d0, acc, dump);
  certify_real(v.il, v.ih, k + N / 2, n, d1, acc, dump);
  dump_prerot(dump, k, N, o, T(1));
}

// QB: the cross pass skips its zero-padding terms in groups of 8 (host picks it
// when n <= m/2 - 8 * 4096, i.e. C3; ivm_v4.cuh cross_fwd)
template <typename T, int M, bool QB = false>
__global__ void __launch_bounds__(512, 1) ivm_v5_kernel(KParams kp, Group5 g) {
  using X = G4<M>;
  using GL = G3<13, 8>;
  using CF = Cfg5<T, M>;
  using V = typename V2t<T>::t;
  constexpr int C = X::C, B = X::B, R = 8, NL = 8192, N = 1 << M;
  constexpr bool TWO = C > 8;  // two-stage last inverse pass
  constexpr int C2 = TWO ? C / 8 : 1;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Cert3 cs;
  __shared__ __align__(8) unsigned long long tbar;
  Buf<T> st{reinterpret_cast<V *>(smem), reinterpret_cast<V *>(smem) + GL::CAP};
  TwC<T> *twb = reinterpret_cast<TwC<T> *>(smem + CF::STATE_BYTES);
  const CI<T> *theta = reinterpret_cast<const CI<T> *>(twb + X::S_TH);
  const TwC<T> *s2tw = twb + X::S_S2;  // w_C^{-j}: s2tw[2 j], upper-half form (G4::S2)
  const TwC<T> *fold = twb + X::S_FO;  // fold[2 r] = z^{4096 r}
  const unsigned crank = blockIdx.x % C;
  const int gi = (int)(blockIdx.x / C), ngr = (int)(gridDim.x / C);
  unsigned *ctr = g.ctr + gi;
  CI<T> *xch = reinterpret_cast<CI<T> *>(g.xch) + (size_t)gi * C * 4096;
  unsigned *link = g.link + (size_t)gi * C * 8;
  unsigned gen = 0;
  const TwC<T> *tw = reinterpret_cast<const TwC<T> *>(kp.tw);
  Buf<T> A{reinterpret_cast<V *>(kp.ascratch) + (size_t)blockIdx.x * NL, nullptr};
  A.im = A.re + NL / 2;
  const int n = kp.n, nc = 2 * n - 1, nout = 2 * n;
  constexpr int RSI1 = GL::iRS(1), SWI1 = GL::iSW(1);
  constexpr unsigned EB = sizeof(TwC<T>);

  if (threadIdx.x == 0) mbar_init(&tbar);
  __syncthreads();
  if (threadIdx.x == 0 && gi < kp.batch) {
    mbar_expect(&tbar, EB * (X::FLAST + X::MF_ENT + X::MI_ENT + 6 * C));
    bulk_copy(twb + X::S_SWAP, tw + X::FWD(crank) + X::FP(4), EB * X::FLAST, &tbar);
    bulk_copy(twb + X::S_MF, tw + X::FWD(crank), EB * X::MF_ENT, &tbar);
    bulk_copy(twb + X::S_MI, tw + X::INV, EB * X::MI_ENT, &tbar);
    bulk_copy(twb + X::S_TH, tw + X::TH(crank), EB * 2 * C, &tbar);
    bulk_copy(twb + X::S_S2, tw + X::S2, EB * 4 * C, &tbar);  // S2 and FO are adjacent
  }
  if (gi < kp.batch) mbar_wait(&tbar, 0);

  // fp64, C >= 16: the cross pass on the tensor cores (exact int8 MMAs, cross_tc)
#ifdef IVM_NO_TC
  constexpr bool TCX = false;
#else
  constexpr bool TCX = sizeof(T) == 8 && C >= 16;
#endif
  int it = 0;
  IVM_PH_DECL
  for (int pair = gi; pair < kp.batch; pair += ngr, it++) {
    const unsigned par = (unsigned)it & 1u;
    if (pair + ngr < kp.batch) {  // L2 prefetch of the next pair's digits (this CTA's slice)
      const int nxt = pair + ngr, sl = (n + C - 1) / C;
      for (int off = (int)crank * sl + (int)threadIdx.x * 128; off < min(n, ((int)crank + 1) * sl);
           off += (int)blockDim.x * 128) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.a + (size_t)nxt * n + off));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kp.b + (size_t)nxt * n + off));
      }
    }
#pragma unroll 1
    for (int op = 0; op < 2; op++) {
      if constexpr (TCX) cross_tc<M>((op == 0 ? kp.a : kp.b) + (size_t)pair * n, n, st, tw + X::LIMB, crank);
      else cross_fwd<T, M, QB>((op == 0 ? kp.a : kp.b) + (size_t)pair * n, n, st, theta, crank, false, true);
      if (op == 1 && threadIdx.x == 0) {
        cs.ok = 1;
        cs.first_bad = 0x7fffffff;
        cs.maxrad = 0ull;
      }
      __syncthreads();
      IVM_PH(2 * op);
#pragma unroll  // (specialised per pass: addresses fold into immediates)
      for (int i = 0; i < 4; i++) {
        const PassRT pp = pick_fwd4<M>(i);
        CI<T> v[R];
        int k0, nu;
        if (op == 0 && i == 3) mbar_wait(&tbar, par);
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
          CI<T> an = A.ld(k0);
#pragma unroll
          for (int r = 0; r < R; r++) {
            const CI<T> a = an;
            if (r + 1 < R) an = A.ld((r + 1) * (pp.L >> 1) + k0);
            v[r] = cmul_ss<T, true>(a, v[r]);
          }
          cdft<T, R, true>(v);
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
#pragma unroll  // (specialised per pass: addresses fold into immediates)
    for (int i = 0; i < 3; i++) {
      const PassRT pp = pick_inv4<M>(i);
      CI<T> v[R];
      int k0, nu;
      if (i == 2) mbar_wait(&tbar, par ^ 1u);
      invR<T, R, false>(st, twb, pp, v, k0, nu);
      if (i < 2) {
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; r++) st.st(sidx(k0 + pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
        __syncthreads();
      } else {  // last local pass: the column goes to the group's exchange scratch (row k0 + L r)
#pragma unroll
        for (int r = 0; r < R; r++) st_ci(xch + (size_t)crank * 4096 + k0 + pp.L * r, v[r]);
      }
    }
    __syncthreads();
    IVM_PH(4);
    if (threadIdx.x == 0) {  // last inverse pass table (this role's rows)
      mbar_expect(&tbar, EB * 4096);
      bulk_copy(twb + X::S_SWAP, tw + X::XINV(crank), EB * 4096, &tbar);
    }
    gsync(ctr, C, gen);  // (1) all columns written
    mbar_wait(&tbar, par);
    IVM_PH(5);
    CertAcc acc;
    // the coefficients (int64): fp64 two-stage into the twiddle swap buffer (free
    // until the next pair's forward-last table, fetched after the carry), else
    // into the state (free once every input is in registers)
    constexpr bool IN_SWAP = TWO && sizeof(TwC<T>) * 4096 >= 8 * 8192;
    long long *coefL = IN_SWAP ? reinterpret_cast<long long *>(twb + X::S_SWAP) : reinterpret_cast<long long *>(smem);
    if constexpr (!TWO) {  // radix C <= 8 in registers: task (g, kl), rows crank B + kl + 512 g
      constexpr int G = 8 / C;
      CI<T> v[G][C];
#pragma unroll
      for (int g = 0; g < G; g++) {
        const int kl = (int)threadIdx.x + 512 * g;
#pragma unroll
        for (int q = 0; q < C; q++) {
          const int src = (2 * q < C) ? 2 * q : 2 * C - 1 - 2 * q;
          const CI<T> z = ldcg_ci(xch + (size_t)src * 4096 + (int)crank * B + kl);
          const TwC<T> w = twb[X::S_SWAP + q * B + kl];
          v[g][q] = (2 * q < C) ? rtmul<T, true, true>(w, z) : rtmul_cd<T, false, true>(w, z);
        }
        cdft<T, C, true>(v[g]);
      }
      double *dump = diag_dump(kp, pair, N);
#pragma unroll
      for (int g = 0; g < G; g++) {
        const int kl = (int)threadIdx.x + 512 * g, k0 = (int)crank * B + kl;
#pragma unroll
        for (int r = 0; r < C; r++)
          emit_tab<T, M>(v[g][r], fold[2 * r], k0 + 4096 * r, n, coefL + r * B + cpos<B / 16>(kl), coefL + (C + r) * B + cpos<B / 16>(kl), acc, dump);
      }
    } else {
      {  // stage 1: task (b, kl): its inputs y_q(kl), q = C2 a + b, gathered straight from
         // the exchange (L2, coalesced over kl) with their input twiddles; DFT8 over a,
         // times w_C^{-b r1}.  The state is free (every local pass finished before the
         // group barrier), so the outputs are stored without a barrier.
        const int b = (int)threadIdx.x / B, kl = (int)threadIdx.x % B;
        CI<T> v[8];
#pragma unroll
        for (int a = 0; a < 8; a++) {
          const int q = C2 * a + b;
          const int src = (2 * q < C) ? 2 * q : 2 * C - 1 - 2 * q;
          const CI<T> z = ldcg_ci(xch + (size_t)src * 4096 + (int)crank * B + kl);
          const TwC<T> w = twb[X::S_SWAP + q * B + kl];
          v[a] = (2 * q < C) ? rtmul<T, true, true>(w, z) : rtmul_cd<T, false, true>(w, z);
        }
        cdft<T, 8, true>(v);
#pragma unroll
        for (int r1 = 1; r1 < 8; r1++) {  // b is warp-uniform (B >= 32)
          const int j = b * r1;
          const TwC<T> w = s2tw[2 * j];
          v[r1] = 2 * j <= C ? rtmul<T, true, true>(w, v[r1]) : rtmul<T, false, true>(w, v[r1]);
        }
#pragma unroll
        for (int r1 = 0; r1 < 8; r1++) st.st((r1 * C2 + b) * B + kl, v[r1]);
        __syncthreads();
      }
      // stage 2: task (r1, kl), DFT_C2 over b, untwist remainder, emit; chunk
      // ch = (h C + r) of B consecutive c_i (fp32, whose swap buffer is too
      // small, waits until every input is in registers)
      constexpr int TASKS = 8 * B / 512;
      {
        double *dump = diag_dump(kp, pair, N);
        if constexpr (IN_SWAP) {
#pragma unroll
          for (int g2 = 0; g2 < TASKS; g2++) {
            const int task = (int)threadIdx.x + 512 * g2, r1 = task / B, kl = task % B;
            const int k0 = (int)crank * B + kl;
            CI<T> v[C2];
#pragma unroll
            for (int b = 0; b < C2; b++) v[b] = st.ld((r1 * C2 + b) * B + kl);
            cdft<T, C2, true>(v);
#pragma unroll
            for (int r2 = 0; r2 < C2; r2++) {
              const int r = r1 + 8 * r2, k = k0 + 4096 * r;
              emit_tab<T, M>(v[r2], fold[2 * r], k, n, coefL + r * B + cpos<B / 16>(kl), coefL + (C + r) * B + cpos<B / 16>(kl), acc, dump);
            }
          }
        } else {
          CI<T> v[TASKS][C2];
#pragma unroll
          for (int g2 = 0; g2 < TASKS; g2++) {
            const int task = (int)threadIdx.x + 512 * g2, r1 = task / B, kl = task % B;
#pragma unroll
            for (int b = 0; b < C2; b++) v[g2][b] = st.ld((r1 * C2 + b) * B + kl);
          }
          __syncthreads();  // the state is free for the coefficients
#pragma unroll
          for (int g2 = 0; g2 < TASKS; g2++) {
            const int task = (int)threadIdx.x + 512 * g2, r1 = task / B, kl = task % B;
            const int k0 = (int)crank * B + kl;
            cdft<T, C2, true>(v[g2]);
#pragma unroll
            for (int r2 = 0; r2 < C2; r2++) {
              const int r = r1 + 8 * r2, k = k0 + 4096 * r;
              emit_tab<T, M>(v[g2][r2], fold[2 * r], k, n, coefL + r * B + cpos<B / 16>(kl), coefL + (C + r) * B + cpos<B / 16>(kl), acc, dump);
            }
          }
        }
      }
    }
    cert_flush(acc, cs);
    __syncthreads();
    IVM_PH(6);
    // chunk ch (global, B coefficients from ch B) is local chunk lc = ch / C of CTA ch % C
    // teams: one warp per chunk and NCH / 16 rounds (C >= 8), else one round of
    // 16 / NCH warps per chunk
    constexpr int NCH = 2 * C, NCHT = 2 * C * C, WB = B / 4;
    constexpr int TPC = WB / 4;  // threads per chunk, four words each (Carry4)
    static_assert(NCH * TPC == 512, "one thread per four words");
    long long *bnd = g.bnd + (size_t)gi * NCHT * 8;
    uint8_t *bits = g.bits + (size_t)gi * NCHT;
    for (int e = (int)threadIdx.x; e < NCH * 8; e += blockDim.x) {  // boundary words of the own chunks
      const int lc = e / 8, ch = lc * C + (int)crank;
      bnd[(size_t)ch * 8 + (e % 8)] = coefL[lc * B + cpos<B / 16>(B - 8 + (e % 8))];
    }
    if (threadIdx.x == 0) {
      link[crank * 8 + 0] = (unsigned)cs.ok;
      link[crank * 8 + 1] = (unsigned)cs.first_bad;
      link[crank * 8 + 2] = (unsigned)(cs.maxrad & 0xffffffffu);
      link[crank * 8 + 3] = (unsigned)(cs.maxrad >> 32);
    }
    gsync(ctr, C, gen);  // (2) certificates and chunk boundaries of every CTA visible
    IVM_PH(7);
    // the group's certificate: warp 0 reads the C link records (L2) and broadcasts;
    // meanwhile the other warps fetch the boundary coefficients before each own chunk
    __shared__ int s_ok, s_bad;
    __shared__ unsigned long long s_rad;
    __shared__ uint8_t s_cin[64];
    __shared__ long long s_prev[64][8];
    if (threadIdx.x >= 32) {
      for (int e = (int)threadIdx.x - 32; e < NCH * 8; e += (int)blockDim.x - 32) {
        const int lc = e / 8, ch = lc * C + (int)crank;
        s_prev[lc][e % 8] = ch > 0 ? __ldcg(bnd + (size_t)(ch - 1) * 8 + e % 8) : 0ll;
      }
    } else {
      const unsigned l = threadIdx.x;
      int okl = 1, badl = 0x7fffffff;
      unsigned long long radl = 0ull;
      if ((int)l < C) {
        const uint4 w = __ldcg(reinterpret_cast<const uint4 *>(link + l * 8));
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
      if (l == 0) {
        s_ok = okl;
        s_bad = badl;
        s_rad = radl;
      }
    }
    __syncthreads();
    IVM_PH(8);
    const int ok = s_ok, bad = s_bad;
    const unsigned long long rad = s_rad;
    const int words = (nout + 3) / 4;
    uint8_t *out = kp.prod + (size_t)pair * nout;
    // thread t carries words 4 tc .. 4 tc + 3 of its chunk lc (cpos layout); the two
    // words below a chunk's first come from s_prev (the chunk below, any CTA)
    const int lc = (int)threadIdx.x / TPC, tc = (int)threadIdx.x % TPC, ch = lc * C + (int)crank;
    __shared__ unsigned s_w[16];  // TPC > 32: per-warp (generate, all-propagate)
    Carry4<TPC> cy;
    if (ok) {
      unsigned long long V[6];
#pragma unroll
      for (int j = 0; j < 6; j++) {
        const int wj = 4 * tc - 2 + j, gi0 = ch * B + 4 * wj;
        unsigned long long c[4];
        if (wj >= 0) {
          const longlong2 *q = reinterpret_cast<const longlong2 *>(coefL + lc * B + cpos<TPC>(4 * wj));
          const longlong2 x = q[0], y = q[1];
          c[0] = (unsigned long long)x.x, c[1] = (unsigned long long)x.y;
          c[2] = (unsigned long long)y.x, c[3] = (unsigned long long)y.y;
        } else {
#pragma unroll
          for (int e = 0; e < 4; e++) c[e] = (unsigned long long)s_prev[lc][4 * (wj + 2) + e];
        }
        V[j] = (wj >= 0 || ch > 0) ? word_of(c[0], c[1], c[2], c[3], gi0, nc) : 0ull;
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
      if (tc == 0) bits[ch] = (uint8_t)cb;
    }
    IVM_PH(9);
    gsync(ctr, C, gen);  // (3) every chunk's generate / all-propagate visible
    IVM_PH(10);
    if (ok) {
      if (threadIdx.x < 32) {  // carries into all 2C^2 chunks: 64 chunks per lane, then across lanes
        const int l = (int)threadIdx.x;
        unsigned long long G = 0ull, P = ~0ull;  // beyond the chunks: propagate
        if (64 * l < NCHT) {
          if constexpr (NCHT % 64 == 0) {  // 4 x 16 B per lane
            P = 0ull;
            const uint4 *bp = reinterpret_cast<const uint4 *>(bits + 64 * l);
#pragma unroll
            for (int q = 0; q < 4; q++) {
              const uint4 w = __ldcg(bp + q);
              const unsigned ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
              for (int e = 0; e < 16; e++) {
                const unsigned bb = (ws[e >> 2] >> (8 * (e & 3))) & 3u;
                G |= (unsigned long long)(bb & 1u) << (16 * q + e);
                P |= (unsigned long long)(bb >> 1) << (16 * q + e);
              }
            }
          } else {  // NCHT = 8, 32: lane 0 only; the bits above NCHT propagate
            P = ~0ull << NCHT;
#pragma unroll
            for (int e = 0; e < NCHT; e++) {
              const unsigned bb = __ldcg(bits + e);
              G |= (unsigned long long)(bb & 1u) << e;
              P |= (unsigned long long)(bb >> 1) << e;
            }
          }
        }
        const unsigned long long X0 = (G | P) + G;
        const bool sg = X0 < (G | P), sp = P == ~0ull;  // segment generate / all-propagate
        const unsigned Gw = __ballot_sync(0xffffffffu, sg), Pw = __ballot_sync(0xffffffffu, sp);
        const unsigned cinl = ((((Gw | Pw) + Gw) ^ Pw) >> l) & 1u;
        const unsigned long long cb = ((G | P) + G + cinl) ^ P;  // carry into each chunk of the segment
        // own chunk lc (global ch = lc C + crank): bit ch % 64 of lane ch / 64's cb
#pragma unroll
        for (int h = 0; h < NCH; h += 32) {
          const int lc = h + l, ch = lc * C + (int)crank;
          const unsigned long long o = __shfl_sync(0xffffffffu, cb, min(ch >> 6, 31));
          if (lc < NCH) s_cin[lc] = (uint8_t)((o >> (ch & 63)) & 1ull);
        }
      }
      __syncthreads();
      unsigned d[4];
      cy.digits(cy.lane_cin(s_cin[lc], s_w), d);
      const int k0 = ch * WB + 4 * tc;
      if (k0 < words) store_words4(out, k0, nout, d);
    } else {
      for (int i = ch * B + 4 * tc; i < min(ch * B + B, nout); i += 4 * TPC)
        for (int b = 0; b < 4 && i + b < nout; b++) out[i + b] = 0;
    }
    if (kp.coeffs) {
      int64_t *co = kp.coeffs + (size_t)pair * nc;
      for (int e = (int)threadIdx.x; e < NCH * B; e += blockDim.x) {
        const int lc2 = e / B, i = (lc2 * C + (int)crank) * B + e % B;
        if (i < nc) co[i] = ok ? coefL[lc2 * B + cpos<B / 16>(e % B)] : 0;
      }
    }
    __syncthreads();  // coefficients read before the next pair's state / table writes
    IVM_PH(11);
    if (threadIdx.x == 0 && pair + ngr < kp.batch) {  // next pair's forward-last table
      mbar_expect(&tbar, EB * X::FLAST);
      bulk_copy(twb + X::S_SWAP, tw + X::FWD(crank) + X::FP(4), EB * X::FLAST, &tbar);
    }
    if (crank == 0 && threadIdx.x == 0) {
      kp.cert[pair] = ok ? 1 : 0;
      if (kp.max_radius) kp.max_radius[pair] = __longlong_as_double((long long)rad);
      if (kp.first_bad) kp.first_bad[pair] = ok ? -1 : bad;
    }
  }
}

}  // namespace v5
}  // namespace ivm
