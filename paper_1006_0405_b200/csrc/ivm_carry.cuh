// ivm_carry.cuh -- carry of snapped coefficients to base-256 digits.
//
// Word form of the carry.  Four digit positions make one 32-bit word:
//   V_k = sum_{b<4} c_{4k+b} 256^b  (< 2^58 for 0 <= c_i < 2^33),  sum_i c_i 256^i = sum_k V_k 2^{32k}.
// With V_k = lo_k + hi_k 2^32 the word sums W_k = lo_k + hi_{k-1} < 2^33 and
// u_k = (W_k mod 2^32) + floor(W_{k-1} / 2^32) <= 2^32 leave carries of 0 or 1:
// generate g_k = (u_k == 2^32), propagate p_k = (u_k == 2^32 - 1), and the
// carry into word k is c_k = g_{k-1} | (p_{k-1} & c_{k-1}).  Inside a warp the
// 32 carries of one step come from the ballot adder cin = ((G|P) + G + c0) ^ P
// (bit l of the sum (G|P) + G + c0 is the carry into lane l, complemented where
// P_l), across warps (and across the CTAs of a cluster) from the same adder on
// the per-warp (per-CTA) generate / all-propagate bits; the digits are the
// bytes of (u_k + c_k) mod 2^32.  Lane l of warp w handles word
// k = k_begin + w 32 J + 32 j + l, so coefficient reads (16 B per lane) and the
// digit stores are contiguous.
#pragma once
#include <stdint.h>

namespace ivm {

// word k of the split: (low 32 bits, high bits) of V_k; c_i = 0 outside [0, nc).
// Src::quad(k, c) fills c_{4k .. 4k+3} (only called when 4k + 3 < nc);
// Src::one(i) returns c_i.  Coefficients are < 2^33 (255^2 n, n <= 2^17), so
// V_k < 2^58 and hi_k < 2^26.
template <typename Src>
static __device__ __forceinline__ void carry_word(const Src &src, int nc, int k, unsigned &lo, unsigned &hi) {
  if (k < 0 || 4 * k >= nc) {
    lo = hi = 0u;
    return;
  }
  unsigned long long c[4];
  if (4 * k + 3 < nc) {
    src.quad(k, c);
  } else {
    c[0] = src.one(4 * k);
    c[1] = 4 * k + 1 < nc ? src.one(4 * k + 1) : 0ull;
    c[2] = 4 * k + 2 < nc ? src.one(4 * k + 2) : 0ull;
    c[3] = 0ull;
  }
  const unsigned long long v = c[0] + (c[1] << 8) + (c[2] << 16) + (c[3] << 24);
  lo = (unsigned)v;
  hi = (unsigned)(v >> 32);
}

// a plain [nc] int32 array (16-byte aligned)
struct CoefLinear {
  const int32_t *c;
  __device__ __forceinline__ void quad(int k, unsigned long long (&o)[4]) const {
    const int4 q = reinterpret_cast<const int4 *>(c)[k];
    o[0] = (unsigned)q.x, o[1] = (unsigned)q.y, o[2] = (unsigned)q.z, o[3] = (unsigned)q.w;
  }
  __device__ __forceinline__ unsigned long long one(int i) const { return (unsigned)c[i]; }
};

// per step: u (mod 2^32) and the generate / propagate bits of this lane's word.
// hprev / eprev: hi_{k-1} and floor(W_{k-1} / 2^32) of the word below lane 0.
struct CarryStep {
  unsigned u;
  bool g, p;
  unsigned hi_top, ov_top;  // lane 31's hi and overflow, for the next step's lane 0
};
template <typename Src>
static __device__ __forceinline__ CarryStep carry_step(const Src &src, int nc, int k, unsigned lane, unsigned hprev,
                                                       unsigned eprev) {
  unsigned lo, hi;
  carry_word(src, nc, k, lo, hi);
  unsigned hp = __shfl_up_sync(0xffffffffu, hi, 1);
  if (lane == 0) hp = hprev;
  const unsigned w = lo + hp;
  const unsigned ov = w < lo ? 1u : 0u;  // floor(W_k / 2^32)
  unsigned ep = __shfl_up_sync(0xffffffffu, ov, 1);
  if (lane == 0) ep = eprev;
  CarryStep s;
  s.u = w + ep;
  s.g = ep != 0u && w == 0xffffffffu;
  s.p = s.u == 0xffffffffu && !s.g;
  s.hi_top = __shfl_sync(0xffffffffu, hi, 31);
  s.ov_top = __shfl_sync(0xffffffffu, ov, 31);
  return s;
}

// Carry over the words [kb, ke) by a team of nw warps (warps w0 .. w0+nw-1 of
// the block; by default the whole block).  Phase 1 (carry_seg_scan): every
// warp scans its sub-segment with carry-in 0; returns the team's generate
// (carry out with carry-in 0) and all-propagate bits.  Phase 2 (carry_seg_emit):
// given the team's carry-in, writes the digits of the words.  Every thread of
// the block calls both (all teams at once: they contain a __syncthreads);
// CarrySeg lives in shared memory.
struct CarrySeg {
  unsigned wg[32], wp[32];
};
template <typename Src>
static __device__ __forceinline__ void carry_seg_scan(const Src &src, int nc, int kb, int ke, CarrySeg &cs,
                                                      unsigned &gen, unsigned &allp, int w0 = 0, int nw = 0) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned nwarps = nw ? (unsigned)nw : blockDim.x >> 5, warp = (threadIdx.x >> 5) - (unsigned)w0;
  const int J = (ke - kb + 32 * (int)nwarps - 1) / (32 * (int)nwarps);
  const int k0 = kb + (int)warp * 32 * J;
  unsigned hp, ep;
  {
    unsigned l1, h1, l2, h2;
    carry_word(src, nc, k0 - 1, l1, h1);
    carry_word(src, nc, k0 - 2, l2, h2);
    hp = h1;
    ep = (l1 + h2) < l1 ? 1u : 0u;
  }
  unsigned c = 0u;
  bool ap = true;
  for (int j = 0; j < J; j++) {
    const int k = k0 + 32 * j + (int)lane;
    const CarryStep s = carry_step(src, nc, k, lane, hp, ep);
    // words beyond the segment neither generate nor propagate
    const bool in = k < ke;
    const unsigned G = __ballot_sync(0xffffffffu, in && s.g), P = __ballot_sync(0xffffffffu, !in || s.p);
    const unsigned long long S = (unsigned long long)(G | P) + G + c;
    c = (unsigned)(S >> 32);
    ap = ap && (P == 0xffffffffu);
    hp = s.hi_top;
    ep = s.ov_top;
  }
  if (nw == 1) {  // a one-warp team: its carry-out is the segment's (no block barrier)
    gen = c;
    allp = ap ? 1u : 0u;
    return;
  }
  if (lane == 0) {
    cs.wg[w0 + warp] = c;
    cs.wp[w0 + warp] = ap ? 1u : 0u;
  }
  __syncthreads();
  // the team's per-warp bits: lane w reads warp w's, two ballots gather them
  const bool gw = lane < nwarps && cs.wg[w0 + lane] != 0u, pw = lane < nwarps && cs.wp[w0 + lane] != 0u;
  const unsigned G2 = __ballot_sync(0xffffffffu, gw), P2 = __ballot_sync(0xffffffffu, pw);
  const unsigned long long S = (unsigned long long)(G2 | P2) + G2;
  gen = (unsigned)(S >> nwarps) & 1u;
  allp = (nwarps == 32 ? P2 == 0xffffffffu : P2 == ((1u << nwarps) - 1u)) ? 1u : 0u;
}

template <typename Src>
static __device__ __forceinline__ void carry_seg_emit(const Src &src, int nc, int nout, int kb, int ke,
                                                      const CarrySeg &cs, unsigned cin, uint8_t *__restrict__ out,
                                                      int w0 = 0, int nw = 0) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned nwarps = nw ? (unsigned)nw : blockDim.x >> 5, warp = (threadIdx.x >> 5) - (unsigned)w0;
  const int J = (ke - kb + 32 * (int)nwarps - 1) / (32 * (int)nwarps);
  const int k0 = kb + (int)warp * 32 * J;
  const bool gw = nw != 1 && lane < nwarps && cs.wg[w0 + lane] != 0u;
  const bool pw = nw != 1 && lane < nwarps && cs.wp[w0 + lane] != 0u;
  const unsigned G2 = __ballot_sync(0xffffffffu, gw), P2 = __ballot_sync(0xffffffffu, pw);
  const unsigned long long S0 = (unsigned long long)(G2 | P2) + G2 + cin;
  unsigned c = nw == 1 ? cin : (unsigned)((S0 ^ P2) >> warp) & 1u;  // carry into this warp's sub-segment
  unsigned hp, ep;
  {
    unsigned l1, h1, l2, h2;
    carry_word(src, nc, k0 - 1, l1, h1);
    carry_word(src, nc, k0 - 2, l2, h2);
    hp = h1;
    ep = (l1 + h2) < l1 ? 1u : 0u;
  }
  const bool wide = (reinterpret_cast<uintptr_t>(out) & 3) == 0;
  for (int j = 0; j < J; j++) {
    const int k = k0 + 32 * j + (int)lane;
    const CarryStep s = carry_step(src, nc, k, lane, hp, ep);
    const bool in = k < ke;
    const unsigned G = __ballot_sync(0xffffffffu, in && s.g), P = __ballot_sync(0xffffffffu, !in || s.p);
    const unsigned long long S = (unsigned long long)(G | P) + G + c;
    const unsigned cl = (((unsigned)S ^ P) >> lane) & 1u;
    c = (unsigned)(S >> 32);
    hp = s.hi_top;
    ep = s.ov_top;
    if (!in) continue;
    const unsigned d = s.u + cl;
    const int i = 4 * k;
    if (i + 3 < nout && wide) {
      *reinterpret_cast<unsigned *>(out + i) = d;
    } else {
#pragma unroll
      for (int b = 0; b < 4; b++)
        if (i + b < nout) out[i + b] = (uint8_t)(d >> (8 * b));
    }
  }
}

// whole product in one CTA.  coef: [2n-1] int32, 16-byte aligned (shared);
// out: [2n] digits (global).  Uncertified pairs get zero digits.
static __device__ __forceinline__ void carry_store(const int32_t *coef, int n, uint8_t *__restrict__ out,
                                                   bool certified) {
  const int nout = 2 * n, nc = 2 * n - 1;
  if (!certified) {
    for (int i = threadIdx.x; i < nout; i += blockDim.x) out[i] = 0;
    return;
  }
  __shared__ CarrySeg seg;
  const CoefLinear src{coef};
  const int words = (nout + 3) / 4;
  unsigned gen, allp;
  carry_seg_scan(src, nc, 0, words, seg, gen, allp);
  carry_seg_emit(src, nc, nout, 0, words, seg, 0u, out);
}

}  // namespace ivm

namespace ivm {

// Coefficient i of the one-CTA kernel lives at cpos<QS>(i): quad Q (c_4Q .. c_4Q+3)
// at quad slot (Q & 3) QS + Q / 4, so that thread t's quads 4t .. 4t+3 (its four
// words) are QS slots apart and a warp's 16-byte reads of them hit consecutive
// slots (no bank conflicts).  QS = 0: linear.
template <int QS>
__device__ __forceinline__ int cpos(int i) {
  if constexpr (QS == 0) {
    return i;
  } else {
    const int Q = i >> 2;
    return ((((Q & 3) * QS) + (Q >> 2)) << 2) | (i & 3);
  }
}

// One-pass carry with four consecutive words per thread (words 4t .. 4t+3, word
// k = c_4k .. c_4k+3, P:229-235 in the word form above): every thread forms its
// u_k, generate and propagate bits in registers (two more words below its own
// come from the quads 4t-2, 4t-1), one ballot adder over the warp's lanes and
// one over the block's warps give each thread its carry-in, and its 16 digit
// bytes are stored at once.  coef: cpos<QS> layout in shared memory, QS =
// blockDim.x (>= the number of words / 4); out: [2n] digits (global).
template <int QS>
static __device__ __forceinline__ void carry_store4(const int32_t *coef, int n, uint8_t *__restrict__ out,
                                                    bool certified) {
  const int nout = 2 * n, nc = 2 * n - 1, words = (nout + 3) / 4;
  const int t = (int)threadIdx.x, lane = t & 31, warp = t >> 5, nwarps = (int)(blockDim.x >> 5);
  if (!certified) {
    for (int i = t; i < nout; i += blockDim.x) out[i] = 0;
    return;
  }
  __shared__ unsigned s_wgp[32];
  unsigned lo[6], hi[6];
#pragma unroll
  for (int j = 0; j < 6; j++) {  // words 4t-2 .. 4t+3
    const int Q = 4 * t - 2 + j;
    unsigned long long v = 0ull;
    if (Q >= 0 && 4 * Q < nc) {
      const int4 q = *reinterpret_cast<const int4 *>(coef + cpos<QS>(4 * Q));
      const unsigned long long c1 = 4 * Q + 1 < nc ? (unsigned)q.y : 0u, c2 = 4 * Q + 2 < nc ? (unsigned)q.z : 0u,
                               c3 = 4 * Q + 3 < nc ? (unsigned)q.w : 0u;
      v = (unsigned long long)(unsigned)q.x + (c1 << 8) + (c2 << 16) + (c3 << 24);
    }
    lo[j] = (unsigned)v;
    hi[j] = (unsigned)(v >> 32);
  }
  // W_k = lo_k + hi_{k-1} = w_k + e_k 2^32;  u_k = w_k + e_{k-1} <= 2^32
  unsigned w[6], e[6];
#pragma unroll
  for (int j = 1; j < 6; j++) {
    w[j] = lo[j] + hi[j - 1];
    e[j] = w[j] < lo[j] ? 1u : 0u;
  }
  unsigned u[4];
  bool g[4], p[4];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    u[i] = w[i + 2] + e[i + 1];
    g[i] = e[i + 1] != 0u && w[i + 2] == 0xffffffffu;
    p[i] = u[i] == 0xffffffffu && !g[i];
  }
  const bool G = g[3] || (p[3] && (g[2] || (p[2] && (g[1] || (p[1] && g[0])))));
  const bool P = p[0] && p[1] && p[2] && p[3];
  const unsigned Gw = __ballot_sync(0xffffffffu, G), Pw = __ballot_sync(0xffffffffu, P);
  if (lane == 0) {
    const unsigned gen = (unsigned)((((unsigned long long)(Gw | Pw)) + Gw) >> 32);
    s_wgp[warp] = gen | ((Pw == 0xffffffffu ? 1u : 0u) << 1);
  }
  __syncthreads();
  const unsigned wb = lane < nwarps ? s_wgp[lane] : 0u;
  const unsigned G2 = __ballot_sync(0xffffffffu, (wb & 1u) != 0u), P2 = __ballot_sync(0xffffffffu, (wb & 2u) != 0u);
  const unsigned cw = ((((G2 | P2) + G2) ^ P2) >> warp) & 1u;  // carry into this warp (0 into the first)
  unsigned c = (unsigned)((((unsigned long long)(Gw | Pw)) + Gw + cw) ^ Pw) >> lane & 1u;
  unsigned d[4];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    d[i] = u[i] + c;
    c = (g[i] || (p[i] && c != 0u)) ? 1u : 0u;
  }
  const int k0 = 4 * t;
  if (k0 >= words) return;
  const int i0 = 4 * k0;  // first digit of this thread
  if (i0 + 15 < nout && ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
    *reinterpret_cast<uint4 *>(out + i0) = make_uint4(d[0], d[1], d[2], d[3]);
  } else {
#pragma unroll
    for (int b = 0; b < 16; b++)
      if (i0 + b < nout) out[i0 + b] = (uint8_t)(d[b >> 2] >> (8 * (b & 3)));
  }
  (void)s_wgp;
}

}  // namespace ivm

namespace ivm {

// Chunked form of the four-words-per-thread carry (the cluster and group
// kernels: every CTA carries 2C chunks of B/4 words, TPC = B/16 threads per
// chunk, chunk carry-ins from a cluster/group-level adder in between).
//   words(V): V = the six words 4t-2 .. 4t+3 of this thread (two below its own);
//   seg_bits(): (generate | all-propagate << 1) of this thread's chunk when
//     TPC <= 32 (a lane segment), of its warp when TPC > 32;
//   chunk_bits(sw): TPC > 32, sw = the block's per-warp seg_bits (shared memory);
//   lane_cin(cin, sw): carry into this thread's first word given the chunk's;
//   digits(c, d): the four digit words.
template <int TPC>
struct Carry4 {
  static_assert(TPC >= 2 && TPC <= 512 && (TPC & (TPC - 1)) == 0, "threads per chunk");
  unsigned u[4];
  unsigned gb, pb;  // bit i: generate / propagate of word i
  unsigned Gw, Pw;  // the warp's ballots of the per-thread composites

  __device__ __forceinline__ void words(const unsigned long long (&V)[6]) {
    unsigned lo[6], hi[6], w[6], e[6];
#pragma unroll
    for (int j = 0; j < 6; j++) {
      lo[j] = (unsigned)V[j];
      hi[j] = (unsigned)(V[j] >> 32);
    }
#pragma unroll
    for (int j = 1; j < 6; j++) {
      w[j] = lo[j] + hi[j - 1];
      e[j] = w[j] < lo[j] ? 1u : 0u;
    }
    gb = pb = 0u;
#pragma unroll
    for (int i = 0; i < 4; i++) {
      u[i] = w[i + 2] + e[i + 1];
      const bool g = e[i + 1] != 0u && w[i + 2] == 0xffffffffu;
      const bool p = u[i] == 0xffffffffu && !g;
      gb |= (g ? 1u : 0u) << i;
      pb |= (p ? 1u : 0u) << i;
    }
    // the thread's composite over its 4 words: the same ballot adder on 4 bits
    const bool G = ((((gb | pb) + gb) >> 4) & 1u) != 0u, P = pb == 15u;
    Gw = __ballot_sync(0xffffffffu, G);
    Pw = __ballot_sync(0xffffffffu, P);
  }
  __device__ __forceinline__ unsigned seg_bits() const {
    if constexpr (TPC >= 32) {
      const unsigned gen = (unsigned)(((unsigned long long)(Gw | Pw) + Gw) >> 32);
      return gen | ((Pw == 0xffffffffu ? 1u : 0u) << 1);
    } else {
      constexpr unsigned MASK = (1u << TPC) - 1u;
      const unsigned sh = (threadIdx.x & 31u) / TPC * TPC;
      const unsigned Gs = (Gw >> sh) & MASK, Ps = (Pw >> sh) & MASK;
      return ((((Gs | Ps) + Gs) >> TPC) & 1u) | ((Ps == MASK ? 1u : 0u) << 1);
    }
  }
  // TPC > 32: fold the chunk's warps (first .. first + TPC/32 - 1) of sw, in word order
  static __device__ __forceinline__ unsigned chunk_bits(const unsigned *sw) {
    constexpr int WPC = TPC / 32;
    const int first = (int)(threadIdx.x >> 5) / WPC * WPC;
    unsigned g = 0u, a = 1u;
#pragma unroll
    for (int j = 0; j < WPC; j++) {
      const unsigned b = sw[first + j];
      g = (b & 1u) | (((b >> 1) & 1u) & g);
      a &= (b >> 1) & 1u;
    }
    return g | (a << 1);
  }
  __device__ __forceinline__ unsigned lane_cin(unsigned cin, const unsigned *sw) const {
    const unsigned lane = threadIdx.x & 31u;
    if constexpr (TPC >= 32) {
      unsigned cw = cin;  // through the chunk's warps below this one
      if constexpr (TPC > 32) {
        constexpr int WPC = TPC / 32;
        const int wi = (int)(threadIdx.x >> 5) % WPC, first = (int)(threadIdx.x >> 5) - wi;
        for (int j = 0; j < wi; j++) {
          const unsigned b = sw[first + j];
          cw = (b & 1u) | (((b >> 1) & 1u) & cw);
        }
      }
      return (unsigned)(((((unsigned long long)(Gw | Pw)) + Gw + cw) ^ Pw) >> lane) & 1u;
    } else {
      constexpr unsigned MASK = (1u << TPC) - 1u;
      const unsigned sh = lane / TPC * TPC;
      const unsigned Gs = (Gw >> sh) & MASK, Ps = (Pw >> sh) & MASK;
      return ((((Gs | Ps) + Gs + cin) ^ Ps) >> (lane - sh)) & 1u;
    }
  }
  __device__ __forceinline__ void digits(unsigned c, unsigned (&d)[4]) const {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      d[i] = u[i] + c;
      c = ((gb >> i) & 1u) | (((pb >> i) & 1u) & c);
    }
  }
};

// the 16 digit bytes of words k0 .. k0+3 (digit 4 k0 on), clipped to nout
__device__ __forceinline__ void store_words4(uint8_t *__restrict__ out, int k0, int nout, const unsigned (&d)[4]) {
  const int i0 = 4 * k0;
  if (i0 >= nout) return;
  if (i0 + 15 < nout && ((reinterpret_cast<uintptr_t>(out + i0) & 15) == 0)) {
    *reinterpret_cast<uint4 *>(out + i0) = make_uint4(d[0], d[1], d[2], d[3]);
  } else {
#pragma unroll
    for (int b = 0; b < 16; b++)
      if (i0 + b < nout) out[i0 + b] = (uint8_t)(d[b >> 2] >> (8 * (b & 3)));
  }
}

// word value V = c0 + c1 2^8 + c2 2^16 + c3 2^24 of four coefficients (those at
// global index >= nc are zero)
__device__ __forceinline__ unsigned long long word_of(unsigned long long c0, unsigned long long c1,
                                                      unsigned long long c2, unsigned long long c3, int i0, int nc) {
  if (i0 >= nc) return 0ull;
  c1 = i0 + 1 < nc ? c1 : 0ull;
  c2 = i0 + 2 < nc ? c2 : 0ull;
  c3 = i0 + 3 < nc ? c3 : 0ull;
  return c0 + (c1 << 8) + (c2 << 16) + (c3 << 24);
}

}  // namespace ivm
