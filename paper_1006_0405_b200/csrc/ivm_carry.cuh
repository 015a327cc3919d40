// ivm_carry.cuh -- carry of snapped coefficients to base-256 digits.
//
// c_i < 2^31 is split into bytes: t_i = sum_b byte_b(c_{i-b}) <= 1020,
// u_i = (t_i & 255) + (t_{i-1} >> 8) <= 258, so sum_i c_i 256^i = sum_i u_i 256^i
// and every remaining carry is 0 or 1: generate g_i = (u_i >= 256), propagate
// p_i = (u_i == 255); carries by a carry-lookahead over warp ballots
// (cin = ((G | P) + G + c0) ^ P), a block scan over warps, then one pass.
#pragma once
#include <stdint.h>

namespace ivm {

// coef: [2n-1] int32 (shared); ubuf: >= 2n+4 uint16 scratch (shared)
static __device__ __forceinline__ void carry_store(const int32_t *coef, int n, uint8_t *__restrict__ out, bool certified,
                                   uint16_t *ubuf) {
  const int nout = 2 * n;
  if (!certified) {
    for (int i = threadIdx.x; i < nout; i += blockDim.x) out[i] = 0;
    return;
  }
  const int nc = 2 * n - 1, npos = 2 * n + 4;
  const int T = blockDim.x, K = (npos + T - 1) / T;
  const int p0 = threadIdx.x * K, p1 = min(p0 + K, npos);
  // sliding window: c_{i-3..i}, t_{i-1}
  auto cget = [&](int i) -> unsigned { return (i >= 0 && i < nc) ? (unsigned)coef[i] : 0u; };
  unsigned c1 = cget(p0 - 1), c2 = cget(p0 - 2), c3 = cget(p0 - 3), c4 = cget(p0 - 4);
  int tprev = (int)((c1 & 255) + ((c2 >> 8) & 255) + ((c3 >> 16) & 255) + (c4 >> 24));
  int c = 0;
  bool allp = true;
  for (int i = p0; i < p1; i++) {
    const unsigned c0 = cget(i);
    const int t = (int)((c0 & 255) + ((c1 >> 8) & 255) + ((c2 >> 16) & 255) + (c3 >> 24));
    const int u = (t & 255) + (tprev >> 8);
    ubuf[i] = (uint16_t)u;
    allp = allp && (u == 255);
    c = (u + c) >> 8;
    tprev = t;
    c3 = c2;
    c2 = c1;
    c1 = c0;
  }
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (T + 31) >> 5;
  const unsigned g = __ballot_sync(0xffffffffu, c != 0), p = __ballot_sync(0xffffffffu, allp);
  __shared__ unsigned wg[32], wp[32], wc[32];
  if (lane == 0) {
    const unsigned long long s = (unsigned long long)(g | p) + g;
    wg[warp] = (unsigned)(s >> 32);
    wp[warp] = (p == 0xffffffffu);
  }
  __syncthreads();
  if (warp == 0) {
    const bool gg = lane < nwarps ? wg[lane] != 0 : false;
    const bool pp = lane < nwarps ? wp[lane] != 0 : true;
    const unsigned G2 = __ballot_sync(0xffffffffu, gg), P2 = __ballot_sync(0xffffffffu, pp);
    const unsigned cin = ((G2 | P2) + G2) ^ P2;
    if (lane < nwarps) wc[lane] = (cin >> lane) & 1u;
  }
  __syncthreads();
  const unsigned long long s = (unsigned long long)(g | p) + g + wc[warp];
  int cc = (int)((((unsigned)s ^ p) >> lane) & 1u);
  for (int i = p0; i < p1; i++) {
    const int u = (int)ubuf[i] + cc;
    if (i < nout) out[i] = (uint8_t)(u & 255);
    cc = u >> 8;
  }
}

}  // namespace ivm
