// ivm_carry.cuh -- carry of snapped coefficients to base-256 digits.
#pragma once
#include <stdint.h>

namespace ivm {

// ---------------------------------------------------------------------------
// carry: c_i < 2^31 split into bytes; t_i = sum_b byte_b(c_{i-b})
// <= 1020; u_i = (t_i & 255) + (t_{i-1} >> 8) <= 258; then binary carries
// with generate u >= 256 / propagate u == 255 (carry-lookahead by ballots).
// ---------------------------------------------------------------------------
static __device__ __forceinline__ int coef_at(const int32_t *coef, int i, int nc) {
  return (i >= 0 && i < nc) ? coef[i] : 0;
}
static __device__ __forceinline__ int t_at(const int32_t *coef, int i, int nc) {
  int t = 0;
#pragma unroll
  for (int b = 0; b < 4; b++) t += (coef_at(coef, i - b, nc) >> (8 * b)) & 255;
  return t;
}
static __device__ __forceinline__ int u_at(const int32_t *coef, int i, int nc) {
  return (t_at(coef, i, nc) & 255) + (t_at(coef, i - 1, nc) >> 8);
}

static __device__ void carry_store(const int32_t *coef, int n, uint8_t *__restrict__ out, bool certified) {
  const int nout = 2 * n;
  if (!certified) {
    for (int i = threadIdx.x; i < nout; i += blockDim.x) out[i] = 0;
    return;
  }
  const int nc = 2 * n - 1, npos = 2 * n + 4;
  const int T = blockDim.x, K = (npos + T - 1) / T;
  const int p0 = threadIdx.x * K, p1 = min(p0 + K, npos);
  // chunk generate / propagate
  int c = 0;
  bool allp = true;
  for (int i = p0; i < p1; i++) {
    int u = u_at(coef, i, nc);
    allp = allp && (u == 255);
    c = (u + c) >> 8;
  }
  const bool G = c != 0, Pp = allp;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (T + 31) >> 5;
  const unsigned g = __ballot_sync(0xffffffffu, G), p = __ballot_sync(0xffffffffu, Pp);
  __shared__ unsigned wg[32], wp[32], wc[32];
  if (lane == 0) {
    unsigned long long s = (unsigned long long)(g | p) + g;
    wg[warp] = (unsigned)(s >> 32);
    wp[warp] = (p == 0xffffffffu);
  }
  __syncthreads();
  if (warp == 0) {
    bool gg = lane < nwarps ? wg[lane] != 0 : false;
    bool pp = lane < nwarps ? wp[lane] != 0 : true;
    unsigned G2 = __ballot_sync(0xffffffffu, gg), P2 = __ballot_sync(0xffffffffu, pp);
    unsigned cin = ((G2 | P2) + G2) ^ P2;
    if (lane < nwarps) wc[lane] = (cin >> lane) & 1u;
  }
  __syncthreads();
  const unsigned c0 = wc[warp];
  const unsigned long long s = (unsigned long long)(g | p) + g + c0;
  const unsigned cin_vec = (unsigned)s ^ p;
  int cc = (cin_vec >> lane) & 1u;
  for (int i = p0; i < p1; i++) {
    int u = u_at(coef, i, nc) + cc;
    if (i < nout) out[i] = (uint8_t)(u & 255);
    cc = u >> 8;
  }
}

}  // namespace ivm
