// ivm_fft.cuh -- in-register interval DFTs (radix-2 DIT-form butterflies).
//
// dft<T,R,INV>(v): v[r] <- sum_q v[q] * w_R^{+-qr}, w_R = e^{2 pi i/R}
// (inverse uses w^-1), computed as the paper's
// Cooley-Tukey recursion unrolled: bit-reversed input order,
// then log2 R stages of butterflies (E + w^j O, E - w^j O) -- the twiddle
// multiplies ONE input and is followed by the add/sub (DIT form).
// Twiddles w_{2h}^j are the optimal enclosures held in __constant__ memory
// (c_w32: w_32^j, j < 32); j = 0 and w = +-i are exact and cost no multiply.
#pragma once
#include "ivm_interval.cuh"

namespace ivm {

// w_32^j optimal enclosures (uploaded by the host planner; this header is
// included by exactly one translation unit, ivm_kernels.cu)
__constant__ CI<double> c_w32_f64[32];
__constant__ CI<float> c_w32_f32[32];

template <typename T> __device__ __forceinline__ const CI<T> &cw32(int j);
template <> __device__ __forceinline__ const CI<double> &cw32<double>(int j) { return c_w32_f64[j]; }
template <> __device__ __forceinline__ const CI<float> &cw32<float>(int j) { return c_w32_f32[j]; }

__host__ __device__ constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x / 2); }
__host__ __device__ constexpr int brev(int i, int bits) {  // non-recursive: folds after unrolling
  int r = 0;
  for (int b = 0; b < bits; b++) r |= ((i >> b) & 1) << (bits - 1 - b);
  return r;
}

// t = w_M^j * o (INV: conj(w)), M a power of two <= 32, j < M/2
template <typename T, bool INV>
__device__ __forceinline__ CI<T> const_twmul(const CI<T> &o, int j, int M) {
  if (j == 0) return o;
  if (4 * j == M) return INV ? mul_mi(o) : mul_i(o);
  CI<T> w = cw32<T>(j * (32 / M));
  if (INV) w = cconj(w);
  return twmul(w, o);
}

template <typename T, int R, bool INV>
__device__ __forceinline__ void dft(CI<T> (&v)[R]) {
  constexpr int B = ilog2c(R);
  CI<T> a[R];
#pragma unroll
  for (int i = 0; i < R; i++) a[i] = v[brev(i, B)];
#pragma unroll
  for (int h = 1; h < R; h *= 2) {
#pragma unroll
    for (int blk = 0; blk < R; blk += 2 * h) {
#pragma unroll
      for (int j = 0; j < h; j++) {
        CI<T> t = const_twmul<T, INV>(a[blk + j + h], j, 2 * h);
        bfly(a[blk + j], a[blk + j + h], t);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < R; i++) v[i] = a[i];
}

}  // namespace ivm
