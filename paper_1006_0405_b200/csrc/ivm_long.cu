// ivm_long.cu -- exact base-256 long multiplication on the GPU: the
// paper's guaranteed-correct comparator and the last tier of the
// precision escalation ("increase the precision ... or use a different
// algorithm").
//
// s_k = sum_{i+j=k} x_i y_j (step 7) is computed exactly: a CTA owns a
// tile of T = 256 consecutive k for one pair (thread t: k = k0 + t) and walks the
// i range in chunks of CH digits staged in shared memory, x forward and y
// reversed, so that x_i y_{k-i} for four consecutive i is one byte dot product
// (__dp4a) of an aligned x word and a byte-shifted (__byte_perm) reversed-y word.
// A chunk's partial sum is < CH 255^2 < 2^32; the tile sums are accumulated in
// 64 bits.  The carry of steps 9-10 is the word-form carry of ivm_carry.cuh over
// the exact sums (one CTA per pair).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ivm_internal.h"
#include "ivm_carry.cuh"

namespace ivm {

namespace lm {

constexpr int T = 256;     // outputs per CTA (one per thread)
constexpr int CH = 4096;   // digits of x per chunk (partial sums < 4096 * 255^2 < 2^32)

__global__ void __launch_bounds__(T) long_coef_kernel(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b,
                                                      int n, long long *__restrict__ coef) {
  __shared__ __align__(16) uint8_t xs[CH];
  __shared__ __align__(16) uint8_t yr[CH + T + 16];
  const int pair = blockIdx.y, k0 = blockIdx.x * T, t = threadIdx.x, nc = 2 * n - 1;
  const uint8_t *x = a + (size_t)pair * n, *y = b + (size_t)pair * n;
  const int k = k0 + t;
  unsigned long long s = 0;
  // chunks of i that meet [k0 - (n-1), k0 + T - 1]
  const int ilo = max(0, k0 - (n - 1)), ihi = min(n - 1, k0 + T - 1);
  for (int i0 = ilo - ilo % 4; i0 <= ihi; i0 += CH) {
    // stage x[i0 .. i0+CH) and yr[u] = y[(k0 + T - 1 - i0) - u] (zero outside [0, n))
    __syncthreads();
    for (int u = t; u < CH; u += T) {
      const int i = i0 + u;
      xs[u] = (i < n) ? x[i] : 0;
    }
    const int top = k0 + T - 1 - i0;
    for (int u = t; u < CH + T + 16; u += T) {
      const int j = top - u;
      yr[u] = (j >= 0 && j < n) ? y[j] : 0;
    }
    __syncthreads();
    // thread t: y_{k-i} = yr[(T-1-t) + (i-i0)]
    const int o = T - 1 - t, sh = o & 3;
    const unsigned *xw = reinterpret_cast<const unsigned *>(xs);
    const unsigned *yw = reinterpret_cast<const unsigned *>(yr) + (o >> 2);
    const unsigned sel = 0x3210u + 0x1111u * (unsigned)sh;  // bytes sh..sh+3 of (w1:w0)
    const int iend = min(CH, ihi - i0 + 1), words = (iend + 3) >> 2;
    unsigned acc = 0, w0 = yw[0];
#pragma unroll 4
    for (int u = 0; u < words; u++) {
      const unsigned w1 = yw[u + 1];
      acc = __dp4a(xw[u], __byte_perm(w0, w1, sel), acc);
      w0 = w1;
    }
    s += acc;
  }
  if (k < nc) coef[(size_t)pair * nc + k] = (long long)s;
}

// exact sums [nc] (int64, global) of one pair -> 2n digits; one CTA per pair
struct Coef64 {
  const long long *c;
  __device__ __forceinline__ void quad(int k, unsigned long long (&o)[4]) const {
#pragma unroll
    for (int e = 0; e < 4; e++) o[e] = (unsigned long long)c[4 * k + e];
  }
  __device__ __forceinline__ unsigned long long one(int i) const { return (unsigned long long)c[i]; }
};

__global__ void __launch_bounds__(512) long_carry_kernel(const long long *__restrict__ coef, int n,
                                                         uint8_t *__restrict__ prod) {
  __shared__ CarrySeg seg;
  const int pair = blockIdx.x, nc = 2 * n - 1, nout = 2 * n, words = (nout + 3) / 4;
  const Coef64 src{coef + (size_t)pair * nc};
  unsigned gen, allp;
  carry_seg_scan(src, nc, 0, words, seg, gen, allp);
  carry_seg_emit(src, nc, nout, 0, words, seg, 0u, prod + (size_t)pair * nout);
}

// ---- precision escalation helpers (ivm_multiply_exact) ----
// pairs whose flag is set get `tier` in method[]; the others are appended to idx
__global__ void mark_kernel(const uint8_t *__restrict__ cert, const int *__restrict__ map, int count, uint8_t tier,
                            uint8_t *__restrict__ method, int *__restrict__ idx, int *__restrict__ nidx) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= count) return;
  const int p = map ? map[j] : j;
  if (cert[j]) {
    if (method) method[p] = tier;
  } else {
    idx[atomicAdd(nidx, 1)] = p;
  }
}
// dst[j][0..len) = src[idx[j]][0..len)
__global__ void gather_rows_kernel(const uint8_t *__restrict__ src, size_t len, const int *__restrict__ idx,
                                   uint8_t *__restrict__ dst) {
  const int j = blockIdx.x;
  const uint8_t *s = src + (size_t)idx[j] * len;
  uint8_t *d = dst + (size_t)j * len;
  for (size_t i = threadIdx.x; i < len; i += blockDim.x) d[i] = s[i];
}
// dst[idx[j]][0..len) = src[j][0..len) where ok == nullptr or ok[j]
__global__ void scatter_rows_kernel(const uint8_t *__restrict__ src, size_t len, const int *__restrict__ idx,
                                    const uint8_t *__restrict__ ok, uint8_t *__restrict__ dst) {
  const int j = blockIdx.x;
  if (ok && !ok[j]) return;
  const uint8_t *s = src + (size_t)j * len;
  uint8_t *d = dst + (size_t)idx[j] * len;
  for (size_t i = threadIdx.x; i < len; i += blockDim.x) d[i] = s[i];
}

// method[map[j]] = tier (map null: method[j])
__global__ void set_method_kernel(const int *__restrict__ map, int count, uint8_t tier, uint8_t *__restrict__ method) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < count) method[map ? map[j] : j] = tier;
}

}  // namespace lm

int esc_set_method(const int *map, int count, int tier, uint8_t *method, cudaStream_t s) {
  if (count <= 0 || !method) return 0;
  lm::set_method_kernel<<<(count + 255) / 256, 256, 0, s>>>(map, count, (uint8_t)tier, method);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

int esc_mark(const uint8_t *cert, const int *map, int count, int tier, uint8_t *method, int *idx, int *nidx,
             cudaStream_t s) {
  if (count <= 0) return 0;
  lm::mark_kernel<<<(count + 255) / 256, 256, 0, s>>>(cert, map, count, (uint8_t)tier, method, idx, nidx);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}
int esc_gather(const uint8_t *src, size_t len, const int *idx, int count, uint8_t *dst, cudaStream_t s) {
  if (count <= 0) return 0;
  lm::gather_rows_kernel<<<count, 256, 0, s>>>(src, len, idx, dst);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}
int esc_scatter(const uint8_t *src, size_t len, const int *idx, const uint8_t *ok, int count, uint8_t *dst,
                cudaStream_t s) {
  if (count <= 0) return 0;
  lm::scatter_rows_kernel<<<count, 256, 0, s>>>(src, len, idx, ok, dst);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

int long_launch(const uint8_t *a, const uint8_t *b, int n, int batch, long long *coef, uint8_t *prod,
                cudaStream_t s) {
  const int nc = 2 * n - 1;
  for (int p0 = 0; p0 < batch; p0 += 65535) {  // grid.y limit
    const int pb = batch - p0 < 65535 ? batch - p0 : 65535;
    lm::long_coef_kernel<<<dim3((nc + lm::T - 1) / lm::T, pb), lm::T, 0, s>>>(
        a + (size_t)p0 * n, b + (size_t)p0 * n, n, coef + (size_t)p0 * nc);
    if (cudaPeekAtLastError() != cudaSuccess) return -1;
  }
  lm::long_carry_kernel<<<batch, 512, 0, s>>>(coef, n, prod);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace ivm
