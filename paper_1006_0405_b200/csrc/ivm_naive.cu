// ivm_naive.cu -- the paper's "naive" fixed-precision SS comparator (P:22,
// P:273-274): the same multiplication with punctual complex numbers,
// round-to-nearest arithmetic and round-to-nearest twiddles, and the
// coefficients rounded to the nearest integer -- no containment sets, no
// certificate, "not guaranteed to be correct ... only useful for speed
// comparisons".  Like the paper's naive SS it transforms a and b
// separately, multiplies pointwise and transforms back
// (P:211); the FFT is an in-place radix-2 DIT of length m in shared memory
// (bit-reversed load, P:143-155's butterflies), one CTA per multiplication.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ivm_internal.h"
#include "ivm_carry.cuh"

namespace ivm {
namespace nv {

template <typename T> struct C2;
template <> struct C2<double> { using t = double2; };
template <> struct C2<float> { using t = float2; };

constexpr int TH = 256;

__device__ __forceinline__ int brev(int j, int bits) { return (int)(__brev((unsigned)j) >> (32 - bits)); }

// in-place radix-2 DIT on bit-reversed input; INV uses the conjugate twiddles
template <typename T, bool INV>
__device__ __forceinline__ void fft_dit(typename C2<T>::t *x, int lg, const typename C2<T>::t *__restrict__ w) {
  const int m = 1 << lg;
  for (int s = 0; s < lg; s++) {
    const int half = 1 << s, stride = m >> (s + 1);  // twiddle w_m^{j stride} = w_{2 half}^j
    for (int b = threadIdx.x; b < m / 2; b += blockDim.x) {
      const int j = b & (half - 1), i0 = ((b >> s) << (s + 1)) + j, i1 = i0 + half;
      const typename C2<T>::t tw = w[j * stride];
      const T wr = tw.x, wi = INV ? -tw.y : tw.y;
      const typename C2<T>::t u = x[i0], v = x[i1];
      const T tr = wr * v.x - wi * v.y, ti = wr * v.y + wi * v.x;  // w * O
      x[i0] = typename C2<T>::t{u.x + tr, u.y + ti};
      x[i1] = typename C2<T>::t{u.x - tr, u.y - ti};
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(TH) naive_kernel(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b, int n,
                                                   int batch, int lg, const typename C2<T>::t *__restrict__ w,
                                                   typename C2<T>::t *__restrict__ scratch,
                                                   uint8_t *__restrict__ prod) {
  using V = typename C2<T>::t;
  extern __shared__ __align__(16) unsigned char smem[];
  V *x = reinterpret_cast<V *>(smem);
  const int m = 1 << lg;
  V *A = scratch + (size_t)blockIdx.x * m;
  for (int pair = blockIdx.x; pair < batch; pair += gridDim.x) {
    for (int op = 0; op < 2; op++) {
      const uint8_t *d = (op == 0 ? a : b) + (size_t)pair * n;
      __syncthreads();
      for (int j = threadIdx.x; j < m; j += blockDim.x) {
        const int s = brev(j, lg);
        x[j] = V{s < n ? (T)d[s] : (T)0, (T)0};
      }
      __syncthreads();
      fft_dit<T, false>(x, lg, w);
      if (op == 0) {
        for (int j = threadIdx.x; j < m; j += blockDim.x) A[j] = x[j];
      } else {
        for (int j = threadIdx.x; j < m; j += blockDim.x) {  // P_k = A_k B_k, then bit-reverse in place
          const V p = A[j], q = x[j];
          x[j] = V{p.x * q.x - p.y * q.y, p.x * q.y + p.y * q.x};
        }
      }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      const int s = brev(j, lg);
      if (j < s) {
        const V t = x[j];
        x[j] = x[s];
        x[s] = t;
      }
    }
    __syncthreads();
    fft_dit<T, true>(x, lg, w);
    // c_k = round(Re(y_k) / m), into the first 4m bytes of x (after a barrier)
    const int nc = 2 * n - 1;
    int32_t cv[32];
    int cnt = 0;
    for (int k = threadIdx.x; k < nc; k += blockDim.x) {
      const double c = rint((double)x[k].x / (double)m);
      cv[cnt++] = c > 2147483647.0 ? 2147483647 : (c < 0.0 ? 0 : (int32_t)c);
    }
    __syncthreads();
    int32_t *coef = reinterpret_cast<int32_t *>(smem);
    cnt = 0;
    for (int k = threadIdx.x; k < nc; k += blockDim.x) coef[k] = cv[cnt++];
    __syncthreads();
    carry_store(coef, n, prod + (size_t)pair * 2 * n, true);
  }
}

}  // namespace nv

int naive_smem(int lg, int prec) { return (1 << lg) * (prec == 0 ? 16 : 8); }

int naive_launch(int prec, const uint8_t *a, const uint8_t *b, int n, int batch, int lg, const void *w, void *scratch,
                 uint8_t *prod, int grid, cudaStream_t s) {
  const int smem = naive_smem(lg, prec);
  if (prec == 0) {
    auto k = nv::naive_kernel<double>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -1;
    k<<<grid, nv::TH, smem, s>>>(a, b, n, batch, lg, (const double2 *)w, (double2 *)scratch, prod);
  } else {
    auto k = nv::naive_kernel<float>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -1;
    k<<<grid, nv::TH, smem, s>>>(a, b, n, batch, lg, (const float2 *)w, (float2 *)scratch, prod);
  }
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace ivm
