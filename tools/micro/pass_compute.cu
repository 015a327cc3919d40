// Microbenchmark: the radix-8 pass body of the one-CTA kernel (7 compact
// twiddle products + the 8-point interval DFT, ivm_v3.cuh fwdR) on register
// data, no shared-memory state and no barriers: cycles per task at 16 warps/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../include -o pass_compute pass_compute.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../paper_1006_0405_b200/csrc/ivm_interval.cuh"
#include "../../paper_1006_0405_b200/csrc/ivm_internal.h"
#include "../../paper_1006_0405_b200/csrc/ivm_carry.cuh"
#include "../../paper_1006_0405_b200/csrc/ivm_v3.cuh"

using namespace ivm;
using namespace ivm::v3;

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int iters, const double *in, double *out, long long *cyc) {
  extern __shared__ TwC<double> tws[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) tws[i] = TwC<double>{0.7071 + 1e-5 * i, 0.3 + 1e-6 * i};
  __syncthreads();
  CI<double> v[8];
  for (int q = 0; q < 8; q++)
    v[q] = CI<double>{in[q], in[q] + 1e-9, -in[q + 1], -in[q + 1] + 1e-9};
  const long long t0 = clock64();
  int k0 = threadIdx.x & 63;
  for (int it = 0; it < iters; it++) {
    if (MODE == 0) {  // twiddle products + DFT
#pragma unroll
      for (int q = 1; q < 8; q++) {
        const TwC<double> w = tws[k0 + 64 * q];
        v[q] = (2 * q <= 8) ? rtmul<double, false, false>(w, v[q]) : rtmul<double, false, true>(w, v[q]);
      }
      cdft<double, 8, false>(v);
    } else if (MODE == 1) {  // DFT only
      cdft<double, 8, false>(v);
    } else {  // twiddle products only
#pragma unroll
      for (int q = 1; q < 8; q++) {
        const TwC<double> w = tws[k0 + 64 * q];
        v[q] = (2 * q <= 8) ? rtmul<double, false, false>(w, v[q]) : rtmul<double, false, true>(w, v[q]);
      }
    }
    k0 = (k0 + 1) & 63;
  }
  const long long t1 = clock64();
  double s = 0;
  for (int q = 0; q < 8; q++) s += v[q].rl + v[q].rh + v[q].il + v[q].ih;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double *in, *out;
  long long *cyc;
  cudaMalloc(&in, 64 * 8);
  cudaMalloc(&out, 148 * 512 * 8);
  cudaMalloc(&cyc, 148 * 8);
  double h[16];
  for (int i = 0; i < 16; i++) h[i] = 0.1 * (i + 1) * (i % 3 == 0 ? -1 : 1);
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  const int iters = 2000;
  const char *names[3] = {"twiddles + DFT", "DFT only", "twiddles only"};
  for (int mode = 0; mode < 3; mode++) {
    auto kern = mode == 0 ? k<0> : (mode == 1 ? k<1> : k<2>);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    kern<<<148, 512, 65536>>>(iters, in, out, cyc);
    kern<<<148, 512, 65536>>>(iters, in, out, cyc);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    // per SM: 16 warps x iters tasks; per SMSP 4 warps
    printf("%-16s %8.1f cycles per pass-equivalent (512 tasks / SM), %.1f per task per SMSP-warp\n", names[mode],
           (double)c / iters, (double)c / iters / 4);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
