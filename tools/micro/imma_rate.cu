// Microbenchmark: throughput of mma.sync.m16n8k32 u8 x s8 -> s32 (IMMA.16832) on one SM
// and on the whole chip (independent accumulator chains per warp).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imma_rate imma_rate.cu && ./imma_rate
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma(int (&d)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3, unsigned b0,
                                    unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int CH>
__global__ void k(int iters, int *out, unsigned seed) {
  int d[CH][4] = {};
  unsigned a = seed ^ threadIdx.x, b = seed * 3u + threadIdx.x;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) mma(d[c], a + c, a, b, a ^ c, b + c, b);
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int *out;
  cudaMalloc(&out, 148 * 1024 * sizeof(int) * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    for (int grid : {1, 148}) {
      k<4><<<grid, warps * 32>>>(iters, out, 1);
      cudaEventRecord(e0);
      k<4><<<grid, warps * 32>>>(iters, out, 2);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double mmas = (double)grid * warps * iters * 4;
      printf("grid %3d warps/CTA %2d: %.3f ms  %.2f IMMA/clk/SM (at 1.965 GHz)  %.1f TOPS\n", grid, warps, ms,
             mmas / grid / (ms * 1e-3 * 1.965e9), mmas * 16 * 8 * 32 * 2 / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
