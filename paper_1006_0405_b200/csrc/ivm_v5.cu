// ivm_v5.cu -- translation unit of the group kernel for m = 2^14 .. 2^18
// (ivm_v5.cuh): launch info and the cooperative launch.  Its twiddle tables are
// the v4 layout (v4_tables, ivm_v4.cu).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "ivm_interval.cuh"
#include "ivm_internal.h"
#include "ivm_carry.cuh"
#include "ivm_v3.cuh"
#include "ivm_v4.cuh"
#include "ivm_v5.cuh"
#include "ivm_v7.cuh"
#include "ivm_d3.cuh"
#include "ivm_d7.cuh"
#include "ivm_twc_host.h"

namespace ivm {

int upload_w64_v5(const double *w64, const float *w32) {  // this TU's DFT-internal constants
  v3::TwC<double> d[17];
  v3::TwC<float> f[17];
  for (int j = 0; j <= 16; j++) {
    double o[2];
    float of[2];
    if (!compact(w64 + 4 * j, o) || !compact(w32 + 4 * j, of)) return -4;
    d[j] = v3::TwC<double>{o[0], o[1]};
    f[j] = v3::TwC<float>{of[0], of[1]};
  }
  if (cudaMemcpyToSymbol(v3::c_w64_f64, d, sizeof(d)) != cudaSuccess) return -1;
  if (cudaMemcpyToSymbol(v3::c_w64_f32, f, sizeof(f)) != cudaSuccess) return -1;
  return 0;
}

template <typename T, int M> static int v5_info_impl(LaunchInfo *li) {
  using CF = v5::Cfg5<T, M>;
  auto k = v5::ivm_v5_kernel<T, M>;
  if constexpr (M == 18) {  // the zero-padding-skipping variant (v5_go)
    if (cudaFuncSetAttribute(v5::ivm_v5_kernel<T, M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)CF::SMEM) != cudaSuccess)
      return -1;
  }
  li->threads = CF::THREADS;
  li->smem = CF::SMEM;
  li->a_smem = false;
  li->a_bytes_per_cta = CF::A_BYTES;
  li->cluster = v4::G4<M>::C;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM) != cudaSuccess) return -1;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, CF::THREADS, CF::SMEM) != cudaSuccess) return -1;
  li->blocks_per_sm = nb;
  li->max_clusters = 0;
  return 0;
}
#define IVM_V5_DISPATCH(FN, ...)         \
  switch (m) {                           \
    case 14: return FN<14>(__VA_ARGS__); \
    case 15: return FN<15>(__VA_ARGS__); \
    case 16: return FN<16>(__VA_ARGS__); \
    case 17: return FN<17>(__VA_ARGS__); \
    case 18: return FN<18>(__VA_ARGS__); \
    default: return -4;                  \
  }
template <int M> static int v5_info_m(int prec, LaunchInfo *li) {
  return prec == 0 ? v5_info_impl<double, M>(li) : v5_info_impl<float, M>(li);
}
int v5_info(int prec, int m, LaunchInfo *li) { IVM_V5_DISPATCH(v5_info_m, prec, li) }

template <typename T, int M>
static int v5_go(const KParams &kp, const Group5Args &ga, int groups, cudaStream_t s, bool coop) {
  using CF = v5::Cfg5<T, M>;
  KParams k2 = kp;
  v5::Group5 g{ga.ctr, ga.xch, ga.link, ga.bnd, ga.bits};
  void *args[] = {(void *)&k2, (void *)&g};
  // m = 2^18 with n <= 2^17 - 8 * 4096 (C3): the cross pass skips whole groups
  // of zero-padding terms (a separate instantiation: ivm_v4.cuh cross_fwd)
  const bool qb = M == 18 && kp.n <= (1 << (M - 1)) - 8 * 4096;
  const void *fn = qb ? (const void *)v5::ivm_v5_kernel<T, M, M == 18> : (const void *)v5::ivm_v5_kernel<T, M>;
  // coop = false: a plain launch beside the cluster kernel, on the SMs its
  // clusters leave free (the group barrier needs the group's CTAs co-resident,
  // which the free SMs give; a CTA placed late only delays its group)
  const cudaError_t e = coop ? cudaLaunchCooperativeKernel(fn, dim3(groups * v4::G4<M>::C), dim3(CF::THREADS), args,
                                                         CF::SMEM, s)
                             : cudaLaunchKernel(fn, dim3(groups * v4::G4<M>::C), dim3(CF::THREADS), args, CF::SMEM, s);
  return e == cudaSuccess ? 0 : -1;
}
template <int M>
static int v5_launch_m(int prec, const KParams &kp, const Group5Args &ga, int groups, cudaStream_t s, bool coop) {
  return prec == 0 ? v5_go<double, M>(kp, ga, groups, s, coop) : v5_go<float, M>(kp, ga, groups, s, coop);
}
int v5_launch(int prec, int m, const KParams &kp, const Group5Args &ga, int groups, cudaStream_t s, bool coop) {
  IVM_V5_DISPATCH(v5_launch_m, prec, kp, ga, groups, s, coop)
}

// ---- pipelined group kernel (ivm_v7.cuh): fp64, m = 2^17, 2^18 ----
template <int M> static int v7_info_m(LaunchInfo *li) {
  using CF = v5::Cfg5<double, M>;
  auto k = v7::ivm_v7_kernel<M>;
  li->threads = CF::THREADS;
  li->smem = CF::SMEM;
  li->a_smem = false;
  li->a_bytes_per_cta = CF::A_BYTES;
  li->cluster = v4::G4<M>::C;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM) != cudaSuccess) return -1;
  if (cudaFuncSetAttribute(v7::ivm_v7_kernel<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM) !=
      cudaSuccess)
    return -1;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, CF::THREADS, CF::SMEM) != cudaSuccess) return -1;
  li->blocks_per_sm = nb;
  li->max_clusters = 0;
  return 0;
}
int v7_info(int m, LaunchInfo *li) {
  switch (m) {
    case 17: return v7_info_m<17>(li);
    case 18: return v7_info_m<18>(li);
    default: return -4;
  }
}
template <int M> static int v7_go(const KParams &kp, const Pipe7Args &pa, int grid, cudaStream_t s) {
  using CF = v5::Cfg5<double, M>;
  KParams k2 = kp;
  v7::Pipe7 g{pa.cnt, pa.xch, pa.wds, pa.rec, pa.link, pa.rp};
  void *args[] = {(void *)&k2, (void *)&g};
  // word-aligned digit rows and no diagnostic outputs: the kernel compiled without those paths
  const bool fast = kp.n % 4 == 0 && ((reinterpret_cast<uintptr_t>(kp.a) | reinterpret_cast<uintptr_t>(kp.b)) % 4 == 0) &&
                    !kp.dump_slot && !kp.coeffs;
  const void *fn = fast ? (const void *)v7::ivm_v7_kernel<M, true> : (const void *)v7::ivm_v7_kernel<M>;
  const cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(CF::THREADS), args, CF::SMEM, s);
  return e == cudaSuccess ? 0 : -1;
}
int v7_launch(int m, const KParams &kp, const Pipe7Args &pa, int grid, cudaStream_t s) {
  switch (m) {
    case 17: return v7_go<17>(kp, pa, grid, s);
    case 18: return v7_go<18>(kp, pa, grid, s);
    default: return -4;
  }
}


// ---- circular containment sets on the pipelined group schedule (ivm_d7.cuh): fp64, m = 2^17, 2^18 ----
template <int M> static int d7_info_m(LaunchInfo *li) {
  using CF = d7::CfgD7<M>;
  auto k = d7::ivm_d7_kernel<M>;
  li->threads = CF::THREADS;
  li->smem = CF::SMEM;
  li->a_smem = false;
  li->a_bytes_per_cta = CF::A_BYTES;
  li->cluster = v4::G4<M>::C;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM) != cudaSuccess) return -1;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, CF::THREADS, CF::SMEM) != cudaSuccess) return -1;
  li->blocks_per_sm = nb > 1 ? 1 : nb;  // one CTA per SM (the persistent grid of ivm_v7.cuh)
  li->max_clusters = 0;
  return 0;
}
int d7_info(int m, LaunchInfo *li) {
  switch (m) {
    case 17: return d7_info_m<17>(li);
    case 18: return d7_info_m<18>(li);
    default: return -4;
  }
}
template <int M> static int d7_go(const KParams &kp, const Pipe7Args &pa, int grid, cudaStream_t s) {
  using CF = d7::CfgD7<M>;
  KParams k2 = kp;
  v7::Pipe7 g{pa.cnt, pa.xch, pa.wds, pa.rec, pa.link, pa.rp};
  void *args[] = {(void *)&k2, (void *)&g};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void *)d7::ivm_d7_kernel<M>, dim3(grid), dim3(CF::THREADS),
                                                    args, CF::SMEM, s);
  return e == cudaSuccess ? 0 : -1;
}
int d7_launch(int m, const KParams &kp, const Pipe7Args &pa, int grid, cudaStream_t s) {
  switch (m) {
    case 17: return d7_go<17>(kp, pa, grid, s);
    case 18: return d7_go<18>(kp, pa, grid, s);
    default: return -4;
  }
}

}  // namespace ivm
