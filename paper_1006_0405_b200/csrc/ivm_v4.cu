// ivm_v4.cu -- translation unit of the cluster kernel (ivm_v4.cuh): host-side
// role tables, launch info and the cluster launch.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <math.h>

#include "ivm_interval.cuh"
#include "ivm_internal.h"
#include "ivm_carry.cuh"
#include "ivm_v3.cuh"
#include "ivm_v4.cuh"
#include "ivm_d3.cuh"
#include "ivm_d4.cuh"
#include "ivm_twc_host.h"

namespace ivm {

// this TU's copy of the DFT-internal constants (ivm_v3.cuh defines them per TU)
int upload_w64_v4(const double *w64, const float *w32) {
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

// Tables of ivm_v4.cuh (G4<M>), exponents as powers of z = e^{2 pi i/(2m)}:
//   forward role c, local pass p (L = fL(p), R = 8, Sp = 8192/(L R)), row kappa:
//     e = q (2 k + 1) Sp,  k = C kappa + (kappa even ? c : C-1-c)
//   inverse local pass p (L = iL(p), Q = 8, Sp = m/(L Q)), row k0 (direct q < 4 / mirror):
//     e = 2 q k0 Sp  /  2 (Q-q) k0 Sp
//   last inverse pass (Q = C, L = 4096, Sp = 2) role c, rows k0 in [c B, c B + B):
//     e = k0 (2 q Sp + 1) (q < C/2)  /  k0 (2 (C-q) Sp - 1)  (the untwist z^{-k0} folded in)
//   theta role c: e = q (1 + 4 r) m / (2C), r = c/2 (c even) or (2C-1-c)/2, full intervals
template <typename F, int M> static int v4_tables_impl(const F *w2N /* [2m][4] */, F *out) {
  using X = v4::G4<M>;
  constexpr int C = X::C, B = X::B;
  constexpr long N = 1L << M, N2 = 2 * N;
  constexpr v3::Plan P = v3::plan_cta(13, 8);
  memset(out, 0, sizeof(F) * 2 * (size_t)X::TOTAL);
  bool ok = true;
  auto put = [&](long idx, long e) { ok = ok && compact(w2N + 4L * (((e % N2) + N2) % N2), out + 2L * idx); };
  for (int c = 0; c < C; c++) {
    for (int p = 1; p <= 4; p++) {
      const int L = v3::fL(P, p), Sp = 8192 / (L * 8);
      for (int q = 1; q < 8; q++)
        for (int kap = 0; kap < L / 2; kap++) {
          const long k = (long)C * kap + ((kap & 1) == 0 ? c : C - 1 - c);
          put(X::FWD(c) + X::FP(p) + (q - 1) * (L / 2) + kap, (long)q * (2 * k + 1) * Sp);
        }
    }
  }
  const int inv_off[3] = {X::INV1, X::INV2, X::INV3};
  for (int p = 1; p <= 3; p++) {
    const int L = v3::iL(P, p), Q = 8;
    const long Sp = N / ((long)L * Q);
    for (int q = 1; q < Q; q++)
      for (int k0 = 0; k0 < L; k0++) {
        const long e = (2 * q < Q) ? 2L * q * k0 * Sp : 2L * (Q - q) * k0 * Sp;
        put(X::INV + inv_off[p - 1] + (q - 1) * L + k0, e);
      }
  }
  for (int c = 0; c < C; c++) {
    const long Sp = 2;
    for (int q = 0; q < C; q++)
      for (int kl = 0; kl < B; kl++) {
        const long k0 = (long)c * B + kl;
        const long e = (2 * q < C) ? k0 * (2 * q * Sp + 1) : k0 * (2 * (C - q) * Sp - 1);
        put(X::XINV(c) + q * B + kl, e);
        out[2L * (X::XINV(c) + q * B + kl)] *= (F)2 / (F)N;  // the exact scale 2/m of P:97
        out[2L * (X::XINV(c) + q * B + kl) + 1] *= (F)2 / (F)N;
      }
    const int r = (c % 2 == 0) ? c / 2 : (2 * C - 1 - c) / 2;
    for (int q = 0; q < C; q++) {
      const long e = ((long)q * (1 + 4 * r) * (N / (2 * C))) % N2;
      memcpy(out + 2L * (X::TH(c) + 2 * q), w2N + 4L * e, 4 * sizeof(F));  // full interval
    }
  }
  for (int c = 0; c < C; c++) {  // TH1: w_j theta_q (odd roles: w_j conj(theta_q)), full intervals
    const int r = (c % 2 == 0) ? c / 2 : (2 * C - 1 - c) / 2;
    for (int j = 0; j < 8; j++)
      for (int q = 0; q < C; q++) {
        const long ew = (long)j * (2 * c + 1) * 512;  // local pass 1, kappa = 0: k = c
        const long et = (long)q * (1 + 4 * r) * (N / (2 * C));
        const long e = (((ew + (c % 2 == 0 ? et : -et)) % N2) + N2) % N2;
        memcpy(out + 2L * (X::TH1(c) + 2 * (j * C + q)), w2N + 4L * e, 4 * sizeof(F));
      }
  }
  for (int j = 0; j < C; j++) {  // compact upper-half roots: w_C^j (2j <= C) or w_C^{C-j}; z^{4096 j}
    put(X::S2 + 2 * j, (long)(2 * j <= C ? j : C - j) * (N2 / C));
    put(X::FO + 2 * j, (long)j * 4096);
  }
  // the tensor-core cross pass (fp64, C >= 16, ivm_v5.cuh cross_tc): theta_q = T_q 2^-54 + err,
  // |err| <= 3 2^-55, T_q = round(mid(theta_q) 2^54) as 7 balanced base-256 digits d_i
  // (T = sum_i d_i 256^i).  B operand s (s < 4) of role c: int8 [8 columns n][32 q] at byte
  // 1024 c + 256 s; column n = 2 u + e holds part (u & 1) (re / im), digit 2 s + e, except
  // (s, e) = (3, 1): ones (sum_q x_q, the error's multiplier)
  if (sizeof(F) == 8 && C >= 16) {
    int8_t *lb = reinterpret_cast<int8_t *>(out + 2L * X::LIMB);
    for (int c = 0; c < C; c++)
      for (int q = 0; q < C; q++)
        for (int p = 0; p < 2; p++) {
          const F *th = out + 2L * (X::TH(c) + 2 * q);  // (re.lo, re.hi, im.lo, im.hi)
          const long double lo = th[2 * p], hi = th[2 * p + 1];
          const long double sc = 18014398509481984.0L;  // 2^54
          const long long T = llroundl((lo + hi) / 2 * sc);
          const long double e = 3.0L / 36028797018963968.0L;  // 3 2^-55
          const long double tv = (long double)T / sc;
          if (!(lo <= hi) || fabsl(lo - tv) > e || fabsl(hi - tv) > e) return -4;
          int8_t d[8];
          long long r = T;
          for (int i = 0; i < 7; i++) {
            long long di = ((r % 256) + 256) % 256;  // balanced digit in [-128, 127]
            if (di >= 128) di -= 256;
            d[i] = (int8_t)di;
            r = (r - di) / 256;
          }
          if (r != 0) return -4;
          d[7] = 1;
          for (int s = 0; s < 4; s++)
            for (int u = p; u < 4; u += 2)
              for (int e2 = 0; e2 < 2; e2++) lb[1024 * c + 256 * s + 32 * (2 * u + e2) + q] = d[2 * s + e2];
        }
  }
  return ok ? X::TOTAL : -4;
}

#define IVM_V4_DISPATCH(FN, ...)       \
  switch (m) {                         \
    case 14: return FN<14>(__VA_ARGS__); \
    case 15: return FN<15>(__VA_ARGS__); \
    case 16: return FN<16>(__VA_ARGS__); \
    default: return -4;                \
  }
#define IVM_V45_DISPATCH(FN, ...)      \
  switch (m) {                         \
    case 14: return FN<14>(__VA_ARGS__); \
    case 15: return FN<15>(__VA_ARGS__); \
    case 16: return FN<16>(__VA_ARGS__); \
    case 17: return FN<17>(__VA_ARGS__); \
    case 18: return FN<18>(__VA_ARGS__); \
    default: return -4;                \
  }

template <int M> static int v4_entries_m() { return v4::G4<M>::TOTAL; }
int v4_table_entries(int m) { IVM_V45_DISPATCH(v4_entries_m) }

template <int M> static int v4_tables_m(int prec, const void *w2N, void *out) {
  return prec == 0 ? v4_tables_impl<double, M>((const double *)w2N, (double *)out)
                   : v4_tables_impl<float, M>((const float *)w2N, (float *)out);
}
int v4_tables(int m, int prec, const void *w2N, void *out) { IVM_V45_DISPATCH(v4_tables_m, prec, w2N, out) }

template <typename T, int M> static int v4_info_impl(LaunchInfo *li) {
  using CF = v4::Cfg4<T, M>;
  constexpr int C = v4::G4<M>::C;
  auto k = v4::ivm_v4_kernel<T, M>;
  li->threads = CF::THREADS;
  li->smem = CF::SMEM;
  li->a_smem = false;
  li->a_bytes_per_cta = CF::A_BYTES;
  li->cluster = C;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM) != cudaSuccess) return -1;
  if constexpr (sizeof(T) == 8) {  // the throughput variant (v4_go)
    if (cudaFuncSetAttribute(v4::ivm_v4_kernel<T, M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)CF::SMEM) != cudaSuccess)
      return -1;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(C * 64);
  cfg.blockDim = dim3(CF::THREADS);
  cfg.dynamicSmemBytes = CF::SMEM;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, (void *)k, &cfg) != cudaSuccess) return -1;
  li->blocks_per_sm = ncl > 0 ? 1 : 0;
  li->max_clusters = ncl;
  return 0;
}
template <int M> static int v4_info_m(int prec, LaunchInfo *li) {
  return prec == 0 ? v4_info_impl<double, M>(li) : v4_info_impl<float, M>(li);
}
int v4_info(int prec, int m, LaunchInfo *li) { IVM_V4_DISPATCH(v4_info_m, prec, li) }

template <typename T, int M> static int v4_go(const KParams &kp, int clusters, cudaStream_t s) {
  using CF = v4::Cfg4<T, M>;
  constexpr int C = v4::G4<M>::C;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(C * clusters);
  cfg.blockDim = dim3(CF::THREADS);
  cfg.dynamicSmemBytes = CF::SMEM;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // fp64, no diagnostic outputs and (where digits are staged) 16-byte aligned rows:
  // the kernel compiled without those paths (same arithmetic)
  if constexpr (sizeof(T) == 8) {
    const bool aligned = CF::DIG_BYTES == 0 || (kp.n % 16 == 0 && ((reinterpret_cast<uintptr_t>(kp.a) |
                                                                    reinterpret_cast<uintptr_t>(kp.b)) % 16 == 0));
    if (aligned && !kp.dump_slot && !kp.coeffs)
      return cudaLaunchKernelEx(&cfg, v4::ivm_v4_kernel<T, M, true>, kp) == cudaSuccess ? 0 : -1;
  }
  return cudaLaunchKernelEx(&cfg, v4::ivm_v4_kernel<T, M>, kp) == cudaSuccess ? 0 : -1;
}
template <int M> static int v4_launch_m(int prec, const KParams &kp, int clusters, cudaStream_t s) {
  return prec == 0 ? v4_go<double, M>(kp, clusters, s) : v4_go<float, M>(kp, clusters, s);
}
int v4_launch(int prec, int m, const KParams &kp, int clusters, cudaStream_t s) {
  IVM_V4_DISPATCH(v4_launch_m, prec, kp, clusters, s)
}


// ---- circular containment sets on the cluster schedule (ivm_d4.cuh): fp64, m = 2^14 .. 2^16 ----
template <int M> static void d4_cfg(cudaLaunchConfig_t &cfg, cudaLaunchAttribute *attr, int clusters, cudaStream_t s) {
  using CF = d4::CfgD4<M>;
  constexpr int C = v4::G4<M>::C;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(C * clusters);
  cfg.blockDim = dim3(CF::THREADS);
  cfg.dynamicSmemBytes = CF::SMEM;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
}
template <int M> static int d4_info_m(LaunchInfo *li) {
  using CF = d4::CfgD4<M>;
  auto k = d4::ivm_d4_kernel<M>;
  li->threads = CF::THREADS;
  li->smem = CF::SMEM;
  li->a_smem = false;
  li->a_bytes_per_cta = CF::A_BYTES;
  li->cluster = v4::G4<M>::C;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM) != cudaSuccess) return -1;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  d4_cfg<M>(cfg, attr, 64, nullptr);
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, (void *)k, &cfg) != cudaSuccess) return -1;
  li->blocks_per_sm = ncl > 0 ? 1 : 0;
  li->max_clusters = ncl;
  return 0;
}
int d4_info(int m, LaunchInfo *li) {
  switch (m) {
    case 14: return d4_info_m<14>(li);
    case 15: return d4_info_m<15>(li);
    case 16: return d4_info_m<16>(li);
    default: return -4;
  }
}
template <int M> static int d4_go(const KParams &kp, int clusters, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  d4_cfg<M>(cfg, attr, clusters, s);
  return cudaLaunchKernelEx(&cfg, d4::ivm_d4_kernel<M>, kp) == cudaSuccess ? 0 : -1;
}
int d4_launch(int m, const KParams &kp, int clusters, cudaStream_t s) {
  switch (m) {
    case 14: return d4_go<14>(kp, clusters, s);
    case 15: return d4_go<15>(kp, clusters, s);
    case 16: return d4_go<16>(kp, clusters, s);
    default: return -4;
  }
}

}  // namespace ivm
