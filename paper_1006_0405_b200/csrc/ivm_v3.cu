// ivm_v3.cu -- translation unit of the balanced odd-frequency kernels (ivm_v3.cuh)
// and their host-side tables / launchers.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "ivm_interval.cuh"
#include "ivm_internal.h"
#include "ivm_carry.cuh"
#include "ivm_v3.cuh"
#include "ivm_v6.cuh"
#include "ivm_d3.cuh"
#include "ivm_twc_host.h"

namespace ivm {

int upload_w64(const double *w64, const float *w32) {  // full-circle w_64^j tables [64][4]
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

// ---- v3 twiddle tables (host): compact entries [2] per twiddle ----
template <typename F, int M, int RK>
static int v3_tables_impl(const F *w2N /* [2N][4] */, F *out) {
  using Gm = v3::G3<M, RK>;
  constexpr int N = Gm::N;
  constexpr v3::Plan P = v3::plan_cta(M, RK);
  const long N2 = 2L * N;
  bool ok = true;
  auto put = [&](int idx, long e) { ok = ok && compact(w2N + 4L * (((e % N2) + N2) % N2), out + 2L * idx); };
  // the last inverse pass's tables also carry the exact scale 2/m of P:97 (a power of
  // two: every product, sum and rounding of that pass scales exactly, so the
  // coefficients are bit-identical to scaling them afterwards)
  auto put_s = [&](int idx, long e) {
    put(idx, e);
    out[2L * idx] *= (F)2 / (F)N;
    out[2L * idx + 1] *= (F)2 / (F)N;
  };
  for (int p = 1; p < P.nf; p++) {  // forward: w_{2LR}^{q(2k0+1)} = w_{2N}^{q(2k0+1)S'}
    const int R = P.f[p], L = v3::fL(P, p), Sp = N / (L * R);
    for (int q = 1; q < R; q++)
      for (int k0 = 0; k0 < L / 2; k0++) put(Gm::tw_fwd(p) + (q - 1) * (L / 2) + k0, (long)q * (2 * k0 + 1) * Sp);
  }
  for (int p = 1; p < P.ni; p++) {  // inverse: w_{LQ} = w_{2N}^{2S'} (direct entries conj'd in-kernel)
    const int Q = P.q[p], L = v3::iL(P, p), Sp = N / (L * Q);
    for (int q = 1; q < Q; q++)
      for (int k0 = 0; k0 < L; k0++) {
        if (2 * q < Q) put(Gm::tw_inv(p) + (q - 1) * L + k0, 2L * q * k0 * Sp);
        else put(Gm::tw_inv(p) + (q - 1) * L + k0, 2L * (Q - q) * k0 * Sp);
      }
  }
  for (int k = 0; k < N / 2; k++) put_s(Gm::tw_fin() + k, k);  // (2/m) z^k (conj'd in-kernel)
  if (Gm::LAST16) {  // last inverse pass (radix RK) with z^{-k0} folded in: [RK][L]
    const int p = P.ni - 1, Q = P.q[p], L = v3::iL(P, p), Sp = N / (L * Q);
    for (int q = 0; q < Q; q++)
      for (int k0 = 0; k0 < L; k0++) {
        // direct (q < 8): conj(u) with u = w_{LQ}^{q k0} z^{k0}; mirror: w_{LQ}^{(Q-q) k0} z^{-k0}
        const long e = (2 * q < Q) ? (long)k0 * (2L * q * Sp + 1) : (long)k0 * (2L * (Q - q) * Sp - 1);
        put_s(Gm::tw_l16() + q * L + k0, e);
      }
  }
  return ok ? Gm::tw_total() : -4;
}

#define IVM_V3_DISPATCH(FN, ...)                    \
  switch (m) {                                      \
    case 4: return FN<4>(__VA_ARGS__);              \
    case 5: return FN<5>(__VA_ARGS__);              \
    case 6: return FN<6>(__VA_ARGS__);              \
    case 7: return FN<7>(__VA_ARGS__);              \
    case 8: return FN<8>(__VA_ARGS__);              \
    case 9: return FN<9>(__VA_ARGS__);              \
    case 10: return FN<10>(__VA_ARGS__);            \
    case 11: return FN<11>(__VA_ARGS__);            \
    case 12: return FN<12>(__VA_ARGS__);            \
    case 13: return FN<13>(__VA_ARGS__);            \
    case 14: return FN<14>(__VA_ARGS__);            \
    case 15: return FN<15>(__VA_ARGS__);            \
    case 16: return FN<16>(__VA_ARGS__);            \
    case 17: return FN<17>(__VA_ARGS__);            \
    case 18: return FN<18>(__VA_ARGS__);            \
    default: return -4;                             \
  }

template <int M> static int v3_table_size_m(int radix) {
  return radix == 8 ? v3::G3<M, 8>::tw_total() : v3::G3<M, 16>::tw_total();
}
int v3_table_entries(int m, int radix) { IVM_V3_DISPATCH(v3_table_size_m, radix) }

template <int M> static int v3_tables_m(int prec, int radix, const void *w2N, void *out) {
  if (radix == 8)
    return prec == 0 ? v3_tables_impl<double, M, 8>((const double *)w2N, (double *)out)
                     : v3_tables_impl<float, M, 8>((const float *)w2N, (float *)out);
  return prec == 0 ? v3_tables_impl<double, M, 16>((const double *)w2N, (double *)out)
                   : v3_tables_impl<float, M, 16>((const float *)w2N, (float *)out);
}
int v3_tables(int m, int prec, int radix, const void *w2N, void *out) {
  IVM_V3_DISPATCH(v3_tables_m, prec, radix, w2N, out)
}

template <typename T, int M, int R>
static int v3_info_impl(LaunchInfo *li) {
  using C = v3::Cfg3<T, M, R>;
  li->threads = C::THREADS;
  li->smem = C::SMEM;
  li->a_smem = false;
  li->a_bytes_per_cta = C::A_BYTES;
  auto k = v3::ivm_v3_kernel<T, M, R>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) != cudaSuccess)
    return -1;
  if constexpr (sizeof(T) == 8) {  // the throughput variants (v3_go)
    if (cudaFuncSetAttribute(v3::ivm_v3_kernel<T, M, R, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)C::SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(v3::ivm_v3_kernel<T, M, R, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)C::SMEM) != cudaSuccess)
      return -1;
  }
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, C::THREADS, C::SMEM) != cudaSuccess) return -1;
  li->blocks_per_sm = nb;
  return 0;
}
template <int M> static int v3_info_m(int prec, int radix, LaunchInfo *li) {
  if constexpr (M > 13 || M < 10) {
    return -4;
  } else {
    if (radix != 8) return -4;  // the one-CTA kernel is radix 8 only
    return prec == 0 ? v3_info_impl<double, M, 8>(li) : v3_info_impl<float, M, 8>(li);
  }
}
int v3_info(int prec, int m, int radix, LaunchInfo *li) { IVM_V3_DISPATCH(v3_info_m, prec, radix, li) }

template <typename T, int M, int R> static void v3_go(const KParams &kp, int grid, cudaStream_t s) {
  using C = v3::Cfg3<T, M, R>;
  // fp64 and no diagnostic outputs: the kernels compiled without the dump / coefficient
  // paths, with staged digits when every row is 16-byte aligned, else without the
  // staging (same arithmetic)
  if constexpr (sizeof(T) == 8) {
    const bool aligned = kp.n % 16 == 0 &&
                         ((reinterpret_cast<uintptr_t>(kp.a) | reinterpret_cast<uintptr_t>(kp.b)) % 16 == 0);
    if (!kp.dump_slot && !kp.coeffs) {
      if (aligned) v3::ivm_v3_kernel<T, M, R, 1><<<grid, C::THREADS, C::SMEM, s>>>(kp);
      else v3::ivm_v3_kernel<T, M, R, 2><<<grid, C::THREADS, C::SMEM, s>>>(kp);
      return;
    }
  }
  v3::ivm_v3_kernel<T, M, R><<<grid, C::THREADS, C::SMEM, s>>>(kp);
}
template <int M> static int v3_launch_m(int prec, int radix, const KParams &kp, int grid, cudaStream_t s) {
  if constexpr (M > 13 || M < 10) {
    return -4;
  } else {
    if (radix != 8) return -4;
    (prec == 0 ? v3_go<double, M, 8> : v3_go<float, M, 8>)(kp, grid, s);
  }
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}
int v3_launch(int prec, int m, int radix, const KParams &kp, int grid, cudaStream_t s) {
  IVM_V3_DISPATCH(v3_launch_m, prec, radix, kp, grid, s)
}



// ---- small m (2^6 .. 2^9): one multiplication per m/16 lanes ----
template <typename T, int M> static int v6_info_impl(LaunchInfo *li) {
  using C = v6::Cfg6<T, M>;
  auto k = v6::ivm_v6_kernel<T, M>;
  li->threads = C::THREADS;
  li->smem = C::SMEM;
  li->a_smem = false;
  li->a_bytes_per_cta = C::A_BYTES;
  li->cluster = C::PPC;  // multiplications per CTA
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) != cudaSuccess) return -1;
  if constexpr (sizeof(T) == 8) {
    if (cudaFuncSetAttribute(v6::ivm_v6_kernel<T, M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)C::SMEM) != cudaSuccess)
      return -1;
  }
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, C::THREADS, C::SMEM) != cudaSuccess) return -1;
  li->blocks_per_sm = nb;
  return 0;
}
template <int M> static int v6_info_m(int prec, LaunchInfo *li) {
  if constexpr (M < 6 || M > 9) {
    return -4;
  } else {
    return prec == 0 ? v6_info_impl<double, M>(li) : v6_info_impl<float, M>(li);
  }
}
int v6_info(int prec, int m, LaunchInfo *li) { IVM_V3_DISPATCH(v6_info_m, prec, li) }

template <typename T, int M> static void v6_go(const KParams &kp, int grid, cudaStream_t s) {
  using C = v6::Cfg6<T, M>;
  if constexpr (sizeof(T) == 8) {  // no diagnostic outputs: the kernel compiled without them
    if (!kp.dump_slot && !kp.coeffs) {
      v6::ivm_v6_kernel<T, M, true><<<grid, C::THREADS, C::SMEM, s>>>(kp);
      return;
    }
  }
  v6::ivm_v6_kernel<T, M><<<grid, C::THREADS, C::SMEM, s>>>(kp);
}
template <int M> static int v6_launch_m(int prec, const KParams &kp, int grid, cudaStream_t s) {
  if constexpr (M < 6 || M > 9) {
    return -4;
  } else {
    (prec == 0 ? v6_go<double, M> : v6_go<float, M>)(kp, grid, s);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
  }
}
int v6_launch(int prec, int m, const KParams &kp, int grid, cudaStream_t s) {
  IVM_V3_DISPATCH(v6_launch_m, prec, kp, grid, s)
}


// ---- circular containment sets on the one-CTA radix-8 schedule (ivm_d3.cuh): m = 2^10 .. 2^13 ----
template <int M> static int d3_info_m(LaunchInfo *li) {
  using C = d3::CfgD<M>;
  auto k = d3::ivm_d3_kernel<M>;
  li->threads = C::THREADS;
  li->smem = C::SMEM;
  li->a_smem = false;
  li->a_bytes_per_cta = C::A_BYTES;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) != cudaSuccess) return -1;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, C::THREADS, C::SMEM) != cudaSuccess) return -1;
  li->blocks_per_sm = nb;
  return 0;
}
int d3_info(int m, LaunchInfo *li) {
  switch (m) {
    case 10: return d3_info_m<10>(li);
    case 11: return d3_info_m<11>(li);
    case 12: return d3_info_m<12>(li);
    case 13: return d3_info_m<13>(li);
    default: return -4;
  }
}
template <int M> static int d3_go(const KParams &kp, int grid, cudaStream_t s) {
  using C = d3::CfgD<M>;
  d3::ivm_d3_kernel<M><<<grid, C::THREADS, C::SMEM, s>>>(kp);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}
int d3_launch(int m, const KParams &kp, int grid, cudaStream_t s) {
  switch (m) {
    case 10: return d3_go<10>(kp, grid, s);
    case 11: return d3_go<11>(kp, grid, s);
    case 12: return d3_go<12>(kp, grid, s);
    case 13: return d3_go<13>(kp, grid, s);
    default: return -4;
  }
}

}  // namespace ivm
