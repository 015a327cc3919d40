// ivm_v6.cuh -- small transforms, m = 64 .. 512: one multiplication per group of
// m/16 lanes of a warp (included by ivm_v3.cu, after ivm_v3.cuh).
//
// The radix-8 odd-frequency schedule of the one-CTA kernel (same plans, passes,
// tables and mirror rules; plan_cta(m, 8) for m = 2^6 .. 2^9), but a pass of a
// multiplication has only m/16 tasks, so 32 / (m/16) multiplications share a
// warp and 8192/m share a 512-thread CTA.  Every group works on its own shared
// state, so the barriers are __syncwarp (all groups of a warp run the same pass
// sequence in lockstep); the whole twiddle table stays in shared memory; a's
// spectrum is parked in L2 as in the one-CTA kernel; certification and the word
// carry are reduced over the group's lanes.
#pragma once

namespace ivm {
namespace v6 {

using namespace v3;

template <int M> struct RT6 {  // pass parameters; tables at their global offsets
  using Gm = G3<M, 8>;
  static constexpr int R = 8;
  static constexpr int nf = plan_cta(M, 8).nf, ni = plan_cta(M, 8).ni;
  static constexpr int NFWD = nf - 2;
  static constexpr bool LAST8 = plan_cta(M, 8).q[ni - 1] == 8;
  static constexpr int NINV = LAST8 ? ni - 1 : ni - 2;
  __host__ __device__ static constexpr PassRT fwd(int i) {
    return PassRT{ilog2r((1 << M) / fL(plan_cta(M, 8), i + 2) / R), fL(plan_cta(M, 8), i + 2), Gm::fRS(i + 2),
                  (i + 3 < nf) ? Gm::fRS(i + 3) : Gm::iRS(1), Gm::fSW(i + 2),
                  (i + 3 < nf) ? Gm::fSW(i + 3) : Gm::iSW(1), Gm::tw_fwd(i + 2), 0, 0};
  }
  __host__ __device__ static constexpr PassRT inv(int i) {
    return PassRT{ilog2r((1 << M) / iL(plan_cta(M, 8), i + 1) / R), iL(plan_cta(M, 8), i + 1), Gm::iRS(i + 1),
                  (i + 2 < ni) ? Gm::iRS(i + 2) : 0, Gm::iSW(i + 1), (i + 2 < ni) ? Gm::iSW(i + 2) : 0,
                  (LAST8 && i == NINV - 1) ? Gm::tw_l16() : Gm::tw_inv(i + 1), 0,
                  (LAST8 && i == NINV - 1) ? 1 : 0};
  }
};

template <typename T, int M> struct Cfg6 {
  using Gm = G3<M, 8>;
  static constexpr int N = 1 << M, TPP = Gm::TASKS;  // lanes per multiplication: 4 .. 32
  static_assert(TPP >= 4 && TPP <= 32, "m = 64 .. 512");
  static constexpr int THREADS = 512, PPC = THREADS / TPP;  // multiplications per CTA
  static constexpr size_t E = sizeof(typename V2t<T>::t);
  // per-multiplication stride in elements: skewed by 16 bytes across the groups
  // of a warp (distinct bank groups), and 16-byte aligned for the carry's reads
  static constexpr int CAPP = Gm::CAP + (int)(16 / E);
  static constexpr size_t STATE_BYTES = 2 * E * (size_t)CAPP * PPC;
  static constexpr size_t TW_BYTES = (sizeof(TwC<T>) * (size_t)Gm::tw_total() + 15) / 16 * 16;
  static constexpr size_t SMEM = STATE_BYTES + TW_BYTES;
  static constexpr size_t A_BYTES = 2 * E * (size_t)(N / 2) * PPC;  // per CTA
  static_assert(4 * N <= (int)(E * CAPP), "coefficients alias the re plane");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

// certificate of a group of TPP lanes (lane-aligned, TPP a power of two <= 32)
template <int TPP> __device__ __forceinline__ void cert_group(CertAcc &acc) {
  int ok = acc.ok, bad = acc.bad;
  double rad = acc.rad;
#pragma unroll
  for (int o = TPP / 2; o; o >>= 1) {
    ok &= __shfl_xor_sync(0xffffffffu, ok, o, TPP);
    bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o, TPP));
    const double r2 = __shfl_xor_sync(0xffffffffu, rad, o, TPP);
    rad = (r2 <= rad) ? rad : r2;  // NaN propagates
  }
  acc.ok = ok, acc.bad = bad, acc.rad = rad;
}

// word carry of one multiplication by a group of TPP lanes (ivm_carry.cuh's
// adder on the group's bits); every lane of the warp calls it
template <int TPP>
__device__ __forceinline__ void carry_group(const int32_t *coef, int n, uint8_t *__restrict__ out, bool certified,
                                            bool write) {
  const int nout = 2 * n, nc = 2 * n - 1, words = (nout + 3) / 4;
  const unsigned lane = threadIdx.x & 31, gl = lane & (TPP - 1), gbase = lane - gl;
  const unsigned tmask = TPP == 32 ? 0xffffffffu : ((1u << TPP) - 1u);
  const CoefLinear src{coef};
  const bool wide = (reinterpret_cast<uintptr_t>(out) & 3) == 0;
  unsigned hp = 0u, ep = 0u, c = 0u;
  const int J = (words + TPP - 1) / TPP;
  for (int j = 0; j < J; j++) {
    const int k = TPP * j + (int)gl;
    unsigned lo, hi;
    carry_word(src, nc, k, lo, hi);
    unsigned h1 = __shfl_up_sync(0xffffffffu, hi, 1);
    if (gl == 0) h1 = hp;
    const unsigned w = lo + h1, ov = w < lo ? 1u : 0u;
    unsigned e1 = __shfl_up_sync(0xffffffffu, ov, 1);
    if (gl == 0) e1 = ep;
    const unsigned u = w + e1;
    const bool g = e1 != 0u && w == 0xffffffffu, p = u == 0xffffffffu && !g, in = k < words;
    const unsigned G = (__ballot_sync(0xffffffffu, in && g) >> gbase) & tmask;
    const unsigned P = (__ballot_sync(0xffffffffu, !in || p) >> gbase) & tmask;
    const unsigned long long S = (unsigned long long)(G | P) + G + c;
    const unsigned cl = (unsigned)((S ^ P) >> gl) & 1u;
    c = (unsigned)(S >> TPP) & 1u;
    hp = __shfl_sync(0xffffffffu, hi, (int)(gbase + TPP - 1));
    ep = __shfl_sync(0xffffffffu, ov, (int)(gbase + TPP - 1));
    if (!in || !write) continue;
    const unsigned d = certified ? u + cl : 0u;
    const int i = 4 * k;
    if (i + 3 < nout && wide) {
      *reinterpret_cast<unsigned *>(out + i) = d;
    } else {
#pragma unroll
      for (int b = 0; b < 4; b++)
        if (i + b < nout) out[i + b] = (uint8_t)(d >> (8 * b));
    }
  }
}

// FAST: no diagnostic outputs (interval dump, snapped coefficients), host-checked
template <typename T, int M, bool FAST = false>
__global__ void __launch_bounds__(512, 1) ivm_v6_kernel(KParams kp) {
  using C = Cfg6<T, M>;
  using Gm = G3<M, 8>;
  using X = RT6<M>;
  using V = typename V2t<T>::t;
  constexpr int N = C::N, TPP = C::TPP, PPC = C::PPC, R = 8;
  constexpr int NFWD = X::NFWD, NINV = X::NINV;
  constexpr bool LAST8 = X::LAST8;
  constexpr int RSI1 = Gm::iRS(1), SWI1 = Gm::iSW(1);
  constexpr int RATIO = 2 * N / Gm::LASTL();
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) unsigned long long tbar;
  const int g = (int)threadIdx.x / TPP, tid = (int)threadIdx.x % TPP;
  V *base = reinterpret_cast<V *>(smem);
  Buf<T> st{base + (size_t)g * C::CAPP, base + (size_t)(PPC + g) * C::CAPP};
  int32_t *coef = reinterpret_cast<int32_t *>(st.re);  // aliases this multiplication's re plane
  TwC<T> *twb = reinterpret_cast<TwC<T> *>(smem + C::STATE_BYTES);
  const TwC<T> *tw = reinterpret_cast<const TwC<T> *>(kp.tw);
  Buf<T> A{reinterpret_cast<V *>(kp.ascratch) + ((size_t)blockIdx.x * PPC + g) * N, nullptr};
  A.im = A.re + N / 2;
  const int n = kp.n;
  constexpr unsigned TB = (unsigned)(sizeof(TwC<T>) * Gm::tw_total());
  if (threadIdx.x == 0) mbar_init(&tbar);
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect(&tbar, (TB + 15u) & ~15u);
    bulk_copy(twb, tw, (TB + 15u) & ~15u, &tbar);
  }
  mbar_wait(&tbar, 0);

  for (int pb = (int)blockIdx.x * PPC; pb < kp.batch; pb += (int)gridDim.x * PPC) {
    const int pair = pb + g;
    const bool valid = pair < kp.batch;
    const int pr = valid ? pair : kp.batch - 1;  // idle groups recompute the last pair, write nothing
    CertAcc acc;
#pragma unroll 1
    for (int op = 0; op < 2; op++) {
      fwd_first<T, M, 8>((op == 0 ? kp.a : kp.b) + (size_t)pr * n, n, st, tw, tid);
      __syncwarp();
#pragma unroll 1
      for (int i = 0; i < NFWD; i++) {
        const PassRT pp = (i == 0) ? X::fwd(0) : X::fwd(NFWD > 1 ? 1 : 0);
        CI<T> v[R];
        int k0, nu;
        fwdR<T, R>(st, twb, pp, v, k0, nu, tid);
        if (i < NFWD - 1) {
          __syncwarp();
#pragma unroll
          for (int r = 0; r < R; r++) {
            if (2 * r < R) st.st(sidx(k0 + pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
            else st.st_conj(sidx(R * pp.L - 1 - k0 - pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
          }
        } else if (op == 0) {
#pragma unroll
          for (int r = 0; r < R; r++) A.st(r * (pp.L >> 1) + k0, v[r]);
        } else {
          CI<T> an = A.ld(k0);
#pragma unroll
          for (int r = 0; r < R; r++) {
            const CI<T> a = an;
            if (r + 1 < R) an = A.ld((r + 1) * (pp.L >> 1) + k0);
            v[r] = cmul_ss(a, v[r]);
          }
          cdft<T, R, true>(v);
          __syncwarp();
#pragma unroll
          for (int r = 0; r < R; r++) st.st(sidx(r, k0, RSI1, SWI1), v[r]);
        }
        __syncwarp();
      }
    }
    double *dump = (!FAST && valid) ? diag_dump(kp, pair, N) : nullptr;
#pragma unroll 1
    for (int i = 0; i < NINV; i++) {
      const PassRT pp = (i == 0) ? X::inv(0) : X::inv(NINV > 1 ? 1 : 0);
      CI<T> v[R];
      int k0, nu;
      if (LAST8 && i == NINV - 1) {
        invR<T, R, true>(st, twb, pp, v, k0, nu, tid);
        __syncwarp();  // every input loaded: the coefficients may overwrite the state
#pragma unroll
        for (int r = 0; r < R; r++) {
          const int k = k0 + pp.L * r;
          emit_fold<T, M, RATIO>(v[r], r, k, n, coef + k, coef + k + N / 2, acc, dump);
        }
      } else {
        invR<T, R, false>(st, twb, pp, v, k0, nu, tid);
        __syncwarp();
#pragma unroll
        for (int r = 0; r < R; r++) st.st(sidx(k0 + pp.L * r, nu, pp.RSo, pp.SWo), v[r]);
      }
      __syncwarp();
    }
    if constexpr (!LAST8) inv_last<T, M, 8, true>(st, tw, n, coef, acc, dump, tid);
    cert_group<TPP>(acc);
    __syncwarp();
    const bool certified = acc.ok != 0;
    carry_group<TPP>(coef, n, kp.prod + (size_t)pr * 2 * n, certified, valid);
    if (valid) {
      if (!FAST && kp.coeffs) {
        int64_t *co = kp.coeffs + (size_t)pair * (2 * n - 1);
        for (int i = tid; i < 2 * n - 1; i += TPP) co[i] = certified ? coef[i] : 0;
      }
      if (tid == 0) {
        kp.cert[pair] = certified ? 1 : 0;
        if (kp.max_radius) kp.max_radius[pair] = acc.rad * 0.5;  // (acc tracks the width)
        if (kp.first_bad) kp.first_bad[pair] = certified ? -1 : acc.bad;
      }
    }
    __syncwarp();
  }
}

}  // namespace v6
}  // namespace ivm
