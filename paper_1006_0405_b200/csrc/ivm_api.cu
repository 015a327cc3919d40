// ivm_api.cu -- the C ABI (include/ivm.h): context, plan cache, launches.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "../../include/ivm.h"

#include "ivm_internal.h"

static const int kMaxLog2M = 18;  // 13: CTA-resident; 14..18: multi-CTA groups

struct ivm_ctx {
  int device = 0;
  int sms = 0;
  int sticky = 0;
  bool consts = false;
  std::map<std::pair<int, int>, void *> tw;  // (log2m, prec) -> device table (v1)
  std::map<std::pair<int, int>, void *> tw3;  // (log2m, prec) -> v3 per-pass tables
  std::map<std::pair<int, int>, ivm::LaunchInfo> info;
  std::map<std::pair<int, int>, ivm::LaunchInfo> info3;
  bool force_v1 = false;
  bool force_v5 = false;   // IVM_KERNEL=v5: the group kernel also for m = 2^14 .. 2^16
  bool v7 = true;          // fp64 m = 2^17, 2^18: the pipelined group kernel (IVM_V7=0: the lockstep one)
  bool disc3 = true;       // circular sets at m = 2^10 .. 2^13 on the radix-8 schedule (IVM_DISC3=0: radix 2)
  void *g7scratch = nullptr;  // its stage counters and per-pair ring
  size_t g7scratch_bytes = 0;
  std::map<std::pair<int, int>, void *> tw4;  // (log2m, prec) -> v4 role tables
  std::map<std::pair<int, int>, ivm::LaunchInfo> info4;
  std::map<std::pair<int, int>, void *> twn;  // (log2m, prec) -> round-to-nearest twiddles (naive SS)
  std::map<int, std::pair<void *, double>> twd;  // log2m -> twiddle disc centers + radius bound
  void *dscratch = nullptr;                  // circular sets: per-CTA spectrum of a
  size_t dscratch_bytes = 0;
  void *nscratch = nullptr;                  // naive SS: per-CTA spectrum of a
  size_t nscratch_bytes = 0;
  int radix = 8;  // radix of the one-CTA kernel
  void *ascratch = nullptr;
  size_t ascratch_bytes = 0;
  int32_t *slot = nullptr;
  size_t slot_cap = 0;
  uint8_t *stage = nullptr;  // host API staging: a | b | prod | cert
  size_t stage_bytes = 0;
  int last_launches = 0;
  void *gscratch = nullptr;  // large-m group scratch
  size_t gscratch_bytes = 0;
  void *lscratch = nullptr;  // long multiplication sums / escalation buffers
  size_t lscratch_bytes = 0;
  // host API pipeline: copy-in / copy-out streams and per-chunk events
  cudaStream_t s_in = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> ev;
  // the scratch buffers above are shared by every call on the context: a call
  // on another stream than the previous call's waits for the previous call
  cudaEvent_t done_ev = nullptr;
  // co-run of the group kernel beside the cluster kernel (corun_split)
  bool corun = true;
  double corun_eff = 0.0;  // group kernel's rate relative to a cluster's; 0: the measured default per m
  cudaStream_t s_co = nullptr;
  cudaEvent_t co_ev[2] = {nullptr, nullptr};
  cudaStream_t last_stream = nullptr;
  bool have_last = false;
};

static int cuda_fail(ivm_ctx_t c) {
  if (c) c->sticky = IVM_ECUDA;
  return IVM_ECUDA;
}

// Orders the calls of one context across streams (include/ivm.h "Streams"):
// the guard makes the call's stream wait for the previous call's work when the
// stream changed, and records the call's completion event when it returns.
struct StreamOrder {
  ivm_ctx_t c;
  cudaStream_t s;
  bool ok = true;
  StreamOrder(ivm_ctx_t c_, void *stream) : c(c_), s((cudaStream_t)stream) {
    if (c->have_last && c->last_stream != s) ok = cudaStreamWaitEvent(s, c->done_ev, 0) == cudaSuccess;
  }
  ~StreamOrder() {
    if (cudaEventRecord(c->done_ev, s) == cudaSuccess) {
      c->last_stream = s;
      c->have_last = true;
    }
  }
};

static int log2m_for(size_t n) {
  if (n <= 1) return 0;
  size_t N = 1;
  int m = 0;
  while (N < 2 * n - 1) {
    N <<= 1;
    m++;
  }
  return m;
}

extern "C" {

const char *ivm_version(void) { return "ivm 0.1.0 sm_100a"; }

#ifdef IVM_PHASES
// experiment build only (tools/phases.py): per-CTA cycle counts of the kernel
// phases (ivm_phase.cuh); slots [0, 1024) the main kernel, [1024, 2048) the co-run
static unsigned long long *g_phases = nullptr;
static constexpr size_t PH_SLOTS = 2048 * 16;
static unsigned long long *phases_buf() {
  if (!g_phases && cudaMalloc(&g_phases, PH_SLOTS * 8) == cudaSuccess) cudaMemset(g_phases, 0, PH_SLOTS * 8);
  return g_phases;
}
extern "C" int ivm_phases_read(unsigned long long *out, size_t count) {
  if (!g_phases || count > PH_SLOTS) return IVM_EINVAL;
  if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpy(out, g_phases, count * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemset(g_phases, 0, PH_SLOTS * 8) != cudaSuccess)
    return IVM_ECUDA;
  return IVM_OK;
}
#endif

const char *ivm_strerror(int s) {
  switch (s) {
    case IVM_OK: return "ok";
    case IVM_EINVAL: return "invalid argument";
    case IVM_ENOMEM: return "out of memory";
    case IVM_ECUDA: return "CUDA error";
    case IVM_EUNSUPPORTED: return "unsupported size or precision";
    case IVM_ENCCL: return "NCCL unavailable or failed";
    case IVM_ENODEV: return "no CUDA device";
    default: return "unknown status";
  }
}

size_t ivm_max_digits(int prec) {
  if (prec != IVM_F64 && prec != IVM_F32) return 0;
  return ((size_t)1 << kMaxLog2M) / 2;  // 2n-1 <= m = 2^18
}

size_t ivm_fft_length(size_t n) { return n == 0 ? 0 : (size_t)1 << log2m_for(n); }

int ivm_twiddle_table(int log2m, int prec, void *out) {
  if (!out || log2m < 0 || log2m > 24 || (prec != IVM_F64 && prec != IVM_F32)) return IVM_EINVAL;
  return ivm::plan_twiddles(log2m, prec, out) == 0 ? IVM_OK : IVM_EUNSUPPORTED;
}

int ivm_create(ivm_ctx_t *ctx, int device) {
  if (!ctx) return IVM_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return IVM_ENODEV;
  if (device < 0 || device >= ndev) return IVM_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return IVM_ECUDA;
  ivm_ctx *c = new ivm_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  double w64[32 * 4];
  float w32[32 * 4];
  if (ivm::plan_twiddles(5, 0, w64) != 0 || ivm::plan_twiddles(5, 1, w32) != 0) {
    delete c;
    return IVM_EUNSUPPORTED;
  }
  if (ivm::upload_w32(w64, w32) != 0) {
    delete c;
    return IVM_ECUDA;
  }
  {
    double t64[64 * 4];
    float t32[64 * 4];
    if (ivm::plan_twiddles(6, 0, t64) != 0 || ivm::plan_twiddles(6, 1, t32) != 0) {
      delete c;
      return IVM_EUNSUPPORTED;
    }
    if (ivm::upload_w64(t64, t32) != 0 || ivm::upload_w64_v4(t64, t32) != 0 ||
        ivm::upload_w64_v5(t64, t32) != 0) {
      delete c;
      return IVM_ECUDA;
    }
  }
  const char *kv = getenv("IVM_KERNEL");
  c->force_v1 = kv && strcmp(kv, "v1") == 0;
  c->force_v5 = kv && strcmp(kv, "v5") == 0;
  {
    const char *e = getenv("IVM_V7");
    c->v7 = !(e && strcmp(e, "0") == 0);
    const char *d = getenv("IVM_DISC3");
    c->disc3 = !(d && strcmp(d, "0") == 0);
  }
  {  // IVM_CORUN=0 disables the co-run; IVM_CORUN_EFF sets the group kernel's relative rate
    const char *e = getenv("IVM_CORUN");
    c->corun = !(e && strcmp(e, "0") == 0);
    const char *f = getenv("IVM_CORUN_EFF");
    if (f && atof(f) > 0.05 && atof(f) <= 2.0) c->corun_eff = atof(f);
  }
  if (cudaEventCreateWithFlags(&c->done_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->co_ev[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->co_ev[1], cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return IVM_ECUDA;
  }
  c->consts = true;
  *ctx = c;
  return IVM_OK;
}

int ivm_destroy(ivm_ctx_t c) {
  if (!c) return IVM_OK;
  cudaSetDevice(c->device);
  for (auto &kv : c->tw) cudaFree(kv.second);
  for (auto &kv : c->tw3) cudaFree(kv.second);
  for (auto &kv : c->tw4) cudaFree(kv.second);
  for (auto &kv : c->twn) cudaFree(kv.second);
  for (auto &kv : c->twd) cudaFree(kv.second.first);
  cudaFree(c->dscratch);
  cudaFree(c->nscratch);
  cudaFree(c->ascratch);
  cudaFree(c->slot);
  cudaFree(c->stage);
  cudaFree(c->gscratch);
  cudaFree(c->g7scratch);
  cudaFree(c->lscratch);
  if (c->s_in) cudaStreamDestroy(c->s_in);
  if (c->s_out) cudaStreamDestroy(c->s_out);
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  if (c->done_ev) cudaEventDestroy(c->done_ev);
  for (cudaEvent_t e : c->co_ev)
    if (e) cudaEventDestroy(e);
  if (c->s_co) cudaStreamDestroy(c->s_co);
  delete c;
  return IVM_OK;
}

static int get_table(ivm_ctx_t c, int m, int prec, const void **out) {
  auto key = std::make_pair(m, prec);
  auto it = c->tw.find(key);
  if (it != c->tw.end()) {
    *out = it->second;
    return IVM_OK;
  }
  const size_t N = (size_t)1 << m, es = prec == IVM_F64 ? 8 : 4;
  std::vector<unsigned char> h(N * 4 * es);
  if (ivm::plan_twiddles(m, prec, h.data()) != 0) return IVM_EUNSUPPORTED;
  void *d = nullptr;
  if (cudaMalloc(&d, h.size()) != cudaSuccess) return IVM_ENOMEM;
  if (cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return cuda_fail(c);
  }
  c->tw[key] = d;
  *out = d;
  return IVM_OK;
}

static bool use_v3(ivm_ctx_t c, int m) { return !c->force_v1 && m >= 10 && m <= 13; }
// fp64 only: at fp32 (C4, the precision-limit sweep) the v1 kernel's full-interval
// twiddles give ~2x tighter enclosures (93 % vs 0 % of 32-digit uniform pairs certified)
static bool use_v6(ivm_ctx_t c, int m, int prec) { return !c->force_v1 && prec == IVM_F64 && m >= 6 && m <= 9; }
static bool use_v4(ivm_ctx_t c, int m) { return !c->force_v5 && m >= 14 && m <= 16; }
static bool use_v5(ivm_ctx_t c, int m) { return m >= 14 && m <= 18 && !use_v4(c, m); }
static bool use_v7(ivm_ctx_t c, int m, int prec) { return c->v7 && prec == IVM_F64 && (m == 17 || m == 18); }

static int get_info5(ivm_ctx_t c, int m, int prec, ivm::LaunchInfo *li) {
  auto key = std::make_pair(m + 100, prec);
  auto it = c->info4.find(key);
  if (it != c->info4.end()) {
    *li = it->second;
    return IVM_OK;
  }
  int r = ivm::v5_info(prec, m, li);
  if (r == -4) return IVM_EUNSUPPORTED;
  if (r != 0 || li->blocks_per_sm < 1) return cuda_fail(c);
  c->info4[key] = *li;
  return IVM_OK;
}

static int get_info7(ivm_ctx_t c, int m, ivm::LaunchInfo *li) {
  auto key = std::make_pair(m + 200, (int)IVM_F64);
  auto it = c->info4.find(key);
  if (it != c->info4.end()) {
    *li = it->second;
    return IVM_OK;
  }
  int r = ivm::v7_info(m, li);
  if (r == -4) return IVM_EUNSUPPORTED;
  if (r != 0 || li->blocks_per_sm < 1) return cuda_fail(c);
  c->info4[key] = *li;
  return IVM_OK;
}

static int get_table4(ivm_ctx_t c, int m, int prec, const void **out) {
  auto key = std::make_pair(m, prec);
  auto it = c->tw4.find(key);
  if (it != c->tw4.end()) {
    *out = it->second;
    return IVM_OK;
  }
  const size_t N2 = (size_t)2 << m, es = prec == IVM_F64 ? 8 : 4;
  std::vector<unsigned char> w2N(N2 * 4 * es);
  if (ivm::plan_twiddles(m + 1, prec, w2N.data()) != 0) return IVM_EUNSUPPORTED;
  const int ent = ivm::v4_table_entries(m);
  if (ent < 0) return IVM_EUNSUPPORTED;
  std::vector<unsigned char> h((size_t)ent * 2 * es);
  if (ivm::v4_tables(m, prec, w2N.data(), h.data()) != ent) return IVM_EUNSUPPORTED;
  void *d = nullptr;
  if (cudaMalloc(&d, h.size()) != cudaSuccess) return IVM_ENOMEM;
  if (cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return cuda_fail(c);
  }
  c->tw4[key] = d;
  *out = d;
  return IVM_OK;
}

static int get_info4(ivm_ctx_t c, int m, int prec, ivm::LaunchInfo *li) {
  auto key = std::make_pair(m, prec);
  auto it = c->info4.find(key);
  if (it != c->info4.end()) {
    *li = it->second;
    return IVM_OK;
  }
  int r = ivm::v4_info(prec, m, li);
  if (r == -4) return IVM_EUNSUPPORTED;
  if (r != 0 || li->max_clusters < 1) return cuda_fail(c);
  c->info4[key] = *li;
  return IVM_OK;
}

static int get_table3(ivm_ctx_t c, int m, int prec, const void **out) {
  const int radix = 8;  // v6 / v3 radix-8 plans
  auto key = std::make_pair(m * 100 + radix, prec);
  auto it = c->tw3.find(key);
  if (it != c->tw3.end()) {
    *out = it->second;
    return IVM_OK;
  }
  const size_t N2 = (size_t)2 << m, es = prec == IVM_F64 ? 8 : 4;
  std::vector<unsigned char> w2N(N2 * 4 * es);
  if (ivm::plan_twiddles(m + 1, prec, w2N.data()) != 0) return IVM_EUNSUPPORTED;
  const int ent = ivm::v3_table_entries(m, radix);
  if (ent < 0) return IVM_EUNSUPPORTED;
  std::vector<unsigned char> h((size_t)ent * 2 * es);  // compact entries
  if (ivm::v3_tables(m, prec, radix, w2N.data(), h.data()) != ent) return IVM_EUNSUPPORTED;
  void *d = nullptr;
  if (cudaMalloc(&d, h.size()) != cudaSuccess) return IVM_ENOMEM;
  if (cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return cuda_fail(c);
  }
  c->tw3[key] = d;
  *out = d;
  return IVM_OK;
}

static int get_info3(ivm_ctx_t c, int m, int prec, ivm::LaunchInfo *li) {
  auto key = std::make_pair(m * 100 + c->radix, prec);
  auto it = c->info3.find(key);
  if (it != c->info3.end()) {
    *li = it->second;
    return IVM_OK;
  }
  int r = ivm::v3_info(prec, m, c->radix, li);
  if (r == -4) return IVM_EUNSUPPORTED;
  if (r != 0 || li->blocks_per_sm < 1) return cuda_fail(c);
  c->info3[key] = *li;
  return IVM_OK;
}

static int get_info6(ivm_ctx_t c, int m, int prec, ivm::LaunchInfo *li) {
  auto key = std::make_pair(m + 200, prec);
  auto it = c->info4.find(key);
  if (it != c->info4.end()) {
    *li = it->second;
    return IVM_OK;
  }
  int r = ivm::v6_info(prec, m, li);
  if (r == -4) return IVM_EUNSUPPORTED;
  if (r != 0 || li->blocks_per_sm < 1) return cuda_fail(c);
  c->info4[key] = *li;
  return IVM_OK;
}

static int get_info(ivm_ctx_t c, int m, int prec, ivm::LaunchInfo *li) {
  auto key = std::make_pair(m, prec);
  auto it = c->info.find(key);
  if (it != c->info.end()) {
    *li = it->second;
    return IVM_OK;
  }
  int r = ivm::cta_info(prec, m, li);
  if (r == -4) return IVM_EUNSUPPORTED;
  if (r != 0 || li->blocks_per_sm < 1) return cuda_fail(c);
  c->info[key] = *li;
  return IVM_OK;
}

// exchange / barrier scratch of the group kernel (v5) for `groups` groups of C CTAs
static int ensure_gscratch5(ivm_ctx_t c, int m, int prec, size_t groups, size_t C) {
  (void)m;
  const size_t al = 256, es = prec == IVM_F64 ? 8 : 4;
  auto up = [&](size_t x) { return (x + al - 1) / al * al; };
  const size_t need = up(groups * C * 4096 * 4 * es) + up(groups * C * 32) + up(groups * 2 * C * C * 8 * 8) +
                      up(groups * 2 * C * C) + up(groups * 4);
  if (c->gscratch_bytes >= need) return IVM_OK;
  cudaFree(c->gscratch);
  c->gscratch = nullptr;
  c->gscratch_bytes = 0;
  if (cudaMalloc(&c->gscratch, need) != cudaSuccess) return IVM_ENOMEM;
  c->gscratch_bytes = need;
  return IVM_OK;
}

// the group kernel on `groups` groups (scratch ensured by the caller); coop:
// cooperative launch (the kernel alone on the device), else a plain launch
// (co-run beside the cluster kernel on the SMs its clusters leave free)
static int launch_v5(ivm_ctx_t c, int m, int prec, const ivm::KParams &kp0, size_t groups, size_t C, void *ascr,
                     cudaStream_t s, bool coop) {
  const size_t al = 256, es = prec == IVM_F64 ? 8 : 4;
  auto up = [&](size_t x) { return (x + al - 1) / al * al; };
  const size_t b_x = up(groups * C * 4096 * 4 * es), b_l = up(groups * C * 32),
               b_b = up(groups * 2 * C * C * 8 * 8), b_bits = up(groups * 2 * C * C), b_ctr = up(groups * 4);
  char *gs = (char *)c->gscratch;
  ivm::Group5Args ga;
  ga.xch = gs;
  ga.link = (unsigned *)(gs + b_x);
  ga.bnd = (long long *)(gs + b_x + b_l);
  ga.bits = (uint8_t *)(gs + b_x + b_l + b_b);
  ga.ctr = (unsigned *)(gs + b_x + b_l + b_b + b_bits);
  if (cudaMemsetAsync(ga.ctr, 0, b_ctr, s) != cudaSuccess) return cuda_fail(c);
  ivm::KParams kp = kp0;
  kp.ascratch = ascr;
  if (ivm::v5_launch(prec, m, kp, ga, (int)groups, s, coop) != 0) return cuda_fail(c);
  return IVM_OK;
}

// The pipelined group kernel (v7): grid, ring size and scratch.  A pair's tasks
// span at most two consecutive slots, its last stage runs three slots after its
// first task's; the L stage of pair p + rp waits for pair p's last stage, which
// must lie at an earlier slot: rp C >= 5 grid + C - 1 (ivm_v7.cuh)
static int ensure_scratch(ivm_ctx_t c, size_t bytes);
static int v7_ring(size_t grid, size_t C, size_t batch, size_t pair_bytes) {
  size_t rp = (5 * grid + C - 1) / C + 1;
  // a larger ring when memory allows (up to 1 GB): no slot reuse, so no ring waits, below 1 GB
  const size_t cap = ((size_t)1 << 30) / pair_bytes;
  if (cap > rp) rp = cap;
  if (rp > batch) rp = batch;
  return (int)rp;
}
static int launch_v7(ivm_ctx_t c, int m, const ivm::KParams &kp0, const ivm::LaunchInfo &li, size_t batch,
                     cudaStream_t s, bool disc = false) {
  const size_t C = (size_t)li.cluster;
  size_t grid = (size_t)c->sms * li.blocks_per_sm;
  if (grid > batch * C) grid = batch * C;
  const size_t per_pair = C * 4096 * 32 + C * 512 * 16 + 2 * C * C * 8 + C * 32;
  const size_t rp = (size_t)v7_ring(grid, C, batch, per_pair);
  const size_t al = 256;
  auto up = [&](size_t x) { return (x + al - 1) / al * al; };
  const size_t b_cnt = up(batch * 16), b_x = up(rp * C * 4096 * 32), b_w = up(rp * C * 512 * 16),
               b_r = up(rp * 2 * C * C * 8), b_l = up(rp * C * 32);
  const size_t need = b_cnt + b_x + b_w + b_r + b_l;
  int r = ensure_scratch(c, grid * li.a_bytes_per_cta);
  if (r) return r;
  if (c->g7scratch_bytes < need) {
    cudaFree(c->g7scratch);
    c->g7scratch = nullptr;
    c->g7scratch_bytes = 0;
    if (cudaMalloc(&c->g7scratch, need) != cudaSuccess) return IVM_ENOMEM;
    c->g7scratch_bytes = need;
  }
  char *gs = (char *)c->g7scratch;
  ivm::Pipe7Args pa;
  pa.cnt = (unsigned *)gs;
  pa.xch = gs + b_cnt;
  pa.wds = (uint4 *)(gs + b_cnt + b_x);
  pa.rec = (uint2 *)(gs + b_cnt + b_x + b_w);
  pa.link = (unsigned *)(gs + b_cnt + b_x + b_w + b_r);
  pa.rp = (int)rp;
  if (cudaMemsetAsync(pa.cnt, 0, b_cnt, s) != cudaSuccess) return cuda_fail(c);
  ivm::KParams kp = kp0;
  kp.ascratch = c->ascratch;
  if ((disc ? ivm::d7_launch(m, kp, pa, (int)grid, s) : ivm::v7_launch(m, kp, pa, (int)grid, s)) != 0) return cuda_fail(c);
  return IVM_OK;
}

// Co-run split of a cluster-kernel batch (m = 2^14 .. 2^16): clusters of C CTAs
// must sit inside one GPC, so `cl` clusters strand sms - cl C SMs; `g5` groups
// of the group kernel (same C, exchange through L2) run there at a per-group
// rate `eff` of a cluster's.  Returns the pairs the group kernel takes so that
// the two finish together (0: no co-run).
static size_t corun_split(size_t batch, size_t cl, size_t g5, double eff) {
  if (g5 == 0 || cl == 0 || batch < 2 * (cl + g5)) return 0;
  size_t best = 0;
  double tbest = (double)((batch + cl - 1) / cl);
  for (size_t r5 = 1; r5 * g5 <= batch; r5++) {
    const size_t b5 = r5 * g5, b4 = batch - b5;
    const double t = std::max((double)((b4 + cl - 1) / cl), (double)r5 / eff);
    if (t < tbest) {
      tbest = t;
      best = b5;
    }
    if ((double)r5 / eff > tbest) break;
  }
  return best;
}

static int grid_for(ivm_ctx_t c, const ivm::LaunchInfo &li, size_t batch) {
  size_t g = (size_t)c->sms * (size_t)li.blocks_per_sm;
  if (g > batch) g = batch;
  return (int)g;
}

static int ensure_scratch(ivm_ctx_t c, size_t bytes) {
  if (bytes <= c->ascratch_bytes) return IVM_OK;
  cudaFree(c->ascratch);
  c->ascratch = nullptr;
  c->ascratch_bytes = 0;
  if (cudaMalloc(&c->ascratch, bytes) != cudaSuccess) return IVM_ENOMEM;
  c->ascratch_bytes = bytes;
  return IVM_OK;
}

static int check_args(ivm_ctx_t c, const void *a, const void *b, size_t n, size_t batch, const void *p,
                      const void *cert, int prec) {
  if (!c || !a || !b || !p || !cert || n == 0 || batch == 0) return IVM_EINVAL;
  if (prec != IVM_F64 && prec != IVM_F32) return IVM_EINVAL;
  if (n > ivm_max_digits(prec)) return IVM_EUNSUPPORTED;
  if (batch > (size_t)0x7fffffff) return IVM_EINVAL;
  if (c->sticky) return c->sticky;
  return IVM_OK;
}

int ivm_reserve(ivm_ctx_t c, size_t n, size_t batch, int prec) {
  if (!c || n == 0 || batch == 0 || (prec != IVM_F64 && prec != IVM_F32)) return IVM_EINVAL;
  if (n > ivm_max_digits(prec)) return IVM_EUNSUPPORTED;
  if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(c);
  int m = log2m_for(n);
  if (m < 2) return IVM_OK;
  if (use_v4(c, m)) {
    const void *t4;
    ivm::LaunchInfo li;
    int r = get_table4(c, m, prec, &t4);
    if (!r) r = get_info4(c, m, prec, &li);
    if (r) return r;
    size_t cl = (size_t)li.max_clusters < batch ? (size_t)li.max_clusters : batch;
    return ensure_scratch(c, cl * li.cluster * li.a_bytes_per_cta);
  }
  if (use_v6(c, m, prec)) {
    const void *t3;
    ivm::LaunchInfo li;
    int r = get_table3(c, m, prec, &t3);
    if (!r) r = get_info6(c, m, prec, &li);
    if (r) return r;
    size_t grid = (batch + li.cluster - 1) / li.cluster, cap = (size_t)c->sms * li.blocks_per_sm;
    if (grid > cap) grid = cap;
    return ensure_scratch(c, grid * li.a_bytes_per_cta);
  }
  if (use_v7(c, m, prec)) {
    const void *t4;
    ivm::LaunchInfo li;
    int r = get_table4(c, m, prec, &t4);
    if (!r) r = get_info7(c, m, &li);
    return r;
  }
  if (use_v5(c, m)) {
    const void *t4;
    ivm::LaunchInfo li;
    int r = get_table4(c, m, prec, &t4);
    if (!r) r = get_info5(c, m, prec, &li);
    return r;
  }
  const void *t;
  ivm::LaunchInfo li;
  int r;
  if (use_v3(c, m)) {
    r = get_table3(c, m, prec, &t);
    if (r) return r;
    r = get_info3(c, m, prec, &li);
  } else {
    r = get_table(c, m, prec, &t);
    if (r) return r;
    r = get_info(c, m, prec, &li);
  }
  if (r) return r;
  if (!li.a_smem) return ensure_scratch(c, (size_t)grid_for(c, li, batch) * li.a_bytes_per_cta);
  return IVM_OK;
}

int ivm_multiply_batched_diag(ivm_ctx_t c, const uint8_t *a, const uint8_t *b, size_t n, size_t batch,
                              uint8_t *prod, uint8_t *cert, int prec, void *stream, double *max_radius,
                              int32_t *first_bad, int64_t *coeffs, const int32_t *dump_pairs,
                              size_t n_dump, double *intervals) {
  int r = check_args(c, a, b, n, batch, prod, cert, prec);
  if (r) return r;
  if (n_dump && (!dump_pairs || !intervals)) return IVM_EINVAL;
  if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(c);
  StreamOrder order(c, stream);
  if (!order.ok) return cuda_fail(c);
  cudaStream_t s = (cudaStream_t)stream;
  ivm::KParams kp{};
  kp.a = a; kp.b = b; kp.prod = prod; kp.cert = cert;
  kp.n = (int)n; kp.batch = (int)batch;
  kp.max_radius = max_radius; kp.first_bad = first_bad; kp.coeffs = coeffs;
  kp.intervals = intervals;
#ifdef IVM_PHASES
  kp.phases = phases_buf();
#endif
  int launches = 0;
  if (n_dump) {
    if (c->slot_cap < batch) {
      cudaFree(c->slot);
      c->slot = nullptr;
      c->slot_cap = 0;
      if (cudaMalloc(&c->slot, batch * sizeof(int32_t)) != cudaSuccess) return IVM_ENOMEM;
      c->slot_cap = batch;
    }
    if (ivm::dump_map_launch(c->slot, (int)batch, dump_pairs, (int)n_dump, s) != 0) return cuda_fail(c);
    launches += 2;
    kp.dump_slot = c->slot;
  }
  int m = log2m_for(n);
  if (m == 0) {
    if (ivm::n1_launch(kp, s) != 0) return cuda_fail(c);
    c->last_launches = launches + 1;
    return IVM_OK;
  }
  if (use_v4(c, m)) {
    const void *tw;
    ivm::LaunchInfo li;
    r = get_table4(c, m, prec, &tw);
    if (!r) r = get_info4(c, m, prec, &li);
    if (r) return r;
    const size_t C = (size_t)li.cluster;
    const size_t cl = (size_t)li.max_clusters < batch ? (size_t)li.max_clusters : batch;
    // the SMs whole clusters leave free take a share of the batch with the group kernel
    ivm::LaunchInfo l5;
    size_t g5 = 0, b5 = 0;
    if (c->corun && cl == (size_t)li.max_clusters && get_info5(c, m, prec, &l5) == IVM_OK && l5.blocks_per_sm >= 1) {
      const size_t used = cl * C, free_sms = (size_t)c->sms > used ? (size_t)c->sms - used : 0;
      g5 = free_sms / C;
      // measured same-box sweeps: m = 2^15 (4 groups of 4 beside 33 clusters)
      // 0.74, m = 2^16 (2 groups of 8 beside 16 clusters) 0.9
      const double eff = c->corun_eff > 0.0 ? c->corun_eff : (m == 15 ? 0.74 : 0.9);
      b5 = corun_split(batch, cl, g5, eff);
    }
    const size_t b4 = batch - b5;
    const size_t a4 = cl * C * li.a_bytes_per_cta;
    r = ensure_scratch(c, a4 + (b5 ? g5 * C * l5.a_bytes_per_cta : 0));
    if (!r && b5) r = ensure_gscratch5(c, m, prec, g5, C);
    if (!r && b5 && !c->s_co && cudaStreamCreateWithFlags(&c->s_co, cudaStreamNonBlocking) != cudaSuccess)
      r = cuda_fail(c);
    if (r) return r;
    kp.tw = tw;
    if (b5) {  // the group kernel's stream starts after the work queued on s
      if (cudaEventRecord(c->co_ev[0], s) != cudaSuccess || cudaStreamWaitEvent(c->s_co, c->co_ev[0], 0) != cudaSuccess)
        return cuda_fail(c);
    }
    kp.batch = (int)b4;
    kp.ascratch = c->ascratch;
    if (ivm::v4_launch(prec, m, kp, (int)(cl < b4 ? cl : b4), s) != 0) return cuda_fail(c);
    launches++;
    if (b5) {
      ivm::KParams k5 = kp;
      k5.batch = (int)b5;
      k5.a = kp.a + b4 * n;
      k5.b = kp.b + b4 * n;
      k5.prod = kp.prod + b4 * 2 * n;
      k5.cert = kp.cert + b4;
      if (kp.max_radius) k5.max_radius = kp.max_radius + b4;
      if (kp.first_bad) k5.first_bad = kp.first_bad + b4;
      if (kp.coeffs) k5.coeffs = kp.coeffs + b4 * (2 * n - 1);
      if (kp.dump_slot) k5.dump_slot = kp.dump_slot + b4;
      if (kp.phases) k5.phases = kp.phases + 1024 * 16;
      r = launch_v5(c, m, prec, k5, g5 < b5 ? g5 : b5, C, (char *)c->ascratch + a4, c->s_co, false);
      if (r) return r;
      launches += 1;
      if (cudaEventRecord(c->co_ev[1], c->s_co) != cudaSuccess || cudaStreamWaitEvent(s, c->co_ev[1], 0) != cudaSuccess)
        return cuda_fail(c);
    }
    c->last_launches = launches;
    return IVM_OK;
  }
  if (use_v6(c, m, prec)) {
    const void *tw;
    ivm::LaunchInfo li;
    r = get_table3(c, m, prec, &tw);
    if (!r) r = get_info6(c, m, prec, &li);
    if (r) return r;
    size_t grid = (batch + li.cluster - 1) / li.cluster, cap = (size_t)c->sms * li.blocks_per_sm;
    if (grid > cap) grid = cap;
    r = ensure_scratch(c, grid * li.a_bytes_per_cta);
    if (r) return r;
    kp.ascratch = c->ascratch;
    kp.tw = tw;
    if (ivm::v6_launch(prec, m, kp, (int)grid, s) != 0) return cuda_fail(c);
    c->last_launches = launches + 1;
    return IVM_OK;
  }
  if (use_v7(c, m, prec)) {
    const void *tw;
    ivm::LaunchInfo li;
    r = get_table4(c, m, prec, &tw);
    if (!r) r = get_info7(c, m, &li);
    if (r) return r;
    kp.tw = tw;
    r = launch_v7(c, m, kp, li, batch, s);
    if (r) return r;
    c->last_launches = launches + 1;
    return IVM_OK;
  }
  if (use_v5(c, m)) {
    const void *tw;
    ivm::LaunchInfo li;
    r = get_table4(c, m, prec, &tw);
    if (!r) r = get_info5(c, m, prec, &li);
    if (r) return r;
    const size_t C = (size_t)li.cluster;
    size_t groups = (size_t)c->sms * li.blocks_per_sm / C;
    if (groups > batch) groups = batch;
    if (groups < 1) return IVM_EUNSUPPORTED;
    r = ensure_scratch(c, groups * C * li.a_bytes_per_cta);
    if (!r) r = ensure_gscratch5(c, m, prec, groups, C);
    if (r) return r;
    kp.tw = tw;
    r = launch_v5(c, m, prec, kp, groups, C, c->ascratch, s, true);
    if (r) return r;
    c->last_launches = launches + 1;
    return IVM_OK;
  }
  const void *tw;
  ivm::LaunchInfo li;
  const bool v3 = use_v3(c, m);
  if (v3) {
    r = get_table3(c, m, prec, &tw);
    if (r) return r;
    r = get_info3(c, m, prec, &li);
  } else {
    r = get_table(c, m, prec, &tw);
    if (r) return r;
    r = get_info(c, m, prec, &li);
  }
  if (r) return r;
  int grid = grid_for(c, li, batch);
  if (!li.a_smem) {
    r = ensure_scratch(c, (size_t)grid * li.a_bytes_per_cta);
    if (r) return r;
    kp.ascratch = c->ascratch;
  }
  kp.tw = tw;
  if ((v3 ? ivm::v3_launch(prec, m, c->radix, kp, grid, s) : ivm::cta_launch(prec, m, kp, grid, s)) != 0)
    return cuda_fail(c);
  c->last_launches = launches + 1;
  return IVM_OK;
}

int ivm_multiply_batched(ivm_ctx_t c, const uint8_t *a, const uint8_t *b, size_t n, size_t batch,
                         uint8_t *prod, uint8_t *cert, int prec, void *stream) {
  return ivm_multiply_batched_diag(c, a, b, n, batch, prod, cert, prec, stream, nullptr, nullptr,
                                   nullptr, nullptr, 0, nullptr);
}

int ivm_multiply(ivm_ctx_t c, const uint8_t *a, const uint8_t *b, size_t n, uint8_t *prod,
                 uint8_t *cert, int prec, void *stream) {
  return ivm_multiply_batched(c, a, b, n, 1, prod, cert, prec, stream);
}

int ivm_multiply_batched_host(ivm_ctx_t c, const uint8_t *a, const uint8_t *b, size_t n, size_t batch,
                              uint8_t *prod, uint8_t *cert, int prec, void *stream) {
  int r = check_args(c, a, b, n, batch, prod, cert, prec);
  if (r) return r;
  if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(c);
  StreamOrder order(c, stream);
  if (!order.ok) return cuda_fail(c);
  const size_t in = n * batch, out = 2 * n * batch;
  const size_t need = 2 * in + out + batch;
  if (c->stage_bytes < need) {
    cudaFree(c->stage);
    c->stage = nullptr;
    c->stage_bytes = 0;
    if (cudaMalloc(&c->stage, need) != cudaSuccess) return IVM_ENOMEM;
    c->stage_bytes = need;
  }
  if (!c->s_in) {
    if (cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking) != cudaSuccess)
      return cuda_fail(c);
  }
  // chunks of whole waves (multiples of the SM count), at most kChunks: the
  // copy-in of chunk i+1 and the copy-out of chunk i-1 overlap the kernel of chunk i
  static const int kChunks = [] {  // IVM_HOST_CHUNKS overrides (tuning)
    const char *e = getenv("IVM_HOST_CHUNKS");
    const int v = e ? atoi(e) : 0;
    return v >= 1 && v <= 64 ? v : 8;
  }();
  const size_t sms = (size_t)(c->sms > 0 ? c->sms : 1);
  size_t chunk = batch;
  if (batch >= 2 * sms) {
    chunk = (batch + kChunks - 1) / kChunks;
    chunk = (chunk + sms - 1) / sms * sms;
  }
  const size_t nchunks = (batch + chunk - 1) / chunk;
  while (c->ev.size() < 3 * nchunks + 1) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return cuda_fail(c);
    c->ev.push_back(e);
  }
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t *da = c->stage, *db = da + in, *dp = db + in, *dc = dp + out;
  // the internal streams start after the work already queued on `stream`
  cudaEvent_t e0 = c->ev[3 * nchunks];
  if (cudaEventRecord(e0, s) != cudaSuccess || cudaStreamWaitEvent(c->s_in, e0, 0) != cudaSuccess)
    return cuda_fail(c);
  int launches = 0;
  // all copy-ins first: a copy-out waiting on its kernel must not sit ahead of
  // a later copy-in in a shared copy queue
  for (size_t k = 0; k < nchunks; k++) {
    const size_t p0 = k * chunk, bk = (batch - p0 < chunk) ? batch - p0 : chunk;
    if (cudaMemcpyAsync(da + p0 * n, a + p0 * n, bk * n, cudaMemcpyHostToDevice, c->s_in) != cudaSuccess ||
        cudaMemcpyAsync(db + p0 * n, b + p0 * n, bk * n, cudaMemcpyHostToDevice, c->s_in) != cudaSuccess ||
        cudaEventRecord(c->ev[3 * k], c->s_in) != cudaSuccess)
      return cuda_fail(c);
  }
  for (size_t k = 0; k < nchunks; k++) {
    const size_t p0 = k * chunk, bk = (batch - p0 < chunk) ? batch - p0 : chunk;
    cudaEvent_t e_in = c->ev[3 * k], e_run = c->ev[3 * k + 1], e_out = c->ev[3 * k + 2];
    if (cudaStreamWaitEvent(s, e_in, 0) != cudaSuccess) return cuda_fail(c);
    r = ivm_multiply_batched(c, da + p0 * n, db + p0 * n, n, bk, dp + p0 * 2 * n, dc + p0, prec, stream);
    if (r) return r;
    launches += c->last_launches;
    if (cudaEventRecord(e_run, s) != cudaSuccess || cudaStreamWaitEvent(c->s_out, e_run, 0) != cudaSuccess ||
        cudaMemcpyAsync(prod + p0 * 2 * n, dp + p0 * 2 * n, bk * 2 * n, cudaMemcpyDeviceToHost, c->s_out) !=
            cudaSuccess ||
        cudaMemcpyAsync(cert + p0, dc + p0, bk, cudaMemcpyDeviceToHost, c->s_out) != cudaSuccess ||
        cudaEventRecord(e_out, c->s_out) != cudaSuccess)
      return cuda_fail(c);
  }
  // `stream` completes after the last copy-out
  if (cudaStreamWaitEvent(s, c->ev[3 * (nchunks - 1) + 2], 0) != cudaSuccess) return cuda_fail(c);
  c->last_launches = launches;
  if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_fail(c);
  return IVM_OK;
}

static int ensure_lscratch(ivm_ctx_t c, size_t bytes) {
  if (bytes <= c->lscratch_bytes) return IVM_OK;
  cudaFree(c->lscratch);
  c->lscratch = nullptr;
  c->lscratch_bytes = 0;
  if (cudaMalloc(&c->lscratch, bytes) != cudaSuccess) return IVM_ENOMEM;
  c->lscratch_bytes = bytes;
  return IVM_OK;
}

static const size_t kLongMaxDigits = (size_t)1 << 18;  // sums < 255^2 n < 2^34 (word carry bound)
static const size_t kLongChunkBytes = (size_t)256 << 20;

static size_t long_chunk(size_t n, size_t batch) {  // pairs per launch (int64 sums <= 256 MiB)
  size_t chunk = kLongChunkBytes / ((2 * n - 1) * 8);
  if (chunk < 1) chunk = 1;
  return chunk > batch ? batch : chunk;
}

// exact products of `batch` pairs; the int64 sums go to the long-multiplication
// scratch at offset `off`, which the caller has sized for long_chunk(n, batch) pairs
static int long_run(ivm_ctx_t c, const uint8_t *a, const uint8_t *b, size_t n, size_t batch, uint8_t *prod,
                    cudaStream_t s, size_t off, int *launches) {
  const size_t nc = 2 * n - 1, chunk = long_chunk(n, batch);
  long long *coef = (long long *)((char *)c->lscratch + off);
  for (size_t p0 = 0; p0 < batch; p0 += chunk) {
    const size_t pb = batch - p0 < chunk ? batch - p0 : chunk;
    if (ivm::long_launch(a + p0 * n, b + p0 * n, (int)n, (int)pb, coef, prod + p0 * 2 * n, s) != 0)
      return cuda_fail(c);
    *launches += 2 + (int)((pb - 1) / 65535);
  }
  return IVM_OK;
}

int ivm_long_multiply_batched(ivm_ctx_t c, const uint8_t *a, const uint8_t *b, size_t n, size_t batch,
                              uint8_t *prod, void *stream) {
  if (!c || !a || !b || !prod || n == 0 || batch == 0) return IVM_EINVAL;
  if (n > kLongMaxDigits || batch > (size_t)0x7fffffff) return IVM_EUNSUPPORTED;
  if (c->sticky) return c->sticky;
  if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(c);
  StreamOrder order(c, stream);
  if (!order.ok) return cuda_fail(c);
  int r = ensure_lscratch(c, long_chunk(n, batch) * (2 * n - 1) * 8);
  if (r) return r;
  int launches = 0;
  r = long_run(c, a, b, n, batch, prod, (cudaStream_t)stream, 0, &launches);
  c->last_launches = launches;
  return r;
}

int ivm_multiply_exact(ivm_ctx_t c, const uint8_t *a, const uint8_t *b, size_t n, size_t batch, uint8_t *prod,
                       uint8_t *method, int policy, void *stream) {
  if (!c || !a || !b || !prod || n == 0 || batch == 0 || (policy != 0 && policy != 1)) return IVM_EINVAL;
  if (n > kLongMaxDigits || batch > (size_t)0x7fffffff) return IVM_EUNSUPPORTED;
  if (c->sticky) return c->sticky;
  if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(c);
  StreamOrder order(c, stream);
  if (!order.ok) return cuda_fail(c);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t al = 256;
  auto up = [&](size_t x) { return (x + al - 1) / al * al; };
  // scratch: cert | idx0 | idx1 | count | a', b' [batch][n] | prod' [batch][2n] | long-multiplication sums
  const size_t o_i0 = up(batch), o_i1 = o_i0 + up(4 * batch), o_cnt = o_i1 + up(4 * batch);
  const size_t o_a = o_cnt + al, o_b = o_a + up(batch * n), o_p = o_b + up(batch * n), o_l = o_p + up(2 * n * batch);
  int r = ensure_lscratch(c, o_l + long_chunk(n, batch) * (2 * n - 1) * 8);
  if (r) return r;
  char *L = (char *)c->lscratch;
  uint8_t *cert = (uint8_t *)L, *ga = (uint8_t *)(L + o_a), *gb = (uint8_t *)(L + o_b), *gp = (uint8_t *)(L + o_p);
  int *idx0 = (int *)(L + o_i0), *idx1 = (int *)(L + o_i1), *cnt = (int *)(L + o_cnt);
  int launches = 0, count = (int)batch, h = 0;
  const int *map = nullptr;  // compact index -> pair (null: identity)
  const bool f32 = policy == 0 && n <= 32;
  // policy 1: below m = 64 (n <= 16) the exact long multiplication outruns the
  // interval FFT on B200 (tools/long_vs_fft.py), so those sizes go to it directly
  const bool fft = n <= ivm_max_digits(IVM_F64) && !(policy == 1 && ivm_fft_length(n) < 64);
  if (fft) {
    // tier 1: fp32 (n <= 32) or fp64 interval FFT on the whole batch
    r = ivm_multiply_batched(c, a, b, n, batch, prod, cert, f32 ? IVM_F32 : IVM_F64, stream);
    if (r) return r;
    launches += c->last_launches;
    if (cudaMemsetAsync(cnt, 0, 4, s) != cudaSuccess) return cuda_fail(c);
    if (ivm::esc_mark(cert, nullptr, count, f32 ? 1 : 2, method, idx0, cnt, s) != 0) return cuda_fail(c);
    launches++;
    if (cudaMemcpyAsync(&h, cnt, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
      return cuda_fail(c);
    count = h;
    map = idx0;
    if (f32 && count > 0) {  // tier 2: fp64 for the pairs fp32 did not certify
      if (ivm::esc_gather(a, n, idx0, count, ga, s) || ivm::esc_gather(b, n, idx0, count, gb, s))
        return cuda_fail(c);
      r = ivm_multiply_batched(c, ga, gb, n, (size_t)count, gp, cert, IVM_F64, stream);
      if (r) return r;
      launches += 2 + c->last_launches;
      if (ivm::esc_scatter(gp, 2 * n, idx0, cert, count, prod, s) != 0) return cuda_fail(c);
      if (cudaMemsetAsync(cnt, 0, 4, s) != cudaSuccess) return cuda_fail(c);
      if (ivm::esc_mark(cert, idx0, count, 2, method, idx1, cnt, s) != 0) return cuda_fail(c);
      launches += 2;
      if (cudaMemcpyAsync(&h, cnt, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
          cudaStreamSynchronize(s) != cudaSuccess)
        return cuda_fail(c);
      count = h;
      map = idx1;
    }
  }
  if (count > 0) {  // tier 3: exact long multiplication
    const uint8_t *la = a, *lb = b;
    uint8_t *lp = prod;
    if (map) {
      if (ivm::esc_gather(a, n, map, count, ga, s) || ivm::esc_gather(b, n, map, count, gb, s))
        return cuda_fail(c);
      launches += 2;
      la = ga, lb = gb, lp = gp;
    }
    r = long_run(c, la, lb, n, (size_t)count, lp, s, o_l, &launches);
    if (r) return r;
    if (map) {
      if (ivm::esc_scatter(gp, 2 * n, map, nullptr, count, prod, s) != 0) return cuda_fail(c);
      launches++;
    }
    if (method) {
      if (ivm::esc_set_method(map, count, 3, method, s) != 0) return cuda_fail(c);
      launches++;
    }
  }
  c->last_launches = launches;
  if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_fail(c);
  return IVM_OK;
}

int ivm_multiply_naive(ivm_ctx_t c, const uint8_t *a, const uint8_t *b, size_t n, size_t batch, uint8_t *prod,
                       int prec, void *stream) {
  if (!c || !a || !b || !prod || n == 0 || batch == 0 || (prec != IVM_F64 && prec != IVM_F32)) return IVM_EINVAL;
  if (n > 4096 || batch > (size_t)0x7fffffff) return IVM_EUNSUPPORTED;
  if (c->sticky) return c->sticky;
  if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(c);
  StreamOrder order(c, stream);
  if (!order.ok) return cuda_fail(c);
  const int lg = log2m_for(n) < 1 ? 1 : log2m_for(n);
  auto key = std::make_pair(lg, prec);
  void *w = nullptr;
  auto it = c->twn.find(key);
  if (it != c->twn.end()) {
    w = it->second;
  } else {
    const size_t es = prec == IVM_F64 ? 8 : 4, bytes = ((size_t)2 << lg) * es;
    std::vector<unsigned char> h(bytes);
    if (ivm::plan_twiddles_rn(lg, prec, h.data()) != 0) return IVM_EUNSUPPORTED;
    if (cudaMalloc(&w, bytes) != cudaSuccess) return IVM_ENOMEM;
    if (cudaMemcpy(w, h.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaFree(w);
      return cuda_fail(c);
    }
    c->twn[key] = w;
  }
  const int smem = ivm::naive_smem(lg, prec);
  size_t grid = (size_t)c->sms * (smem > 114 * 1024 ? 1 : (smem > 56 * 1024 ? 2 : 4));
  if (grid > batch) grid = batch;
  const size_t need = grid * ((size_t)1 << lg) * (prec == IVM_F64 ? 16 : 8);
  if (c->nscratch_bytes < need) {
    cudaFree(c->nscratch);
    c->nscratch = nullptr;
    c->nscratch_bytes = 0;
    if (cudaMalloc(&c->nscratch, need) != cudaSuccess) return IVM_ENOMEM;
    c->nscratch_bytes = need;
  }
  if (ivm::naive_launch(prec, a, b, (int)n, (int)batch, lg, w, c->nscratch, prod, (int)grid, (cudaStream_t)stream) != 0)
    return cuda_fail(c);
  c->last_launches = 1;
  return IVM_OK;
}

int ivm_multiply_disc(ivm_ctx_t c, const uint8_t *a, const uint8_t *b, size_t n, size_t batch, uint8_t *prod,
                      uint8_t *cert, double *max_radius, void *stream) {
  if (!c || !a || !b || !prod || !cert || n == 0 || batch == 0) return IVM_EINVAL;
  if (n > ivm_max_digits(IVM_F64) || batch > (size_t)0x7fffffff) return IVM_EUNSUPPORTED;
  if (c->sticky) return c->sticky;
  if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(c);
  StreamOrder order(c, stream);
  if (!order.ok) return cuda_fail(c);
  const int lg = log2m_for(n);  // n = 1: m = 1 (no FFT stage)
  if (lg >= 10 && lg <= 13 && c->disc3) {
    // the one-CTA odd-frequency radix-8 schedule in disc arithmetic (ivm_d3.cuh),
    // on the rectangular kernels' tables (IVM_DISC3=0: the radix-2 kernel below)
    const void *tw3;
    ivm::LaunchInfo li;
    int r = get_table3(c, lg, IVM_F64, &tw3);
    if (r) return r;
    if (ivm::d3_info(lg, &li) != 0 || li.blocks_per_sm < 1) return cuda_fail(c);
    size_t grid = (size_t)c->sms * (size_t)li.blocks_per_sm;
    if (grid > batch) grid = batch;
    r = ensure_scratch(c, grid * li.a_bytes_per_cta);
    if (r) return r;
    ivm::KParams kp = {};
    kp.a = a;
    kp.b = b;
    kp.prod = prod;
    kp.cert = cert;
    kp.n = (int)n;
    kp.batch = (int)batch;
    kp.tw = tw3;
    kp.ascratch = c->ascratch;
    kp.max_radius = max_radius;
    if (ivm::d3_launch(lg, kp, (int)grid, (cudaStream_t)stream) != 0) return cuda_fail(c);
    c->last_launches = 1;
    return IVM_OK;
  }
  if (lg >= 14 && lg <= 16 && c->disc3) {
    // the cluster schedule in disc arithmetic (ivm_d4.cuh), on the rectangular cluster
    // kernel's tables (IVM_DISC3=0: the radix-2 group kernel below)
    const void *tw4;
    ivm::LaunchInfo li;
    int r = get_table4(c, lg, IVM_F64, &tw4);
    if (r) return r;
    if (ivm::d4_info(lg, &li) != 0 || li.max_clusters < 1) return cuda_fail(c);
    size_t cl = (size_t)li.max_clusters;
    if (cl > batch) cl = batch;
    r = ensure_scratch(c, cl * (size_t)li.cluster * li.a_bytes_per_cta);
    if (r) return r;
    ivm::KParams kp = {};
    kp.a = a;
    kp.b = b;
    kp.prod = prod;
    kp.cert = cert;
    kp.n = (int)n;
    kp.batch = (int)batch;
    kp.tw = tw4;
    kp.ascratch = c->ascratch;
    kp.max_radius = max_radius;
    if (ivm::d4_launch(lg, kp, (int)cl, (cudaStream_t)stream) != 0) return cuda_fail(c);
    c->last_launches = 1;
    return IVM_OK;
  }
  if ((lg == 17 || lg == 18) && c->disc3) {
    // the pipelined group schedule in disc arithmetic (ivm_d7.cuh), on the rectangular
    // kernel's tables and scratch layout (IVM_DISC3=0: the radix-2 group kernel below)
    const void *tw4;
    ivm::LaunchInfo li;
    int r = get_table4(c, lg, IVM_F64, &tw4);
    if (r) return r;
    if (ivm::d7_info(lg, &li) != 0 || li.blocks_per_sm < 1) return cuda_fail(c);
    ivm::KParams kp = {};
    kp.a = a;
    kp.b = b;
    kp.prod = prod;
    kp.cert = cert;
    kp.n = (int)n;
    kp.batch = (int)batch;
    kp.tw = tw4;
    kp.max_radius = max_radius;
    r = launch_v7(c, lg, kp, li, batch, (cudaStream_t)stream, true);
    if (r) return r;
    c->last_launches = 1;
    return IVM_OK;
  }
  void *w = nullptr;
  double rw = 0.0;
  auto it = c->twd.find(lg);
  if (it != c->twd.end()) {
    w = it->second.first;
    rw = it->second.second;
  } else {  // twiddle discs from the optimal rectangles: c = lower corner, r >= its diagonal (max over j)
    const size_t m = (size_t)1 << lg;
    std::vector<double> rect(m * 4), h(m < 2 ? 2 : m, 0.0);
    if (ivm::plan_twiddles(lg, IVM_F64, rect.data()) != 0) return IVM_EUNSUPPORTED;
    for (size_t j = 0; j < m / 2; j++) {
      const double *t = &rect[4 * j];
      h[2 * j] = t[0];
      h[2 * j + 1] = t[2];
      const double r = std::nextafter((t[1] - t[0]) + (t[3] - t[2]), 1.0);  // exact differences, sum rounded up
      rw = r > rw ? r : rw;
    }
    if (cudaMalloc(&w, h.size() * sizeof(double)) != cudaSuccess) return IVM_ENOMEM;
    if (cudaMemcpy(w, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaFree(w);
      return cuda_fail(c);
    }
    c->twd[lg] = std::make_pair(w, rw);
  }
  if (lg > 13) {  // groups of m/8192 co-resident CTAs (ivm_disc.cu disc_group_kernel)
    const int nb = ivm::disc_group_blocks_per_sm();
    if (nb < 1) return cuda_fail(c);
    const size_t C = (size_t)1 << (lg - 13);
    size_t groups = (size_t)c->sms * nb / C;
    if (groups > batch) groups = batch;
    if (groups < 1) return IVM_EUNSUPPORTED;
    const size_t need = ivm::disc_group_scratch(lg, groups);
    if (c->dscratch_bytes < need) {
      cudaFree(c->dscratch);
      c->dscratch = nullptr;
      c->dscratch_bytes = 0;
      if (cudaMalloc(&c->dscratch, need) != cudaSuccess) return IVM_ENOMEM;
      c->dscratch_bytes = need;
    }
    if (ivm::disc_group_launch(a, b, (int)n, (int)batch, lg, w, rw, c->dscratch, groups, prod, cert, max_radius,
                               (cudaStream_t)stream) != 0)
      return cuda_fail(c);
    c->last_launches = 1;
    return IVM_OK;
  }
  size_t grid = (size_t)c->sms;
  if (grid > batch) grid = batch;
  const size_t need = grid * ((size_t)32 << lg);
  if (c->dscratch_bytes < need) {
    cudaFree(c->dscratch);
    c->dscratch = nullptr;
    c->dscratch_bytes = 0;
    if (cudaMalloc(&c->dscratch, need) != cudaSuccess) return IVM_ENOMEM;
    c->dscratch_bytes = need;
  }
  if (ivm::disc_launch(a, b, (int)n, (int)batch, lg, w, rw, c->dscratch, prod, cert, max_radius, (int)grid,
                       (cudaStream_t)stream) != 0)
    return cuda_fail(c);
  c->last_launches = 1;
  return IVM_OK;
}

int ivm_generate_digits(ivm_ctx_t c, uint8_t *out, size_t n, size_t batch, uint64_t seed, uint64_t pair0,
                        int operand, int kind, const uint8_t *kinds, void *stream) {
  if (!c || !out || n == 0 || batch == 0 || kind < 0 || kind > 3 || (operand != 0 && operand != 1))
    return IVM_EINVAL;
  if (n > 0x7fffffff) return IVM_EINVAL;
  if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(c);
  if (ivm::digits_launch(out, (int)n, (long long)batch, seed, pair0, operand, kind, kinds, c->sms,
                         (cudaStream_t)stream) != 0)
    return cuda_fail(c);
  return IVM_OK;
}

int ivm_peak_probe(ivm_ctx_t c, int prec, int iters, double *sink, uint64_t *count, void *stream) {
  if (!c || !sink || !count || iters <= 0 || (prec != IVM_F64 && prec != IVM_F32)) return IVM_EINVAL;
  if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(c);
  if (ivm::probe_launch(prec, iters, sink, c->sms, (cudaStream_t)stream, count) != 0) return cuda_fail(c);
  return IVM_OK;
}

int ivm_last_launch_count(ivm_ctx_t c) { return c ? c->last_launches : 0; }

}  // extern "C"
