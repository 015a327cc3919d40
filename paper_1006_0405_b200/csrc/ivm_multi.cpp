// ivm_multi.cpp -- single-process multi-GPU API (include/ivm.h, SURVEY §8(b),
// §8(e)): one context per device, the batch sharded by the caller (independent
// multiplications, no data-path collective), an optional NCCL gather of the
// products and flags to the root device (grouped ncclSend / ncclRecv, chunk k
// on a communication stream while chunk k+1 multiplies on the compute stream),
// and the step summary {certified pairs, max radius} all-reduced over devices.
//
// NCCL is opened with dlopen("libnccl.so.2") on ivm_multi_create, so the
// library has no link-time NCCL dependency and a process that already loaded
// an NCCL (PyTorch's) shares it (same soname).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#include <cmath>

#include <vector>

#include "../../include/ivm.h"
#include "ivm_internal.h"

namespace {

// the few NCCL entry points used (ABI of nccl.h, stable across 2.x)
typedef void *ncclComm_t;
typedef int ncclResult_t;
enum { ncclUint8 = 1, ncclFloat64 = 8 };
enum { ncclSum = 0, ncclMax = 2 };
typedef ncclResult_t (*CommInitAll_t)(ncclComm_t *, int, const int *);
typedef ncclResult_t (*CommDestroy_t)(ncclComm_t);
typedef ncclResult_t (*Group_t)(void);
typedef ncclResult_t (*Send_t)(const void *, size_t, int, int, ncclComm_t, cudaStream_t);
typedef ncclResult_t (*Recv_t)(void *, size_t, int, int, ncclComm_t, cudaStream_t);
typedef ncclResult_t (*AllReduce_t)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t);

struct Nccl {
  void *h = nullptr;
  CommInitAll_t init = nullptr;
  CommDestroy_t destroy = nullptr;
  Group_t gstart = nullptr, gend = nullptr;
  Send_t send = nullptr;
  Recv_t recv = nullptr;
  AllReduce_t allreduce = nullptr;
  bool load() {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    init = (CommInitAll_t)dlsym(h, "ncclCommInitAll");
    destroy = (CommDestroy_t)dlsym(h, "ncclCommDestroy");
    gstart = (Group_t)dlsym(h, "ncclGroupStart");
    gend = (Group_t)dlsym(h, "ncclGroupEnd");
    send = (Send_t)dlsym(h, "ncclSend");
    recv = (Recv_t)dlsym(h, "ncclRecv");
    allreduce = (AllReduce_t)dlsym(h, "ncclAllReduce");
    return init && destroy && gstart && gend && send && recv && allreduce;
  }
};
Nccl g_nccl;

}  // namespace

struct ivm_multi {
  int ngpu = 0;
  std::vector<int> dev;
  std::vector<ivm_ctx_t> ctx;
  std::vector<cudaStream_t> st;   // compute
  std::vector<cudaStream_t> cst;  // communication (gather)
  std::vector<std::vector<cudaEvent_t>> ev;  // [g][chunk]: chunk computed
  std::vector<double *> sum;      // [g]: {certified, max radius} (device)
  std::vector<ncclComm_t> comm;
};

static const int kMultiChunks = 4;

extern "C" {

int ivm_multi_create(ivm_multi_t *m, int ngpu, const int *devices) {
  if (!m || ngpu < 1 || !devices) return IVM_EINVAL;
  *m = nullptr;
  int have = 0;
  if (cudaGetDeviceCount(&have) != cudaSuccess || have < 1) return IVM_ENODEV;
  for (int g = 0; g < ngpu; g++)
    if (devices[g] < 0 || devices[g] >= have) return IVM_EINVAL;
  if (!g_nccl.load()) return IVM_ENCCL;
  ivm_multi *mm = new ivm_multi;
  mm->ngpu = ngpu;
  mm->dev.assign(devices, devices + ngpu);
  mm->ctx.assign(ngpu, nullptr);
  mm->st.assign(ngpu, nullptr);
  mm->cst.assign(ngpu, nullptr);
  mm->ev.assign(ngpu, std::vector<cudaEvent_t>(kMultiChunks, nullptr));
  mm->sum.assign(ngpu, nullptr);
  mm->comm.assign(ngpu, nullptr);
  int r = IVM_OK;
  for (int g = 0; g < ngpu && r == IVM_OK; g++) {
    r = ivm_create(&mm->ctx[g], devices[g]);
    if (r != IVM_OK) break;
    if (cudaSetDevice(devices[g]) != cudaSuccess ||
        cudaStreamCreateWithFlags(&mm->st[g], cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&mm->cst[g], cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&mm->sum[g], 2 * sizeof(double)) != cudaSuccess)
      r = IVM_ECUDA;
    for (int k = 0; k < kMultiChunks && r == IVM_OK; k++)
      if (cudaEventCreateWithFlags(&mm->ev[g][k], cudaEventDisableTiming) != cudaSuccess) r = IVM_ECUDA;
  }
  if (r == IVM_OK && g_nccl.init(mm->comm.data(), ngpu, devices) != 0) r = IVM_ENCCL;
  if (r != IVM_OK) {
    ivm_multi_destroy(mm);
    return r;
  }
  *m = mm;
  return IVM_OK;
}

int ivm_multi_multiply(ivm_multi_t m, const uint8_t *const *a_shards, const uint8_t *const *b_shards, size_t n,
                       size_t batch_per_gpu, uint8_t *const *prod_shards, uint8_t *const *cert_shards, int prec,
                       int gather_to_root, uint8_t *root_prod, uint8_t *root_cert) {
  if (!m || !a_shards || !b_shards || !prod_shards || !cert_shards || n == 0 || batch_per_gpu == 0) return IVM_EINVAL;
  if (gather_to_root && (!root_prod || !root_cert)) return IVM_EINVAL;
  const int G = m->ngpu;
  const size_t bpg = batch_per_gpu;
  // without a gather the shard is one launch; with it, kMultiChunks chunks so
  // the gather of chunk k overlaps the multiplication of chunk k+1
  const int K = gather_to_root && bpg >= (size_t)kMultiChunks ? kMultiChunks : 1;
  for (int k = 0; k < K; k++) {
    const size_t p0 = bpg * k / K, cnt = bpg * (k + 1) / K - p0;
    for (int g = 0; g < G; g++) {  // independent shards: one batched multiply per device
      int r = ivm_multiply_batched(m->ctx[g], a_shards[g] + p0 * n, b_shards[g] + p0 * n, n, cnt,
                                   prod_shards[g] + p0 * 2 * n, cert_shards[g] + p0, prec, m->st[g]);
      if (r) return r;
      if (gather_to_root && (cudaSetDevice(m->dev[g]) != cudaSuccess ||
                             cudaEventRecord(m->ev[g][k], m->st[g]) != cudaSuccess ||
                             cudaStreamWaitEvent(m->cst[g], m->ev[g][k], 0) != cudaSuccess))
        return IVM_ECUDA;
    }
    if (!gather_to_root) continue;
    // chunk k of every shard to the root, in shard order, on the comm streams
    if (cudaSetDevice(m->dev[0]) != cudaSuccess ||
        cudaMemcpyAsync(root_prod + p0 * 2 * n, prod_shards[0] + p0 * 2 * n, cnt * 2 * n, cudaMemcpyDeviceToDevice,
                        m->cst[0]) != cudaSuccess ||
        cudaMemcpyAsync(root_cert + p0, cert_shards[0] + p0, cnt, cudaMemcpyDeviceToDevice, m->cst[0]) != cudaSuccess)
      return IVM_ECUDA;
    if (G > 1) {
      if (g_nccl.gstart() != 0) return IVM_ENCCL;
      for (int g = 1; g < G; g++) {
        const size_t q = g * bpg + p0;
        if (g_nccl.send(prod_shards[g] + p0 * 2 * n, cnt * 2 * n, ncclUint8, 0, m->comm[g], m->cst[g]) != 0 ||
            g_nccl.send(cert_shards[g] + p0, cnt, ncclUint8, 0, m->comm[g], m->cst[g]) != 0 ||
            g_nccl.recv(root_prod + q * 2 * n, cnt * 2 * n, ncclUint8, g, m->comm[0], m->cst[0]) != 0 ||
            g_nccl.recv(root_cert + q, cnt, ncclUint8, g, m->comm[0], m->cst[0]) != 0) {
          g_nccl.gend();
          return IVM_ENCCL;
        }
      }
      if (g_nccl.gend() != 0) return IVM_ENCCL;
    }
  }
  for (int g = 0; g < G; g++)
    if (cudaSetDevice(m->dev[g]) != cudaSuccess || cudaStreamSynchronize(m->st[g]) != cudaSuccess ||
        cudaStreamSynchronize(m->cst[g]) != cudaSuccess)
      return IVM_ECUDA;
  return IVM_OK;
}

int ivm_multi_summary(ivm_multi_t m, const uint8_t *const *cert_shards, const double *const *radius_shards,
                      size_t batch_per_gpu, uint64_t *certified_total, double *max_radius) {
  if (!m || !cert_shards || batch_per_gpu == 0 || batch_per_gpu > (size_t)0x7fffffff || !certified_total)
    return IVM_EINVAL;
  const int G = m->ngpu;
  for (int g = 0; g < G; g++) {
    if (cudaSetDevice(m->dev[g]) != cudaSuccess) return IVM_ECUDA;
    if (ivm::summary_launch(cert_shards[g], radius_shards ? radius_shards[g] : nullptr, (int)batch_per_gpu,
                            m->sum[g], m->st[g]) != 0)
      return IVM_ECUDA;
  }
  if (g_nccl.gstart() != 0) return IVM_ENCCL;
  for (int g = 0; g < G; g++)
    if (g_nccl.allreduce(m->sum[g], m->sum[g], 1, ncclFloat64, ncclSum, m->comm[g], m->st[g]) != 0 ||
        g_nccl.allreduce(m->sum[g] + 1, m->sum[g] + 1, 1, ncclFloat64, ncclMax, m->comm[g], m->st[g]) != 0) {
      g_nccl.gend();
      return IVM_ENCCL;
    }
  if (g_nccl.gend() != 0) return IVM_ENCCL;
  double h[2];
  if (cudaSetDevice(m->dev[0]) != cudaSuccess ||
      cudaMemcpyAsync(h, m->sum[0], sizeof(h), cudaMemcpyDeviceToHost, m->st[0]) != cudaSuccess)
    return IVM_ECUDA;
  for (int g = 0; g < G; g++)
    if (cudaSetDevice(m->dev[g]) != cudaSuccess || cudaStreamSynchronize(m->st[g]) != cudaSuccess) return IVM_ECUDA;
  *certified_total = (uint64_t)h[0];
  if (max_radius) *max_radius = radius_shards ? h[1] : NAN;
  return IVM_OK;
}

int ivm_multi_destroy(ivm_multi_t m) {
  if (!m) return IVM_OK;
  for (int g = 0; g < m->ngpu; g++) {
    if (m->comm[g]) g_nccl.destroy(m->comm[g]);
    cudaSetDevice(m->dev[g]);
    if (m->st[g]) cudaStreamDestroy(m->st[g]);
    if (m->cst[g]) cudaStreamDestroy(m->cst[g]);
    for (cudaEvent_t e : m->ev[g])
      if (e) cudaEventDestroy(e);
    cudaFree(m->sum[g]);
    ivm_destroy(m->ctx[g]);
  }
  delete m;
  return IVM_OK;
}

}  // extern "C"
