// ivm_multi.cpp -- single-process multi-GPU API (include/ivm.h, SURVEY §8(b),
// §8(e)): one context per device, the batch sharded by the caller (independent
// multiplications, no data-path collective), and an optional NCCL gather of the
// products and flags to the root device (grouped ncclSend / ncclRecv).
//
// NCCL is opened with dlopen("libnccl.so.2") on ivm_multi_create, so the
// library has no link-time NCCL dependency and a process that already loaded
// an NCCL (PyTorch's) shares it (same soname).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#include <vector>

#include "../../include/ivm.h"

namespace {

// the few NCCL entry points used (ABI of nccl.h, stable across 2.x)
typedef void *ncclComm_t;
typedef int ncclResult_t;
enum { ncclUint8 = 1 };
typedef ncclResult_t (*CommInitAll_t)(ncclComm_t *, int, const int *);
typedef ncclResult_t (*CommDestroy_t)(ncclComm_t);
typedef ncclResult_t (*Group_t)(void);
typedef ncclResult_t (*Send_t)(const void *, size_t, int, int, ncclComm_t, cudaStream_t);
typedef ncclResult_t (*Recv_t)(void *, size_t, int, int, ncclComm_t, cudaStream_t);

struct Nccl {
  void *h = nullptr;
  CommInitAll_t init = nullptr;
  CommDestroy_t destroy = nullptr;
  Group_t gstart = nullptr, gend = nullptr;
  Send_t send = nullptr;
  Recv_t recv = nullptr;
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
    return init && destroy && gstart && gend && send && recv;
  }
};
Nccl g_nccl;

}  // namespace

struct ivm_multi {
  int ngpu = 0;
  std::vector<int> dev;
  std::vector<ivm_ctx_t> ctx;
  std::vector<cudaStream_t> st;
  std::vector<ncclComm_t> comm;
};

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
  mm->comm.assign(ngpu, nullptr);
  int r = IVM_OK;
  for (int g = 0; g < ngpu && r == IVM_OK; g++) {
    r = ivm_create(&mm->ctx[g], devices[g]);
    if (r == IVM_OK && (cudaSetDevice(devices[g]) != cudaSuccess ||
                        cudaStreamCreateWithFlags(&mm->st[g], cudaStreamNonBlocking) != cudaSuccess))
      r = IVM_ECUDA;
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
  for (int g = 0; g < G; g++) {  // independent shards: one batched multiply per device
    int r = ivm_multiply_batched(m->ctx[g], a_shards[g], b_shards[g], n, batch_per_gpu, prod_shards[g],
                                 cert_shards[g], prec, m->st[g]);
    if (r) return r;
  }
  if (gather_to_root) {
    const size_t pb = 2 * n * batch_per_gpu;
    if (cudaSetDevice(m->dev[0]) != cudaSuccess ||
        cudaMemcpyAsync(root_prod, prod_shards[0], pb, cudaMemcpyDeviceToDevice, m->st[0]) != cudaSuccess ||
        cudaMemcpyAsync(root_cert, cert_shards[0], batch_per_gpu, cudaMemcpyDeviceToDevice, m->st[0]) != cudaSuccess)
      return IVM_ECUDA;
    if (G > 1) {
      if (g_nccl.gstart() != 0) return IVM_ENCCL;
      for (int g = 1; g < G; g++) {
        if (g_nccl.send(prod_shards[g], pb, ncclUint8, 0, m->comm[g], m->st[g]) != 0 ||
            g_nccl.send(cert_shards[g], batch_per_gpu, ncclUint8, 0, m->comm[g], m->st[g]) != 0 ||
            g_nccl.recv(root_prod + g * pb, pb, ncclUint8, g, m->comm[0], m->st[0]) != 0 ||
            g_nccl.recv(root_cert + g * batch_per_gpu, batch_per_gpu, ncclUint8, g, m->comm[0], m->st[0]) != 0) {
          g_nccl.gend();
          return IVM_ENCCL;
        }
      }
      if (g_nccl.gend() != 0) return IVM_ENCCL;
    }
  }
  for (int g = 0; g < G; g++)
    if (cudaSetDevice(m->dev[g]) != cudaSuccess || cudaStreamSynchronize(m->st[g]) != cudaSuccess) return IVM_ECUDA;
  return IVM_OK;
}

int ivm_multi_destroy(ivm_multi_t m) {
  if (!m) return IVM_OK;
  for (int g = 0; g < m->ngpu; g++) {
    if (m->comm[g]) g_nccl.destroy(m->comm[g]);
    if (m->st[g]) {
      cudaSetDevice(m->dev[g]);
      cudaStreamDestroy(m->st[g]);
    }
    ivm_destroy(m->ctx[g]);
  }
  delete m;
  return IVM_OK;
}

}  // extern "C"
