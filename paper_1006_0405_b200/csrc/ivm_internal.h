// ivm_internal.h -- declarations shared by ivm_api.cu and ivm_kernels.cu.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace ivm {

struct KParams {
  const uint8_t *a, *b;
  uint8_t *prod, *cert;
  int n, batch;
  const void *tw;            // CI<T>[m]: omega_m^j
  void *ascratch;            // [gridDim.x][2][m/2+1] split re/im when A is not in SMEM
  double *max_radius;        // [batch] nullable
  int32_t *first_bad;        // [batch] nullable
  int64_t *coeffs;           // [batch][2n-1] nullable
  const int32_t *dump_slot;  // [batch] slot or -1 (nullable)
  double *intervals;         // [n_dump][m][4]
  unsigned long long *phases;  // [grid][16] SM cycles per phase (-DIVM_PHASES experiment builds only)
};

struct LaunchInfo {
  int threads;
  size_t smem;
  bool a_smem;
  size_t a_bytes_per_cta;
  int blocks_per_sm;
  int cluster = 1;       // CTAs per multiplication (v4)
  int max_clusters = 0;  // co-resident clusters (v4)
};

int upload_w32(const double *w64, const float *w32);
int cta_info(int prec, int m, LaunchInfo *li);
int cta_launch(int prec, int m, const KParams &kp, int grid, cudaStream_t s);
int n1_launch(const KParams &kp, cudaStream_t s);
int digits_launch(uint8_t *out, int n, long long batch, uint64_t seed, uint64_t pair0, int operand,
                  int kind, const uint8_t *kinds, int sms, cudaStream_t s);
int probe_launch(int prec, int iters, void *sink, int sms, cudaStream_t s, uint64_t *count);
int dump_map_launch(int32_t *slot, int batch, const int32_t *pairs, int n_dump, cudaStream_t s);
int plan_twiddles(int m, int prec, void *out);
int plan_twiddles_rn(int m, int prec, void *out);
// v3 (odd-frequency, balanced) path
int upload_w64(const double *w64, const float *w32);
int v3_table_entries(int m, int radix);
int v3_tables(int m, int prec, int radix, const void *w2N, void *out);
int v3_info(int prec, int m, int radix, LaunchInfo *li);
int v3_launch(int prec, int m, int radix, const KParams &kp, int grid, cudaStream_t s);
// small m (2^6 .. 2^9): 8192/m multiplications per 512-thread CTA
int v6_info(int prec, int m, LaunchInfo *li);
int v6_launch(int prec, int m, const KParams &kp, int grid, cudaStream_t s);
// circular containment sets on the one-CTA radix-8 schedule: m = 2^10 .. 2^13 (fp64)
int d3_info(int m, LaunchInfo *li);
int d3_launch(int m, const KParams &kp, int grid, cudaStream_t s);
// ... and on the cluster schedule: m = 2^14 .. 2^16 (fp64, 16-byte aligned digit rows)
int d4_info(int m, LaunchInfo *li);
int d4_launch(int m, const KParams &kp, int clusters, cudaStream_t s);
// m = 2^14 .. 2^16: one thread-block cluster of m/8192 CTAs per multiplication
int upload_w64_v4(const double *w64, const float *w32);
int v4_table_entries(int m);
int v4_tables(int m, int prec, const void *w2N, void *out);
int v4_info(int prec, int m, LaunchInfo *li);
int v4_launch(int prec, int m, const KParams &kp, int clusters, cudaStream_t s);
// m = 2^17, 2^18: co-resident groups of m/8192 CTAs exchanging through L2 scratch
struct Group5Args {
  unsigned *ctr;   // [groups], zeroed before every launch
  void *xch;       // [groups][C][4096] complex intervals
  unsigned *link;  // [groups][C][8]
  long long *bnd;  // [groups][2 C^2][8]
  uint8_t *bits;   // [groups][2 C^2]
};
int upload_w64_v5(const double *w64, const float *w32);
int v5_info(int prec, int m, LaunchInfo *li);
int v5_launch(int prec, int m, const KParams &kp, const Group5Args &ga, int groups, cudaStream_t s, bool coop);
// m = 2^17, 2^18, fp64: the pipelined group kernel (ivm_v7.cuh): a persistent
// grid of one CTA per SM dealing the batch's batch x C tasks; per-pair scratch in
// a ring of rp pairs (v7_ring)
struct Pipe7Args {
  unsigned *cnt;     // [batch][4], zeroed before every launch
  void *xch;         // [rp][C][4096] complex intervals
  uint4 *wds;        // [rp][C][512]
  uint2 *rec;        // [rp][2 C^2]
  unsigned *link;    // [rp][C][8]
  int rp;
};
int v7_info(int m, LaunchInfo *li);
int v7_launch(int m, const KParams &kp, const Pipe7Args &pa, int grid, cudaStream_t s);
// circular containment sets on the same pipeline (ivm_d7.cuh; word-aligned digit rows)
int d7_info(int m, LaunchInfo *li);
int d7_launch(int m, const KParams &kp, const Pipe7Args &pa, int grid, cudaStream_t s);

// batch summary {certified count, max radius} into out[2] (device), zeroed first
int summary_launch(const uint8_t *cert, const double *rad, int batch, double *out, cudaStream_t s);
// circular containment sets, m = 2^14 .. 2^18: groups of m/8192 CTAs
int disc_group_blocks_per_sm();
size_t disc_group_scratch(int lg, size_t groups);
int disc_group_launch(const uint8_t *a, const uint8_t *b, int n, int batch, int lg, const void *tw, double rw,
                      void *scratch, size_t groups, uint8_t *prod, uint8_t *cert, double *max_radius, cudaStream_t s);
// circular containment sets, m <= 8192
int disc_smem(int lg);
int disc_launch(const uint8_t *a, const uint8_t *b, int n, int batch, int lg, const void *tw, double rw,
                void *scratch, uint8_t *prod, uint8_t *cert, double *max_radius, int grid, cudaStream_t s);
// the naive (punctual, round-to-nearest) SS comparator
int naive_smem(int lg, int prec);
int naive_launch(int prec, const uint8_t *a, const uint8_t *b, int n, int batch, int lg, const void *w, void *scratch,
                 uint8_t *prod, int grid, cudaStream_t s);
// exact long multiplication and the precision escalation helpers
int long_launch(const uint8_t *a, const uint8_t *b, int n, int batch, long long *coef, uint8_t *prod,
                cudaStream_t s);
int esc_mark(const uint8_t *cert, const int *map, int count, int tier, uint8_t *method, int *idx, int *nidx,
             cudaStream_t s);
int esc_set_method(const int *map, int count, int tier, uint8_t *method, cudaStream_t s);
int esc_gather(const uint8_t *src, size_t len, const int *idx, int count, uint8_t *dst, cudaStream_t s);
int esc_scatter(const uint8_t *src, size_t len, const int *idx, const uint8_t *ok, int count, uint8_t *dst,
                cudaStream_t s);

}  // namespace ivm
