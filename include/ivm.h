/*
 * ivm.h -- C ABI of the B200-native certified interval-FFT multiplier.
 *
 * The operation is the paper's "rigorous extension of the Schoenhage-Strassen
 * algorithm" (arXiv 1006.0405, /root/reference/PAPER.md, cited P:<line>):
 *   input  x, y in Z_b^n, b = 256,
 *   output z in Z_b^{2n} with z = x*y,
 * computed as: zero-pad to m = 2^k, k = ceil(log2(2n-1)),
 * forward FFT of both, pointwise product,
 * inverse FFT, all on rectangular complex interval
 * containment sets with directed rounding; then each coefficient
 * interval must contain exactly one integer -- "choose the unique integer in
 * the containment set ... if [it] contains multiple integers, then we report
 * an error" -- and the certified coefficients are carried back to
 * base 256.  A product is returned only when certified; an
 * uncertified pair is not an error of the call: its flag is 0 and its digits
 * are zero ("increase the precision ... or use a different algorithm").
 *
 * Conventions for every entry point:
 *   - digits are base 256, little-endian (digit i has weight 256^i), uint8;
 *     both operands have the same length n >= 1 (the caller zero-pads the
 *     shorter one); the product has exactly 2n digits (z_{2n-1} is the final
 *     carry) and is not canonicalised;
 *   - batched arrays are row-major: a, b = [batch][n], prod = [batch][2n],
 *     certified = [batch] (1 = certified, 0 = needs more precision);
 *   - pointers passed to ivm_multiply* are DEVICE pointers on the context's
 *     device; the caller allocates and owns them (the context owns only its
 *     twiddle tables and scratch);
 *   - calls are asynchronous on `cuda_stream` (a cudaStream_t, NULL = legacy
 *     default stream); outputs are valid after the stream is synchronised;
 *   - precision: IVM_F64 = binary64 intervals (P:5), IVM_F32 = binary32
 *     (P:22);
 *   - errors: argument errors (n == 0, batch == 0, NULL required pointer,
 *     unknown precision, n beyond the supported maximum) return before any
 *     launch and write nothing; CUDA failures return IVM_ECUDA and are
 *     sticky for the context;
 *   - determinism: identical inputs give bitwise identical outputs;
 *   - thread safety: one host thread per context at a time;
 *   - streams: every call on a context uses the context's scratch buffers,
 *     so calls on one context are ordered even across streams: a call on a
 *     different stream than the previous call's first makes its stream wait
 *     for the previous call's work (cudaStreamWaitEvent on an event the
 *     previous call recorded).  Calls on distinct contexts run concurrently.
 */
#ifndef IVM_H
#define IVM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ivm_ctx *ivm_ctx_t;
typedef struct ivm_multi *ivm_multi_t;  /* G device contexts + NCCL communicators */

enum { IVM_F64 = 0, IVM_F32 = 1 };

enum {
    IVM_OK = 0,
    IVM_EINVAL = -1,        /* bad argument */
    IVM_ENOMEM = -2,        /* device or host allocation failed */
    IVM_ECUDA = -3,         /* CUDA runtime / launch error (sticky) */
    IVM_EUNSUPPORTED = -4,  /* size / precision not supported by this build */
    IVM_ENCCL = -5,         /* NCCL missing or failed (multi-GPU API) */
    IVM_ENODEV = -6         /* no CUDA device */
};

/* Version string of the library ("ivm <semver> sm_100a"). */
const char *ivm_version(void);

/* Human-readable text of a status code. */
const char *ivm_strerror(int status);

/* Largest supported operand length n for a precision (0 if none). */
size_t ivm_max_digits(int prec);

/* FFT length m = 2^ceil(log2(2n-1)) used for operands of n digits. */
size_t ivm_fft_length(size_t n);

/* Create a context on CUDA device `device` (selects it on the calling
 * thread).  *ctx is set on success. */
int ivm_create(ivm_ctx_t *ctx, int device);

/* Destroy a context; frees tables and scratch.  NULL is a no-op. */
int ivm_destroy(ivm_ctx_t ctx);

/* Optional: build the twiddle table for (n, prec) and size the scratch for
 * `batch` so that the first multiply does no allocation. */
int ivm_reserve(ivm_ctx_t ctx, size_t n, size_t batch, int prec);

/* One multiplication (the paper's problem):
 * a, b: [n] device digits; prod: [2n] device digits; certified: 1 device byte. */
int ivm_multiply(ivm_ctx_t ctx, const uint8_t *a, const uint8_t *b, size_t n,
                 uint8_t *prod, uint8_t *certified, int prec, void *cuda_stream);

/* Batched independent multiplications: a, b [batch][n], prod [batch][2n],
 * certified [batch] (all device pointers).  Any alignment and any n are
 * accepted and give the same results; rows that are 16-byte aligned (a, b
 * 16-byte aligned and n a multiple of 16) take the staged-digit kernels
 * (bulk copies into shared memory one pair ahead), the fastest path. */
int ivm_multiply_batched(ivm_ctx_t ctx, const uint8_t *a, const uint8_t *b, size_t n,
                         size_t batch, uint8_t *prod, uint8_t *certified, int prec,
                         void *cuda_stream);

/* Diagnostics for parity tests; every output is nullable (device pointers):
 *   max_radius [batch]   : max over coefficients i < 2n-1 of (hi-lo)/2 of the
 *                          real and imaginary parts (binary64, rounded up);
 *   first_bad  [batch]   : smallest i < 2n-1 whose interval does not certify,
 *                          -1 if certified;
 *   coeffs [batch][2n-1] : the snapped integer coefficients c_i (valid where
 *                          the pair is certified);
 *   dump_pairs [n_dump]  : pair indices whose final coefficient intervals are
 *                          written to intervals [n_dump][m][4] as binary64
 *                          (re.lo, re.hi, im.lo, im.hi), m = ivm_fft_length(n).
 *                          The odd-frequency kernels (binary64 with m >= 64,
 *                          binary32 with m >= 1024) compute each coefficient
 *                          as a real interval: their im.lo / im.hi are NaN. */
int ivm_multiply_batched_diag(ivm_ctx_t ctx, const uint8_t *a, const uint8_t *b, size_t n,
                              size_t batch, uint8_t *prod, uint8_t *certified, int prec,
                              void *cuda_stream, double *max_radius, int32_t *first_bad,
                              int64_t *coeffs, const int32_t *dump_pairs, size_t n_dump,
                              double *intervals);

/* Host-pointer convenience (end-to-end path): copies a, b (host, [batch][n])
 * to the device, multiplies, and copies prod / certified back to host
 * buffers; returns after `cuda_stream` is synchronised.  The batch is cut into
 * at most 8 chunks of whole waves (multiples of the SM count): chunk i's
 * kernel runs on `cuda_stream` while chunk i+1 is copied in and chunk i-1
 * copied out on two context-owned streams (event-ordered; work queued on
 * `cuda_stream` before the call is waited for).  Host buffers should be
 * pinned for the copies to overlap.  Uses context-owned device staging
 * buffers (2 n batch + 2 n batch + batch bytes). */
int ivm_multiply_batched_host(ivm_ctx_t ctx, const uint8_t *a, const uint8_t *b, size_t n,
                              size_t batch, uint8_t *prod, uint8_t *certified, int prec,
                              void *cuda_stream);

/* Exact long multiplication on the device (the paper's
 * guaranteed-correct comparator): prod[p] = a[p] * b[p] exactly, no FFT
 * and no rounding.  a, b: device [batch][n] digits (least significant first);
 * prod: device [batch][2n].  The sums s_k = sum_{i+j=k} a_i b_j are formed
 * exactly (byte dot products, 64-bit accumulation) in context-owned device
 * scratch (<= 256 MiB per launch, pairs chunked), then carried.
 * Requires n <= 2^18 (IVM_EUNSUPPORTED otherwise).  Asynchronous on
 * `cuda_stream`. */
int ivm_long_multiply_batched(ivm_ctx_t ctx, const uint8_t *a, const uint8_t *b, size_t n,
                              size_t batch, uint8_t *prod, void *cuda_stream);

/* Exact products with the paper's escalation (when an error is
 * detected, "increase the precision being used or ... use a different
 * algorithm").  policy 0 (the paper's order): the fp32 interval FFT when
 * n <= 32, else the fp64 one; the fp64 interval FFT for the pairs fp32 did not
 * certify; exact long multiplication for the pairs fp64 did not certify (and
 * for n > ivm_max_digits(IVM_F64)).  policy 1 (fastest exact): long
 * multiplication when the FFT length is below 64 (n <= 16, where it is faster
 * on B200), else fp64 then long multiplication.
 * prod: device [batch][2n], always the exact product.  method: device
 * [batch] or NULL; receives 1 (fp32 interval), 2 (fp64 interval) or 3 (long
 * multiplication) per pair.  Synchronises `cuda_stream` (the uncertified
 * counts size the later tiers).  Uses context-owned device scratch.
 * IVM_EINVAL for a bad policy. */
int ivm_multiply_exact(ivm_ctx_t ctx, const uint8_t *a, const uint8_t *b, size_t n, size_t batch,
                       uint8_t *prod, uint8_t *method, int policy, void *cuda_stream);

/* The paper's naive fixed-precision SS: the same FFT
 * multiplication with punctual complex numbers, round-to-nearest arithmetic
 * and twiddles, coefficients rounded to the nearest integer.  NOT guaranteed
 * to be correct -- a speed and error-rate comparator for the certified
 * path.  a, b: device [batch][n]; prod: device [batch][2n].  prec IVM_F64 or
 * IVM_F32; n <= 4096 (IVM_EUNSUPPORTED otherwise).  Asynchronous on
 * `cuda_stream`. */
int ivm_multiply_naive(ivm_ctx_t ctx, const uint8_t *a, const uint8_t *b, size_t n, size_t batch,
                       uint8_t *prod, int prec, void *cuda_stream);

/* Circular containment sets (the paper's suggested future work;
 * SURVEY §8(f) rank 4): the same multiplication (radix-2 DIT FFT P:143-155,
 * pointwise product P:210, inverse P:97/P:211, unique-integer rule P:24, carry
 * P:229-235) with every complex value a disc <c, r> = {z : |z - c| <= r}:
 * round-to-nearest centers, round-up radius bounds (reading R15).
 * fp64.  a, b: device [batch][n]; prod: device [batch][2n] (zero digits where
 * not certified); cert: device [batch] (1 = proved exact); max_radius:
 * device [batch] largest disc radius over the 2n-1 used coefficients, or NULL.
 * n <= ivm_max_digits(IVM_F64) (m <= 2^18; IVM_EUNSUPPORTED otherwise).
 * Kernels: for m >= 2^10 the odd-frequency radix-8 schedules of
 * ivm_multiply_batched (one CTA, a thread-block cluster, or pipelined CTA
 * groups per multiplication) with a disc as the element (fastest with aligned
 * digit rows: a, b and n multiples of 16 bytes); below, and everywhere under
 * IVM_DISC3=0, the radix-2 DIT (one CTA for m <= 8192, else a group of m/8192
 * co-resident CTAs, the DIT factored as 8192 x m/8192 through device scratch).
 * Same results contract either way (certified => exact; the radii differ
 * within a small factor).  Asynchronous on `cuda_stream`; uses
 * context-owned device scratch. */
int ivm_multiply_disc(ivm_ctx_t ctx, const uint8_t *a, const uint8_t *b, size_t n, size_t batch,
                      uint8_t *prod, uint8_t *cert, double *max_radius, void *cuda_stream);

/* Single-process multi-GPU: one context per device plus NCCL
 * communicators (ncclCommInitAll; NCCL is dlopen'ed, "libnccl.so.2").
 * devices: [ngpu] CUDA ordinals, devices[0] is the root.  IVM_ENCCL if NCCL
 * cannot be loaded or initialised.  (One process per GPU under
 * torch.distributed is the other supported launch model: bench.py.) */
int ivm_multi_create(ivm_multi_t *m, int ngpu, const int *devices);

/* Independent multiplications sharded by the caller: shard g (device
 * devices[g]) multiplies a_shards[g], b_shards[g] ([batch_per_gpu][n], device
 * memory of that GPU) into prod_shards[g] ([batch_per_gpu][2n]) and
 * cert_shards[g] ([batch_per_gpu]); no data-path collective.  If
 * gather_to_root, the products and flags are gathered in shard order into
 * root_prod ([ngpu * batch_per_gpu][2n]) and root_cert ([ngpu *
 * batch_per_gpu]) on the root device (grouped ncclSend / ncclRecv).  The
 * gather is pipelined: each shard runs as 4 chunks, and chunk k's sends run on
 * a communication stream while chunk k+1 multiplies.  Returns after every
 * device's work (and the gather) completed. */
int ivm_multi_multiply(ivm_multi_t m, const uint8_t *const *a_shards, const uint8_t *const *b_shards,
                       size_t n, size_t batch_per_gpu, uint8_t *const *prod_shards,
                       uint8_t *const *cert_shards, int prec, int gather_to_root, uint8_t *root_prod,
                       uint8_t *root_cert);

/* The step summary over all devices: *certified_total = the
 * number of nonzero flags in cert_shards[g][0 .. batch_per_gpu) summed over
 * the devices, *max_radius = the largest radius_shards[g][i] (device arrays,
 * e.g. ivm_multiply_batched_diag's max_radius; NaN counts as +inf), or NaN if
 * radius_shards is NULL (max_radius nullable).  A per-device reduction kernel,
 * then ncclAllReduce (SUM, MAX) across the devices; synchronous. */
int ivm_multi_summary(ivm_multi_t m, const uint8_t *const *cert_shards, const double *const *radius_shards,
                      size_t batch_per_gpu, uint64_t *certified_total, double *max_radius);

/* Destroy the communicators and contexts; NULL is a no-op. */
int ivm_multi_destroy(ivm_multi_t m);

/* Seeded synthetic digits on the device (the counter-based SplitMix64
 * generator of SURVEY.md §8(d.2); same bits as
 * paper_1006_0405_b200/inputs.py).  kind: 0 uniform, 1 all-255, 2 sparse
 * (90 % zeros), 3 uniform with nonzero most significant digit; kinds: NULL
 * (use `kind` for all pairs) or [batch] device bytes.  Writes [batch][n]
 * digits of operand `operand` (0 = a, 1 = b) for pairs pair0 .. pair0+batch-1. */
int ivm_generate_digits(ivm_ctx_t ctx, uint8_t *out, size_t n, size_t batch, uint64_t seed,
                        uint64_t pair0, int operand, int kind, const uint8_t *kinds,
                        void *cuda_stream);

/* Directed-rounding FP64 / FP32 throughput probe: runs `iters` dependent
 * chains of DFMA.RP / FFMA.RP on every SM; writes the number of executed
 * FMA instructions (thread level) to *fma_count (host).  The caller times
 * the call with events on `cuda_stream`.  sink: device buffer of
 * >= 148*1024 doubles. */
int ivm_peak_probe(ivm_ctx_t ctx, int prec, int iters, double *sink, uint64_t *fma_count,
                   void *cuda_stream);

/* Number of kernels launched by the last ivm_multiply* call on this context. */
int ivm_last_launch_count(ivm_ctx_t ctx);

/* Host-side copy of the twiddle table the kernels use for m = 2^log2m:
 * out = [m][4] (re.lo, re.hi, im.lo, im.hi) of omega_m^j = e^{2 pi i j/m}
 * (P:68), the optimal enclosures [RD, RU] of cos and sin; out is double[m][4]
 * for IVM_F64 and float[m][4] for IVM_F32 (host memory, caller-owned).
 * Returns IVM_EUNSUPPORTED if an entry cannot be rounded rigorously.
 * Needs no device. */
int ivm_twiddle_table(int log2m, int prec, void *out);

#ifdef __cplusplus
}
#endif

#endif /* IVM_H */
