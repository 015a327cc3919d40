/*
 * ivm_oracle.c -- CPU ORACLE for the certified interval-FFT multiplication.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1006_0405_b200/csrc); neither side includes or links the other.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, cited as P:<line>):
 *   - long multiplication, literally P:44-56 (§2.1), and the exact
 *     coefficient sums z_i = sum_j x_j y_{i-j} of P:37;
 *   - the paper's interval Schoenhage-Strassen multiply (§2.3-§2.5):
 *       fast convolution P:203-211 with the recursive Cooley-Tukey FFT
 *       P:143-155, every complex operation on rectangular complex
 *       intervals P:261-265 built from the real interval operations
 *       P:250-253, with directed rounding;
 *       inverse DFT P:97: the same FFT with omega^-1, then 1/n;
 *       the "unique integer in the containment set" rule P:24/P:247;
 *       the carry loop P:229-235.
 *
 * Directed rounding: every worker thread calls fesetround(FE_UPWARD) once;
 * RU(x op y) is the plain C operation, RD(x op y) = -RU(-x op' y) (exact
 * negation).  Compiled with -frounding-math -ffp-contract=off, no fast-math.
 * A self-check at every entry point verifies lo < hi for 1/3 and 0.1+0.2 and
 * aborts otherwise (catches code motion across fesetround).
 *
 * Twiddles omega_N^j = e^{2 pi i j/N} are INPUTS: the optimal enclosures
 * [RD(cos), RU(cos)] + i[RD(sin), RU(sin)] are computed by oracle/twiddles.py
 * from mpmath (reading R2: the paper's recurrence P:163 is replaced
 * by "other efficient methods" P:164).
 *
 * Interval vectors are arrays of T[4] = (re.lo, re.hi, im.lo, im.hi).
 * T = double (binary64) or float (binary32); the code below is written once
 * as a macro template and instantiated for both (P:22 binary32, P:5 binary64).
 */
#include <fenv.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#pragma STDC FENV_ACCESS ON

/* ------------------------------------------------------------------ */
/* rounding-mode discipline                                             */
/* ------------------------------------------------------------------ */

static int set_upward(void) { return fesetround(FE_UPWARD); }

/* volatile operands defeat constant folding of the self-check */
static int rounding_self_check(void) {
    volatile double one = 1.0, three = 3.0, p1 = 0.1, p2 = 0.2;
    volatile float onef = 1.0f, threef = 3.0f;
    double hi = one / three, lo = -((-one) / three);
    double shi = p1 + p2, slo = -((-p1) + (-p2));
    float hif = onef / threef, lof = -((-onef) / threef);
    if (!(lo < hi) || !(slo < shi) || !(lof < hif)) return -1;
    return 0;
}

static void enter(void) {
    if (set_upward() != 0 || rounding_self_check() != 0) {
        fprintf(stderr, "ivm_oracle: directed rounding unavailable, aborting\n");
        abort();
    }
}

int oracle_self_check(void) {
    int old = fegetround();
    set_upward();
    int r = rounding_self_check();
    fesetround(old);
    return r;
}

/* ------------------------------------------------------------------ */
/* §2.1 long multiplication and the coefficient sums   */
/* ------------------------------------------------------------------ */

/* P:44-56 literally: z in Z_b^{n+m}, b = 256. */
void oracle_long_multiply(const uint8_t *x, size_t n, const uint8_t *y, size_t m, uint8_t *z) {
    uint64_t c = 0;                                           /* 3. carry */
    for (size_t i = 0; i < n + m; i++) {                      /* 4. */
        uint64_t s = 0;                                       /* 5. */
        size_t jlo = (i + 1 > m) ? i + 1 - m : 0;             /* max{0, i-m+1} */
        size_t jhi = (i < n - 1) ? i : n - 1;                 /* min{n-1, i} */
        for (size_t j = jlo; j <= jhi && j < n; j++)          /* 6. */
            s += (uint64_t)x[j] * (uint64_t)y[i - j];         /* 7. */
        z[i] = (uint8_t)((s + c) % 256u);                     /* 9. */
        c = (s + c) / 256u;                                   /* 10. */
    }
}

/* z_i = sum_{j=max(0,i-m+1)}^{min(n-1,i)} x_j y_{i-j}, i < n+m-1 */
void oracle_coefficients(const uint8_t *x, size_t n, const uint8_t *y, size_t m, int64_t *z) {
    for (size_t i = 0; i + 1 < n + m; i++) {
        uint64_t s = 0;
        size_t jlo = (i + 1 > m) ? i + 1 - m : 0;
        size_t jhi = (i < n - 1) ? i : n - 1;
        for (size_t j = jlo; j <= jhi; j++) s += (uint64_t)x[j] * (uint64_t)y[i - j];
        z[i] = (int64_t)s;
    }
}

/* carry the 2n-1 coefficients into 2n base-256 digits. */
void oracle_carry(const int64_t *v, size_t n, uint8_t *z) {
    uint64_t c = 0;
    for (size_t i = 0; i + 1 < 2 * n; i++) {                  /* 5. i = 0 .. 2n-2 */
        uint64_t t = (uint64_t)v[i] + c;
        z[i] = (uint8_t)(t % 256u);                           /* 6. */
        c = t / 256u;                                         /* 7. */
    }
    z[2 * n - 1] = (uint8_t)c;                                /* 9. z_{2n-1} = c */
}

/* ------------------------------------------------------------------ */
/* P:24 / P:247 round-and-certify and the radius (one definition each)  */
/* ------------------------------------------------------------------ */

/* P:24 "choose the unique integer in the containment set; if there are
 * multiple, report an error" with DESIGN.md R8/R18: the real part [lo, hi]
 * holds exactly one integer iff ceil(lo) == floor(hi); the imaginary part
 * must hold only 0.  NaN never certifies (comparisons fail).
 * Intervals are [len][4] binary64 (re.lo, re.hi, im.lo, im.hi).  Writes the
 * unique integers to coeff (nullable; 0 where not certified) and returns the
 * first failing index, or -1 if every entry certifies. */
int32_t oracle_certify_span(const double *iv, size_t len, int64_t *coeff) {
    int32_t bad = -1;
    for (size_t i = 0; i < len; i++) {
        double cl = ceil(iv[4 * i]), fh = floor(iv[4 * i + 1]);
        double il = ceil(iv[4 * i + 2]), ih = floor(iv[4 * i + 3]);
        int unique = (cl == fh) && (il == 0.0) && (ih == 0.0);
        if (coeff) coeff[i] = unique ? (int64_t)cl : 0;
        if (!unique && bad < 0) bad = (int32_t)i;
    }
    return bad;
}

/* DESIGN.md R10: the radius of an interval is (hi - lo)/2, here rounded up
 * (the caller is in FE_UPWARD; the halving is exact), NaN counted as +inf;
 * the max is taken over both parts of every entry of [len][4]. */
static double max_radius_span(const double *iv, size_t len) {
    double rad = 0.0;
    for (size_t i = 0; i < 2 * len; i++) {
        double r = (iv[2 * i + 1] - iv[2 * i]) / 2.0;
        if (r != r) r = INFINITY;
        if (r > rad) rad = r;
    }
    return rad;
}

/* ------------------------------------------------------------------ */
/* §2.5 interval arithmetic, instantiated for T = double and T = float  */
/* ------------------------------------------------------------------ */

#define DEFINE_INTERVAL(T, S)                                                  \
typedef struct { T lo, hi; } iv_##S;                                           \
typedef struct { iv_##S re, im; } civ_##S;                                     \
                                                                               \
/* rounding mode is FE_UPWARD: RU is the plain op, RD negates */               \
static T ru_add_##S(T a, T b) { return a + b; }                                \
static T rd_add_##S(T a, T b) { return -((-a) + (-b)); }                       \
static T ru_sub_##S(T a, T b) { return a - b; }                                \
static T rd_sub_##S(T a, T b) { return -((-a) + b); }                          \
static T ru_mul_##S(T a, T b) { return a * b; }                                \
static T rd_mul_##S(T a, T b) { return -((-a) * b); }                          \
static T ru_div_##S(T a, T b) { return a / b; }                                \
static T rd_div_##S(T a, T b) { return -((-a) / b); }                          \
                                                                               \
/* P:251 */                                                                    \
static iv_##S iadd_##S(iv_##S a, iv_##S b) {                                   \
    iv_##S r = { rd_add_##S(a.lo, b.lo), ru_add_##S(a.hi, b.hi) }; return r; } \
/* P:252 */                                                                    \
static iv_##S isub_##S(iv_##S a, iv_##S b) {                                   \
    iv_##S r = { rd_sub_##S(a.lo, b.hi), ru_sub_##S(a.hi, b.lo) }; return r; } \
/* min / max over the four endpoint products, each product rounded  */  \
/* down for the min and up for the max. */                                     \
static iv_##S imul_##S(iv_##S a, iv_##S b) {                                   \
    T l1 = rd_mul_##S(a.lo, b.lo), l2 = rd_mul_##S(a.lo, b.hi);                \
    T l3 = rd_mul_##S(a.hi, b.lo), l4 = rd_mul_##S(a.hi, b.hi);                \
    T h1 = ru_mul_##S(a.lo, b.lo), h2 = ru_mul_##S(a.lo, b.hi);                \
    T h3 = ru_mul_##S(a.hi, b.lo), h4 = ru_mul_##S(a.hi, b.hi);                \
    T lo = l1; if (l2 < lo) lo = l2; if (l3 < lo) lo = l3; if (l4 < lo) lo = l4; \
    T hi = h1; if (h2 > hi) hi = h2; if (h3 > hi) hi = h3; if (h4 > hi) hi = h4; \
    /* NaN propagates: a comparison with NaN is false, keep NaN visible */     \
    if (l1 != l1 || l2 != l2 || l3 != l3 || l4 != l4) lo = l1 + l2 + l3 + l4;  \
    if (h1 != h1 || h2 != h2 || h3 != h3 || h4 != h4) hi = h1 + h2 + h3 + h4;  \
    iv_##S r = { lo, hi }; return r; }                                         \
/* P:264 division by a positive integer k */                                   \
static iv_##S idivk_##S(iv_##S a, T k) {                                       \
    iv_##S r = { rd_div_##S(a.lo, k), ru_div_##S(a.hi, k) }; return r; }       \
                                                                               \
/* P:264 */                                                                    \
static civ_##S cadd_##S(civ_##S z, civ_##S w) {                                \
    civ_##S r = { iadd_##S(z.re, w.re), iadd_##S(z.im, w.im) }; return r; }    \
static civ_##S csub_##S(civ_##S z, civ_##S w) {                                \
    civ_##S r = { isub_##S(z.re, w.re), isub_##S(z.im, w.im) }; return r; }    \
/* P:265 */                                                                    \
static civ_##S cmul_##S(civ_##S z, civ_##S w) {                                \
    civ_##S r;                                                                 \
    r.re = isub_##S(imul_##S(z.re, w.re), imul_##S(z.im, w.im));               \
    r.im = iadd_##S(imul_##S(z.re, w.im), imul_##S(z.im, w.re));               \
    return r; }                                                                \
static civ_##S cdivk_##S(civ_##S z, T k) {                                     \
    civ_##S r = { idivk_##S(z.re, k), idivk_##S(z.im, k) }; return r; }        \
static civ_##S cconj_##S(civ_##S z) {                                          \
    civ_##S r = { z.re, { -z.im.hi, -z.im.lo } }; return r; }                  \
                                                                               \
static civ_##S load_##S(const T *p) {                                          \
    civ_##S r = { { p[0], p[1] }, { p[2], p[3] } }; return r; }                \
static void store_##S(T *p, civ_##S z) {                                       \
    p[0] = z.re.lo; p[1] = z.re.hi; p[2] = z.im.lo; p[3] = z.im.hi; }          \
                                                                               \
/* P:143-155 The Cooley-Tukey FFT, recursive, literally.                    */ \
/*   x: n = 2^k complex intervals.  tw: omega_N^j, j < N (N >= n), so the   */ \
/*   n-th root omega = e^{2 pi i/n} has powers omega^i = tw[i * N/n].        */ \
/*   inverse != 0 uses omega^-1 = conj; the 1/n is applied by caller. */ \
static void fft_rec_##S(int k, const civ_##S *x, civ_##S *out,                 \
                        const civ_##S *tw, size_t N, int inverse) {            \
    size_t n = (size_t)1 << k;                                                 \
    if (k == 0) { out[0] = x[0]; return; }                       /* 4. */      \
    size_t h = n / 2;                                                          \
    civ_##S *buf = (civ_##S *)malloc(sizeof(civ_##S) * 2 * n);                 \
    civ_##S *xe = buf, *xo = buf + h, *Xe = buf + n, *Xo = buf + n + h;        \
    for (size_t i = 0; i < h; i++) { xe[i] = x[2 * i]; xo[i] = x[2 * i + 1]; } /* 5. */ \
    fft_rec_##S(k - 1, xe, Xe, tw, N, inverse);                  /* 6. */      \
    fft_rec_##S(k - 1, xo, Xo, tw, N, inverse);                  /* 7. */      \
    size_t stride = N / n;                                       /* 8. */      \
    for (size_t i = 0; i < n; i++) {                             /* 9. */      \
        civ_##S w = tw[i * stride];                                            \
        if (inverse) w = cconj_##S(w);                                         \
        out[i] = cadd_##S(Xe[i % h], cmul_##S(w, Xo[i % h]));    /* 10. */     \
    }                                                                          \
    free(buf);                                                                 \
}                                                                              \
                                                                               \
/* One multiplication, §2.4 + §2.3 with containment sets (§2.5).           */  \
/* Returns the certified flag; fills prod (2n digits, zero if not certified), */ \
/* coeff (2n-1 snapped coefficients, valid if certified), the max radius over */ \
/* the used coefficients (real and imag), the first failing index (-1), and   */ \
/* optionally the N output intervals. */                                       \
static int ss_multiply_##S(const uint8_t *a, const uint8_t *b, size_t n,       \
                           const T *twraw, size_t N, uint8_t *prod,            \
                           int64_t *coeff, double *maxrad, int32_t *first_bad, \
                           T *intervals_out) {                                 \
    int k = 0; while (((size_t)1 << k) < N) k++;                               \
    const civ_##S *tw = (const civ_##S *)twraw;                                \
    civ_##S *ap = (civ_##S *)calloc(N, sizeof(civ_##S));                       \
    civ_##S *bp = (civ_##S *)calloc(N, sizeof(civ_##S));                       \
    civ_##S *A = (civ_##S *)malloc(N * sizeof(civ_##S));                       \
    civ_##S *Bv = (civ_##S *)malloc(N * sizeof(civ_##S));                      \
    /* P:208 pad: a' = (a_0..a_{n-1}, 0..0) as thin intervals */       \
    for (size_t j = 0; j < n; j++) {                                           \
        ap[j].re.lo = ap[j].re.hi = (T)a[j];                                   \
        bp[j].re.lo = bp[j].re.hi = (T)b[j];                                   \
    }                                                                          \
    fft_rec_##S(k, ap, A, tw, N, 0);                             /* P:209 */   \
    fft_rec_##S(k, bp, Bv, tw, N, 0);                                          \
    for (size_t i = 0; i < N; i++) ap[i] = cmul_##S(A[i], Bv[i]); /* P:210 */  \
    fft_rec_##S(k, ap, A, tw, N, 1);                             /* P:211 */   \
    for (size_t i = 0; i < N; i++) A[i] = cdivk_##S(A[i], (T)N); /* P:97 1/n */\
    if (intervals_out)                                                         \
        for (size_t i = 0; i < N; i++) store_##S(intervals_out + 4 * i, A[i]); \
    /* P:24 / P:247: the unique integer in each containment set, over the   */ \
    /* 2n-1 used coefficients; the same two functions the pins call. */ \
    size_t used = 2 * n - 1;                                                   \
    double *ud = (double *)malloc(used * 4 * sizeof(double));                  \
    for (size_t i = 0; i < used; i++) {    /* binary32 -> binary64 is exact */ \
        ud[4 * i] = (double)A[i].re.lo; ud[4 * i + 1] = (double)A[i].re.hi;    \
        ud[4 * i + 2] = (double)A[i].im.lo; ud[4 * i + 3] = (double)A[i].im.hi; \
    }                                                                          \
    int32_t bad = oracle_certify_span(ud, used, coeff);                               \
    int ok = bad < 0;                                                          \
    double rad = max_radius_span(ud, used);                                    \
    if (ok) {                                                                  \
        int64_t *c = coeff ? coeff : (int64_t *)malloc((2 * n - 1) * sizeof(int64_t)); \
        if (!coeff) oracle_certify_span(ud, used, c);                                 \
        oracle_carry(c, n, prod);                                /* P:229-235 */ \
        if (!coeff) free(c);                                                   \
    } else {                                                                   \
        memset(prod, 0, 2 * n);                                                \
    }                                                                          \
    if (maxrad) *maxrad = rad;                                                 \
    if (first_bad) *first_bad = bad;                                           \
    free(ud);                                                                  \
    free(ap); free(bp); free(A); free(Bv);                                     \
    return ok;                                                                 \
}

DEFINE_INTERVAL(double, f64)
DEFINE_INTERVAL(float, f32)

static size_t fft_len(size_t n) {                 /* k = ceil(log2(2n-1)), m = 2^k */
    size_t N = 1;
    while (N < 2 * n - 1) N <<= 1;
    return N;
}

size_t oracle_fft_length(size_t n) { return fft_len(n); }

/* ------------------------------------------------------------------ */
/* exported entry points (ctypes)                                       */
/* ------------------------------------------------------------------ */

/* Batched interval multiply.  prec 0 = binary64 (tw: double[N][4]),
 * prec 1 = binary32 (tw: float[N][4]).  Arrays are [batch][n] digits,
 * [batch][2n] products, [batch] flags / radii / first-bad,
 * coeffs [batch][2n-1] (nullable), intervals [batch][N][4] in the
 * precision's type (nullable).  nthreads <= 0: OpenMP default. */
int oracle_ivmul_batch(const uint8_t *a, const uint8_t *b, size_t n, size_t batch, int prec,
                       const void *tw, uint8_t *prod, uint8_t *cert, double *maxrad,
                       int32_t *first_bad, int64_t *coeffs, void *intervals, int nthreads) {
    if (n == 0 || batch == 0) return -1;
    size_t N = fft_len(n);
    int old = fegetround();
    (void)nthreads;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        enter();
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (long long p = 0; p < (long long)batch; p++) {
            int ok;
            int64_t *cf = coeffs ? coeffs + (size_t)p * (2 * n - 1) : NULL;
            if (prec == 0) {
                double *iv = intervals ? (double *)intervals + (size_t)p * N * 4 : NULL;
                ok = ss_multiply_f64(a + (size_t)p * n, b + (size_t)p * n, n, (const double *)tw, N,
                                     prod + (size_t)p * 2 * n, cf, maxrad ? maxrad + p : NULL,
                                     first_bad ? first_bad + p : NULL, iv);
            } else {
                float *iv = intervals ? (float *)intervals + (size_t)p * N * 4 : NULL;
                ok = ss_multiply_f32(a + (size_t)p * n, b + (size_t)p * n, n, (const float *)tw, N,
                                     prod + (size_t)p * 2 * n, cf, maxrad ? maxrad + p : NULL,
                                     first_bad ? first_bad + p : NULL, iv);
            }
            cert[p] = (uint8_t)ok;
        }
        fesetround(old);
    }
    fesetround(old);
    return 0;
}

/* P:24 / P:247 rule and the radius on their own (for the pins): the very
 * functions ss_multiply_* calls.  iv: [len][4] (binary64, or binary32 for
 * the _f32 twins, widened exactly); flag[i] = 1 and coeff[i] = the unique
 * integer where entry i certifies. */
void oracle_certify_f64(const double *iv, size_t len, int64_t *coeff, uint8_t *flag) {
    for (size_t i = 0; i < len; i++) {
        int64_t c;
        flag[i] = (uint8_t)(oracle_certify_span(iv + 4 * i, 1, &c) < 0);
        coeff[i] = c;
    }
}
void oracle_certify_f32(const float *iv, size_t len, int64_t *coeff, uint8_t *flag) {
    for (size_t i = 0; i < len; i++) {
        double d[4] = { iv[4 * i], iv[4 * i + 1], iv[4 * i + 2], iv[4 * i + 3] };
        int64_t c;
        flag[i] = (uint8_t)(oracle_certify_span(d, 1, &c) < 0);
        coeff[i] = c;
    }
}
double oracle_max_radius_f64(const double *iv, size_t len) {
    int old = fegetround(); enter();
    double r = max_radius_span(iv, len);
    fesetround(old);
    return r;
}
double oracle_max_radius_f32(const float *iv, size_t len) {
    int old = fegetround(); enter();
    double *d = (double *)malloc((len ? len : 1) * 4 * sizeof(double));
    for (size_t i = 0; i < 4 * len; i++) d[i] = iv[i];
    double r = max_radius_span(d, len);
    free(d);
    fesetround(old);
    return r;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Batched long multiplication and coefficient sums. */
void oracle_long_multiply_batch(const uint8_t *a, const uint8_t *b, size_t n, size_t batch,
                                uint8_t *z, int nthreads) {
    (void)nthreads;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (long long p = 0; p < (long long)batch; p++)
        oracle_long_multiply(a + (size_t)p * n, n, b + (size_t)p * n, n, z + (size_t)p * 2 * n);
}

void oracle_coefficients_batch(const uint8_t *a, const uint8_t *b, size_t n, size_t batch,
                               int64_t *z, int nthreads) {
    (void)nthreads;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (long long p = 0; p < (long long)batch; p++)
        oracle_coefficients(a + (size_t)p * n, n, b + (size_t)p * n, n, z + (size_t)p * (2 * n - 1));
}

/* S:432 "residues modulo 61-bit primes": a product z (2n digits) of x, y
 * (n digits each) is checked as (x mod p)(y mod p) == z mod p for each given
 * modulus p < 2^62 (primes, drawn by the caller).  Horner's rule over the
 * base-256 digits, most significant first, seven digits per reduction.
 * ok[pair] = 1 iff every modulus agrees.  A wrong product passes one random
 * 61-bit prime with probability < 2^-40 at these sizes (a nonzero difference
 * below 2^(16 n) has at most 16n/60 prime factors of 61 bits). */
static uint64_t mod_digits(const uint8_t *d, size_t len, uint64_t p) {
    unsigned __int128 r = 0;
    size_t i = len;
    while (i > 0) {
        size_t k = i >= 7 ? 7 : i;
        i -= k;
        uint64_t chunk = 0;
        for (size_t j = k; j-- > 0;) chunk = (chunk << 8) | d[i + j];
        r = ((r << (8 * k)) + chunk) % p;
    }
    return (uint64_t)r;
}

void oracle_residue_check_batch(const uint8_t *a, const uint8_t *b, const uint8_t *z, size_t n, size_t batch,
                                const uint64_t *primes, int nprimes, uint8_t *ok, int nthreads) {
    (void)nthreads;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
    for (long long q = 0; q < (long long)batch; q++) {
        int good = 1;
        for (int k = 0; k < nprimes; k++) {
            uint64_t p = primes[k];
            unsigned __int128 xy = (unsigned __int128)mod_digits(a + (size_t)q * n, n, p) *
                                   mod_digits(b + (size_t)q * n, n, p);
            if ((uint64_t)(xy % p) != mod_digits(z + (size_t)q * 2 * n, 2 * n, p)) good = 0;
        }
        ok[q] = (uint8_t)good;
    }
}

/* --- single steps, for the pins (each one operation of §2.5 / §2.2) --- */

/* op: 0 add, 1 sub, 2 mul; vectors of [len][2] */
void oracle_interval_op_f64(int op, const double *a, const double *b, double *r, size_t len) {
    int old = fegetround(); enter();
    for (size_t i = 0; i < len; i++) {
        iv_f64 x = { a[2 * i], a[2 * i + 1] }, y = { b[2 * i], b[2 * i + 1] }, z;
        z = op == 0 ? iadd_f64(x, y) : op == 1 ? isub_f64(x, y) : imul_f64(x, y);
        r[2 * i] = z.lo; r[2 * i + 1] = z.hi;
    }
    fesetround(old);
}
void oracle_interval_op_f32(int op, const float *a, const float *b, float *r, size_t len) {
    int old = fegetround(); enter();
    for (size_t i = 0; i < len; i++) {
        iv_f32 x = { a[2 * i], a[2 * i + 1] }, y = { b[2 * i], b[2 * i + 1] }, z;
        z = op == 0 ? iadd_f32(x, y) : op == 1 ? isub_f32(x, y) : imul_f32(x, y);
        r[2 * i] = z.lo; r[2 * i + 1] = z.hi;
    }
    fesetround(old);
}

/* complex op: 0 cadd, 1 csub, 2 cmul; vectors of [len][4] */
void oracle_cinterval_op_f64(int op, const double *a, const double *b, double *r, size_t len) {
    int old = fegetround(); enter();
    for (size_t i = 0; i < len; i++) {
        civ_f64 x = load_f64(a + 4 * i), y = load_f64(b + 4 * i), z;
        z = op == 0 ? cadd_f64(x, y) : op == 1 ? csub_f64(x, y) : cmul_f64(x, y);
        store_f64(r + 4 * i, z);
    }
    fesetround(old);
}

/* Interval FFT of length N = 2^k, forward (inverse = 0) or the
 * unscaled inverse (P:97 without 1/n, inverse = 1) or scaled (inverse = 2).
 * x, out: [N][4]; tw: omega_N^j, j < N, as [N][4]. */
void oracle_fft_f64(const double *x, double *out, const double *tw, size_t N, int inverse) {
    int old = fegetround(); enter();
    int k = 0; while (((size_t)1 << k) < N) k++;
    fft_rec_f64(k, (const civ_f64 *)x, (civ_f64 *)out, (const civ_f64 *)tw, N, inverse != 0);
    if (inverse == 2)
        for (size_t i = 0; i < N; i++) ((civ_f64 *)out)[i] = cdivk_f64(((civ_f64 *)out)[i], (double)N);
    fesetround(old);
}
void oracle_fft_f32(const float *x, float *out, const float *tw, size_t N, int inverse) {
    int old = fegetround(); enter();
    int k = 0; while (((size_t)1 << k) < N) k++;
    fft_rec_f32(k, (const civ_f32 *)x, (civ_f32 *)out, (const civ_f32 *)tw, N, inverse != 0);
    if (inverse == 2)
        for (size_t i = 0; i < N; i++) ((civ_f32 *)out)[i] = cdivk_f32(((civ_f32 *)out)[i], (float)N);
    fesetround(old);
}
