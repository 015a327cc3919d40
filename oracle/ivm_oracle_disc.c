/*
 * ivm_oracle_disc.c -- CPU ORACLE for the circular-containment-set variant.
 *
 * TEST INFRASTRUCTURE ONLY (same rules as ivm_oracle.c: only tests/,
 * __graft_entry__.smoke() and bench.py's reference legs may load it; it shares
 * no code, header or table with the CUDA path).
 *
 * PAPER.md P:290 (§4, conclusion): "It may also be interesting to use circular
 * containment sets rather than rectangular containment sets.  The advantage of
 * circular containment sets is that they easily deal with complex rotations".
 * The paper defines no arithmetic for them; reading R15 fixes it:
 *
 *   a disc <c, r> = { z : |z - c| <= r }, c = (cr, ci) binary64, r >= 0;
 *   every center operation is one rounded binary64 operation (here: the
 *   FE_UPWARD mode the whole oracle runs in); every radius is an upper bound
 *   computed with upward rounding;
 *   a rounded result x~ of an exact x satisfies |x~ - x| <= U |x~| + ETA with
 *   U = 2^-52 (one ulp, any rounding direction) and ETA = 2^-1000 (subnormal
 *   guard);
 *   sum:      <a.c + b.c, a.r + b.r + E>,  E = U (|sr| + |si|) + 2 ETA;
 *   product:  t1 = ar br, t2 = ai bi, t3 = ar bi, t4 = ai br (rounded),
 *             pr = t1 - t2, pi = t3 + t4 (rounded),
 *             E = U (|t1| + |t2| + |pr| + |t3| + |t4| + |pi|) + 6 ETA,
 *             r = |a.c| b.r + |b.c| a.r + a.r b.r + E,  |c| = sqrt(cr^2 + ci^2) rounded up;
 *   conjugate: <(cr, -ci), r>;  division by N = 2^L: exact on c and r;
 *   twiddle: omega_N^j from the optimal rectangular enclosure [lo, hi] + i[lo, hi]
 *            (oracle/twiddles.py): c = (re.lo, im.lo), r = (re.hi - re.lo) + (im.hi - im.lo);
 *   certify: the real part [cr - r, cr + r] (directed) holds exactly one
 *            integer and the imaginary part [ci - r, ci + r] holds only 0.
 *
 * The FFT is the paper's recursive Cooley-Tukey and the
 * multiplication the fast convolution P:203-211, exactly as in ivm_oracle.c
 * with discs in place of rectangular intervals.  binary64 only.
 */
#include <fenv.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#pragma STDC FENV_ACCESS ON

void oracle_carry(const int64_t *v, size_t n, uint8_t *z); /* ivm_oracle.c */

typedef struct { double cr, ci, r; } disc;

static const double U = 0x1p-52, ETA = 0x1p-1000;

/* all arithmetic below runs with fesetround(FE_UPWARD): radii are upper bounds */
static double absu(double x) { return fabs(x); }
static double normu(double cr, double ci) { return sqrt(cr * cr + ci * ci); }

static disc d_add(disc a, disc b) {
    disc s;
    s.cr = a.cr + b.cr;
    s.ci = a.ci + b.ci;
    double e = U * (absu(s.cr) + absu(s.ci)) + 2 * ETA;
    s.r = a.r + b.r + e;
    return s;
}

static disc d_sub(disc a, disc b) {
    disc s;
    s.cr = a.cr - b.cr;
    s.ci = a.ci - b.ci;
    double e = U * (absu(s.cr) + absu(s.ci)) + 2 * ETA;
    s.r = a.r + b.r + e;
    return s;
}

static disc d_mul(disc a, disc b) {
    disc p;
    double t1 = a.cr * b.cr, t2 = a.ci * b.ci, t3 = a.cr * b.ci, t4 = a.ci * b.cr;
    p.cr = t1 - t2;
    p.ci = t3 + t4;
    double e = U * (absu(t1) + absu(t2) + absu(p.cr) + absu(t3) + absu(t4) + absu(p.ci)) + 6 * ETA;
    p.r = normu(a.cr, a.ci) * b.r + normu(b.cr, b.ci) * a.r + a.r * b.r + e;
    return p;
}

static disc d_conj(disc a) { a.ci = -a.ci; return a; }

static disc d_scale(disc a, double s) { a.cr *= s; a.ci *= s; a.r *= s; return a; } /* s = 2^-L: exact */

static disc d_twiddle(const double *t) {  /* t = (re.lo, re.hi, im.lo, im.hi) */
    disc w;
    w.cr = t[0];
    w.ci = t[2];
    w.r = (t[1] - t[0]) + (t[3] - t[2]);
    return w;
}

/* P:143-155, recursive radix-2 DIT; tw: omega_N^j rectangular table, j < N */
static void d_fft_rec(int k, const disc *x, disc *out, const double *tw, size_t N, int inverse) {
    size_t n = (size_t)1 << k;
    if (k == 0) { out[0] = x[0]; return; }
    size_t h = n / 2;
    disc *buf = (disc *)malloc(sizeof(disc) * 2 * n);
    disc *xe = buf, *xo = buf + h, *Xe = buf + n, *Xo = buf + n + h;
    for (size_t i = 0; i < h; i++) { xe[i] = x[2 * i]; xo[i] = x[2 * i + 1]; }
    d_fft_rec(k - 1, xe, Xe, tw, N, inverse);
    d_fft_rec(k - 1, xo, Xo, tw, N, inverse);
    size_t stride = N / n;
    for (size_t i = 0; i < n; i++) {
        disc w = d_twiddle(tw + 4 * (i * stride));
        if (inverse) w = d_conj(w);
        out[i] = d_add(Xe[i % h], d_mul(w, Xo[i % h]));
    }
    free(buf);
}

static size_t d_fft_len(size_t n) {
    size_t N = 1;
    while (N < 2 * n - 1) N <<= 1;
    return N;
}

/* ivm_oracle.c: the P:24 certify rule (one definition for both oracles) */
int32_t oracle_certify_span(const double *iv, size_t len, int64_t *coeff);

/* one multiplication (P:203-211 with discs); returns the certified flag */
static int d_multiply(const uint8_t *a, const uint8_t *b, size_t n, const double *tw, size_t N,
                      uint8_t *prod, int64_t *coeff, double *maxrad, int32_t *first_bad, double *discs_out) {
    int k = 0;
    while (((size_t)1 << k) < N) k++;
    disc *ap = (disc *)calloc(N, sizeof(disc)), *bp = (disc *)calloc(N, sizeof(disc));
    disc *A = (disc *)malloc(N * sizeof(disc)), *B = (disc *)malloc(N * sizeof(disc));
    for (size_t j = 0; j < n; j++) { ap[j].cr = a[j]; bp[j].cr = b[j]; }  /* P:208, radius 0 */
    d_fft_rec(k, ap, A, tw, N, 0);
    d_fft_rec(k, bp, B, tw, N, 0);
    for (size_t i = 0; i < N; i++) ap[i] = d_mul(A[i], B[i]);
    d_fft_rec(k, ap, A, tw, N, 1);
    for (size_t i = 0; i < N; i++) A[i] = d_scale(A[i], 1.0 / (double)N);
    if (discs_out)
        for (size_t i = 0; i < N; i++) {
            discs_out[3 * i] = A[i].cr; discs_out[3 * i + 1] = A[i].ci; discs_out[3 * i + 2] = A[i].r;
        }
    /* P:24 on the enclosing rectangle [cr - r, cr + r] + i[ci - r, ci + r]
     * (rounded outward), by the rectangular oracle's certify function */
    size_t used = 2 * n - 1;
    double *box = (double *)malloc(used * 4 * sizeof(double));
    double rad = 0.0;
    for (size_t i = 0; i < used; i++) {
        disc z = A[i];
        if (z.r > rad || z.r != z.r) rad = (z.r != z.r) ? INFINITY : z.r;
        box[4 * i] = -((-z.cr) + z.r); box[4 * i + 1] = z.cr + z.r;   /* RD(cr - r), RU(cr + r) */
        box[4 * i + 2] = -((-z.ci) + z.r); box[4 * i + 3] = z.ci + z.r;
    }
    int64_t *c = coeff ? coeff : (int64_t *)malloc(used * sizeof(int64_t));
    int32_t bad = oracle_certify_span(box, used, c);
    int ok = bad < 0;
    if (ok) oracle_carry(c, n, prod);
    else memset(prod, 0, 2 * n);
    if (!coeff) free(c);
    free(box);
    if (maxrad) *maxrad = rad;
    if (first_bad) *first_bad = bad;
    free(ap); free(bp); free(A); free(B);
    return ok;
}

/* batched disc multiply: tw = rectangular double[N][4] table (oracle/twiddles.py);
 * prod [batch][2n], cert/maxrad/first_bad [batch], coeffs [batch][2n-1] and
 * discs [batch][N][3] nullable */
int oracle_disc_batch(const uint8_t *a, const uint8_t *b, size_t n, size_t batch, const double *tw,
                      uint8_t *prod, uint8_t *cert, double *maxrad, int32_t *first_bad, int64_t *coeffs,
                      double *discs, int nthreads) {
    if (n == 0 || batch == 0) return -1;
    size_t N = d_fft_len(n);
    int old = fegetround();
    (void)nthreads;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        fesetround(FE_UPWARD);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (long long p = 0; p < (long long)batch; p++) {
            cert[p] = (uint8_t)d_multiply(a + (size_t)p * n, b + (size_t)p * n, n, tw, N, prod + (size_t)p * 2 * n,
                                          coeffs ? coeffs + (size_t)p * (2 * n - 1) : NULL,
                                          maxrad ? maxrad + p : NULL, first_bad ? first_bad + p : NULL,
                                          discs ? discs + (size_t)p * N * 3 : NULL);
        }
        fesetround(old);
    }
    fesetround(old);
    return 0;
}

/* the primitives on their own (pins): op 0 add, 1 sub, 2 mul, 3 conj; [len][3] */
void oracle_disc_op(int op, const double *a, const double *b, double *r, size_t len) {
    int old = fegetround();
    fesetround(FE_UPWARD);
    for (size_t i = 0; i < len; i++) {
        disc x = {a[3 * i], a[3 * i + 1], a[3 * i + 2]}, y = {b[3 * i], b[3 * i + 1], b[3 * i + 2]}, z;
        z = op == 0 ? d_add(x, y) : op == 1 ? d_sub(x, y) : op == 2 ? d_mul(x, y) : d_conj(x);
        r[3 * i] = z.cr; r[3 * i + 1] = z.ci; r[3 * i + 2] = z.r;
    }
    fesetround(old);
}

/* the disc FFT on its own: x, out [N][3]; tw rectangular [N][4]; unscaled */
void oracle_disc_fft(const double *x, double *out, const double *tw, size_t N, int inverse) {
    int old = fegetround();
    fesetround(FE_UPWARD);
    int k = 0;
    while (((size_t)1 << k) < N) k++;
    d_fft_rec(k, (const disc *)x, (disc *)out, tw, N, inverse);
    fesetround(old);
}
