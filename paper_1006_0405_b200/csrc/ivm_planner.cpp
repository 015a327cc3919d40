// ivm_planner.cpp -- optimal twiddle enclosures for the device tables.
//
// omega_m^j = e^{2 pi i j/m} enclosed as
// [RD(cos), RU(cos)] + i [RD(sin), RU(sin)] in binary64 or binary32.  The
// paper's recurrence omega_{2n} = (1+omega_n)/|1+omega_n| is replaced
// by "other efficient methods": each first-octant value is evaluated
// once in binary128 (libquadmath cosq/sinq, error < 2^-108 including the
// rounding of the angle), and rounded down/up only when that error ball
// cannot straddle a target-format number -- otherwise the plan fails loudly.
// The remaining octants follow from exact symmetries (swap, negation), which
// commute with directed rounding.  Exact entries 1, i, -1, -i at j = 0, m/4,
// m/2, 3m/4 (omega_1 = 1, omega_2 = -1, omega_4 = i); exact zeros are
// stored as [+0, +0].
//
// Independent of oracle/twiddles.py (mpmath); tests check bit equality.
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <string.h>

namespace {

const __float128 kErr = 0x1p-108Q;

template <typename F> struct Fmt;
template <> struct Fmt<double> {
  static double down(__float128 v) {  // largest double <= v
    double d = (double)v;
    while ((__float128)d > v) d = nextafter(d, -INFINITY);
    while ((__float128)nextafter(d, INFINITY) <= v) d = nextafter(d, INFINITY);
    return d;
  }
  static double up(__float128 v) { return -down(-v); }
};
template <> struct Fmt<float> {
  static float down(__float128 v) {
    float d = (float)v;
    while ((__float128)d > v) d = nextafterf(d, -INFINITY);
    while ((__float128)nextafterf(d, INFINITY) <= v) d = nextafterf(d, INFINITY);
    return d;
  }
  static float up(__float128 v) { return -down(-v); }
};

// enclosure of an irrational value known within +-kErr of v
template <typename F> bool enclose(__float128 v, F *lo, F *hi) {
  F l1 = Fmt<F>::down(v - kErr), l2 = Fmt<F>::down(v + kErr);
  F h1 = Fmt<F>::up(v - kErr), h2 = Fmt<F>::up(v + kErr);
  if (l1 != l2 || h1 != h2) return false;
  *lo = l1;
  *hi = h1;
  return true;
}

template <typename F> int build(int m, F *out /* [N][4] */) {
  const long N = 1L << m;
  if (N == 1) {
    out[0] = 1; out[1] = 1; out[2] = 0; out[3] = 0;
    return 0;
  }
  if (N == 2) {
    F t[8] = {1, 1, 0, 0, -1, -1, 0, 0};
    memcpy(out, t, sizeof(t));
    return 0;
  }
  const long Q = N / 4;
  // first quadrant j in [0, Q]: (clo, chi, slo, shi)
  F *cq = new F[4 * (Q + 1)];
  for (long j = 0; j <= N / 8; j++) {
    F *e = cq + 4 * j;
    if (j == 0) {
      e[0] = 1; e[1] = 1; e[2] = 0; e[3] = 0;
      continue;
    }
    __float128 th = 2 * M_PIq * (__float128)j / (__float128)N;
    __float128 c = cosq(th), s = sinq(th);
    if (!enclose<F>(c, &e[0], &e[1]) || !enclose<F>(s, &e[2], &e[3])) {
      delete[] cq;
      return -1;
    }
    if (8 * j == N) {  // pi/4: cos = sin exactly
      e[2] = e[0];
      e[3] = e[1];
    }
  }
  for (long j = N / 8 + 1; j <= Q; j++) {  // angle pi/2 - t: swap
    const F *s = cq + 4 * (Q - j);
    F *e = cq + 4 * j;
    e[0] = s[2]; e[1] = s[3]; e[2] = s[0]; e[3] = s[1];
  }
  for (long j = 0; j < N; j++) {
    long quad = j / Q, r = j % Q;
    const F *c = cq + 4 * r;
    F *o = out + 4 * j;
    switch (quad) {
      case 0: o[0] = c[0]; o[1] = c[1]; o[2] = c[2]; o[3] = c[3]; break;
      case 1: o[0] = -c[3]; o[1] = -c[2]; o[2] = c[0]; o[3] = c[1]; break;     // (-s, c)
      case 2: o[0] = -c[1]; o[1] = -c[0]; o[2] = -c[3]; o[3] = -c[2]; break;   // (-c, -s)
      default: o[0] = c[2]; o[1] = c[3]; o[2] = -c[1]; o[3] = -c[0]; break;    // (s, -c)
    }
    for (int k = 0; k < 4; k++)
      if (o[k] == 0) o[k] = 0;  // canonical +0 for exact zeros
  }
  delete[] cq;
  return 0;
}

// nearest-rounded points (cos, sin) of omega_N^j for the naive (punctual) SS
// comparator: binary128 values rounded to nearest; exact at multiples of pi/2
template <typename F> int build_rn(int m, F *out /* [N][2] */) {
  const long N = 1L << m;
  for (long j = 0; j < N; j++) {
    F c, s;
    if (N >= 4 && j % (N / 4) == 0) {
      const long q = j / (N / 4);
      c = (q == 0) ? 1 : (q == 2 ? -1 : 0);
      s = (q == 1) ? 1 : (q == 3 ? -1 : 0);
    } else if (N < 4) {
      c = (j == 0) ? 1 : -1;
      s = 0;
    } else {
      const __float128 th = 2 * M_PIq * (__float128)j / (__float128)N;
      c = (F)cosq(th);
      s = (F)sinq(th);
    }
    out[2 * j] = c;
    out[2 * j + 1] = s;
  }
  return 0;
}

}  // namespace

namespace ivm {
// prec 0: double[N][4]; prec 1: float[N][4]
int plan_twiddles(int m, int prec, void *out) {
  if (m < 0 || m > 26) return -1;
  return prec == 0 ? build<double>(m, (double *)out) : build<float>(m, (float *)out);
}
// prec 0: double[N][2]; prec 1: float[N][2] (round to nearest, no enclosure)
int plan_twiddles_rn(int m, int prec, void *out) {
  if (m < 0 || m > 26) return -1;
  return prec == 0 ? build_rn<double>(m, (double *)out) : build_rn<float>(m, (float *)out);
}
}  // namespace ivm
