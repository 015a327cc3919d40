// ivm_interval.cuh -- device-side rectangular complex interval arithmetic with
// directed rounding (§2.5), binary64 and binary32.
//
// Every endpoint is computed by ONE directed-rounding instruction
// (DADD/DMUL/DFMA .RM/.RP, FADD/FMUL/FFMA .RM/.RP): lower endpoints round
// toward -inf, upper endpoints toward +inf, so each result interval contains
// the exact result of the real operation on any points of the operands.
// Real interval products select their endpoint pair by the sign classes of
// the operands (Moore's nine cases) instead of P:253's min/max over four
// rounded products: the selected pair is the exact argmin/argmax, so the
// result is contained in P:253's (never wider) and never chosen by comparing
// rounded values.  Complex products fuse the subtraction/addition of P:265
// into an FMA: re.lo = RD(RD(x1*y1) - x2*y2) etc.
//
// Shares nothing with oracle/ (which is plain C with fesetround).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ivm {

template <typename T> struct CI { T rl, rh, il, ih; };  // [rl,rh] + i[il,ih]

template <typename T> struct DR;
template <> struct DR<double> {
  static __device__ __forceinline__ double add_rd(double a, double b) { return __dadd_rd(a, b); }
  static __device__ __forceinline__ double add_ru(double a, double b) { return __dadd_ru(a, b); }
  static __device__ __forceinline__ double mul_rd(double a, double b) { return __dmul_rd(a, b); }
  static __device__ __forceinline__ double mul_ru(double a, double b) { return __dmul_ru(a, b); }
  static __device__ __forceinline__ double fma_rd(double a, double b, double c) { return __fma_rd(a, b, c); }
  static __device__ __forceinline__ double fma_ru(double a, double b, double c) { return __fma_ru(a, b, c); }
  // sign bit set (x < 0 or x == -0.0): a test of the high word only (a 64-bit
  // compare costs two ISETPs)
  static __device__ __forceinline__ bool neg(double x) { return __double2hiint(x) < 0; }
};
template <> struct DR<float> {
  static __device__ __forceinline__ float add_rd(float a, float b) { return __fadd_rd(a, b); }
  static __device__ __forceinline__ float add_ru(float a, float b) { return __fadd_ru(a, b); }
  static __device__ __forceinline__ float mul_rd(float a, float b) { return __fmul_rd(a, b); }
  static __device__ __forceinline__ float mul_ru(float a, float b) { return __fmul_ru(a, b); }
  static __device__ __forceinline__ float fma_rd(float a, float b, float c) { return __fmaf_rd(a, b, c); }
  static __device__ __forceinline__ float fma_ru(float a, float b, float c) { return __fmaf_ru(a, b, c); }
  static __device__ __forceinline__ bool neg(float x) { return __float_as_int(x) < 0; }
};

// ---- exact operations --------------------------------------------------
template <typename T> __device__ __forceinline__ CI<T> cconj(const CI<T> &z) {
  return CI<T>{z.rl, z.rh, -z.ih, -z.il};
}
template <typename T> __device__ __forceinline__ CI<T> mul_i(const CI<T> &z) {  // i*z
  return CI<T>{-z.ih, -z.il, z.rl, z.rh};
}
template <typename T> __device__ __forceinline__ CI<T> mul_mi(const CI<T> &z) {  // -i*z
  return CI<T>{z.il, z.ih, -z.rh, -z.rl};
}
template <typename T> __device__ __forceinline__ CI<T> punctual(T re) {
  return CI<T>{re, re, T(0), T(0)};
}

// ---- P:264 addition / subtraction ---------------------------------------
template <typename T> __device__ __forceinline__ CI<T> cadd(const CI<T> &a, const CI<T> &b) {
  return CI<T>{DR<T>::add_rd(a.rl, b.rl), DR<T>::add_ru(a.rh, b.rh),
               DR<T>::add_rd(a.il, b.il), DR<T>::add_ru(a.ih, b.ih)};
}
template <typename T> __device__ __forceinline__ CI<T> csub(const CI<T> &a, const CI<T> &b) {
  return CI<T>{DR<T>::add_rd(a.rl, -b.rh), DR<T>::add_ru(a.rh, -b.rl),
               DR<T>::add_rd(a.il, -b.ih), DR<T>::add_ru(a.ih, -b.il)};
}
// butterfly (E + t, E - t)  (PAPER.md P:153 with omega^{i+n/2} = -omega^i)
template <typename T>
__device__ __forceinline__ void bfly(CI<T> &e, CI<T> &o, const CI<T> &t) {
  CI<T> s = cadd(e, t);
  o = csub(e, t);
  e = s;
}

// ---- twiddle product t = w * d ------------------------------------------
// w: twiddle enclosure whose real and imaginary parts each have one sign
// (exact zeros are stored as [+0,+0]); d: any interval.  For a single-signed
// w-component [wl,wh] and data [yl,yh] (P:253 by sign cases):
//   lo(w*y) = y1*(y1 >= 0 ? wl : wh),  y1 = (w >= 0 ? yl : yh)
//   hi(w*y) = y2*(y2 >= 0 ? wh : wl),  y2 = (w >= 0 ? yh : yl)
template <typename T> struct Pair { T x, y; };
template <typename T>
__device__ __forceinline__ Pair<T> tw_lo(T wl, T wh, bool wneg, T yl, T yh) {
  T y = wneg ? yh : yl;
  return Pair<T>{DR<T>::neg(y) ? wh : wl, y};
}
template <typename T>
__device__ __forceinline__ Pair<T> tw_hi(T wl, T wh, bool wneg, T yl, T yh) {
  T y = wneg ? yl : yh;
  return Pair<T>{DR<T>::neg(y) ? wl : wh, y};
}

template <typename T>
__device__ __forceinline__ CI<T> twmul(const CI<T> &w, const CI<T> &d) {
  const bool rn = DR<T>::neg(w.rh), in = DR<T>::neg(w.ih);
  // re = wr*dr - wi*di ; im = wr*di + wi*dr
  Pair<T> a1 = tw_lo(w.rl, w.rh, rn, d.rl, d.rh), a2 = tw_hi(w.il, w.ih, in, d.il, d.ih);
  Pair<T> b1 = tw_hi(w.rl, w.rh, rn, d.rl, d.rh), b2 = tw_lo(w.il, w.ih, in, d.il, d.ih);
  Pair<T> c1 = tw_lo(w.rl, w.rh, rn, d.il, d.ih), c2 = tw_lo(w.il, w.ih, in, d.rl, d.rh);
  Pair<T> e1 = tw_hi(w.rl, w.rh, rn, d.il, d.ih), e2 = tw_hi(w.il, w.ih, in, d.rl, d.rh);
  CI<T> t;
  t.rl = DR<T>::fma_rd(-a2.x, a2.y, DR<T>::mul_rd(a1.x, a1.y));
  t.rh = DR<T>::fma_ru(-b2.x, b2.y, DR<T>::mul_ru(b1.x, b1.y));
  t.il = DR<T>::fma_rd(c2.x, c2.y, DR<T>::mul_rd(c1.x, c1.y));
  t.ih = DR<T>::fma_ru(e2.x, e2.y, DR<T>::mul_ru(e1.x, e1.y));
  return t;
}

// ---- general complex interval product (pointwise step, P:210 / P:265) ----
// Sign classes: P = x >= 0 (sign bit of lo clear), N = x <= 0 (sign bit of
// hi set), S = straddles.  Endpoint pairs (Moore):
//   lo: x_sel = (yP ? xl : yN ? xh : (xP ? xh : xl)), y_sel = (xP ? yl : xN ? yh : (yP ? yh : yl))
//   hi: x_sel = (yP ? xh : yN ? xl : (xP ? xh : xl)), y_sel = (xP ? yh : xN ? yl : (yP ? yh : yl))
// except S x S, where lo = min(xl*yh, xh*yl), hi = max(xl*yl, xh*yh).
template <typename T> struct RPairs { Pair<T> lo, hi; bool ss; };
template <typename T>
__device__ __forceinline__ RPairs<T> rpairs(T xl, T xh, T yl, T yh) {
  // sign bits (-0 counts as negative: harmless, its products are 0)
  const bool xln = DR<T>::neg(xl), xhn = DR<T>::neg(xh), yln = DR<T>::neg(yl), yhn = DR<T>::neg(yh);
  RPairs<T> r;
  r.lo.x = (!yln || (!yhn && xhn)) ? xl : xh;
  r.lo.y = (!xln || (!xhn && yln)) ? yl : yh;
  r.hi.x = (!yln || (!yhn && !xln)) ? xh : xl;
  r.hi.y = (!xln || (!xhn && !yln)) ? yh : yl;
  r.ss = xln && !xhn && yln && !yhn;  // both straddle zero
  return r;
}
template <typename T>
__device__ __forceinline__ T rlo_exact_ss(T xl, T xh, T yl, T yh) {  // RD(min(xl*yh, xh*yl))
  return fmin(DR<T>::mul_rd(xl, yh), DR<T>::mul_rd(xh, yl));
}
template <typename T>
__device__ __forceinline__ T rhi_exact_ss(T xl, T xh, T yl, T yh) {  // RU(max(xl*yl, xh*yh))
  return fmax(DR<T>::mul_ru(xl, yl), DR<T>::mul_ru(xh, yh));
}

template <typename T>
__device__ __forceinline__ CI<T> cmul(const CI<T> &z, const CI<T> &w) {
  RPairs<T> p_rr = rpairs(z.rl, z.rh, w.rl, w.rh);
  RPairs<T> p_ii = rpairs(z.il, z.ih, w.il, w.ih);
  RPairs<T> p_ri = rpairs(z.rl, z.rh, w.il, w.ih);
  RPairs<T> p_ir = rpairs(z.il, z.ih, w.rl, w.rh);
  CI<T> t;
  if (!(p_rr.ss || p_ii.ss || p_ri.ss || p_ir.ss)) {
    t.rl = DR<T>::fma_rd(-p_ii.hi.x, p_ii.hi.y, DR<T>::mul_rd(p_rr.lo.x, p_rr.lo.y));
    t.rh = DR<T>::fma_ru(-p_ii.lo.x, p_ii.lo.y, DR<T>::mul_ru(p_rr.hi.x, p_rr.hi.y));
    t.il = DR<T>::fma_rd(p_ir.lo.x, p_ir.lo.y, DR<T>::mul_rd(p_ri.lo.x, p_ri.lo.y));
    t.ih = DR<T>::fma_ru(p_ir.hi.x, p_ir.hi.y, DR<T>::mul_ru(p_ri.hi.x, p_ri.hi.y));
  } else {
    // unfused fallback: each real product as a rounded interval, then P:265
    T rr_l = p_rr.ss ? rlo_exact_ss(z.rl, z.rh, w.rl, w.rh) : DR<T>::mul_rd(p_rr.lo.x, p_rr.lo.y);
    T rr_h = p_rr.ss ? rhi_exact_ss(z.rl, z.rh, w.rl, w.rh) : DR<T>::mul_ru(p_rr.hi.x, p_rr.hi.y);
    T ii_l = p_ii.ss ? rlo_exact_ss(z.il, z.ih, w.il, w.ih) : DR<T>::mul_rd(p_ii.lo.x, p_ii.lo.y);
    T ii_h = p_ii.ss ? rhi_exact_ss(z.il, z.ih, w.il, w.ih) : DR<T>::mul_ru(p_ii.hi.x, p_ii.hi.y);
    T ri_l = p_ri.ss ? rlo_exact_ss(z.rl, z.rh, w.il, w.ih) : DR<T>::mul_rd(p_ri.lo.x, p_ri.lo.y);
    T ri_h = p_ri.ss ? rhi_exact_ss(z.rl, z.rh, w.il, w.ih) : DR<T>::mul_ru(p_ri.hi.x, p_ri.hi.y);
    T ir_l = p_ir.ss ? rlo_exact_ss(z.il, z.ih, w.rl, w.rh) : DR<T>::mul_rd(p_ir.lo.x, p_ir.lo.y);
    T ir_h = p_ir.ss ? rhi_exact_ss(z.il, z.ih, w.rl, w.rh) : DR<T>::mul_ru(p_ir.hi.x, p_ir.hi.y);
    t.rl = DR<T>::add_rd(rr_l, -ii_h);
    t.rh = DR<T>::add_ru(rr_h, -ii_l);
    t.il = DR<T>::add_rd(ri_l, ir_l);
    t.ih = DR<T>::add_ru(ri_h, ir_h);
  }
  return t;
}

// Pointwise product with a single-sign fast path.  When no component of z or w
// straddles zero (the sign bits of each lower and upper endpoint agree; -0 counts
// as negative, so [-0, x] takes the general path), the exact argmin / argmax pair
// of a real product x*y follows from the two signs alone:
//   lo = (y < 0 ? xh : xl) * (x < 0 ? yh : yl),  hi = (y < 0 ? xl : xh) * (x < 0 ? yl : yh),
// i.e. four predicates (the signs of z.re, z.im, w.re, w.im) and 16 double selects for
// the complex product instead of cmul's nine-case classes; the FMA fusion and the
// rounding are cmul's, so the result is bit-identical.  Anything else goes to cmul.
template <typename T> __device__ __forceinline__ unsigned sgnw(T x);
template <> __device__ __forceinline__ unsigned sgnw<double>(double x) { return (unsigned)__double2hiint(x); }
template <> __device__ __forceinline__ unsigned sgnw<float>(float x) { return (unsigned)__float_as_int(x); }

// (the general product out of line: the cold straddle path keeps its registers
// out of the hot passes' allocation)
template <typename T>
__device__ __noinline__ CI<T> cmul_cold(const CI<T> z, const CI<T> w) {
  return cmul(z, w);
}

template <typename T, bool COLD_CALL = false>
__device__ __forceinline__ CI<T> cmul_ss(const CI<T> &z, const CI<T> &w) {
  const unsigned a = sgnw(z.rl), b = sgnw(z.rh), c = sgnw(z.il), d = sgnw(z.ih);
  const unsigned e = sgnw(w.rl), f = sgnw(w.rh), g = sgnw(w.il), h = sgnw(w.ih);
  if ((int)((a ^ b) | (c ^ d) | (e ^ f) | (g ^ h)) < 0) return COLD_CALL ? cmul_cold(z, w) : cmul(z, w);
  const bool zr = (int)a < 0, zi = (int)c < 0, wr = (int)e < 0, wi = (int)g < 0;
  CI<T> t;
  // re = z.re w.re - z.im w.im ; im = z.re w.im + z.im w.re
  t.rl = DR<T>::fma_rd(-(wi ? z.il : z.ih), zi ? w.il : w.ih, DR<T>::mul_rd(wr ? z.rh : z.rl, zr ? w.rh : w.rl));
  t.rh = DR<T>::fma_ru(-(wi ? z.ih : z.il), zi ? w.ih : w.il, DR<T>::mul_ru(wr ? z.rl : z.rh, zr ? w.rl : w.rh));
  t.il = DR<T>::fma_rd(wr ? z.ih : z.il, zi ? w.rh : w.rl, DR<T>::mul_rd(wi ? z.rh : z.rl, zr ? w.ih : w.il));
  t.ih = DR<T>::fma_ru(wr ? z.il : z.ih, zi ? w.rl : w.rh, DR<T>::mul_ru(wi ? z.rl : z.rh, zr ? w.il : w.ih));
  return t;
}

}  // namespace ivm
