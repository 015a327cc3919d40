// ivm_twc_host.h -- host helpers for the compact twiddle entries of ivm_v3.cuh.
#pragma once
#include <stdint.h>
#include <string.h>

namespace ivm {

// compact first-quadrant entry (lower endpoints); the upper endpoints must be
// the next representable numbers with the same high 32-bit word (double) --
// otherwise the plan fails (never observed for m <= 15; tested).
template <typename F> static inline bool hi_ok(F lo, F hi) {
  if (lo == hi) return true;  // exact: the kernel uses next(lo) >= hi, sound
  if (sizeof(F) == 8) {
    uint64_t l, h;
    memcpy(&l, &lo, 8);
    memcpy(&h, &hi, 8);
    return h == l + 1 && (h >> 32) == (l >> 32);
  }
  uint32_t l, h;
  memcpy(&l, &lo, 4);
  memcpy(&h, &hi, 4);
  return h == l + 1;
}

// w = full-circle enclosure (re.lo, re.hi, im.lo, im.hi) in the upper half
// plane -> (c.lo, s.lo with the sign bit = k) where w = i^k (c + i s)
template <typename F> static inline bool compact(const F *w, F *o) {
  F cl = w[0], ch = w[1], sl = w[2], sh = w[3];
  if (!(sl >= 0)) return false;  // not in the upper half plane
  unsigned k = 0;
  if (ch < 0 || (ch == 0 && cl < 0)) {  // second quadrant: w = i (s - i c)
    F ncl = -ch, nch = -cl;
    cl = sl; ch = sh; sl = ncl; sh = nch;
    k = 1;
  }
  if (cl == 0) cl = 0;
  if (sl == 0) sl = 0;
  if (!hi_ok(cl, ch) || !hi_ok(sl, sh)) return false;
  o[0] = cl;
  o[1] = k ? -sl : sl;
  if (k && sl == 0) {  // -0.0 carries the flag
    F z = 0;
    o[1] = -z;
  }
  return true;
}

}  // namespace ivm
