// Number formatting shared by host and device code (report emission, §8(f)-4).
//
// fmt_double writes exactly what the reference's format_double writes
// (report.cpp:42-47: std::to_chars(double) with no format, i.e. the shortest
// digit string that round-trips, printed in fixed or scientific notation,
// whichever is shorter, fixed on a tie). The shortest digits come from Ryu
// (U. Adams, PLDI 2018: exact base-10 interval arithmetic with 128-bit
// multipliers, csrc/ryu_tables.h), which is what libstdc++ uses as well; the
// layout follows printf's %f / %e rules. fmt_u64 / fmt_i64 are std::to_string.
// Every function returns the number of bytes written; a nullptr buffer only
// counts (the size pass of a two-pass writer).
#pragma once

#include <cstdint>
#include <cstring>

#include "ryu_tables.h"

namespace xsp {

XSP_HD inline uint64_t umul128_hi(uint64_t a, uint64_t b, uint64_t* lo) {
#ifdef __CUDA_ARCH__
  *lo = a * b;
  return __umul64hi(a, b);
#else
  const unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  return (uint64_t)(p >> 64);
#endif
}

// (m * mul) >> j for a 128-bit multiplier, j >= 64
XSP_HD inline uint64_t ryu_mul_shift(uint64_t m, const uint64_t* mul, int j) {
  uint64_t lo0, lo2;
  const uint64_t hi0 = umul128_hi(m, mul[0], &lo0);
  const uint64_t hi2 = umul128_hi(m, mul[1], &lo2);
  const uint64_t sum_lo = hi0 + lo2;
  const uint64_t sum_hi = hi2 + (sum_lo < hi0 ? 1 : 0);
  const int s = j - 64;  // shift of the 128-bit (sum_hi:sum_lo)
  return s == 0 ? sum_lo : (sum_hi << (64 - s)) | (sum_lo >> s);
}

XSP_HD inline int ryu_pow5bits(int e) { return (int)(((uint32_t)e * 1217359u) >> 19) + 1; }
XSP_HD inline int ryu_log10_pow2(int e) { return (int)(((uint32_t)e * 78913u) >> 18); }
XSP_HD inline int ryu_log10_pow5(int e) { return (int)(((uint32_t)e * 732923u) >> 20); }

XSP_HD inline int ryu_pow5_factor(uint64_t v) {
  int c = 0;
  while (v % 5 == 0) {
    v /= 5;
    ++c;
  }
  return c;
}
XSP_HD inline bool ryu_multiple_of_pow5(uint64_t v, int p) { return ryu_pow5_factor(v) >= p; }
XSP_HD inline bool ryu_multiple_of_pow2(uint64_t v, int p) { return (v & ((1ull << p) - 1)) == 0; }

// Shortest decimal (digits, exponent) of a finite, nonzero |x|: x = digits * 10^exp.
XSP_HD inline void ryu_d2d(uint64_t bits, uint64_t& digits, int& exp10) {
  const uint64_t mant = bits & ((1ull << 52) - 1);
  const int e_bits = (int)((bits >> 52) & 0x7FF);
  int e2;
  uint64_t m2;
  if (e_bits == 0) {
    e2 = 1 - 1023 - 52 - 2;
    m2 = mant;
  } else {
    e2 = e_bits - 1023 - 52 - 2;
    m2 = (1ull << 52) | mant;
  }
  const bool even = (m2 & 1) == 0;
  const bool accept = even;
  const uint64_t mv = 4 * m2;
  const uint32_t mm_shift = (mant != 0 || e_bits <= 1) ? 1 : 0;
  uint64_t vr, vp, vm;
  int e10;
  bool vm_tz = false, vr_tz = false;
  if (e2 >= 0) {
    const int q = ryu_log10_pow2(e2) - (e2 > 3 ? 1 : 0);
    e10 = q;
    const int k = kRyuPow5InvBits + ryu_pow5bits(q) - 1;
    const int i = -e2 + q + k;
    const uint64_t* mul = ryu_pow5_inv(q);
    vr = ryu_mul_shift(4 * m2, mul, i);
    vp = ryu_mul_shift(4 * m2 + 2, mul, i);
    vm = ryu_mul_shift(4 * m2 - 1 - mm_shift, mul, i);
    if (q <= 21) {
      if (mv % 5 == 0) {
        vr_tz = ryu_multiple_of_pow5(mv, q);
      } else if (accept) {
        vm_tz = ryu_multiple_of_pow5(mv - 1 - mm_shift, q);
      } else {
        vp -= ryu_multiple_of_pow5(mv + 2, q) ? 1 : 0;
      }
    }
  } else {
    const int q = ryu_log10_pow5(-e2) - (-e2 > 1 ? 1 : 0);
    e10 = q + e2;
    const int i = -e2 - q;
    const int k = ryu_pow5bits(i) - kRyuPow5Bits;
    const int j = q - k;
    const uint64_t* mul = ryu_pow5(i);
    vr = ryu_mul_shift(4 * m2, mul, j);
    vp = ryu_mul_shift(4 * m2 + 2, mul, j);
    vm = ryu_mul_shift(4 * m2 - 1 - mm_shift, mul, j);
    if (q <= 1) {
      vr_tz = true;
      if (accept) {
        vm_tz = mm_shift == 1;
      } else {
        --vp;
      }
    } else if (q < 63) {
      vr_tz = ryu_multiple_of_pow2(mv, q);
    }
  }
  int removed = 0;
  uint8_t last = 0;
  uint64_t out;
  if (vm_tz || vr_tz) {
    for (;;) {
      const uint64_t vp10 = vp / 10, vm10 = vm / 10;
      if (vp10 <= vm10) break;
      const uint64_t vr10 = vr / 10;
      vm_tz &= vm - vm10 * 10 == 0;
      vr_tz &= last == 0;
      last = (uint8_t)(vr - vr10 * 10);
      vr = vr10;
      vp = vp10;
      vm = vm10;
      ++removed;
    }
    if (vm_tz) {
      for (;;) {
        const uint64_t vm10 = vm / 10;
        if (vm - vm10 * 10 != 0) break;
        const uint64_t vp10 = vp / 10, vr10 = vr / 10;
        vr_tz &= last == 0;
        last = (uint8_t)(vr - vr10 * 10);
        vr = vr10;
        vp = vp10;
        vm = vm10;
        ++removed;
      }
    }
    if (vr_tz && last == 5 && vr % 2 == 0) last = 4;  // round half to even
    out = vr + (((vr == vm && (!accept || !vm_tz)) || last >= 5) ? 1 : 0);
  } else {
    bool round_up = false;
    if (vp / 100 > vm / 100) {
      round_up = vr % 100 >= 50;
      vr /= 100;
      vp /= 100;
      vm /= 100;
      removed += 2;
    }
    for (;;) {
      const uint64_t vp10 = vp / 10, vm10 = vm / 10;
      if (vp10 <= vm10) break;
      round_up = vr % 10 >= 5;
      vr /= 10;
      vp = vp10;
      vm = vm10;
      ++removed;
    }
    out = vr + ((vr == vm || round_up) ? 1 : 0);
  }
  digits = out;
  exp10 = e10 + removed;
}

XSP_HD inline int fmt_ndigits(uint64_t v) {
  int n = 1;
  while (v >= 10) {
    v /= 10;
    ++n;
  }
  return n;
}

// writes the decimal digits of v (exactly n of them) at p
XSP_HD inline void fmt_put_digits(char* p, uint64_t v, int n) {
  for (int i = n - 1; i >= 0; --i) {
    p[i] = (char)('0' + v % 10);
    v /= 10;
  }
}

XSP_HD inline int fmt_u64(char* p, uint64_t v) {
  const int n = fmt_ndigits(v);
  if (p) fmt_put_digits(p, v, n);
  return n;
}

XSP_HD inline int fmt_i64(char* p, int64_t v) {
  if (v >= 0) return fmt_u64(p, (uint64_t)v);
  const uint64_t a = (uint64_t)0 - (uint64_t)v;
  if (p) *p++ = '-';
  return 1 + fmt_u64(p, a);
}

XSP_HD inline int fmt_str(char* p, const char* s, int n) {
  if (p)
    for (int i = 0; i < n; ++i) p[i] = s[i];
  return n;
}

// std::to_chars(double) (shortest round trip; %f or %e, the shorter, %f on a tie)
XSP_HD inline int fmt_double(char* p, double x) {
  uint64_t bits;
  memcpy(&bits, &x, 8);
  const bool neg = (bits >> 63) != 0;
  const uint64_t ab = bits & ~(1ull << 63);
  int w = 0;
  if (ab >= 0x7FF0000000000000ull) {  // inf / nan
    if (ab == 0x7FF0000000000000ull) {
      if (neg) w += fmt_str(p ? p + w : nullptr, "-", 1);
      return w + fmt_str(p ? p + w : nullptr, "inf", 3);
    }
    if (neg) w += fmt_str(p ? p + w : nullptr, "-", 1);
    return w + fmt_str(p ? p + w : nullptr, "nan", 3);
  }
  if (neg) w += fmt_str(p ? p + w : nullptr, "-", 1);
  if (ab == 0) return w + fmt_str(p ? p + w : nullptr, "0", 1);
  uint64_t d;
  int e;
  ryu_d2d(ab, d, e);
  const int n = fmt_ndigits(d);
  const int sci_exp = e + n - 1;
  const int abs_se = sci_exp < 0 ? -sci_exp : sci_exp;
  const int len_sci = n + (n > 1 ? 1 : 0) + 2 + (abs_se >= 100 ? 3 : 2);
  int len_fix;
  if (e >= 0)
    len_fix = n + e;
  else if (-e < n)
    len_fix = n + 1;
  else
    len_fix = 2 + (-e);
  if (!p) return w + (len_fix <= len_sci ? len_fix : len_sci);
  char* q = p + w;
  if (len_fix <= len_sci) {
    if (e > 0) {
      // an integer-valued double: the exact value (same length, no error) is
      // preferred over the shortest digits padded with zeros; fixed notation is
      // only chosen below 10^22, so it fits 128 bits
      const uint64_t mant = ab & ((1ull << 52) - 1);
      const int eb = (int)(ab >> 52);
      const unsigned __int128 m2 = eb ? (mant | (1ull << 52)) : mant;
      const int sh = (eb ? eb : 1) - 1075;
      unsigned __int128 v = sh >= 0 ? m2 << sh : m2 >> -sh;
      for (int i = len_fix - 1; i >= 0; --i) {
        q[i] = (char)('0' + (int)(v % 10));
        v /= 10;
      }
    } else if (e == 0) {
      fmt_put_digits(q, d, n);
    } else if (-e < n) {
      const int ip = n + e;  // integer digits
      char tmp[20];
      fmt_put_digits(tmp, d, n);
      for (int i = 0; i < ip; ++i) q[i] = tmp[i];
      q[ip] = '.';
      for (int i = ip; i < n; ++i) q[i + 1] = tmp[i];
    } else {
      q[0] = '0';
      q[1] = '.';
      const int z = -e - n;
      for (int i = 0; i < z; ++i) q[2 + i] = '0';
      fmt_put_digits(q + 2 + z, d, n);
    }
    return w + len_fix;
  }
  char tmp[20];
  fmt_put_digits(tmp, d, n);
  int k = 0;
  q[k++] = tmp[0];
  if (n > 1) {
    q[k++] = '.';
    for (int i = 1; i < n; ++i) q[k++] = tmp[i];
  }
  q[k++] = 'e';
  q[k++] = sci_exp < 0 ? '-' : '+';
  if (abs_se >= 100) {
    q[k++] = (char)('0' + abs_se / 100);
    q[k++] = (char)('0' + (abs_se / 10) % 10);
    q[k++] = (char)('0' + abs_se % 10);
  } else {
    q[k++] = (char)('0' + abs_se / 10);
    q[k++] = (char)('0' + abs_se % 10);
  }
  return w + k;
}

}  // namespace xsp
