// Line formatting of the GPU .tns writer (tns.cu, write side).  Header-only,
// __host__ __device__: the CPU self-check (tests/cpp/tns_format_check.cpp)
// runs exactly this code against std::to_chars.
//
// The reference writer (io.cpp:128-152) prints each row as the 1-based
// indices (std::to_chars(uint32_t + 1)) separated by ' ', then ' ', the value
// by std::to_chars(double) — the shortest round-trip form, fixed or
// scientific, whichever is shorter (fixed on a tie); in fixed form an
// integer-valued double prints its exact digits — and '\n'.
// Shortest digits: Ryu (Adams, PLDI 2018) with the 125-bit tables of
// gen/ryu_tables.py.
#pragma once

#include <cstdint>

#include "tns_parse.cuh"  // QD_HD, QD_TABLE, mul64

namespace qb200 {
namespace tns {

#include "tns_ryu.inc"

QD_HD uint32_t pow5bits(int32_t e) { return (uint32_t)(((e * 1217359) >> 19) + 1); }
QD_HD uint32_t log10Pow2(int32_t e) { return (uint32_t)((e * 78913) >> 18); }
QD_HD uint32_t log10Pow5(int32_t e) { return (uint32_t)((e * 732923) >> 20); }

QD_HD uint32_t pow5Factor(uint64_t v) {
  uint32_t c = 0;
  while (v % 5 == 0 && v) {
    v /= 5;
    ++c;
  }
  return c;
}
QD_HD bool multipleOfPowerOf5(uint64_t v, uint32_t p) { return pow5Factor(v) >= p; }
QD_HD bool multipleOfPowerOf2(uint64_t v, uint32_t p) { return (v & ((1ull << p) - 1)) == 0; }

// (m * mul) >> j for a 128-bit mul {lo, hi}, j >= 64
QD_HD uint64_t mulShift64(uint64_t m, const uint64_t* mul, int32_t j) {
  uint64_t h0, l0, h1, l1;
  mul64(m, mul[0], &h0, &l0);
  mul64(m, mul[1], &h1, &l1);
  // (h0 + (h1:l1)) >> (j - 64)
  uint64_t lo = l1 + h0;
  uint64_t hi = h1 + (lo < h0 ? 1 : 0);
  const int s = j - 64;
  if (s == 0) return lo;
  if (s >= 64) return hi >> (s - 64);
  return (lo >> s) | (hi << (64 - s));
}

struct Decimal {
  uint64_t digits;  // no trailing zeros
  int32_t exp10;    // value = digits * 10^exp10
};

// Shortest round-trip digits of a positive finite double (Ryu d2d).
QD_HD Decimal shortest(uint64_t ieeeMantissa, uint32_t ieeeExponent) {
  int32_t e2;
  uint64_t m2;
  if (ieeeExponent == 0) {
    e2 = 1 - 1023 - 52 - 2;
    m2 = ieeeMantissa;
  } else {
    e2 = (int32_t)ieeeExponent - 1023 - 52 - 2;
    m2 = (1ull << 52) | ieeeMantissa;
  }
  const bool acceptBounds = (m2 & 1) == 0;
  const uint64_t mv = 4 * m2;
  const uint32_t mmShift = ieeeMantissa != 0 || ieeeExponent <= 1;
  uint64_t vr, vp, vm;
  int32_t e10;
  bool vmIsTrailingZeros = false, vrIsTrailingZeros = false;
  if (e2 >= 0) {
    const uint32_t q = log10Pow2(e2) - (e2 > 3);
    e10 = (int32_t)q;
    const int32_t k = 125 + (int32_t)pow5bits((int32_t)q) - 1;
    const int32_t i = -e2 + (int32_t)q + k;
    const uint64_t* mul = kRyuPow5Inv[q];
    vr = mulShift64(4 * m2, mul, i);
    vp = mulShift64(4 * m2 + 2, mul, i);
    vm = mulShift64(4 * m2 - 1 - mmShift, mul, i);
    if (q <= 21) {
      if (mv % 5 == 0) {
        vrIsTrailingZeros = multipleOfPowerOf5(mv, q);
      } else if (acceptBounds) {
        vmIsTrailingZeros = multipleOfPowerOf5(mv - 1 - mmShift, q);
      } else {
        vp -= multipleOfPowerOf5(mv + 2, q);
      }
    }
  } else {
    const uint32_t q = log10Pow5(-e2) - (-e2 > 1);
    e10 = (int32_t)q + e2;
    const int32_t i = -e2 - (int32_t)q;
    const int32_t k = (int32_t)pow5bits(i) - 125;
    const int32_t j = (int32_t)q - k;
    const uint64_t* mul = kRyuPow5[i];
    vr = mulShift64(4 * m2, mul, j);
    vp = mulShift64(4 * m2 + 2, mul, j);
    vm = mulShift64(4 * m2 - 1 - mmShift, mul, j);
    if (q <= 1) {
      vrIsTrailingZeros = true;
      if (acceptBounds) vmIsTrailingZeros = mmShift == 1;
      else --vp;
    } else if (q < 63) {
      vrIsTrailingZeros = multipleOfPowerOf2(mv, q);
    }
  }
  int32_t removed = 0;
  uint32_t lastRemovedDigit = 0;
  uint64_t output;
  if (vmIsTrailingZeros || vrIsTrailingZeros) {
    for (;;) {
      const uint64_t vpDiv10 = vp / 10, vmDiv10 = vm / 10;
      if (vpDiv10 <= vmDiv10) break;
      const uint32_t vmMod10 = (uint32_t)(vm - 10 * vmDiv10);
      const uint64_t vrDiv10 = vr / 10;
      const uint32_t vrMod10 = (uint32_t)(vr - 10 * vrDiv10);
      vmIsTrailingZeros &= vmMod10 == 0;
      vrIsTrailingZeros &= lastRemovedDigit == 0;
      lastRemovedDigit = vrMod10;
      vr = vrDiv10;
      vp = vpDiv10;
      vm = vmDiv10;
      ++removed;
    }
    if (vmIsTrailingZeros) {
      for (;;) {
        const uint64_t vmDiv10 = vm / 10;
        const uint32_t vmMod10 = (uint32_t)(vm - 10 * vmDiv10);
        if (vmMod10 != 0) break;
        const uint64_t vpDiv10 = vp / 10, vrDiv10 = vr / 10;
        const uint32_t vrMod10 = (uint32_t)(vr - 10 * vrDiv10);
        vrIsTrailingZeros &= lastRemovedDigit == 0;
        lastRemovedDigit = vrMod10;
        vr = vrDiv10;
        vp = vpDiv10;
        vm = vmDiv10;
        ++removed;
      }
    }
    if (vrIsTrailingZeros && lastRemovedDigit == 5 && vr % 2 == 0) lastRemovedDigit = 4;
    output = vr + ((vr == vm && (!acceptBounds || !vmIsTrailingZeros)) || lastRemovedDigit >= 5);
  } else {
    bool roundUp = false;
    const uint64_t vpDiv100 = vp / 100, vmDiv100 = vm / 100;
    if (vpDiv100 > vmDiv100) {
      const uint64_t vrDiv100 = vr / 100;
      const uint32_t vrMod100 = (uint32_t)(vr - 100 * vrDiv100);
      roundUp = vrMod100 >= 50;
      vr = vrDiv100;
      vp = vpDiv100;
      vm = vmDiv100;
      removed += 2;
    }
    for (;;) {
      const uint64_t vpDiv10 = vp / 10, vmDiv10 = vm / 10;
      if (vpDiv10 <= vmDiv10) break;
      const uint64_t vrDiv10 = vr / 10;
      const uint32_t vrMod10 = (uint32_t)(vr - 10 * vrDiv10);
      roundUp = vrMod10 >= 5;
      vr = vrDiv10;
      vp = vpDiv10;
      vm = vmDiv10;
      ++removed;
    }
    output = vr + (vr == vm || roundUp);
  }
  Decimal d{output, e10 + removed};
  // Ryu may leave trailing zeros in the output digits; strip them
  while (d.digits && d.digits % 10 == 0) {
    d.digits /= 10;
    ++d.exp10;
  }
  return d;
}

QD_HD uint32_t dec_len(uint64_t v) {
  uint32_t n = 1;
  while (v >= 10) {
    v /= 10;
    ++n;
  }
  return n;
}

// Writes v's decimal digits (exactly `n` of them) ending at out + n.
QD_HD void put_digits(char* out, uint64_t v, uint32_t n) {
  for (uint32_t i = n; i-- > 0;) {
    out[i] = (char)('0' + v % 10);
    v /= 10;
  }
}

// std::to_chars(double) (shortest, plain format).  out must hold 32 chars;
// returns the length.  When out is null only the length is computed.
QD_HD uint32_t format_f64(double x, char* out) {
  union {
    double d;
    uint64_t u;
  } b;
  b.d = x;
  const bool neg = b.u >> 63;
  const uint32_t ex = (uint32_t)((b.u >> 52) & 0x7FF);
  const uint64_t man = b.u & ((1ull << 52) - 1);
  uint32_t p = 0;
  auto put = [&](char c) {
    if (out) out[p] = c;
    ++p;
  };
  if (neg) put('-');
  if (ex == 0x7FF) {
    const char* s = man ? "nan" : "inf";
    for (int i = 0; i < 3; ++i) put(s[i]);
    return p;
  }
  if (ex == 0 && man == 0) {
    put('0');
    return p;
  }
  const Decimal d = shortest(man, ex);
  const uint32_t n = dec_len(d.digits);
  const int32_t X = d.exp10 + (int32_t)n - 1;  // scientific exponent
  const uint32_t ax = (uint32_t)(X < 0 ? -X : X);
  const uint32_t sci = n + (n > 1 ? 1 : 0) + 2 + (ax >= 100 ? 3 : 2);
  uint32_t fix;
  if (X >= (int32_t)n - 1) fix = (uint32_t)X + 1;
  else if (X >= 0) fix = n + 1;
  else fix = n + 1 + (uint32_t)(-X);
  if (fix <= sci) {
    if (X >= (int32_t)n - 1) {
      // integer value: the exact digits of the double (< 10^22 here, so the
      // value fits in 128 bits)
      const int32_t e2 = (ex == 0 ? -1074 : (int32_t)ex - 1075);
      const uint64_t m2 = ex == 0 ? man : (man | (1ull << 52));
      uint64_t hi = 0, lo = m2;
      if (e2 >= 0) {
        const int s = e2;
        if (s >= 64) { hi = lo << (s - 64); lo = 0; }
        else if (s > 0) { hi = lo >> (64 - s); lo <<= s; }
      } else {
        lo >>= -e2;  // exact: the value is an integer
      }
      char tmp[40];
      uint32_t k = 0;
      do {  // 128-bit by 10
        const uint64_t rh = hi % 10;
        hi /= 10;
        // (rh * 2^64 + lo) / 10 without 128-bit types: split lo in 32-bit halves
        const uint64_t a = (rh << 32) | (lo >> 32);
        const uint64_t qa = a / 10, ra = a % 10;
        const uint64_t bb = (ra << 32) | (lo & 0xFFFFFFFFull);
        const uint64_t qb = bb / 10, rb = bb % 10;
        lo = (qa << 32) | qb;
        tmp[k++] = (char)('0' + rb);
      } while (hi || lo);
      while (k) put(tmp[--k]);
      return p;
    }
    if (X >= 0) {
      char dg[20];
      put_digits(dg, d.digits, n);
      for (uint32_t i = 0; i < n; ++i) {
        if (i == (uint32_t)X + 1) put('.');
        put(dg[i]);
      }
      return p;
    }
    put('0');
    put('.');
    for (int32_t i = 0; i < -X - 1; ++i) put('0');
    char dg[20];
    put_digits(dg, d.digits, n);
    for (uint32_t i = 0; i < n; ++i) put(dg[i]);
    return p;
  }
  char dg[20];
  put_digits(dg, d.digits, n);
  put(dg[0]);
  if (n > 1) {
    put('.');
    for (uint32_t i = 1; i < n; ++i) put(dg[i]);
  }
  put('e');
  put(X < 0 ? '-' : '+');
  if (ax >= 100) put((char)('0' + ax / 100));
  put((char)('0' + (ax / 10) % 10));
  put((char)('0' + ax % 10));
  return p;
}

// std::to_chars(uint32_t) of v (out: 10 chars, or null for the length).
QD_HD uint32_t format_u64(uint64_t v, char* out) {
  const uint32_t n = dec_len(v);
  if (out) put_digits(out, v, n);
  return n;
}

}  // namespace tns
}  // namespace qb200
