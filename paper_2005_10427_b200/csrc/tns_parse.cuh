// Token parsers of the GPU .tns reader (tns.cu).  Header-only and
// __host__ __device__ so the exact same code is exercised by the CPU
// self-check (tests/cpp/tns_parse_check.cpp, compiled with g++) and by the
// kernels.
//
// Semantics follow the reference reader (io.cpp:42-126), which tokenises on
// ' ', '\t', '\r' (io.cpp:22-34) and converts every token with std::from_chars:
//   * indices: std::from_chars(uint32_t) — decimal digits only, no sign, the
//     whole token consumed, no overflow (io.cpp:83-88);
//   * values:  std::from_chars(double), chars_format::general (io.cpp:108-113):
//     optional '-', "inf"/"infinity"/"nan"/"nan(chars)" case-insensitive, or
//     digits with an optional '.' and an optional exponent (an incomplete
//     exponent is not consumed, so the token is rejected); correctly rounded
//     (ties to even); a finite token that overflows to infinity or a nonzero
//     token that underflows to zero is result_out_of_range, i.e. rejected.
// Conversion: Eisel-Lemire (128-bit products with a table of normalised
// powers of five, gen/pow5_table.py) on the first 19 significant digits; when
// later digits were dropped and w and w+1 round differently, an exact
// big-integer comparison against the halfway points decides.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define QD_HD __host__ __device__ __forceinline__
#define QD_TABLE __device__ __constant__
#else
#define QD_HD inline
#define QD_TABLE
#endif

namespace qb200 {
namespace tns {

QD_TABLE static const uint64_t kPow5[] = {
#include "tns_pow5.inc"
};
constexpr int kSmallestPow10 = -342;
constexpr int kLargestPow10 = 308;

QD_HD bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r'; }

// std::from_chars(uint32_t) over the whole token.
QD_HD bool parse_u32(const char* s, uint32_t n, uint32_t* out) {
  if (n == 0) return false;
  uint64_t v = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const unsigned d = (unsigned char)s[i] - '0';
    if (d > 9) return false;
    v = v * 10 + d;
    if (v > 0xFFFFFFFFull) return false;
  }
  *out = (uint32_t)v;
  return true;
}

QD_HD void mul64(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
#if defined(__CUDA_ARCH__)
  *lo = a * b;
  *hi = __umul64hi(a, b);
#else
  const unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
#endif
}

QD_HD int clz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
  return __clzll((long long)x);
#else
  return __builtin_clzll(x);
#endif
}

struct Adjusted {
  uint64_t mantissa;  // 52 explicit bits
  int32_t power2;     // biased exponent field; 0x7FF = infinity
};

// Eisel-Lemire: w * 10^q rounded to nearest-even binary64 (w != 0 exact).
QD_HD Adjusted compute_float(int64_t q, uint64_t w) {
  Adjusted a{0, 0};
  if (w == 0 || q < kSmallestPow10) return a;
  if (q > kLargestPow10) return Adjusted{0, 0x7FF};
  const int lz = clz64(w);
  w <<= lz;
  const int idx = 2 * (int)(q - kSmallestPow10);
  uint64_t hi, lo;
  mul64(w, kPow5[idx], &hi, &lo);
  const uint64_t mask = 0xFFFFFFFFFFFFFFFFull >> 55;
  if ((hi & mask) == mask) {
    uint64_t hi2, lo2;
    mul64(w, kPow5[idx + 1], &hi2, &lo2);
    lo += hi2;
    if (hi2 > lo) ++hi;
  }
  const int upper = (int)(hi >> 63);
  a.mantissa = hi >> (upper + 64 - 52 - 3);
  const int32_t p10 = (int32_t)(((152170 + 65536) * q) >> 16) + 63;
  a.power2 = p10 + upper - lz + 1023;
  if (a.power2 <= 0) {  // subnormal or zero
    if (-a.power2 + 1 >= 64) return Adjusted{0, 0};
    a.mantissa >>= -a.power2 + 1;
    a.mantissa += (a.mantissa & 1);
    a.mantissa >>= 1;
    a.power2 = (a.mantissa < (1ull << 52)) ? 0 : 1;
    a.mantissa &= ~(1ull << 52);
    return a;
  }
  if (lo <= 1 && q >= -4 && q <= 23 && (a.mantissa & 3) == 1) {
    if ((a.mantissa << (upper + 64 - 52 - 3)) == hi) a.mantissa &= ~1ull;  // tie: to even
  }
  a.mantissa += (a.mantissa & 1);
  a.mantissa >>= 1;
  if (a.mantissa >= (2ull << 52)) {
    a.mantissa = 1ull << 52;
    a.power2++;
  }
  a.mantissa &= ~(1ull << 52);
  if (a.power2 >= 0x7FF) return Adjusted{0, 0x7FF};
  return a;
}

// ---- exact slow path: big-integer comparison --------------------------------
constexpr int kBigWords = 176;     // 5632 bits: 780 digits + 5^1125 + shifts
constexpr int kMaxBigDigits = 780;  // digits beyond are folded into a sticky bit

struct Big {
  uint32_t w[kBigWords];
  int n;
};

QD_HD void big_set(Big& b, uint64_t v) {
  b.n = 0;
  while (v) {
    b.w[b.n++] = (uint32_t)v;
    v >>= 32;
  }
}
QD_HD void big_muladd(Big& b, uint32_t m, uint32_t add) {
  uint64_t carry = add;
  for (int i = 0; i < b.n; ++i) {
    const uint64_t t = (uint64_t)b.w[i] * m + carry;
    b.w[i] = (uint32_t)t;
    carry = t >> 32;
  }
  if (carry && b.n < kBigWords) b.w[b.n++] = (uint32_t)carry;
}
QD_HD void big_mulpow5(Big& b, int p) {
  while (p >= 13) {
    big_muladd(b, 1220703125u, 0);  // 5^13
    p -= 13;
  }
  uint32_t m = 1;
  while (p-- > 0) m *= 5;
  if (m != 1) big_muladd(b, m, 0);
}
QD_HD void big_shl(Big& b, int s) {
  if (b.n == 0 || s == 0) return;
  const int ws = s >> 5, bs = s & 31;
  int n = b.n + ws + 1;
  if (n > kBigWords) n = kBigWords;  // cannot happen within the documented bounds
  for (int i = n - 1; i >= 0; --i) {
    const int src = i - ws;
    uint32_t v = 0;
    if (src >= 0 && src < b.n) v = b.w[src] << bs;
    if (bs && src - 1 >= 0 && src - 1 < b.n) v |= b.w[src - 1] >> (32 - bs);
    b.w[i] = v;
  }
  b.n = n;
  while (b.n && b.w[b.n - 1] == 0) --b.n;
}
QD_HD int big_cmp(const Big& a, const Big& b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int i = a.n - 1; i >= 0; --i)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
  return 0;
}

// Significant digits of a validated numeral, in order (skips '.').
struct Digits {
  const char* s;      // numeral text (after the sign)
  uint32_t n;         // up to the exponent marker
  uint32_t first;     // index of the first significant (nonzero) digit
};

// Compares X = D * 10^qd (D = the first kMaxBigDigits significant digits;
// `sticky` = a nonzero digit was dropped after them) with Y = h * 2^f.
QD_HD int compare_halfway(const Digits& dg, int64_t qd, bool sticky, uint64_t h, int64_t f,
                          Big& A, Big& B) {
  A.n = 0;
  uint32_t taken = 0, chunk = 0, cm = 1;
  for (uint32_t i = dg.first; i < dg.n && taken < (uint32_t)kMaxBigDigits; ++i) {
    const char c = dg.s[i];
    if (c == '.') continue;
    chunk = chunk * 10 + (uint32_t)(c - '0');
    cm *= 10;
    ++taken;
    if (cm == 1000000000u) {
      big_muladd(A, cm, chunk);
      chunk = 0;
      cm = 1;
    }
  }
  if (cm != 1) big_muladd(A, cm, chunk);
  if (A.n == 0 && chunk) big_set(A, chunk);
  big_set(B, h);
  if (qd >= 0) {
    big_mulpow5(A, (int)qd);
    const int64_t s = qd - f;
    if (s >= 0) big_shl(A, (int)s); else big_shl(B, (int)-s);
  } else {
    big_mulpow5(B, (int)-qd);
    const int64_t t = f - qd;
    if (t >= 0) big_shl(B, (int)t); else big_shl(A, (int)-t);
  }
  const int c = big_cmp(A, B);
  return (c == 0 && sticky) ? 1 : c;
}

// ---- std::from_chars(double) over a whole token ------------------------------
QD_HD bool ieq(char c, char lower) { return c == lower || c == (char)(lower - 32); }

// 1 = parsed, 0 = rejected, 2 = the exact slow path is needed but kSlow is
// false (kernels without it keep no big-integer stack frame).
template <bool kSlow>
QD_HD int parse_f64_impl(const char* s, uint32_t n, double* out) {
  uint32_t i = 0;
  bool neg = false;
  if (i < n && s[i] == '-') {
    neg = true;
    ++i;
  }
  const uint64_t sign = neg ? (1ull << 63) : 0;
  union {
    uint64_t u;
    double d;
  } r;
  // inf / infinity / nan / nan(n-char-sequence)
  if (i < n && (ieq(s[i], 'i') || ieq(s[i], 'n'))) {
    const uint32_t m = n - i;
    const char* t = s + i;
    if (ieq(t[0], 'i')) {
      if (m == 3 && ieq(t[1], 'n') && ieq(t[2], 'f')) { r.u = sign | 0x7FF0000000000000ull; *out = r.d; return 1; }
      if (m == 8 && ieq(t[1], 'n') && ieq(t[2], 'f') && ieq(t[3], 'i') && ieq(t[4], 'n') &&
          ieq(t[5], 'i') && ieq(t[6], 't') && ieq(t[7], 'y')) {
        r.u = sign | 0x7FF0000000000000ull; *out = r.d; return 1;
      }
      return 0;
    }
    if (m < 3 || !ieq(t[1], 'a') || !ieq(t[2], 'n')) return 0;
    if (m > 3) {
      if (t[3] != '(' || t[m - 1] != ')') return 0;
      for (uint32_t k = 4; k + 1 < m; ++k) {
        const char c = t[k];
        const bool ok = (c >= '0' && c <= '9') || (c >= 'a' && c <= 'z') ||
                        (c >= 'A' && c <= 'Z') || c == '_';
        if (!ok) return 0;
      }
    }
    r.u = sign | 0x7FF8000000000000ull;
    *out = r.d;
    return 1;
  }
  // digits [. digits]
  const uint32_t num_begin = i;
  uint64_t w = 0;
  uint32_t nsig = 0, ndig = 0, first = 0xFFFFFFFFu;
  int64_t adj = 0;
  bool frac = false, sticky = false;
  for (; i < n; ++i) {
    const char c = s[i];
    if (c == '.') {
      if (frac) break;
      frac = true;
      continue;
    }
    const unsigned d = (unsigned char)c - '0';
    if (d > 9) break;
    ++ndig;
    if (nsig == 0 && d == 0) {
      if (frac) --adj;
      continue;
    }
    if (nsig == 0) first = i - num_begin;
    ++nsig;
    if (nsig <= 19) {
      w = w * 10 + d;
      if (frac) --adj;
    } else {
      if (d) sticky = true;
      if (!frac) ++adj;
    }
  }
  if (ndig == 0) return 0;
  const uint32_t mant_end = i;
  int64_t e10 = 0;
  if (i < n && (s[i] == 'e' || s[i] == 'E')) {
    uint32_t j = i + 1;
    bool eneg = false;
    if (j < n && (s[j] == '+' || s[j] == '-')) {
      eneg = s[j] == '-';
      ++j;
    }
    if (j < n && (unsigned)((unsigned char)s[j] - '0') <= 9) {
      for (; j < n; ++j) {
        const unsigned d = (unsigned char)s[j] - '0';
        if (d > 9) break;
        if (e10 < 100000000) e10 = e10 * 10 + d;
      }
      if (eneg) e10 = -e10;
      i = j;
    }
  }
  if (i != n) return 0;
  if (w == 0) {  // every digit is zero
    r.u = sign;
    *out = r.d;
    return 1;
  }
  const int64_t q = e10 + adj;
  Adjusted a = compute_float(q, w);
  if (sticky) {
    const Adjusted b = compute_float(q, w + 1);
    if (a.mantissa != b.mantissa || a.power2 != b.power2) {
      if constexpr (!kSlow) return 2;
      // Exact decision between a and its successor: X vs the upper halfway.
      Digits dg{s + num_begin, mant_end - num_begin, first};
      // significant digits all count; D has min(nsig, kMaxBigDigits) digits
      const uint32_t taken = nsig < (uint32_t)kMaxBigDigits ? nsig : (uint32_t)kMaxBigDigits;
      // value = D_taken * 10^qd: the first digit's weight is 10^(q + nsig... )
      // q is the exponent of w (19 digits); shift by the digits beyond 19 taken
      const int64_t qd = q - (int64_t)(taken - 19);
      bool st = false;
      if (nsig > taken) {
        // any nonzero among the digits after the first `taken` significant ones
        uint32_t seen = 0;
        for (uint32_t k = first; k < dg.n; ++k) {
          const char c = dg.s[k];
          if (c == '.') continue;
          if (seen++ >= taken && c != '0') { st = true; break; }
        }
      }
      uint64_t m2;
      int64_t e2;
      if (a.power2 == 0) { m2 = a.mantissa; e2 = -1074; }
      else { m2 = a.mantissa | (1ull << 52); e2 = (int64_t)a.power2 - 1075; }
      int c = 0;
      if constexpr (kSlow) {
        Big A, B;
        c = compare_halfway(dg, qd, st, 2 * m2 + 1, e2 - 1, A, B);
      }
      if (c > 0 || (c == 0 && (m2 & 1))) {  // round up to the successor
        uint64_t bits = ((uint64_t)a.power2 << 52) | a.mantissa;
        ++bits;
        a.power2 = (int32_t)(bits >> 52);
        a.mantissa = bits & ((1ull << 52) - 1);
      }
    }
  }
  if (a.power2 >= 0x7FF) return 0;              // overflow: out_of_range
  if (a.power2 == 0 && a.mantissa == 0) return 0;  // underflow: out_of_range
  r.u = sign | ((uint64_t)a.power2 << 52) | a.mantissa;
  *out = r.d;
  return 1;
}

QD_HD bool parse_f64(const char* s, uint32_t n, double* out) {
  return parse_f64_impl<true>(s, n, out) == 1;
}

}  // namespace tns
}  // namespace qb200
