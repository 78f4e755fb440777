// TEST INFRASTRUCTURE: CPU self-check of the GPU .tns token parsers
// (paper_2005_10427_b200/csrc/tns_parse.cuh, compiled here as host code)
// against the reference reader's conversion, std::from_chars (io.cpp:83-88,
// 108-113), on random and adversarial tokens.  Prints the mismatch count.
//   g++ -O2 -std=c++20 -I paper_2005_10427_b200/csrc tests/cpp/tns_parse_check.cpp
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "tns_parse.cuh"

using qb200::tns::parse_f64;
using qb200::tns::parse_u32;

static long bad = 0, total = 0;

static void check_f64(const std::string& s) {
  double ref = 0, got = 0;
  auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), ref);
  const bool ref_ok = ec == std::errc{} && p == s.data() + s.size();
  const bool ok = parse_f64(s.data(), (uint32_t)s.size(), &got);
  ++total;
  uint64_t a, b;
  std::memcpy(&a, &ref, 8);
  std::memcpy(&b, &got, 8);
  if (ref_ok != ok || (ok && a != b)) {
    if (++bad < 20)
      std::printf("MISMATCH f64 '%s': ref ok=%d %016llx  got ok=%d %016llx\n", s.c_str(), ref_ok,
                  (unsigned long long)a, ok, (unsigned long long)b);
  }
}

static void check_u32(const std::string& s) {
  uint32_t ref = 0, got = 0;
  auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), ref);
  const bool ref_ok = ec == std::errc{} && p == s.data() + s.size();
  const bool ok = parse_u32(s.data(), (uint32_t)s.size(), &got);
  ++total;
  if (ref_ok != ok || (ok && ref != got)) {
    if (++bad < 20) std::printf("MISMATCH u32 '%s'\n", s.c_str());
  }
}

int main(int argc, char** argv) {
  const long iters = argc > 1 ? std::atol(argv[1]) : 200000;
  std::mt19937_64 rng(12345);
  const char* fixed[] = {"1e400", "1e-400", "4.9e-324", "2.4703282292062328e-324",
                         "2.4703282292062327e-324", "2.5e-324", "-0", "+1", ".5", "5.", ".",
                         "-.e1", "1e", "1e+", "1E+5", "inf", "-Infinity", "INF", "nan", "-nan",
                         "nan(abc)", "nan()", "nan(", "nan(a)b", "nanx", "infinit", "0x10",
                         "1.7976931348623157e308", "1.7976931348623158e308",
                         "1.7976931348623159e308", "00012", "1e-5000", "0e99999", "-1e-400",
                         "1e999999999999999999", "", "-", "1..2", "1.2.3", "9007199254740993",
                         "9007199254740993.0000000000000000000000000001",
                         "2.2250738585072011e-308", "2.2250738585072012e-308",
                         "0.1", "0.30000000000000004", "123456789012345678901234567890e-20",
                         "1e23", "8.98846567431158e307", "4.4501477170144023e-308"};
  for (const char* s : fixed) check_f64(s);
  const char* fu[] = {"0", "1", "4294967295", "4294967296", "-1", "+1", "", "00001", "1a", "99999999999"};
  for (const char* s : fu) check_u32(s);
  char buf[2048];
  for (long it = 0; it < iters; ++it) {
    // (1) random doubles printed shortest and with extra digits
    uint64_t bits = rng();
    double d;
    std::memcpy(&d, &bits, 8);
    if (std::isnan(d)) continue;
    auto r = std::to_chars(buf, buf + sizeof buf, d);
    check_f64(std::string(buf, r.ptr));
    std::snprintf(buf, sizeof buf, "%.*e", (int)(rng() % 30), d);
    check_f64(buf);
    // (2) exact halfway points between neighbours (long double holds them),
    //     printed exactly, then nudged in the last digits / truncated
    if (std::isfinite(d) && d != 0) {
      double e = std::nextafter(d, INFINITY);
      if (std::isfinite(e)) {
        long double mid = ((long double)d + (long double)e) / 2;
        int prec = 20 + (int)(rng() % 760);
        std::snprintf(buf, sizeof buf, "%.*Le", prec, mid);
        std::string s(buf);
        check_f64(s);
        size_t epos = s.find('e');
        std::string m = s.substr(0, epos), ex = s.substr(epos);
        // truncate the mantissa at a random point
        size_t cut = 3 + rng() % (m.size() - 2);
        check_f64(m.substr(0, cut) + ex);
        // add a trailing 1 (just above halfway) and trailing zeros
        check_f64(m + "1" + ex);
        check_f64(m + "000" + ex);
        // decrement the last nonzero digit (just below halfway)
        std::string m2 = m;
        for (size_t k = m2.size(); k-- > 0;) {
          if (m2[k] >= '1' && m2[k] <= '9') { m2[k]--; break; }
        }
        check_f64(m2 + "999" + ex);
      }
    }
    // (3) random digit strings with random dots and exponents
    std::string s;
    if (rng() % 4 == 0) s += '-';
    int nd = 1 + (int)(rng() % 45);
    int dot = (int)(rng() % (nd + 2)) - 1;
    for (int k = 0; k < nd; ++k) {
      if (k == dot) s += '.';
      s += (char)('0' + (rng() % 10 < 3 ? 0 : rng() % 10));
    }
    if (rng() % 2) {
      s += (rng() % 2) ? 'e' : 'E';
      int sgn = rng() % 3;
      if (sgn == 1) s += '-';
      if (sgn == 2) s += '+';
      s += std::to_string(rng() % 360);
    }
    check_f64(s);
    // (4) junk characters
    if (rng() % 8 == 0) {
      std::string j = s;
      j[rng() % j.size()] = "x+-.e_( "[rng() % 8];
      check_f64(j);
    }
    // (5) indices
    std::string u = std::to_string(rng() % 6000000000ull);
    if (rng() % 10 == 0) u = "0" + u;
    check_u32(u);
  }
  std::printf("tns_parse_check: %ld tokens, %ld mismatches\n", total, bad);
  return bad ? 1 : 0;
}
