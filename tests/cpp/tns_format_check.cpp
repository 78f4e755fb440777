// TEST INFRASTRUCTURE: CPU self-check of the GPU .tns writer's formatting
// (paper_2005_10427_b200/csrc/tns_format.cuh, compiled here as host code)
// against the reference writer's conversion, std::to_chars (io.cpp:138-147),
// on random bit patterns, random decimals, integers, powers of two and
// boundary values.  Prints the mismatch count.
//   g++ -O2 -std=c++20 -I paper_2005_10427_b200/csrc tests/cpp/tns_format_check.cpp
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "tns_format.cuh"

static long bad = 0, total = 0;

static void check(double x) {
  char a[64], b[64];
  auto r = std::to_chars(a, a + 64, x);
  const uint32_t n = qb200::tns::format_f64(x, b);
  const uint32_t n2 = qb200::tns::format_f64(x, nullptr);
  ++total;
  if ((size_t)(r.ptr - a) != n || n2 != n || std::memcmp(a, b, n) != 0) {
    if (++bad < 20) {
      uint64_t u;
      std::memcpy(&u, &x, 8);
      std::printf("MISMATCH %016llx ref '%.*s' got '%.*s' (len %u/%u)\n", (unsigned long long)u,
                  (int)(r.ptr - a), a, (int)n, b, n, n2);
    }
  }
}

int main(int argc, char** argv) {
  const long iters = argc > 1 ? std::atol(argv[1]) : 1000000;
  std::mt19937_64 rng(99);
  const double fixed[] = {0.0, -0.0, INFINITY, -INFINITY, NAN, -NAN, 1.0, 0.1, 0.001, 0.0001,
                          1e-5, 1e16, 1e21, 1e22, 1e23, 12300000.0, 5e-324, 2.2250738585072014e-308,
                          1.7976931348623157e308, 9007199254740992.0, 4503599627370497.5,
                          1.2345678901234567e21, 123456789012345680000.0, 0.5, 100.0, 1e15,
                          123456.0, 1234567.0, 0.3, 2.0 / 3.0};
  for (double x : fixed) check(x);
  for (int e = -1074; e <= 1023; ++e) {
    check(std::ldexp(1.0, e));
    check(std::nextafter(std::ldexp(1.0, e), 0.0));
    check(std::nextafter(std::ldexp(1.0, e), INFINITY));
  }
  for (int e = -325; e <= 308; ++e) {
    check(std::pow(10.0, e));
    for (int k = 1; k < 10; ++k) check(k * std::pow(10.0, e));
  }
  for (long it = 0; it < iters; ++it) {
    uint64_t u = rng();
    double x;
    std::memcpy(&x, &u, 8);
    check(x);
    // integers and short decimals (fixed / scientific boundary cases)
    check((double)(int64_t)(rng() >> (rng() % 64)));
    const double base = (double)(rng() % 100000000) * std::pow(10.0, (int)(rng() % 40) - 20);
    check(base);
    check(std::uniform_real_distribution<double>(0, 1)(rng));
    check((double)(rng() >> 11) * 0x1.0p-53);
  }
  std::printf("tns_format_check: %ld values, %ld mismatches\n", total, bad);
  return bad ? 1 : 0;
}
