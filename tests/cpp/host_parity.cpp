// Host-utility parity (no GPU needed): the drop-in header's string parsers and
// formatters against the reference library's own, on valid strings and on the
// edge cases std::from_chars decides (overflow, signs, spaces, empty tokens).
// Built by oracle/Makefile into oracle/_ref/host_parity; run by
// tests/test_abi.py on CPU.  Reference: ordering.cpp:68-112, transpose.cpp:21-41.
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "quesadilla/ordering.hpp"
#include "quesadilla/transpose.hpp"
#include "quesadilla_b200.hpp"

namespace Q = quesadilla;
namespace B = quesadilla_b200;

static int failures = 0, checks = 0;

// outcome of a call as a string: the value it returned, or the exception class
// and message it threw (both must match the reference)
template <class F>
static std::string outcome(F&& f) {
  try {
    return "ok:" + f();
  } catch (const std::invalid_argument& e) {
    return std::string("invalid_argument:") + e.what();
  } catch (const std::out_of_range& e) {
    return std::string("out_of_range:") + e.what();
  } catch (const std::exception& e) {
    return std::string("other:") + e.what();
  }
}

static void expect_same(const std::string& a, const std::string& b, const std::string& what) {
  ++checks;
  if (a != b) {
    ++failures;
    std::printf("FAIL %s: reference '%s' vs drop-in '%s'\n", what.c_str(), a.c_str(), b.c_str());
  }
}

template <class M>
static std::string join(const M& modes) {
  std::string s;
  for (auto m : modes) s += std::to_string(m) + ".";
  return s;
}

int main() {
  const std::vector<std::string> orderings = {
      "1", "21", "321", "2134", "123456789", "1,2", "2,1,3", "10,9,8,7,6,5,4,3,2,1",
      // from_chars edge cases
      "4294967297,2", "4294967296,1", "4294967295,1", "99999999999999999999,1", "1,4294967297",
      "+1,2", "-1,2", " 1,2", "1 ,2", "1,,2", ",1", "1,", "0,1", "1,0", "01,2", "1,2a", "a",
      "0", "12a", "1 2", "", "11", "1,1", "3,1", "2,3"};
  for (const std::string& s : orderings)
    expect_same(outcome([&] { return join(Q::parse_ordering(s).modes()); }),
                outcome([&] { return join(B::parse_ordering(s).modes()); }),
                "parse_ordering('" + s + "')");
  for (Q::Mode r = 1; r <= 5; ++r)
    for (const Q::Ordering& t : Q::all_orderings(r))
      expect_same(Q::format_ordering(t), B::format_ordering(B::Ordering(t.modes())),
                  "format_ordering");
  const std::vector<std::string> strategies = {
      "quesadilla", "radix", "comparison", "qsort", "splatt", "top1", "top2", "top12",
      "top0", "top", "top-1", "top+2", "top 2", "top2 ", "top4294967295", "top4294967296",
      "top99999999999999999999", "top2x", "Top2", "", "radixx"};
  for (const std::string& s : strategies)
    expect_same(outcome([&] {
                  const auto st = Q::parse_strategy(s);
                  return std::string(st.name()) + "/" + std::to_string(st.k);
                }),
                outcome([&] {
                  const auto st = B::parse_strategy(s);
                  return std::string(st.name()) + "/" + std::to_string(st.k);
                }),
                "parse_strategy('" + s + "')");
  std::printf("%s: %d checks, %d failures\n", failures ? "FAIL" : "PASS", checks, failures);
  return failures ? 1 : 0;
}
