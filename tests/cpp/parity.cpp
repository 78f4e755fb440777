// C++ parity binary: the reference library (namespace quesadilla, compiled
// from /root/reference/proj/src into oracle/_ref/libqref.so) and the B200
// drop-in (namespace quesadilla_b200, include/quesadilla_b200.hpp over the
// C ABI) called side by side on identical tensors; every output compared bit
// for bit, pass logs and exception classes too.  Built by oracle/Makefile
// (test infrastructure), run by tests/test_cpp_gpu.py on the GPU box.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "quesadilla/io.hpp"
#include "quesadilla/planner.hpp"
#include "quesadilla/sort.hpp"
#include "quesadilla/transpose.hpp"
#include "quesadilla_b200.hpp"

namespace Q = quesadilla;
namespace B = quesadilla_b200;

static int failures = 0, checks = 0;

static B::CooTensor to_b(const Q::CooTensor& t) { return {t.dims, t.coords, t.values}; }

static bool same(const Q::CooTensor& a, const B::CooTensor& b) {
  return a.dims == b.dims && a.coords == b.coords && a.values.size() == b.values.size() &&
         std::memcmp(a.values.data(), b.values.data(), a.values.size() * 8) == 0;
}

static void expect(bool ok, const std::string& what) {
  ++checks;
  if (!ok) {
    ++failures;
    std::printf("FAIL %s\n", what.c_str());
  }
}

template <class F>
static int exc_class(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::out_of_range&) {
    return 2;
  } catch (...) {
    return 3;
  }
}

int main() {
  std::mt19937_64 rng(20261019);
  B::Workspace ws;
  // randomised equivalence over strategies (acceptance.cpp:128-184 style)
  for (Q::Mode r = 1; r <= 5; ++r) {
    for (int i = 0; i < 6; ++i) {
      Q::GenSpec spec;
      for (Q::Mode m = 0; m < r; ++m) spec.dims.push_back(1 + rng() % (i % 2 ? 9 : 3000));
      spec.nnz = rng() % 20000;
      spec.seed = rng();
      const Q::CooTensor t = Q::generate(spec);
      std::vector<Q::Mode> tm(r);
      for (Q::Mode m = 0; m < r; ++m) tm[m] = m;
      std::shuffle(tm.begin(), tm.end(), rng);
      const Q::Ordering qt(tm);
      const B::Ordering bt(tm);
      std::vector<std::pair<Q::SortStrategy, B::SortStrategy>> strats{
          {Q::SortStrategy::quesadilla(), B::SortStrategy::quesadilla()},
          {Q::SortStrategy::full_radix(), B::SortStrategy::full_radix()},
          {Q::SortStrategy::comparison_sort(), B::SortStrategy::comparison_sort()},
          {Q::SortStrategy::top_k(1), B::SortStrategy::top_k(1)}};
      for (auto& [qs, bs] : strats) {
        std::vector<Q::PlanStep> qlog;
        std::vector<B::PlanStep> blog;
        Q::TransposeOptions qo;
        qo.pass_log = &qlog;
        qo.parallel.workers = 4;
        B::TransposeOptions bo;
        bo.pass_log = &blog;
        const Q::CooTensor qa = Q::transpose(t, qt, qs, qo);
        B::CooTensor ba = to_b(t);
        B::transpose_inplace(ba, bt, bs, ws, bo);
        expect(same(qa, ba), "transpose " + qs.name() + " r=" + std::to_string(r));
        bool logs = qlog.size() == blog.size();
        for (std::size_t k = 0; logs && k < qlog.size(); ++k)
          logs = qlog[k].prefix_len == blog[k].prefix_len && qlog[k].mode == blog[k].mode;
        expect(logs, "pass_log " + qs.name());
      }
      // the per-step primitive with an arbitrary prefix
      if (r >= 2) {
        std::vector<Q::Mode> pre(tm.begin(), tm.begin() + rng() % r);
        const Q::Mode mode = tm.back();
        Q::CooTensor qa = t;
        Q::Workspace qws;
        Q::partial_sort(qa, pre, mode, qws);
        B::CooTensor ba = to_b(t);
        B::partial_sort(ba, pre, mode, ws);
        expect(same(qa, ba), "partial_sort r=" + std::to_string(r));
      }
    }
  }
  // planner equality for every ordering up to rank 6
  for (Q::Mode r = 1; r <= 6; ++r)
    for (const Q::Ordering& o : Q::all_orderings(r)) {
      const auto qp = Q::quesadilla_plan(o).steps;
      const auto bp = B::quesadilla_plan(B::Ordering(o.modes())).steps;
      bool eq = qp.size() == bp.size();
      for (std::size_t k = 0; eq && k < qp.size(); ++k)
        eq = qp[k].prefix_len == bp[k].prefix_len && qp[k].mode == bp[k].mode;
      expect(eq, "plan");
    }
  // exception classes (sort.cpp:153-166, 26-30; transpose.cpp:83-103)
  {
    Q::CooTensor q{{2, 2}, {0, 1}, {1.0}};
    B::CooTensor b = to_b(q);
    Q::Workspace qws;
    expect(exc_class([&] { Q::partial_sort(q, std::vector<Q::Mode>{1}, 1, qws); }) ==
               exc_class([&] { B::partial_sort(b, {1}, 1, ws); }),
           "exc prefix contains mode");
    Q::CooTensor q2{{4, 4}, {0, 9, 1, 0}, {1.0, 2.0}};
    B::CooTensor b2 = to_b(q2);
    expect(exc_class([&] { Q::partial_sort(q2, {}, 1, qws); }) == 2 &&
               exc_class([&] { B::partial_sort(b2, {}, 1, ws); }) == 2,
           "exc out_of_range");
    expect(exc_class([&] { Q::topk_transpose(q, Q::Ordering({1, 0}), 0); }) ==
               exc_class([&] { B::topk_transpose(b, B::Ordering({1, 0}), 0); }),
           "exc top-k");
  }
  // sort_rows_by over row ranges (sort.cpp:203-235), any key list
  for (int i = 0; i < 20; ++i) {
    Q::GenSpec spec;
    const Q::Mode r = 1 + rng() % 4;
    for (Q::Mode m = 0; m < r; ++m) spec.dims.push_back(1 + rng() % 500);
    spec.nnz = rng() % 30000;
    spec.seed = rng();
    Q::CooTensor q = Q::generate(spec);
    B::CooTensor b = to_b(q);
    std::vector<Q::Mode> keys(rng() % (2 * r + 1));
    for (auto& k : keys) k = rng() % r;
    const std::size_t lo = q.nnz() ? rng() % (q.nnz() + 1) : 0;
    const std::size_t hi = lo + (q.nnz() - lo ? rng() % (q.nnz() - lo + 1) : 0);
    Q::sort_rows_by(q, lo, hi, keys);
    B::sort_rows_by(b, lo, hi, keys, ws);
    expect(same(q, b), "sort_rows_by r=" + std::to_string(r));
  }
  // host utilities of the public headers
  for (Q::Mode r = 1; r <= 4; ++r)
    for (const Q::Ordering& s : Q::all_orderings(r))
      for (const Q::Ordering& t : Q::all_orderings(r)) {
        expect(Q::relabel_target(s, t).modes() ==
                   B::relabel_target(B::Ordering(s.modes()), B::Ordering(t.modes())).modes(),
               "relabel_target");
        expect(Q::format_ordering(t) == B::format_ordering(B::Ordering(t.modes())), "format");
        expect(Q::parse_ordering(Q::format_ordering(t)).modes() ==
                   B::parse_ordering(Q::format_ordering(t)).modes(),
               "parse");
      }
  for (const char* name : {"quesadilla", "top2", "radix", "comparison", "splatt", "qsort"})
    expect(Q::parse_strategy(name).name() == B::parse_strategy(name).name(), "parse_strategy");
  expect(exc_class([&] { Q::parse_strategy("top0"); }) ==
             exc_class([&] { B::parse_strategy("top0"); }),
         "parse_strategy error");
  {
    Q::GenSpec spec;
    spec.dims = {30, 40, 50};
    spec.nnz = 5000;
    spec.seed = 7;
    const Q::CooTensor q = Q::generate(spec);
    const B::CooTensor b = to_b(q);
    for (const Q::Ordering& o : Q::all_orderings(3))
      expect(Q::is_sorted_under(q, o) == B::is_sorted_under(b, B::Ordering(o.modes())),
             "is_sorted_under");
    Q::CooTensor qb = q;
    B::CooTensor bb = b;
    qb.coords[7] = 99;
    bb.coords[7] = 99;
    expect(exc_class([&] { qb.check_valid(); }) == exc_class([&] { bb.check_valid(); }) &&
               exc_class([&] { bb.check_valid(); }) == 1,
           "check_valid");
  }
  {  // io.hpp read_tns: reference reader vs the GPU reader on the same files
    Q::GenSpec spec;
    spec.dims = {300, 20, 4000};
    spec.nnz = 20000;
    spec.seed = 11;
    Q::CooTensor q = Q::generate(spec);
    std::shuffle(q.values.begin(), q.values.end(), rng);
    for (auto& v : q.values) v = std::ldexp(v, (int)(rng() % 400) - 200);
    const std::string path = "/tmp/qd_parity_read.tns";
    Q::write_tns(q, path);
    for (int canon = 0; canon < 2; ++canon) {
      Q::ReadOptions qo;
      qo.canonicalize = canon;
      B::ReadOptions bo;
      bo.canonicalize = canon;
      expect(same(Q::read_tns(path, qo), B::read_tns(path, bo)), "read_tns rows");
      qo.declared_dims = std::vector<std::uint32_t>{300, 25, 4000};
      bo.declared_dims = qo.declared_dims;
      expect(same(Q::read_tns(path, qo), B::read_tns(path, bo)), "read_tns declared");
    }
    {
      std::ofstream f(path, std::ios::trunc);
      f << "1 1 1 1.0\n# c\n2 2 2 2.0\n3 0 3 3.0\n";
    }
    std::string qw, bw;
    std::size_t ql = 0, bl = 0;
    try { Q::read_tns(path); } catch (const Q::ParseError& e) { qw = e.what(); ql = e.line(); }
    try { B::read_tns(path); } catch (const B::ParseError& e) { bw = e.what(); bl = e.line(); }
    expect(!qw.empty() && qw == bw && ql == bl && ql == 4, "read_tns ParseError");
    // write_tns: the GPU writer's bytes equal the reference writer's
    {
      const std::string p1 = "/tmp/qd_parity_w1.tns", p2 = "/tmp/qd_parity_w2.tns";
      Q::write_tns(q, p1);
      B::write_tns(to_b(q), p2);
      std::ifstream f1(p1, std::ios::binary), f2(p2, std::ios::binary);
      const std::string s1((std::istreambuf_iterator<char>(f1)), std::istreambuf_iterator<char>());
      const std::string s2((std::istreambuf_iterator<char>(f2)), std::istreambuf_iterator<char>());
      expect(!s1.empty() && s1 == s2, "write_tns bytes");
      std::remove(p1.c_str());
      std::remove(p2.c_str());
    }
    std::remove(path.c_str());
  }
  std::printf("%s %d checks, %d failures\n", failures ? "FAIL" : "PASS", checks, failures);
  return failures ? 1 : 0;
}
