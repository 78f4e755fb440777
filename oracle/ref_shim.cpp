// TEST INFRASTRUCTURE ONLY — never linked into or called by the product.
//
// A C-ABI shim over the UNMODIFIED reference library (arxiv 2005.10427
// artifact, /root/reference/proj/src/*.cpp compiled in place by
// oracle/Makefile into oracle/_ref/libqref.so).  It lets the Python parity
// tests, the golden-fixture script and bench.py's cpu_baseline / --impl
// reference arm drive the reference's own public API:
//   quesadilla::transpose_inplace   (proj/include/quesadilla/transpose.hpp:59-61)
//   quesadilla::partial_sort         (proj/include/quesadilla/sort.hpp:32-33)
//   quesadilla::parallel_partial_sort(proj/include/quesadilla/parallel.hpp:35-37)
//   quesadilla::quesadilla_plan / prefix_plan (planner.hpp:27-34)
//   quesadilla::generate             (io.hpp:64)
//   quesadilla::detail::bucket_starts (sort.hpp:71-74)
//   quesadilla::pass_histogram / min_plan_bruteforce (planner.hpp:47-52)
// Exceptions are mapped to status codes: 0 ok, 1 std::invalid_argument,
// 2 std::out_of_range, 3 anything else.

#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "quesadilla/io.hpp"
#include "quesadilla/parallel.hpp"
#include "quesadilla/planner.hpp"
#include "quesadilla/sort.hpp"
#include "quesadilla/transpose.hpp"

using namespace quesadilla;

namespace {

thread_local std::string g_msg;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_msg = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_msg = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 3;
  }
}

CooTensor wrap(uint32_t rank, const uint32_t* dims, uint64_t nnz,
               const uint32_t* coords, const double* values) {
  CooTensor t;
  t.dims.assign(dims, dims + rank);
  t.coords.assign(coords, coords + nnz * rank);
  t.values.assign(values, values + nnz);
  return t;
}

void unwrap(const CooTensor& t, uint32_t* coords, double* values) {
  std::memcpy(coords, t.coords.data(), t.coords.size() * sizeof(uint32_t));
  std::memcpy(values, t.values.data(), t.values.size() * sizeof(double));
}

SortStrategy strategy_of(int kind, uint32_t k) {
  switch (kind) {
    case 0: return SortStrategy::quesadilla();
    case 1: return SortStrategy::top_k(k);
    case 2: return SortStrategy::full_radix();
    case 3: return SortStrategy::comparison_sort();
  }
  throw std::invalid_argument("bad strategy kind");
}

}  // namespace

extern "C" {

const char* qref_last_error(void) { return g_msg.c_str(); }

// In place on the caller's buffers.  steps_out (2 x max_steps u32: prefix_len,
// mode) receives opts.pass_log.  kind: 0 quesadilla, 1 topk, 2 radix, 3 cmp.
int qref_transpose(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                   uint32_t* coords, double* values, const uint32_t* target,
                   int kind, uint32_t k, uint32_t workers, int verify_input,
                   uint32_t* steps_out, uint32_t max_steps,
                   uint32_t* nsteps_out) {
  return guard([&] {
    CooTensor t = wrap(rank, dims, nnz, coords, values);
    std::vector<PlanStep> log;
    TransposeOptions opts;
    opts.verify_input = verify_input != 0;
    opts.parallel.workers = workers;
    opts.pass_log = &log;
    Workspace ws;
    Ordering tgt(std::vector<Mode>(target, target + rank));
    transpose_inplace(t, tgt, strategy_of(kind, k), ws, opts);
    unwrap(t, coords, values);
    if (nsteps_out) *nsteps_out = static_cast<uint32_t>(log.size());
    for (std::size_t i = 0; i < log.size() && i < max_steps; ++i) {
      steps_out[2 * i] = log[i].prefix_len;
      steps_out[2 * i + 1] = log[i].mode;
    }
  });
}

// The timed CPU baseline: the caller's tensor is restored by the caller; the
// Workspace handle is reused across calls like the CLI bench
// (proj/tools/main.cpp:198-213).
struct qref_ctx {
  CooTensor t;
  Workspace ws;
};

void* qref_ctx_create(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                      const uint32_t* coords, const double* values) {
  auto* c = new qref_ctx;
  c->t = wrap(rank, dims, nnz, coords, values);
  return c;
}

void qref_ctx_destroy(void* p) { delete static_cast<qref_ctx*>(p); }

// Copies the pristine buffers back into the context tensor (untimed part).
void qref_ctx_reset(void* p, const uint32_t* coords, const double* values) {
  auto* c = static_cast<qref_ctx*>(p);
  std::memcpy(c->t.coords.data(), coords, c->t.coords.size() * 4);
  std::memcpy(c->t.values.data(), values, c->t.values.size() * 8);
}

int qref_ctx_transpose(void* p, const uint32_t* target, uint32_t workers) {
  auto* c = static_cast<qref_ctx*>(p);
  return guard([&] {
    TransposeOptions opts;
    opts.parallel.workers = workers;
    Ordering tgt(std::vector<Mode>(target, target + c->t.rank()));
    transpose_inplace(c->t, tgt, SortStrategy::quesadilla(), c->ws, opts);
  });
}

void qref_ctx_read(void* p, uint32_t* coords, double* values) {
  unwrap(static_cast<qref_ctx*>(p)->t, coords, values);
}

int qref_partial_sort(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                      uint32_t* coords, double* values, const uint32_t* prefix,
                      uint32_t prefix_len, uint32_t mode, uint32_t workers) {
  return guard([&] {
    CooTensor t = wrap(rank, dims, nnz, coords, values);
    Workspace ws;
    std::vector<Mode> pre(prefix, prefix + prefix_len);
    if (workers == 1) {
      partial_sort(t, pre, mode, ws);
    } else {
      parallel_partial_sort(t, pre, mode, ws, ParallelConfig::with_workers(workers));
    }
    unwrap(t, coords, values);
  });
}

int qref_sort_rows_by(uint32_t rank, const uint32_t* dims, uint64_t nnz, uint32_t* coords,
                      double* values, uint64_t row_begin, uint64_t row_end,
                      const uint32_t* keys, uint32_t nkeys) {
  return guard([&] {
    CooTensor t = wrap(rank, dims, nnz, coords, values);
    std::vector<Mode> k(keys, keys + nkeys);
    sort_rows_by(t, row_begin, row_end, k);
    unwrap(t, coords, values);
  });
}

int qref_relabel_target(const uint32_t* source, const uint32_t* target, uint32_t rank,
                        uint32_t* out) {
  return guard([&] {
    Ordering s(std::vector<Mode>(source, source + rank));
    Ordering t(std::vector<Mode>(target, target + rank));
    Ordering o = relabel_target(s, t);
    for (uint32_t i = 0; i < rank; ++i) out[i] = o.at(i);
  });
}

// want == 0 selects quesadilla_plan, else prefix_plan(target, want).
int qref_plan(const uint32_t* target, uint32_t rank, uint32_t want,
              uint32_t* steps_out, uint32_t max_steps, uint32_t* nsteps_out) {
  return guard([&] {
    Ordering tgt(std::vector<Mode>(target, target + rank));
    SortPlan plan = want == 0 ? quesadilla_plan(tgt) : prefix_plan(tgt, want);
    *nsteps_out = static_cast<uint32_t>(plan.steps.size());
    for (std::size_t i = 0; i < plan.steps.size() && i < max_steps; ++i) {
      steps_out[2 * i] = plan.steps[i].prefix_len;
      steps_out[2 * i + 1] = plan.steps[i].mode;
    }
  });
}

int qref_min_plan_bruteforce(const uint32_t* target, uint32_t rank,
                             int* total, int* bucketed) {
  return guard([&] {
    PlanCost c = min_plan_bruteforce(Ordering(std::vector<Mode>(target, target + rank)));
    *total = c.total_passes;
    *bucketed = c.bucketed_passes;
  });
}

int qref_required_sort_count(const uint32_t* source, const uint32_t* target,
                             uint32_t rank, int* out) {
  return guard([&] {
    *out = required_sort_count(Ordering(std::vector<Mode>(source, source + rank)),
                               Ordering(std::vector<Mode>(target, target + rank)));
  });
}

// hist_out[i] = number of rank-r orderings needing i passes (i < max_len).
int qref_pass_histogram(uint32_t rank, long long* hist_out, uint32_t max_len) {
  return guard([&] {
    for (uint32_t i = 0; i < max_len; ++i) hist_out[i] = 0;
    for (auto [k, v] : pass_histogram(rank)) {
      if (static_cast<uint32_t>(k) < max_len) hist_out[k] = v;
    }
  });
}

// Reference generator (io.cpp:154-204), mt19937_64, canonicalised.
int qref_generate(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                  uint64_t seed, int distinct, uint32_t* coords_out,
                  double* values_out) {
  return guard([&] {
    GenSpec spec;
    spec.dims.assign(dims, dims + rank);
    spec.nnz = nnz;
    spec.seed = seed;
    spec.duplicates = distinct ? GenSpec::Duplicates::Distinct
                               : GenSpec::Duplicates::Allow;
    CooTensor t = generate(spec);
    unwrap(t, coords_out, values_out);
  });
}

// Start rows of maximal runs agreeing on `modes` (sort.cpp:136-147).
int qref_bucket_starts(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                       const uint32_t* coords, const double* values,
                       const uint32_t* modes, uint32_t nmodes,
                       uint64_t* starts_out, uint64_t* nstarts_out) {
  return guard([&] {
    CooTensor t = wrap(rank, dims, nnz, coords, values);
    std::vector<Mode> m(modes, modes + nmodes);
    auto s = detail::bucket_starts(t, m, 0, nnz);
    *nstarts_out = s.size();
    for (std::size_t i = 0; i < s.size(); ++i) starts_out[i] = s[i];
  });
}

int qref_is_sorted(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                   const uint32_t* coords, const double* values,
                   const uint32_t* order, int* out) {
  return guard([&] {
    CooTensor t = wrap(rank, dims, nnz, coords, values);
    *out = is_sorted_under(t, Ordering(std::vector<Mode>(order, order + rank)));
  });
}

unsigned qref_default_workers(void) { return ParallelConfig::default_workers(); }


// read_tns / write_tns (io.hpp:24-47).  ParseError -> 4 with its line().
static uint64_t g_parse_line = 0;
uint64_t qref_parse_error_line(void) { return g_parse_line; }
void* qref_read_tns(const char* path, const uint32_t* declared, uint32_t declared_rank,
                    int has_declared, int canonicalize, int* status) {
  CooTensor* out = nullptr;
  g_parse_line = 0;
  *status = guard([&] {
    try {
      ReadOptions o;
      o.canonicalize = canonicalize != 0;
      if (has_declared) o.declared_dims = std::vector<uint32_t>(declared, declared + declared_rank);
      out = new CooTensor(read_tns(path, o));
    } catch (const ParseError& e) {
      g_parse_line = e.line();
      throw std::runtime_error(std::string("PARSE:") + e.what());
    }
  });
  if (*status == 3 && g_msg.rfind("PARSE:", 0) == 0) {
    g_msg = g_msg.substr(6);
    *status = 4;
  }
  return out;
}
void qref_tensor_info(void* h, uint32_t* rank, uint64_t* nnz) {
  auto* t = static_cast<CooTensor*>(h);
  *rank = (uint32_t)t->rank();
  *nnz = t->nnz();
}
void qref_tensor_copy(void* h, uint32_t* dims, uint32_t* coords, double* values) {
  auto* t = static_cast<CooTensor*>(h);
  std::memcpy(dims, t->dims.data(), t->dims.size() * 4);
  std::memcpy(coords, t->coords.data(), t->coords.size() * 4);
  std::memcpy(values, t->values.data(), t->values.size() * 8);
}
void qref_tensor_free(void* h) { delete static_cast<CooTensor*>(h); }
int qref_write_tns(uint32_t rank, const uint32_t* dims, uint64_t nnz, const uint32_t* coords,
                   const double* values, const char* path) {
  return guard([&] { write_tns(wrap(rank, dims, nnz, coords, values), path); });
}

}  // extern "C"
