// quesadilla_b200.hpp — C++ drop-in for the reference's transpose API
// (arxiv 2005.10427 artifact, proj/include/quesadilla/*.hpp), header-only
// over the C ABI in quesadilla_b200.h.  Same names, argument meaning and
// exception classes as namespace quesadilla; a caller switches by changing
// the namespace (and linking libquesadilla_b200.so).  Every transpose runs as
// sm_100a kernels; there is no CPU path.
//
//   reference                                  here
//   quesadilla::Ordering (ordering.hpp:38)     quesadilla_b200::Ordering
//   quesadilla::CooTensor (coo.hpp:16)         quesadilla_b200::CooTensor
//   quesadilla::PlanStep / SortPlan (plan.hpp) quesadilla_b200::PlanStep / SortPlan
//   quesadilla_plan / prefix_plan (planner.hpp:27-34)
//   SortStrategy / TransposeOptions (transpose.hpp:18-54)
//   Workspace (sort.hpp:14)                    device workspace (one GPU)
//   transpose_inplace / transpose (transpose.hpp:59-66)
//   partial_sort (sort.hpp:32) / parallel_partial_sort (parallel.hpp:35)
//   read_tns / write_tns / ParseError / ReadOptions (io.hpp:15-47)
#pragma once

#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <utility>
#include <vector>

#include "quesadilla_b200.h"

namespace quesadilla_b200 {

using Mode = std::uint32_t;
inline constexpr Mode kMaxRank = QD_MAX_RANK;

namespace detail {
inline void check(qd_status s) {
  switch (s) {
    case QD_OK: return;
    case QD_INVALID_ARGUMENT: throw std::invalid_argument(qd_last_error());
    case QD_OUT_OF_RANGE: throw std::out_of_range(qd_last_error());
    default: throw std::runtime_error(std::string("quesadilla_b200: ") + qd_last_error());
  }
}
}  // namespace detail

class Ordering {
 public:
  explicit Ordering(std::vector<Mode> modes) : modes_(std::move(modes)) {
    const std::size_t r = modes_.size();
    // the reference's checks and messages (ordering.cpp:13-31)
    if (r == 0 || r > kMaxRank)
      throw std::invalid_argument("ordering rank must be in 1.." + std::to_string(kMaxRank));
    std::uint64_t seen = 0;
    for (Mode m : modes_) {
      if (m >= r)
        throw std::invalid_argument("ordering contains mode " + std::to_string(m) + " outside 0.." +
                                    std::to_string(r - 1));
      if (seen & (std::uint64_t{1} << m))
        throw std::invalid_argument("ordering repeats mode " + std::to_string(m));
      seen |= std::uint64_t{1} << m;
    }
  }
  static Ordering simple(Mode rank) {
    std::vector<Mode> m(rank);
    for (Mode i = 0; i < rank; ++i) m[i] = i;
    return Ordering(std::move(m));
  }
  Mode rank() const { return static_cast<Mode>(modes_.size()); }
  Mode at(std::size_t i) const { return modes_[i]; }
  const std::vector<Mode>& modes() const { return modes_; }
  auto begin() const { return modes_.begin(); }
  auto end() const { return modes_.end(); }
  std::size_t position_of(Mode m) const {
    for (std::size_t i = 0; i < modes_.size(); ++i)
      if (modes_[i] == m) return i;
    throw std::invalid_argument("mode not in ordering");
  }
  bool is_simple() const {
    for (std::size_t i = 0; i < modes_.size(); ++i)
      if (modes_[i] != i) return false;
    return true;
  }
  friend bool operator==(const Ordering&, const Ordering&) = default;

 private:
  std::vector<Mode> modes_;
};

// all rank! orderings in lexicographic order (ordering.cpp all_orderings)
inline std::vector<Ordering> all_orderings(Mode rank) {
  if (rank < 1 || rank > 8) throw std::invalid_argument("all_orderings supports rank 1..8");
  std::vector<Mode> m(rank);
  for (Mode i = 0; i < rank; ++i) m[i] = i;
  std::vector<Ordering> out;
  do out.emplace_back(m);
  while (std::next_permutation(m.begin(), m.end()));
  return out;
}

// "2134" (1-based digits) or "10,2,1" (ordering.hpp parse_ordering)
inline Ordering parse_ordering(std::string_view text) {
  if (text.empty()) throw std::invalid_argument("empty ordering");
  std::vector<Mode> m;
  if (text.find(',') != std::string_view::npos) {
    std::size_t pos = 0;
    for (;;) {
      const std::size_t comma = text.find(',', pos);
      const std::string_view tok = text.substr(pos, comma == std::string_view::npos
                                                        ? std::string_view::npos : comma - pos);
      // std::from_chars like ordering.cpp:77-83: no sign, no spaces, and a
      // value that overflows unsigned is rejected (not wrapped)
      unsigned v = 0;
      const auto [ptr, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
      if (ec != std::errc{} || ptr != tok.data() + tok.size() || v == 0) throw std::invalid_argument("bad ordering element '" + std::string(tok) + "'");
      m.push_back(static_cast<Mode>(v - 1));
      if (comma == std::string_view::npos) break;
      pos = comma + 1;
    }
  } else {
    for (char ch : text) {
      if (ch < '1' || ch > '9')
        throw std::invalid_argument("ordering digits must be 1-9; use the comma form for larger ranks");
      m.push_back(static_cast<Mode>(ch - '1'));
    }
  }
  return Ordering(std::move(m));
}

inline std::string format_ordering(const Ordering& o) {
  std::string out;
  for (Mode m : o) {
    if (o.rank() <= 9) {
      out.push_back(static_cast<char>('1' + m));
    } else {
      if (!out.empty()) out.push_back(',');
      out += std::to_string(m + 1);
    }
  }
  return out;
}

// f(ordering, p): the modes placed before p (planner.cpp follow_set), as a bit set
class ModeSet {
 public:
  constexpr ModeSet() = default;
  constexpr void insert(Mode m) { bits_ |= std::uint64_t{1} << m; }
  constexpr bool contains(Mode m) const { return (bits_ >> m) & 1u; }
  constexpr bool subset_of(ModeSet o) const { return (bits_ & ~o.bits_) == 0; }
  constexpr bool empty() const { return bits_ == 0; }
  int size() const { return __builtin_popcountll(bits_); }
  constexpr std::uint64_t bits() const { return bits_; }
  friend constexpr bool operator==(ModeSet, ModeSet) = default;

 private:
  std::uint64_t bits_ = 0;
};
inline ModeSet follow_set(const Ordering& ord, Mode p) {
  ModeSet s;
  for (Mode m : ord) {
    if (m == p) return s;
    s.insert(m);
  }
  throw std::invalid_argument("mode not in ordering");
}

// Planning from a non-simple source (planner.hpp relabel_target)
inline Ordering relabel_target(const Ordering& source, const Ordering& target) {
  if (source.rank() != target.rank()) throw std::invalid_argument("source and target ranks differ");
  std::vector<Mode> out(target.rank());
  detail::check(qd_relabel_target(source.modes().data(), target.modes().data(), target.rank(),
                                  out.data()));
  return Ordering(std::move(out));
}

struct PlanStep {
  Mode prefix_len = 0;
  Mode mode = 0;
  bool bucketed() const { return prefix_len > 0; }
  friend bool operator==(const PlanStep&, const PlanStep&) = default;
};

struct SortPlan {
  Ordering target;
  std::vector<PlanStep> steps;
};

struct PlanCost {
  int total_passes = 0;
  int bucketed_passes = 0;
  friend bool operator==(const PlanCost&, const PlanCost&) = default;
};

struct CooTensor {
  std::vector<std::uint32_t> dims;
  std::vector<std::uint32_t> coords;  // nnz * rank, row-major
  std::vector<double> values;         // nnz
  Mode rank() const { return static_cast<Mode>(dims.size()); }
  std::size_t nnz() const { return values.size(); }
  std::uint32_t coord(std::size_t row, Mode mode) const { return coords[row * dims.size() + mode]; }
  // coo.cpp check_valid: shapes, positive dims, every coordinate < its dim
  void check_valid() const {
    const std::size_t r = dims.size();
    if (r == 0) throw std::invalid_argument("tensor rank must be positive");
    for (std::size_t m = 0; m < r; ++m)
      if (dims[m] == 0)
        throw std::invalid_argument("dimension of mode " + std::to_string(m) + " must be positive");
    if (coords.size() != values.size() * r)
      throw std::invalid_argument("coordinate storage does not match value count");
    for (std::size_t j = 0; j < values.size(); ++j)
      for (std::size_t m = 0; m < r; ++m)
        if (coords[j * r + m] >= dims[m])
          throw std::invalid_argument("coordinate out of range in row " + std::to_string(j) +
                                      ", mode " + std::to_string(m));
  }
  friend bool operator==(const CooTensor&, const CooTensor&) = default;
};

// coo.hpp is_sorted_under (host); the device check is qd_is_sorted_device
inline bool is_sorted_under(const CooTensor& t, const Ordering& ord) {
  if (ord.rank() != t.rank()) throw std::invalid_argument("ordering rank does not match tensor rank");
  const std::size_t r = t.rank();
  for (std::size_t j = 1; j < t.nnz(); ++j)
    for (Mode m : ord) {
      const std::uint32_t a = t.coords[(j - 1) * r + m], b = t.coords[j * r + m];
      if (a != b) {
        if (a > b) return false;
        break;
      }
    }
  return true;
}

namespace detail {
inline SortPlan plan_call(const Ordering& target, Mode want) {
  std::vector<qd_plan_step> buf(4096);
  std::uint32_t n = 0;
  if (want == 0)
    check(qd_quesadilla_plan(target.modes().data(), target.rank(), buf.data(), 4096, &n));
  else
    check(qd_prefix_plan(target.modes().data(), target.rank(), want, buf.data(), 4096, &n));
  SortPlan p{target, {}};
  for (std::uint32_t i = 0; i < n; ++i) p.steps.push_back({buf[i].prefix_len, buf[i].mode});
  return p;
}
}  // namespace detail

inline SortPlan quesadilla_plan(const Ordering& target) { return detail::plan_call(target, 0); }
inline SortPlan prefix_plan(const Ordering& target, Mode prefix_len) {
  if (prefix_len < 1 || prefix_len > target.rank())
    throw std::invalid_argument("prefix length must be in 1..rank");
  return detail::plan_call(target, prefix_len);
}
inline int required_sort_count(const Ordering& source, const Ordering& target) {
  if (source.rank() != target.rank()) throw std::invalid_argument("source and target ranks differ");
  int out = 0;
  detail::check(qd_required_sort_count(source.modes().data(), target.modes().data(),
                                       target.rank(), &out));
  return out;
}
inline Ordering apply_transition(const Ordering& current, const PlanStep& step) {
  std::vector<Mode> next(current.rank());
  detail::check(qd_apply_transition(current.modes().data(), current.rank(),
                                    qd_plan_step{step.prefix_len, step.mode}, next.data()));
  return Ordering(std::move(next));
}
inline Ordering simulate_plan(const SortPlan& plan) {
  Ordering o = Ordering::simple(plan.target.rank());
  for (const PlanStep& s : plan.steps) o = apply_transition(o, s);
  return o;
}
inline PlanCost plan_cost(const SortPlan& plan) {
  PlanCost c;
  c.total_passes = static_cast<int>(plan.steps.size());
  for (const PlanStep& s : plan.steps) c.bucketed_passes += s.bucketed();
  return c;
}

struct SortStrategy {
  enum class Kind { Quesadilla, TopK, FullRadix, ComparisonSort };
  Kind kind = Kind::Quesadilla;
  Mode k = 0;
  static SortStrategy quesadilla() { return {Kind::Quesadilla, 0}; }
  static SortStrategy top_k(Mode k) { return {Kind::TopK, k}; }
  static SortStrategy splatt_style() { return top_k(1); }
  static SortStrategy full_radix() { return {Kind::FullRadix, 0}; }
  static SortStrategy comparison_sort() { return {Kind::ComparisonSort, 0}; }
  std::string name() const {
    switch (kind) {
      case Kind::Quesadilla: return "quesadilla";
      case Kind::TopK: return "top" + std::to_string(k);
      case Kind::FullRadix: return "radix";
      case Kind::ComparisonSort: return "comparison";
    }
    return "?";
  }
  qd_strategy_kind c_kind() const {
    switch (kind) {
      case Kind::Quesadilla: return QD_QUESADILLA;
      case Kind::TopK: return QD_TOPK;
      case Kind::FullRadix: return QD_FULL_RADIX;
      default: return QD_COMPARISON_SORT;
    }
  }
  friend bool operator==(const SortStrategy&, const SortStrategy&) = default;
};

// transpose.hpp parse_strategy: quesadilla, top<K>, radix, comparison, splatt, qsort
inline SortStrategy parse_strategy(std::string_view name) {
  if (name == "quesadilla") return SortStrategy::quesadilla();
  if (name == "radix") return SortStrategy::full_radix();
  if (name == "comparison" || name == "qsort") return SortStrategy::comparison_sort();
  if (name == "splatt") return SortStrategy::splatt_style();
  if (name.size() > 3 && name.substr(0, 3) == "top") {
    // std::from_chars like transpose.cpp:30-36 (overflow rejected)
    unsigned k = 0;
    const char* last = name.data() + name.size();
    const auto [ptr, ec] = std::from_chars(name.data() + 3, last, k);
    if (ec == std::errc{} && ptr == last && k >= 1) return SortStrategy::top_k(static_cast<Mode>(k));
  }
  throw std::invalid_argument("unknown strategy '" + std::string(name) +
                              "' (expected quesadilla, top<K>, radix, comparison, splatt or qsort)");
}

inline PlanCost strategy_pass_cost(const SortStrategy& s, const Ordering& target) {
  PlanCost c;
  detail::check(qd_strategy_pass_cost(s.c_kind(), s.k, target.modes().data(), target.rank(),
                                      &c.total_passes, &c.bucketed_passes));
  return c;
}

struct ParallelConfig {
  unsigned workers = 1;  // accepted for API parity; 0 is rejected like the reference
  static ParallelConfig serial() { return {}; }
  static ParallelConfig with_workers(unsigned p) { return {p}; }
  // QUESADILLA_WORKERS or the host's hardware threads (parallel.cpp); the
  // GPU ignores the count, but callers that size CPU work by it keep working
  static unsigned default_workers() {
    if (const char* e = std::getenv("QUESADILLA_WORKERS")) {
      const long v = std::strtol(e, nullptr, 10);
      if (v >= 1) return static_cast<unsigned>(v);
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? hw : 1u;
  }
};

struct TransposeOptions {
  bool verify_input = false;
  ParallelConfig parallel = ParallelConfig::serial();
  std::vector<PlanStep>* pass_log = nullptr;
  // device extra: the output's leading-mode run starts + nnz (CSF pos array)
  std::vector<std::uint64_t>* boundaries = nullptr;
};

// Device workspace (cached HBM buffers on one GPU); reuse across calls,
// never concurrently.
class Workspace {
 public:
  explicit Workspace(int device = 0) { detail::check(qd_workspace_create(device, &ws_)); }
  ~Workspace() { qd_workspace_destroy(ws_); }
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;
  qd_workspace* get() const { return ws_; }
  // wait for every transpose_inplace_async on this workspace
  void synchronize() { detail::check(qd_workspace_synchronize(ws_)); }
  // slices the last synchronous host-buffer call was pipelined in (1: whole tensor)
  std::uint64_t slices() const { return qd_workspace_slices(ws_); }

 private:
  qd_workspace* ws_ = nullptr;
};

// transpose_inplace that returns after enqueueing the input copy; the device
// work and output copy complete by ws.synchronize(), which throws the first
// device-side error (that call's tensor untouched).  Consecutive calls
// overlap copies with device work.  t must outlive the synchronize; no
// bucket boundaries in this form.
inline void transpose_inplace_async(CooTensor& t, const Ordering& target, const SortStrategy& s,
                                    Workspace& ws, const TransposeOptions& opts = {}) {
  if (target.rank() != t.rank())
    throw std::invalid_argument("target ordering rank does not match tensor");
  if (opts.boundaries)
    throw std::invalid_argument("bucket boundaries are only reported by transpose_inplace");
  std::vector<qd_plan_step> log(4096);
  std::uint32_t nlog = 0;
  qd_options o{};
  o.verify_input = opts.verify_input;
  o.workers = opts.parallel.workers;
  o.pass_log = log.data();
  o.pass_log_capacity = 4096;
  o.pass_log_len = &nlog;
  detail::check(qd_transpose_inplace_async(t.rank(), t.dims.data(), t.nnz(), t.coords.data(),
                                           t.values.data(), target.modes().data(), s.c_kind(),
                                           s.k, &o, ws.get()));
  if (opts.pass_log)
    for (std::uint32_t i = 0; i < nlog; ++i) opts.pass_log->push_back({log[i].prefix_len, log[i].mode});
}

inline void transpose_inplace(CooTensor& t, const Ordering& target, const SortStrategy& s,
                              Workspace& ws, const TransposeOptions& opts = {}) {
  if (target.rank() != t.rank())
    throw std::invalid_argument("target ordering rank does not match tensor");
  std::vector<qd_plan_step> log(4096);
  std::uint32_t nlog = 0;
  std::vector<std::uint64_t> bounds;
  std::uint64_t nb = 0;
  qd_options o{};
  o.verify_input = opts.verify_input;
  o.workers = opts.parallel.workers;
  o.pass_log = log.data();
  o.pass_log_capacity = 4096;
  o.pass_log_len = &nlog;
  if (opts.boundaries) {
    bounds.resize(t.nnz() + 1);
    o.boundaries = bounds.data();
    o.n_boundaries = &nb;
  }
  detail::check(qd_transpose_inplace(t.rank(), t.dims.data(), t.nnz(), t.coords.data(),
                                     t.values.data(), target.modes().data(), s.c_kind(), s.k, &o,
                                     ws.get()));
  if (opts.pass_log)
    for (std::uint32_t i = 0; i < nlog; ++i) opts.pass_log->push_back({log[i].prefix_len, log[i].mode});
  if (opts.boundaries) opts.boundaries->assign(bounds.begin(), bounds.begin() + nb);
}

inline CooTensor transpose(const CooTensor& t, const Ordering& target, const SortStrategy& s,
                           const TransposeOptions& opts = {}) {
  CooTensor out = t;
  Workspace ws;
  transpose_inplace(out, target, s, ws, opts);
  return out;
}

inline CooTensor full_radix_transpose(const CooTensor& t, const Ordering& target,
                                      const TransposeOptions& opts = {}) {
  return transpose(t, target, SortStrategy::full_radix(), opts);
}
inline CooTensor comparison_transpose(const CooTensor& t, const Ordering& target) {
  return transpose(t, target, SortStrategy::comparison_sort());
}
inline CooTensor topk_transpose(const CooTensor& t, const Ordering& target, Mode k,
                                const TransposeOptions& opts = {}) {
  return transpose(t, target, SortStrategy::top_k(k), opts);
}

// sort.hpp sort_rows_by: stable sort of rows [row_begin, row_end) by key_modes
inline void sort_rows_by(CooTensor& t, std::size_t row_begin, std::size_t row_end,
                         const std::vector<Mode>& key_modes, Workspace& ws) {
  detail::check(qd_sort_rows_by(t.rank(), t.dims.data(), t.nnz(), t.coords.data(), t.values.data(),
                                row_begin, row_end, key_modes.data(),
                                static_cast<std::uint32_t>(key_modes.size()), ws.get()));
}

inline void partial_sort(CooTensor& t, const std::vector<Mode>& prefix, Mode mode, Workspace& ws) {
  detail::check(qd_partial_sort(t.rank(), t.dims.data(), t.nnz(), t.coords.data(),
                                t.values.data(), prefix.data(),
                                static_cast<std::uint32_t>(prefix.size()), mode, ws.get()));
}
inline void parallel_partial_sort(CooTensor& t, const std::vector<Mode>& prefix, Mode mode,
                                  Workspace& ws, const ParallelConfig& cfg) {
  if (cfg.workers == 0) throw std::invalid_argument("worker count must be at least 1");
  partial_sort(t, prefix, mode, ws);
}

// ---- io.hpp: the .tns text format -------------------------------------------
class ParseError : public std::runtime_error {  // io.hpp:15-22
 public:
  ParseError(std::size_t line, const std::string& what_text)
      : std::runtime_error(what_text), line_(line) {}
  std::size_t line() const { return line_; }

 private:
  std::size_t line_;
};

struct ReadOptions {  // io.hpp:24-35
  bool canonicalize = true;
  std::optional<std::vector<std::uint32_t>> declared_dims;
};

// read_tns over bytes already in memory; parsing and canonicalisation on the GPU.
inline CooTensor read_tns_text(std::string_view text, const ReadOptions& opts, Workspace& ws) {
  qd_tns_tensor t{};
  qd_tns_error e{};
  const auto& d = opts.declared_dims;
  const qd_status s = qd_read_tns(text.data(), text.size(), d ? d->data() : nullptr,
                                  d ? static_cast<std::uint32_t>(d->size()) : 0, d ? 1 : 0,
                                  opts.canonicalize ? 1 : 0, &t, &e, ws.get());
  if (s == QD_PARSE_ERROR) throw ParseError(e.line, qd_last_error());
  detail::check(s);
  CooTensor out;
  out.dims.assign(t.dims, t.dims + t.rank);
  out.coords.assign(t.coords, t.coords + t.nnz * t.rank);
  out.values.assign(t.values, t.values + t.nnz);
  qd_tns_free(&t);
  return out;
}

// io.hpp:40-41 read_tns(path, opts): the file is read on the host.
inline CooTensor read_tns(const std::filesystem::path& path, const ReadOptions& opts = {}) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open '" + path.string() + "' for reading");
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  Workspace ws;
  return read_tns_text(text, opts, ws);
}

// io.hpp:47 write_tns: the text is formatted on the GPU, then written here.
inline void write_tns(const CooTensor& tensor, const std::filesystem::path& path) {
  std::ofstream out(path, std::ios::trunc | std::ios::binary);
  if (!out) throw std::runtime_error("cannot open '" + path.string() + "' for writing");
  Workspace ws;
  char* text = nullptr;
  std::uint64_t n = 0;
  detail::check(qd_write_tns(tensor.rank(), tensor.nnz(), tensor.coords.data(),
                             tensor.values.data(), &text, &n, ws.get()));
  out.write(text, static_cast<std::streamsize>(n));
  qd_text_free(text);
  if (!out) throw std::runtime_error("failed writing '" + path.string() + "'");
}

}  // namespace quesadilla_b200
