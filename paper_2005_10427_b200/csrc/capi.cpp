// extern "C" layer: the drop-in boundary (include/quesadilla_b200.h).
// Validation mirrors the reference's argument checks so the same calls fail
// with the same exception class (mapped to qd_status):
//   transpose.cpp:83-89 (rank, verify_input), transpose.cpp:101-103 (top-K),
//   sort.cpp:153-166 (partial_sort args), parallel.cpp:161-163 (workers).
#include <sys/mman.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cstring>
#include <string>
#include <vector>

#include "internal.hpp"

using namespace qb200;

namespace {

thread_local std::string g_msg;
thread_local uint64_t g_row = 0;
thread_local uint32_t g_mode = 0;

template <class F>
qd_status guard(F&& f) {
  try {
    f();
    g_msg.clear();
    return QD_OK;
  } catch (const Error& e) {
    g_msg = e.what();
    g_row = e.row;
    g_mode = e.mode;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_msg = "host allocation failed";
    return QD_CUDA_ERROR;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return QD_CUDA_ERROR;
  }
}

void check_tensor(uint32_t rank, const uint32_t* dims, uint64_t nnz, const void* c,
                  const void* v) {
  if (rank == 0 || rank > QD_MAX_RANK) invalid("tensor rank must be in 1..64");
  if (!dims) invalid("dims is null");
  for (uint32_t m = 0; m < rank; ++m)
    if (dims[m] == 0) invalid("dimension of mode " + std::to_string(m) + " must be positive");
  if (nnz && (!c || !v)) invalid("coordinate or value buffer is null");
  if (nnz >= (uint64_t{1} << 32))
    invalid("nnz must be below 2^32 (the reference's u32 counters, sort.hpp:15-18)");
}

void log_steps(const qd_options* o, const std::vector<Step>& steps) {
  if (!o || !o->pass_log_len) return;
  *o->pass_log_len = static_cast<uint32_t>(steps.size());
  if (!o->pass_log) return;
  for (size_t i = 0; i < steps.size() && i < o->pass_log_capacity; ++i)
    o->pass_log[i] = {steps[i].prefix_len, steps[i].mode};
}

// ParallelConfig{0} is rejected where the reference would reach
// parallel_partial_sort (any executed step, parallel.cpp:161-163) or the
// top-K bucket phase (parallel.cpp:194-196); elsewhere it is never read.
void check_workers(const qd_options* o, qd_strategy_kind kind, const std::vector<Step>& steps) {
  if (o && o->workers == 0 && (!steps.empty() || kind == QD_TOPK))
    invalid("worker count must be at least 1");
}

void copy_steps(const std::vector<Step>& s, qd_plan_step* out, uint32_t cap, uint32_t* n) {
  if (n) *n = static_cast<uint32_t>(s.size());
  for (size_t i = 0; i < s.size() && i < cap && out; ++i) out[i] = {s[i].prefix_len, s[i].mode};
}

std::vector<Group> partial_sort_group(uint32_t rank, const uint32_t* prefix, uint32_t plen,
                                      uint32_t mode) {
  // validate_sort_args, sort.cpp:153-166
  if (mode >= rank) invalid("sort mode out of range");
  if (plen >= rank) invalid("prefix length out of range");
  for (uint32_t i = 0; i < plen; ++i) {
    if (prefix[i] >= rank) invalid("prefix mode out of range");
    if (prefix[i] == mode) invalid("sort mode lies inside the bucketing prefix");
  }
  Group g;
  g.prefix.assign(prefix, prefix + plen);
  g.keys = {mode};
  g.n_steps = 1;
  return {g};
}

// sort_rows_by's group: no prefix, the key modes (later repeats of a mode
// cannot change the order and are dropped), no range check (sort.cpp:203-211)
std::vector<Group> sort_rows_group(uint32_t rank, const uint32_t* keys, uint32_t nk) {
  if (nk && !keys) invalid("key_modes is null");
  Group g;
  uint64_t seen = 0;
  for (uint32_t i = 0; i < nk; ++i) {
    if (keys[i] >= rank) invalid("key mode out of range");
    if (seen & (uint64_t{1} << keys[i])) continue;
    seen |= uint64_t{1} << keys[i];
    g.keys.push_back(keys[i]);
  }
  g.check_range = false;
  g.n_steps = 0;
  if (g.keys.empty()) return {};
  return {g};
}

// The workspace for a synchronous call: first wait until its async worker
// is idle, so the two never touch the workspace's buffers at the same time.
Workspace& W(qd_workspace* ws) {
  auto* w = reinterpret_cast<Workspace*>(ws);
  async_drain(w);
  return *w;
}
const Workspace* Wc(const qd_workspace* ws) {
  auto* w = const_cast<Workspace*>(reinterpret_cast<const Workspace*>(ws));
  async_drain(w);
  return w;
}

}  // namespace

extern "C" {

int qd_abi_version(void) { return QD_ABI_VERSION; }
const char* qd_last_error(void) { return g_msg.c_str(); }
void qd_last_error_detail(uint64_t* row, uint32_t* mode) {
  if (row) *row = g_row;
  if (mode) *mode = g_mode;
}

qd_status qd_workspace_create(int device, qd_workspace** out) {
  return guard([&] {
    if (!out) invalid("out is null");
    *out = reinterpret_cast<qd_workspace*>(workspace_create(device));
  });
}
void qd_workspace_destroy(qd_workspace* ws) {
  workspace_destroy(reinterpret_cast<Workspace*>(ws));
}
uint64_t qd_workspace_bytes(const qd_workspace* ws) {
  return ws ? workspace_bytes(Wc(ws)) : 0;
}
uint64_t qd_workspace_launches(const qd_workspace* ws) {
  return ws ? workspace_launches(Wc(ws)) : 0;
}
uint64_t qd_workspace_slices(const qd_workspace* ws) {
  return ws ? workspace_slices(Wc(ws)) : 0;
}

void qd_profile_enable(qd_workspace* ws, int enable) {
  if (ws) workspace_profile(&W(ws), enable);
}
void qd_profile_reset(qd_workspace* ws) {
  if (ws) workspace_profile_reset(&W(ws));
}
qd_status qd_profile_get(const qd_workspace* ws, int kernel_class, uint64_t* launches,
                         double* total_ms, double* bytes) {
  return guard([&] {
    if (!ws || !launches || !total_ms || !bytes) invalid("null argument");
    if (!workspace_profile_get(Wc(ws), kernel_class, launches,
                               total_ms, bytes))
      invalid("kernel class must be in 0..4");
  });
}

qd_status qd_quesadilla_plan(const uint32_t* target, uint32_t rank, qd_plan_step* steps,
                             uint32_t capacity, uint32_t* n_steps) {
  return guard([&] { copy_steps(plan_to_prefix(target, rank, rank), steps, capacity, n_steps); });
}

qd_status qd_prefix_plan(const uint32_t* target, uint32_t rank, uint32_t prefix_len,
                         qd_plan_step* steps, uint32_t capacity, uint32_t* n_steps) {
  return guard([&] {
    check_ordering(target, rank);
    if (prefix_len < 1 || prefix_len > rank) invalid("prefix length must be in 1..rank");
    copy_steps(plan_to_prefix(target, rank, prefix_len), steps, capacity, n_steps);
  });
}

qd_status qd_required_sort_count(const uint32_t* source, const uint32_t* target, uint32_t rank,
                                 int* out) {
  return guard([&] { *out = required_sort_count(source, target, rank); });
}

qd_status qd_apply_transition(const uint32_t* current, uint32_t rank, qd_plan_step step,
                              uint32_t* next) {
  return guard([&] {
    auto v = apply_transition(current, rank, Step{step.prefix_len, step.mode});
    std::memcpy(next, v.data(), rank * sizeof(uint32_t));
  });
}

qd_status qd_strategy_pass_cost(qd_strategy_kind kind, uint32_t k, const uint32_t* target,
                                uint32_t rank, int* total, int* bucketed) {
  return guard([&] {
    std::vector<Step> steps;
    if (kind == QD_TOPK && (k < 1 || k > rank)) invalid("prefix length must be in 1..rank");
    strategy_groups(target, rank, kind, k, &steps);
    int b = 0;
    for (auto& s : steps) b += s.prefix_len > 0;
    *total = static_cast<int>(steps.size());
    *bucketed = b;
  });
}

qd_status qd_transpose_inplace(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                               uint32_t* coords, double* values, const uint32_t* target,
                               qd_strategy_kind kind, uint32_t k, const qd_options* opts,
                               qd_workspace* ws) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    check_tensor(rank, dims, nnz, coords, values);
    check_ordering(target, rank);
    std::vector<Step> steps;
    auto groups = strategy_groups(target, rank, kind, k, &steps);
    check_workers(opts, kind, steps);
    TensorView t{rank, dims, nnz};
    run_groups_host(W(ws), t, coords, values, groups,
                    opts && opts->verify_input, opts ? opts->boundaries : nullptr,
                    opts ? opts->n_boundaries : nullptr, target[0]);
    log_steps(opts, steps);
  });
}

qd_status qd_transpose_inplace_async(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                                     uint32_t* coords, double* values, const uint32_t* target,
                                     qd_strategy_kind kind, uint32_t k, const qd_options* opts,
                                     qd_workspace* ws) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    check_tensor(rank, dims, nnz, coords, values);
    check_ordering(target, rank);
    if (opts && (opts->boundaries || opts->n_boundaries))
      invalid("bucket boundaries are only reported by the synchronous calls");
    std::vector<Step> steps;
    auto groups = strategy_groups(target, rank, kind, k, &steps);
    check_workers(opts, kind, steps);
    TensorView t{rank, dims, nnz};
    run_groups_host_async(*reinterpret_cast<Workspace*>(ws), t, coords, values, groups,
                          opts && opts->verify_input);
    log_steps(opts, steps);
  });
}

qd_status qd_workspace_synchronize(qd_workspace* ws) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    workspace_synchronize(reinterpret_cast<Workspace*>(ws));
  });
}

qd_status qd_transpose_device(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                              const uint32_t* d_coords_in, const double* d_values_in,
                              uint32_t* d_coords_out, double* d_values_out,
                              const uint32_t* target, qd_strategy_kind kind, uint32_t k,
                              const qd_options* opts, qd_workspace* ws, void* stream) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    check_tensor(rank, dims, nnz, d_coords_in, d_values_in);
    if (nnz && (!d_coords_out || !d_values_out)) invalid("output buffer is null");
    if (nnz && (d_coords_out == d_coords_in || d_values_out == d_values_in))
      invalid("device transpose is out of place: input and output must differ");
    check_ordering(target, rank);
    std::vector<Step> steps;
    auto groups = strategy_groups(target, rank, kind, k, &steps);
    check_workers(opts, kind, steps);
    TensorView t{rank, dims, nnz};
    run_groups(W(ws), t, d_coords_in, d_values_in, d_coords_out,
               d_values_out, groups, opts && opts->verify_input,
               opts ? opts->boundaries : nullptr, opts ? opts->n_boundaries : nullptr, target[0],
               stream);
    log_steps(opts, steps);
  });
}

qd_status qd_partial_sort(uint32_t rank, const uint32_t* dims, uint64_t nnz, uint32_t* coords,
                          double* values, const uint32_t* prefix, uint32_t prefix_len,
                          uint32_t mode, qd_workspace* ws) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    check_tensor(rank, dims, nnz, coords, values);
    auto groups = partial_sort_group(rank, prefix, prefix_len, mode);
    TensorView t{rank, dims, nnz};
    run_groups_host(W(ws), t, coords, values, groups, false, nullptr,
                    nullptr, 0);
  });
}

qd_status qd_sort_rows_by(uint32_t rank, const uint32_t* dims, uint64_t nnz, uint32_t* coords,
                          double* values, uint64_t row_begin, uint64_t row_end,
                          const uint32_t* key_modes, uint32_t n_keys, qd_workspace* ws) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    check_tensor(rank, dims, nnz, coords, values);
    auto groups = sort_rows_group(rank, key_modes, n_keys);
    if (row_begin > row_end || row_end > nnz) invalid("row range outside [0, nnz]");
    const uint64_t m = row_end - row_begin;
    if (m < 2 || groups.empty()) return;
    TensorView t{rank, dims, m};
    run_groups_host(W(ws), t, coords + row_begin * rank,
                    values + row_begin, groups, false, nullptr, nullptr, 0);
  });
}

qd_status qd_sort_rows_by_device(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                                 const uint32_t* d_coords_in, const double* d_values_in,
                                 uint32_t* d_coords_out, double* d_values_out,
                                 uint64_t row_begin, uint64_t row_end,
                                 const uint32_t* key_modes, uint32_t n_keys, qd_workspace* ws,
                                 void* stream) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    check_tensor(rank, dims, nnz, d_coords_in, d_values_in);
    if (nnz && (!d_coords_out || !d_values_out)) invalid("output buffer is null");
    if (nnz && (d_coords_out == d_coords_in || d_values_out == d_values_in))
      invalid("device sort is out of place: input and output must differ");
    auto groups = sort_rows_group(rank, key_modes, n_keys);
    if (row_begin > row_end || row_end > nnz) invalid("row range outside [0, nnz]");
    const uint64_t m = row_end - row_begin;
    copy_rows_device(W(ws), rank, nnz, d_coords_in, d_values_in,
                     d_coords_out, d_values_out, row_begin, row_end,
                     m < 2 || groups.empty(), stream);
    if (m < 2 || groups.empty()) return;
    TensorView t{rank, dims, m};
    run_groups(W(ws), t, d_coords_in + row_begin * rank,
               d_values_in + row_begin, d_coords_out + row_begin * rank, d_values_out + row_begin,
               groups, false, nullptr, nullptr, 0, stream);
  });
}

// read_tns (io.cpp:42-126): parse on the device (tns.cu), canonicalise with
// the engine's sort_rows_by group (io.cpp:36-38), copy the rows out.
qd_status qd_read_tns(const char* text, uint64_t n_bytes, const uint32_t* declared_dims,
                      uint32_t declared_rank, int has_declared, int canonicalize,
                      qd_tns_tensor* out, qd_tns_error* err, qd_workspace* ws) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    if (!out) invalid("output is null");
    *out = qd_tns_tensor{};
    struct Scope {
      cudaStream_t st = nullptr;
      std::vector<void*> dev;
      ~Scope() {
        if (st) cudaStreamSynchronize(st);
        for (void* p : dev) tns_dev_free(p, st);
        if (st) cudaStreamSynchronize(st);
        if (st) cudaStreamDestroy(st);
      }
    } sc;
    auto ck = [](cudaError_t e) {
      if (e != cudaSuccess) throw Error(QD_CUDA_ERROR, cudaGetErrorString(e));
    };
    ck(cudaStreamCreateWithFlags(&sc.st, cudaStreamNonBlocking));
    // QD_TNS_TIMING=1: phase times on stderr (diagnostics; adds stream syncs)
    static const bool timing = std::getenv("QD_TNS_TIMING") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
      if (!timing) return;
      cudaStreamSynchronize(sc.st);
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "qd_read_tns %-12s %8.2f ms\n", what,
                   std::chrono::duration<double, std::milli>(now - t_last).count());
      t_last = now;
    };
    TnsParsed p;
    parse_tns_device(text, n_bytes, declared_dims, declared_rank, has_declared != 0, &p, err,
                     sc.st);
    sc.dev.push_back(p.d_coords);
    sc.dev.push_back(p.d_values);
    mark("parse");
    const uint32_t R = p.rank;
    const uint64_t N = p.nnz;
    qd_tns_tensor t{R, N, nullptr, nullptr, nullptr};
    // rows in 2 MB-aligned, huge-page-advised memory: first touch costs one
    // fault per 2 MB instead of per 4 KB page
    auto big = [](uint64_t bytes) -> void* {
      const uint64_t a = 2ull << 20;
      bytes = std::max<uint64_t>(bytes, 1);
      if (bytes < a) return std::malloc(bytes);
      void* p = std::aligned_alloc(a, (bytes + a - 1) / a * a);
      if (p) madvise(p, (bytes + a - 1) / a * a, MADV_HUGEPAGE);
      return p;
    };
    t.dims = static_cast<uint32_t*>(std::malloc(std::max<size_t>(R, 1) * 4));
    t.coords = static_cast<uint32_t*>(big(N * R * 4));
    t.values = static_cast<double*>(big(N * 8));
    if (!t.dims || !t.coords || !t.values) {
      qd_tns_free(&t);
      throw std::bad_alloc();
    }
    std::copy(p.dims.begin(), p.dims.end(), t.dims);
    mark("host alloc");
    const uint32_t* c_src = p.d_coords;
    const double* v_src = p.d_values;
    try {
      if (canonicalize && N >= 2) {
        std::vector<uint32_t> simple(R);
        for (uint32_t m = 0; m < R; ++m) simple[m] = m;
        auto groups = sort_rows_group(R, simple.data(), R);
        uint32_t* c2 = nullptr;
        double* v2 = nullptr;
        c2 = static_cast<uint32_t*>(tns_dev_alloc(N * R * 4, sc.st));
        sc.dev.push_back(c2);
        v2 = static_cast<double*>(tns_dev_alloc(N * 8, sc.st));
        sc.dev.push_back(v2);
        TensorView tv{R, p.dims.data(), N};
        run_groups(W(ws), tv, p.d_coords, p.d_values, c2, v2, groups, false, nullptr, nullptr, 0,
                   sc.st);
        c_src = c2;
        v_src = v2;
        mark("canonicalise");
      }
      if (N) {
        staged_d2h(t.coords, c_src, N * R * 4, sc.st);
        staged_d2h(t.values, v_src, N * 8, sc.st);
      }
      ck(cudaStreamSynchronize(sc.st));
      mark("copy out");
    } catch (...) {
      qd_tns_free(&t);
      throw;
    }
    *out = t;
  });
}

void qd_tns_free(qd_tns_tensor* t) {
  if (!t) return;
  std::free(t->dims);
  std::free(t->coords);
  std::free(t->values);
  t->dims = nullptr;
  t->coords = nullptr;
  t->values = nullptr;
  t->nnz = 0;
}

qd_status qd_write_tns(uint32_t rank, uint64_t nnz, const uint32_t* coords,
                       const double* values, char** text, uint64_t* n_bytes,
                       qd_workspace* ws) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    if (!text || !n_bytes) invalid("output is null");
    *text = nullptr;
    *n_bytes = 0;
    if (rank == 0 && nnz) invalid("tensor rank must be positive");
    if (nnz && (!coords || !values)) invalid("coordinate or value buffer is null");
    cudaStream_t st = nullptr;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
      throw Error(QD_CUDA_ERROR, "stream creation failed");
    try {
      format_tns_device(rank, nnz, coords, values, text, n_bytes, st);
    } catch (...) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
      throw;
    }
    cudaStreamDestroy(st);
  });
}

void qd_text_free(char* text) { std::free(text); }

qd_status qd_relabel_target(const uint32_t* source, const uint32_t* target, uint32_t rank,
                            uint32_t* out) {
  return guard([&] {
    check_ordering(source, rank);
    check_ordering(target, rank);
    if (!out) invalid("output is null");
    for (uint32_t i = 0; i < rank; ++i)
      for (uint32_t j = 0; j < rank; ++j)
        if (source[j] == target[i]) out[i] = j;
  });
}

qd_status qd_partial_sort_device(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                                 const uint32_t* d_coords_in, const double* d_values_in,
                                 uint32_t* d_coords_out, double* d_values_out,
                                 const uint32_t* prefix, uint32_t prefix_len, uint32_t mode,
                                 qd_workspace* ws, void* stream) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    check_tensor(rank, dims, nnz, d_coords_in, d_values_in);
    if (nnz && (d_coords_out == d_coords_in || d_values_out == d_values_in))
      invalid("device partial sort is out of place: input and output must differ");
    auto groups = partial_sort_group(rank, prefix, prefix_len, mode);
    TensorView t{rank, dims, nnz};
    run_groups(W(ws), t, d_coords_in, d_values_in, d_coords_out,
               d_values_out, groups, false, nullptr, nullptr, 0, stream);
  });
}

qd_status qd_is_sorted_device(uint32_t rank, uint64_t nnz, const uint32_t* d_coords,
                              const uint32_t* order, int* out, qd_workspace* ws, void* stream) {
  return guard([&] {
    if (!ws || !out) invalid("null argument");
    check_ordering(order, rank);
    *out = is_sorted_device(W(ws), rank, nnz, d_coords, order, stream);
  });
}

qd_status qd_csf_device(uint32_t rank, uint64_t nnz, const uint32_t* d_coords,
                        const uint32_t* order, uint64_t* const* d_pos, uint32_t* const* d_crd,
                        uint64_t* n_fibers, qd_workspace* ws, void* stream) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    if (rank == 0 || rank > QD_MAX_RANK) invalid("tensor rank must be in 1..64");
    if (nnz && !d_coords) invalid("coordinate buffer is null");
    if (nnz >= (uint64_t{1} << 32)) invalid("nnz must be below 2^32");
    check_ordering(order, rank);
    if (!d_pos || !d_crd || !n_fibers) invalid("output arrays are null");
    for (uint32_t k = 0; k < rank; ++k)
      if (!d_pos[k] || (nnz && !d_crd[k])) invalid("output array of a level is null");
    csf_device(W(ws), rank, nnz, d_coords, order, d_pos, d_crd, n_fibers, stream);
  });
}

qd_status qd_bucket_starts_device(uint32_t rank, uint64_t nnz, const uint32_t* d_coords,
                                  const uint32_t* modes, uint32_t n_modes, uint64_t* d_starts,
                                  uint64_t* n_starts, qd_workspace* ws, void* stream) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    for (uint32_t i = 0; i < n_modes; ++i)
      if (modes[i] >= rank) invalid("mode out of range");
    const uint64_t n = bucket_starts_device(W(ws), rank, nnz,
                                            d_coords, modes, n_modes, d_starts, stream);
    if (n_starts) *n_starts = n;
  });
}

qd_status qd_mode_histogram_device(uint32_t rank, uint64_t nnz, const uint32_t* d_coords,
                                   uint32_t mode, uint32_t dim, uint64_t* d_hist,
                                   qd_workspace* ws, void* stream) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    if (mode >= rank) invalid("mode out of range");
    mode_histogram_device(W(ws), rank, nnz, d_coords, mode, dim,
                          d_hist, stream);
  });
}

qd_status qd_partition_rows_device(uint32_t rank, uint64_t nnz, const uint32_t* d_coords_in,
                                   const double* d_values_in, uint32_t mode, uint32_t dim,
                                   const uint32_t* d_lookup, uint32_t n_parts,
                                   uint32_t* d_coords_out, double* d_values_out,
                                   uint64_t* part_counts, qd_workspace* ws, void* stream) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    partition_rows_device(W(ws), rank, nnz, d_coords_in, d_values_in,
                          mode, dim, d_lookup, n_parts, d_coords_out, d_values_out, part_counts,
                          stream);
  });
}

qd_status qd_partition_rows_to_peers_device(uint32_t rank, uint64_t nnz,
                                            const uint32_t* d_coords_in,
                                            const double* d_values_in, uint32_t mode,
                                            uint32_t dim, const uint32_t* d_lookup,
                                            uint32_t n_parts, const uint64_t* peer_coords,
                                            const uint64_t* peer_values,
                                            const uint64_t* peer_row_offsets,
                                            uint64_t* part_counts, qd_workspace* ws,
                                            void* stream) {
  return guard([&] {
    if (!ws) invalid("workspace is null");
    if (!peer_coords || !peer_values || !peer_row_offsets) invalid("peer tables are null");
    for (uint32_t p = 0; p < n_parts; ++p)
      if (!peer_coords[p] || !peer_values[p]) invalid("null peer destination");
    partition_rows_device(W(ws), rank, nnz, d_coords_in, d_values_in, mode, dim, d_lookup,
                          n_parts, nullptr, nullptr, part_counts, stream, peer_coords,
                          peer_values, peer_row_offsets);
  });
}

}  // extern "C"

// ---- sharded transpose (shard.cu) ----------------------------------------------
struct qd_comm {
  Comm* c;
};
struct qd_hub {
  Hub* h;
};

qd_status qd_comm_unique_id(uint8_t out[128]) {
  return guard([&] {
    if (!out) invalid("output buffer is null");
    comm_unique_id(out);
  });
}

qd_status qd_comm_create(const uint8_t id[128], int nranks, int rank, int device, qd_comm** out) {
  return guard([&] {
    if (!id || !out) invalid("null argument");
    *out = new qd_comm{comm_create_nccl(id, nranks, rank, device)};
  });
}

qd_status qd_hub_create(int nranks, qd_hub** out) {
  return guard([&] {
    if (!out) invalid("null argument");
    *out = new qd_hub{hub_create(nranks)};
  });
}

qd_status qd_hub_destroy(qd_hub* hub) {
  return guard([&] {
    if (hub) hub_destroy(hub->h);
    delete hub;
  });
}

qd_status qd_comm_create_emulated(qd_hub* hub, int rank, qd_workspace* ws, qd_comm** out) {
  return guard([&] {
    if (!hub || !ws || !out) invalid("null argument");
    *out = new qd_comm{comm_create_emulated(hub->h, rank, workspace_device(W(ws)), &W(ws))};
  });
}

qd_status qd_comm_destroy(qd_comm* comm) {
  return guard([&] {
    if (comm) comm_destroy(comm->c);
    delete comm;
  });
}

qd_status qd_sharded_transpose_device(qd_comm* comm, uint32_t rank, const uint32_t* dims,
                                      uint64_t nnz, const uint32_t* d_coords_in,
                                      const double* d_values_in, uint32_t* d_coords_out,
                                      double* d_values_out, uint64_t out_capacity,
                                      uint64_t* nnz_out, const uint32_t* target,
                                      qd_strategy_kind kind, uint32_t k, qd_workspace* ws,
                                      void* stream, qd_shard_stats* stats) {
  return guard([&] {
    if (!comm || !ws || !nnz_out) invalid("null argument");
    check_tensor(rank, dims, nnz, d_coords_in, d_values_in);
    if (out_capacity && (!d_coords_out || !d_values_out)) invalid("output buffer is null");
    check_ordering(target, rank);
    std::vector<Step> steps;
    auto groups = strategy_groups(target, rank, kind, k, &steps);
    TensorView t{rank, dims, nnz};
    sharded_transpose_device(*comm->c, W(ws), t, d_coords_in, d_values_in, d_coords_out,
                             d_values_out, out_capacity, nnz_out, groups, target, stream, stats);
  });
}
