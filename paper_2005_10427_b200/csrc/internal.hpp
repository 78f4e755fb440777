// Internal interfaces of libquesadilla_b200 (host C++; not part of the ABI).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "quesadilla_b200.h"

namespace qb200 {

// Error carrying a C-ABI status; thrown inside the library, caught at the
// extern "C" boundary (capi.cpp) and turned into a qd_status.
struct Error : std::runtime_error {
  qd_status code;
  uint64_t row = 0;
  uint32_t mode = 0;
  Error(qd_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void invalid(const std::string& m) {
  throw Error(QD_INVALID_ARGUMENT, m);
}

// ---- planner (planner.cpp) -------------------------------------------------
struct Step {
  uint32_t prefix_len;
  uint32_t mode;
};

void check_ordering(const uint32_t* ord, uint32_t rank);  // ordering.cpp:13-31
std::vector<Step> plan_to_prefix(const uint32_t* target, uint32_t rank,
                                 uint32_t want);          // planner.cpp:37-56
int required_sort_count(const uint32_t* source, const uint32_t* target,
                        uint32_t rank);                   // planner.cpp:19-29
std::vector<uint32_t> apply_transition(const uint32_t* cur, uint32_t rank,
                                       Step s);           // plan.cpp:7-27

// One device "group": a segmented stable sort.  Rows are partitioned into
// maximal runs agreeing on `prefix` (in the current order; empty prefix =
// one run) and each run is stably sorted by the combined key `keys`
// (priority order, keys[0] most significant).  A run of consecutive plan
// steps with the same prefix_len is exactly one group (LSD composition).
struct Group {
  std::vector<uint32_t> prefix;
  std::vector<uint32_t> keys;
  uint32_t first_step = 0, n_steps = 0;  // logical plan steps it covers
  // Histogram passes range-check their key (sort.cpp:26-30 -> out_of_range);
  // comparison phases (sort_rows_by) do not, and then key widths come from
  // the data instead of the dimensions.
  bool check_range = true;
  // Hint from the planner (a simply sorted source assumed): the least
  // significant key mode is the fastest-varying mode of the rows' current
  // order, so the first digit pass sees nearly random digits within a tile
  // (the engine then ranks that pass with ballots instead of MATCH.ANY).
  bool first_digit_scattered = false;
};

// Groups for a whole strategy (transpose.cpp:79-112): the LOGICAL steps go to
// `steps` (pass_log semantics), the device work to the returned groups.
std::vector<Group> strategy_groups(const uint32_t* target, uint32_t rank,
                                   qd_strategy_kind kind, uint32_t k,
                                   std::vector<Step>* steps);

// ---- device engine (engine.cu) ----------------------------------------------
struct Workspace;
Workspace* workspace_create(int device);
void workspace_destroy(Workspace* ws);
uint64_t workspace_bytes(const Workspace* ws);
uint64_t workspace_launches(const Workspace* ws);
uint64_t workspace_slices(const Workspace* ws);  // of the last synchronous host-buffer call
void* workspace_buffer(Workspace& ws, const char* name, size_t bytes);  // cached by name
int workspace_device(const Workspace& ws);
int workspace_sms(const Workspace& ws);
void workspace_count_launch(Workspace& ws);
void workspace_profile(Workspace* ws, int enable);
void workspace_profile_reset(Workspace* ws);
bool workspace_profile_get(const Workspace* ws, int cls, uint64_t* launches, double* ms,
                           double* bytes);

struct TensorView {
  uint32_t rank;
  const uint32_t* dims;  // host
  uint64_t nnz;
};

// Runs the groups in order, src -> dst (device pointers, distinct).  Checks
// verify_input (simple order) first when asked.  Synchronises `stream` and
// throws Error on invalid input / out-of-range coordinates / CUDA errors.
void run_groups(Workspace& ws, const TensorView& t, const uint32_t* d_c_in,
                const double* d_v_in, uint32_t* d_c_out, double* d_v_out,
                const std::vector<Group>& groups, bool verify_input,
                uint64_t* d_boundaries, uint64_t* n_boundaries,
                uint32_t boundary_mode, void* stream);

// Host-buffer convenience: H2D, run_groups, D2H (only on success).
// Device copies of the rows outside [row_begin, row_end) (all rows when
// `whole`) from in to out, on `stream`.
void copy_rows_device(Workspace& ws, uint32_t rank, uint64_t nnz, const uint32_t* c_in,
                      const double* v_in, uint32_t* c_out, double* v_out, uint64_t row_begin,
                      uint64_t row_end, bool whole, void* stream);
void run_groups_host_async(Workspace& ws, const TensorView& t, uint32_t* coords, double* values,
                           const std::vector<Group>& groups, bool verify_input);
void workspace_synchronize(Workspace* ws);
void async_drain(Workspace* ws);
void run_groups_host(Workspace& ws, const TensorView& t, uint32_t* coords,
                     double* values, const std::vector<Group>& groups,
                     bool verify_input, uint64_t* h_boundaries,
                     uint64_t* n_boundaries, uint32_t boundary_mode);

bool is_sorted_device(Workspace& ws, uint32_t rank, uint64_t nnz,
                      const uint32_t* d_coords, const uint32_t* order,
                      void* stream);
void csf_device(Workspace& ws, uint32_t rank, uint64_t nnz, const uint32_t* d_coords,
                const uint32_t* order, uint64_t* const* d_pos, uint32_t* const* d_crd,
                uint64_t* n_fibers, void* stream);
uint64_t bucket_starts_device(Workspace& ws, uint32_t rank, uint64_t nnz,
                              const uint32_t* d_coords, const uint32_t* modes,
                              uint32_t n_modes, uint64_t* d_starts, void* stream);
void mode_histogram_device(Workspace& ws, uint32_t rank, uint64_t nnz,
                           const uint32_t* d_coords, uint32_t mode, uint32_t dim,
                           uint64_t* d_hist, void* stream);
void partition_rows_device(Workspace& ws, uint32_t rank, uint64_t nnz,
                           const uint32_t* d_c_in, const double* d_v_in,
                           uint32_t mode, uint32_t dim, const uint32_t* d_lookup,
                           uint32_t n_parts, uint32_t* d_c_out, double* d_v_out,
                           uint64_t* part_counts, void* stream,
                           const uint64_t* peer_c = nullptr, const uint64_t* peer_v = nullptr,
                           const uint64_t* peer_off = nullptr);

// ---- multi-GPU (shard.cu) ----------------------------------------------------
struct Comm;  // one rank of a communicator (NCCL, or the emulated hub)
struct Hub;   // emulated ranks: threads of one process on one device (tests)
void comm_unique_id(unsigned char* out128);
Comm* comm_create_nccl(const unsigned char* id128, int nranks, int rank, int device);
Hub* hub_create(int nranks);
void hub_destroy(Hub* h);
Comm* comm_create_emulated(Hub* hub, int rank, int device, Workspace* ws);
void comm_destroy(Comm* c);
int comm_size(const Comm& c);
int comm_rank(const Comm& c);
const char* comm_kind(const Comm& c);
void sharded_transpose_device(Comm& comm, Workspace& ws, const TensorView& t,
                              const uint32_t* d_c_in, const double* d_v_in, uint32_t* d_c_out,
                              double* d_v_out, uint64_t out_capacity, uint64_t* n_out,
                              const std::vector<Group>& groups, const uint32_t* target,
                              void* stream, qd_shard_stats* stats);

// .tns reader (tns.cu): io.cpp:42-126 minus canonicalisation.  Parses the
// host text on the device; on success the rows are in device buffers the
// caller frees (tns_dev_free on the same stream), in file order.  Throws Error(QD_PARSE_ERROR) with
// the reference's ParseError text and fills *err.
// Large host<->device copies through a pinned chunk ring with parallel host
// memcpy (tns.cu); synchronous with respect to the host buffer.
void* tns_dev_alloc(uint64_t bytes, void* stream);  // stream-ordered, pooled
void tns_dev_free(void* p, void* stream);
void staged_h2d(void* d_dst, const void* h_src, uint64_t n, void* stream);
void staged_d2h(void* h_dst, const void* d_src, uint64_t n, void* stream);
struct StageSeg {
  void* h;
  const void* d;
  uint64_t n;
};
void staged_d2h_multi(const StageSeg* segs, int nseg, void* stream);

// write_tns's text (io.cpp:128-152) formatted on the device from host rows;
// *h_text is malloc-family memory (free()), null when nnz == 0.
void format_tns_device(uint32_t rank, uint64_t nnz, const uint32_t* h_coords,
                       const double* h_values, char** h_text, uint64_t* n_text, void* stream);

struct TnsParsed {
  uint32_t rank = 0;
  uint64_t nnz = 0;
  std::vector<uint32_t> dims;
  uint32_t* d_coords = nullptr;
  double* d_values = nullptr;
};
void parse_tns_device(const char* h_text, uint64_t n, const uint32_t* declared,
                      uint32_t declared_rank, bool has_declared, TnsParsed* out,
                      qd_tns_error* err, void* stream);

}  // namespace qb200
