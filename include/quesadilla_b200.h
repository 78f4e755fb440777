/* quesadilla_b200 — C ABI of the B200-native Quesadilla COO transpose.
 *
 * The drop-in boundary for the reference's transpose path
 * (arxiv 2005.10427 artifact, /root/reference/proj).  Plain pointers and
 * sizes only; no C++ or torch types cross this boundary; no exceptions cross
 * it either — every reference exception maps to a status code:
 *
 *   QD_INVALID_ARGUMENT  <-> std::invalid_argument
 *   QD_OUT_OF_RANGE      <-> std::out_of_range   (coordinate >= dimension)
 *   QD_CUDA_ERROR / QD_NO_DEVICE: device failures (no CPU fallback exists).
 *
 * Layout (identical to quesadilla::CooTensor, coo.hpp:16-24):
 *   coords : nnz * rank uint32, row-major AoS (row j, mode m at j*rank+m)
 *   values : nnz float64
 *   dims   : rank uint32, each >= 1
 * A target ordering is a permutation of 0..rank-1, highest priority first
 * (quesadilla::Ordering, ordering.hpp:38-61).
 *
 * Semantics are bit-exact with the reference: the output rows are exactly
 * what quesadilla::transpose_inplace produces (stable; values only moved).
 * Functions are synchronous with respect to the host (like the reference);
 * the *_device variants enqueue on `stream` (a cudaStream_t, may be NULL for
 * the legacy stream) and synchronise it before returning the status.
 */
#ifndef QUESADILLA_B200_H
#define QUESADILLA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QD_ABI_VERSION 1
#define QD_MAX_RANK 64 /* quesadilla::kMaxRank, ordering.hpp:14 */

typedef enum qd_status {
  QD_OK = 0,
  QD_INVALID_ARGUMENT = 1,
  QD_OUT_OF_RANGE = 2,
  QD_CUDA_ERROR = 3,
  QD_NCCL_ERROR = 4,
  QD_NO_DEVICE = 5,
  QD_PARSE_ERROR = 6 /* quesadilla::ParseError (io.hpp:15-22), .tns reader */
} qd_status;

/* quesadilla::SortStrategy::Kind, transpose.hpp:22. */
typedef enum qd_strategy_kind {
  QD_QUESADILLA = 0,
  QD_TOPK = 1,
  QD_FULL_RADIX = 2,
  QD_COMPARISON_SORT = 3
} qd_strategy_kind;

/* quesadilla::PlanStep, plan.hpp:13-20. */
typedef struct qd_plan_step {
  uint32_t prefix_len;
  uint32_t mode;
} qd_plan_step;

/* quesadilla::TransposeOptions, transpose.hpp:45-54, plus device extras. */
typedef struct qd_options {
  int verify_input;            /* throw invalid_argument unless simply sorted */
  uint32_t workers;            /* ParallelConfig::workers; 0 rejected like the
                                  reference (parallel.cpp:161-163), otherwise
                                  the GPU uses all of its SMs */
  qd_plan_step* pass_log;      /* optional: receives the executed LOGICAL steps */
  uint32_t pass_log_capacity;
  uint32_t* pass_log_len;      /* out: number of steps executed */
  /* optional: output segment/pos boundaries = start rows of the maximal runs
   * of the leading target mode in the output (detail::bucket_starts(out,
   * {target[0]}), sort.cpp:136-147) followed by nnz.  Host pointer for the
   * host API, device pointer for the device API; capacity nnz + 1. */
  uint64_t* boundaries;
  uint64_t* n_boundaries;      /* out: number of entries written (incl. nnz) */
} qd_options;

typedef struct qd_workspace qd_workspace; /* quesadilla::Workspace, sort.hpp:14-21 */

/* ---- runtime ------------------------------------------------------------ */
int qd_abi_version(void);
const char* qd_last_error(void);          /* thread-local message */
/* Row / mode of the last QD_OUT_OF_RANGE (input row index). */
void qd_last_error_detail(uint64_t* row, uint32_t* mode);

qd_status qd_workspace_create(int device, qd_workspace** out);
void qd_workspace_destroy(qd_workspace* ws);
/* Bytes of device memory currently held by the workspace. */
uint64_t qd_workspace_bytes(const qd_workspace* ws);
/* Number of CUDA kernels this workspace has launched since creation. */
uint64_t qd_workspace_launches(const qd_workspace* ws);
/* Slices the last synchronous host-buffer call (qd_transpose_inplace,
 * qd_partial_sort, qd_sort_rows_by) was pipelined in: 1 = whole tensor; > 1 when
 * every pass keeps a common prefix mode (Alg. 2 only, sort.cpp:80-134), so the
 * tensor is cut where that mode changes and the slices' input copies, passes
 * and output copies overlap.  QD_SLICE_ROWS=<rows> sets the slice size (0: never). */
uint64_t qd_workspace_slices(const qd_workspace* ws);

/* Live per-kernel-class timing with CUDA events recorded on the launch
 * stream (off by default).  Classes: 0 chunk-ordered digit scatter, 1 chunk histogram,
 * 2 local (in-CTA) run sort, 3 run discovery / scans, 4 other.  bytes is the
 * algorithmic traffic of the class (rows moved x 2 x row bytes for
 * classes 0 and 2, coordinates read for class 1). */
void qd_profile_enable(qd_workspace* ws, int enable);
void qd_profile_reset(qd_workspace* ws);
qd_status qd_profile_get(const qd_workspace* ws, int kernel_class,
                         uint64_t* launches, double* total_ms, double* bytes);

/* ---- planner (host; planner.hpp:13-55, plan.hpp:27-36) ------------------ */
qd_status qd_quesadilla_plan(const uint32_t* target, uint32_t rank,
                             qd_plan_step* steps, uint32_t capacity,
                             uint32_t* n_steps);
qd_status qd_prefix_plan(const uint32_t* target, uint32_t rank,
                         uint32_t prefix_len, qd_plan_step* steps,
                         uint32_t capacity, uint32_t* n_steps);
qd_status qd_required_sort_count(const uint32_t* source, const uint32_t* target,
                                 uint32_t rank, int* out);
qd_status qd_apply_transition(const uint32_t* current, uint32_t rank,
                              qd_plan_step step, uint32_t* next);
/* relabel_target (planner.cpp:148-158): for a tensor sorted under `source`,
 * the target ordering in source-relabelled modes (position of each target
 * mode within source), written to out[rank]. */
qd_status qd_relabel_target(const uint32_t* source, const uint32_t* target, uint32_t rank,
                            uint32_t* out);
qd_status qd_strategy_pass_cost(qd_strategy_kind kind, uint32_t k,
                                const uint32_t* target, uint32_t rank,
                                int* total, int* bucketed);

/* ---- transpose (transpose.hpp:59-80) ------------------------------------ */

/* Host buffers, in place: quesadilla::transpose_inplace (transpose.cpp:79-112).
 * Copies H2D, runs the planned passes on the GPU, copies D2H.  Pinned host
 * buffers give full link bandwidth.  On error the host buffers are left
 * unmodified (strong guarantee; the reference gives the basic one). */
qd_status qd_transpose_inplace(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                               uint32_t* coords, double* values,
                               const uint32_t* target, qd_strategy_kind kind,
                               uint32_t k, const qd_options* opts,
                               qd_workspace* ws);

/* Asynchronous form of qd_transpose_inplace for pipelines of host-buffer
 * calls (e.g. the CLI bench's loop over targets, main.cpp:198-213).  The
 * call validates its arguments (invalid_argument is returned at once),
 * enqueues the host->device copy and returns; a worker thread of the
 * workspace runs the device transpose and enqueues the device->host copy.
 * Input copies of consecutive calls run back to back while earlier calls
 * sort and copy out (PCIe is full duplex).  (coords, values) hold the result
 * after qd_workspace_synchronize, which also returns the FIRST device-side
 * error (out_of_range, ...) of the calls since the last synchronize; a
 * failing call leaves its tensor untouched, the others complete.  Buffers
 * must stay valid (and should be pinned) until then.  Calls that read host
 * bytes the previous call writes (chained in-place calls) are ordered after
 * it.  Synchronous calls on the same workspace first wait for its worker.
 * Bucket boundaries are not reported by this form. */
qd_status qd_transpose_inplace_async(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                                     uint32_t* coords, double* values,
                                     const uint32_t* target, qd_strategy_kind kind,
                                     uint32_t k, const qd_options* opts,
                                     qd_workspace* ws);
/* Wait for every asynchronous call on this workspace; returns the first
 * device-side error among them (then cleared). */
qd_status qd_workspace_synchronize(qd_workspace* ws);

/* sort_rows_by (sort.cpp:203-235): stable sort of rows [row_begin, row_end)
 * by key_modes in priority order, rows outside the range untouched.  Like the
 * reference (a comparison sort) it never range-checks coordinates; a key
 * mode >= rank is invalid_argument (so is a row range outside [0, nnz], which
 * the reference leaves undefined).  Host buffers, in place; the device form
 * writes the whole tensor out of place.  This is the canonicalisation
 * read_tns applies (io.cpp:36-38) when key_modes is the simple ordering. */
qd_status qd_sort_rows_by(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                          uint32_t* coords, double* values, uint64_t row_begin,
                          uint64_t row_end, const uint32_t* key_modes, uint32_t n_keys,
                          qd_workspace* ws);
qd_status qd_sort_rows_by_device(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                                 const uint32_t* d_coords_in, const double* d_values_in,
                                 uint32_t* d_coords_out, double* d_values_out,
                                 uint64_t row_begin, uint64_t row_end,
                                 const uint32_t* key_modes, uint32_t n_keys,
                                 qd_workspace* ws, void* stream);

/* Device-resident, out of place (in and out must not overlap). */
qd_status qd_transpose_device(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                              const uint32_t* d_coords_in,
                              const double* d_values_in, uint32_t* d_coords_out,
                              double* d_values_out, const uint32_t* target,
                              qd_strategy_kind kind, uint32_t k,
                              const qd_options* opts, qd_workspace* ws,
                              void* stream);

/* ---- one partial sort (sort.hpp:32-33, parallel.hpp:35-37) -------------- */
qd_status qd_partial_sort(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                          uint32_t* coords, double* values,
                          const uint32_t* prefix, uint32_t prefix_len,
                          uint32_t mode, qd_workspace* ws);
qd_status qd_partial_sort_device(uint32_t rank, const uint32_t* dims,
                                 uint64_t nnz, const uint32_t* d_coords_in,
                                 const double* d_values_in,
                                 uint32_t* d_coords_out, double* d_values_out,
                                 const uint32_t* prefix, uint32_t prefix_len,
                                 uint32_t mode, qd_workspace* ws, void* stream);

/* ---- checks and boundaries ---------------------------------------------- */
/* is_sorted_under (coo.cpp:32-49) on device coords; *out = 0/1. */
qd_status qd_is_sorted_device(uint32_t rank, uint64_t nnz,
                              const uint32_t* d_coords, const uint32_t* order,
                              int* out, qd_workspace* ws, void* stream);
/* detail::bucket_starts (sort.cpp:136-147) on device coords, followed by nnz:
 * d_starts (device, capacity nnz + 1) receives the run starts + nnz. */
/* CSF levels of a tensor sorted under `order` (the emitted
 * boundaries turned into level pointers; the paper's motivation).  Level k
 * (0 <= k < rank) has n_fibers[k] fibers = maximal runs of equal
 * (order[0..k]) coordinates; d_crd[k][f] is coordinate order[k] of fiber f;
 * d_pos[0] = {0, n_fibers[0]} and for k >= 1 d_pos[k][j] is the first
 * level-k fiber of level-(k-1) fiber j (n_fibers[k-1] + 1 entries).  The
 * leaf level is the distinct coordinates (duplicates share a leaf; values
 * stay per row).  Capacities: d_pos[k] max(nnz + 1, 2), d_crd[k] nnz entries. */
qd_status qd_csf_device(uint32_t rank, uint64_t nnz, const uint32_t* d_coords,
                        const uint32_t* order, uint64_t* const* d_pos,
                        uint32_t* const* d_crd, uint64_t* n_fibers,
                        qd_workspace* ws, void* stream);
qd_status qd_bucket_starts_device(uint32_t rank, uint64_t nnz,
                                  const uint32_t* d_coords,
                                  const uint32_t* modes, uint32_t n_modes,
                                  uint64_t* d_starts, uint64_t* n_starts,
                                  qd_workspace* ws, void* stream);

/* ---- multi-GPU sharding helpers (device) -------------- */
/* Histogram of mode `mode` over rows (device, n_bins = dims[mode] counters,
 * uint64), accumulated into d_hist. */
qd_status qd_mode_histogram_device(uint32_t rank, uint64_t nnz,
                                   const uint32_t* d_coords, uint32_t mode,
                                   uint32_t dim, uint64_t* d_hist,
                                   qd_workspace* ws, void* stream);
/* Stable partition of rows into n_parts destination parts by
 * part = lookup[coords[row*rank+mode]] (d_lookup: dim uint32 entries < n_parts).
 * Writes the rows grouped by part, input order kept inside each part, and
 * part_counts[n_parts] (host). */
qd_status qd_partition_rows_device(uint32_t rank, uint64_t nnz,
                                   const uint32_t* d_coords_in,
                                   const double* d_values_in, uint32_t mode,
                                   uint32_t dim, const uint32_t* d_lookup,
                                   uint32_t n_parts, uint32_t* d_coords_out,
                                   double* d_values_out, uint64_t* part_counts,
                                   qd_workspace* ws, void* stream);
/* The same partition fused with the exchange that follows it (SURVEY §8e
 * steps 3-4): part p's rows are written straight into destination p — device
 * addresses peer_coords[p] / peer_values[p] (on a multi-GPU box: NVLink peer
 * mappings of rank p's receive buffer, e.g. torch symmetric memory), starting
 * at row peer_row_offsets[p] (this rank's place among the senders to p, in
 * source-rank order) — instead of a local buffer followed by an all-to-all.
 * Replaces the ncclSend/ncclRecv group of the exchange step; the caller
 * orders the receivers' reads after every sender's kernel (stream sync +
 * barrier). */
qd_status qd_partition_rows_to_peers_device(uint32_t rank, uint64_t nnz,
                                            const uint32_t* d_coords_in,
                                            const double* d_values_in, uint32_t mode,
                                            uint32_t dim, const uint32_t* d_lookup,
                                            uint32_t n_parts, const uint64_t* peer_coords,
                                            const uint64_t* peer_values,
                                            const uint64_t* peer_row_offsets,
                                            uint64_t* part_counts, qd_workspace* ws,
                                            void* stream);

/* ---- sharded transpose over NCCL ------------
 * One communicator rank per device: every rank holds a contiguous slice of
 * the global (simply sorted) input rows, slices in rank order; after the
 * call rank g holds the slice of the global output whose leading target mode
 * falls in g's range, so the rank outputs concatenated in rank order equal
 * transpose(global, target) bit for bit.  Lifts parallel.cpp:113-154's
 * bucket-aligned regions to GPUs: target[0] == 0 with mode-0-aligned slices
 * needs no communication; otherwise one exchange (ncclAllReduce of the
 * leading mode's histogram, splitters on the device, one grouped
 * ncclSend/ncclRecv per peer, received in source-rank order).  Collective:
 * every rank calls it with the same target and strategy. */
typedef struct qd_comm qd_comm;
typedef struct qd_hub qd_hub;
typedef struct qd_shard_stats {
  int exchanged;            /* 1 when the rows were exchanged */
  uint64_t rows_out;        /* rows of this rank's output slice */
  uint64_t bytes_sent;      /* to other ranks */
  uint64_t bytes_received;  /* from other ranks */
  float exchange_ms;        /* device time of the grouped send/recv (CUDA events) */
} qd_shard_stats;
/* ncclGetUniqueId: 128 bytes for rank 0 to broadcast to every rank */
qd_status qd_comm_unique_id(uint8_t out[128]);
/* ncclCommInitRank on `device` (NCCL loaded at run time: libnccl.so.2) */
qd_status qd_comm_create(const uint8_t id[128], int nranks, int rank, int device,
                         qd_comm** out);
/* Test transport: `nranks` ranks emulated as threads of one process on one
 * device (device copies + host barriers; no NCCL).  The hub must outlive
 * its comms; each rank uses its own workspace. */
qd_status qd_hub_create(int nranks, qd_hub** out);
qd_status qd_hub_destroy(qd_hub* hub);
qd_status qd_comm_create_emulated(qd_hub* hub, int rank, qd_workspace* ws, qd_comm** out);
qd_status qd_comm_destroy(qd_comm* comm);
/* this rank's input slice (device) -> its output slice (device, capacity
 * out_capacity rows; *nnz_out = the slice's rows, also when it does not fit:
 * then every rank fails with QD_INVALID_ARGUMENT).  stats may be null. */
qd_status qd_sharded_transpose_device(qd_comm* comm, uint32_t rank, const uint32_t* dims,
                                      uint64_t nnz, const uint32_t* d_coords_in,
                                      const double* d_values_in, uint32_t* d_coords_out,
                                      double* d_values_out, uint64_t out_capacity,
                                      uint64_t* nnz_out, const uint32_t* target,
                                      qd_strategy_kind kind, uint32_t k, qd_workspace* ws,
                                      void* stream, qd_shard_stats* stats);

/* ---- .tns text format (io.hpp:24-47, io.cpp:42-126) --------------------- */
/* A tensor owned by the library (host memory; release with qd_tns_free). */
typedef struct qd_tns_tensor {
  uint32_t rank;
  uint64_t nnz;
  uint32_t* dims;   /* rank entries */
  uint32_t* coords; /* AoS, nnz * rank, 0-based */
  double* values;   /* nnz */
} qd_tns_tensor;

/* Where a QD_PARSE_ERROR was found: `line` is ParseError::line() (1-based);
 * kind 1 first data line has < 2 fields, 2 rank != declared rank, 3 field
 * count differs from the first data line, 4 invalid index token, 5 index 0,
 * 6 index beyond its declared dimension, 7 invalid value token, 8 empty
 * file without declared dims.  `field` is the 0-based field, the token is
 * text[token_offset, +token_len).  qd_last_error() holds the reference's
 * ParseError::what() text ("line N: ..."). */
typedef struct qd_tns_error {
  uint64_t line;
  uint32_t kind;
  uint32_t field;
  uint32_t got;
  uint32_t expected;
  uint64_t token_offset;
  uint64_t token_len;
} qd_tns_error;

/* read_tns over a file's bytes (the caller reads the file): tokens are split
 * on ' ', '\t', '\r'; blank lines and lines whose first field starts with
 * '#' are skipped; indices are 1-based std::from_chars(uint32_t), values
 * std::from_chars(double) (correctly rounded, out-of-range rejected).
 * `declared_dims` (has_declared != 0) plays ReadOptions::declared_dims;
 * canonicalize != 0 stably sorts the rows into the simple ordering
 * (io.cpp:36-38) on the device.  Parsing runs on the GPU (text copied to
 * HBM once); `err` (nullable) receives the failure location.  Differences
 * from the reference: a file of rank > QD_MAX_RANK is QD_INVALID_ARGUMENT
 * (the reference reads it, but no transpose accepts it). */
qd_status qd_read_tns(const char* text, uint64_t n_bytes, const uint32_t* declared_dims,
                      uint32_t declared_rank, int has_declared, int canonicalize,
                      qd_tns_tensor* out, qd_tns_error* err, qd_workspace* ws);
void qd_tns_free(qd_tns_tensor* t);

/* write_tns's text (io.cpp:128-152): per row the 1-based indices and the
 * value (std::to_chars shortest round-trip, fixed or scientific) separated by
 * ' ', '\n'-terminated, in storage order; formatted on the GPU.  *text is
 * library-owned (qd_text_free); the caller writes it to the file.  Like the
 * reference, the tensor is not validated. */
qd_status qd_write_tns(uint32_t rank, uint64_t nnz, const uint32_t* coords,
                       const double* values, char** text, uint64_t* n_bytes,
                       qd_workspace* ws);
void qd_text_free(char* text);

#ifdef __cplusplus
}
#endif
#endif /* QUESADILLA_B200_H */
