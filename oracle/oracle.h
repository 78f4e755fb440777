/* TEST INFRASTRUCTURE ONLY — the CPU parity oracle.
 *
 * A plain-C restatement of the reference's transpose path (arxiv 2005.10427
 * artifact, /root/reference/proj).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the checker.  The
 * product path (paper_2005_10427_b200) never links or calls it.
 *
 * Pinned: tests/test_oracle.py checks it against the reference's own golden
 * vectors (tests/golden/, produced by oracle/make_golden.py from the
 * unmodified reference library oracle/_ref/libqref.so) and, when
 * oracle/_ref is built, bit-for-bit against the reference on random cases.
 *
 * Status codes: 0 ok, 1 invalid_argument, 2 out_of_range.
 */
#ifndef QD_ORACLE_H
#define QD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Strategy kinds, transpose.hpp:22 (Kind { Quesadilla, TopK, FullRadix,
 * ComparisonSort }). */
enum { QO_QUESADILLA = 0, QO_TOPK = 1, QO_RADIX = 2, QO_COMPARISON = 3 };

/* Alg. 3 planner, planner.cpp:37-69.  want == 0 -> quesadilla_plan, else
 * prefix_plan(target, want).  steps: pairs (prefix_len, mode). */
int qo_plan(const uint32_t* target, uint32_t rank, uint32_t want,
            uint32_t* steps, uint32_t max_steps, uint32_t* nsteps);

/* One serial partial sort, sort.cpp:170-201 (Alg. 1 when plen == 0,
 * Alg. 2 otherwise).  In place on AoS coords[nnz*rank], values[nnz]. */
int qo_partial_sort(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                    uint32_t* coords, double* values, const uint32_t* prefix,
                    uint32_t plen, uint32_t mode);

/* transpose_inplace, transpose.cpp:79-112 (serial path). */
int qo_transpose(uint32_t rank, const uint32_t* dims, uint64_t nnz,
                 uint32_t* coords, double* values, const uint32_t* target,
                 int kind, uint32_t k, int verify_input, uint32_t* steps_out,
                 uint32_t max_steps, uint32_t* nsteps_out);

/* detail::bucket_starts, sort.cpp:136-147 (rows [0, nnz)). */
uint64_t qo_bucket_starts(uint32_t rank, uint64_t nnz, const uint32_t* coords,
                          const uint32_t* modes, uint32_t nmodes,
                          uint64_t* starts_out);

/* sort_rows_by, sort.cpp:203-235: stable comparison sort of rows [b, e) by
 * `keys` in priority order (no range check). */
int qo_sort_rows_by(uint32_t rank, uint64_t nnz, uint32_t* coords, double* values,
                    uint64_t b, uint64_t e, const uint32_t* keys, uint32_t nkeys);

/* relabel_target, planner.cpp:148-158. */
int qo_relabel_target(const uint32_t* source, const uint32_t* target, uint32_t rank,
                      uint32_t* out);

/* is_sorted_under, coo.cpp:32-49. */
int qo_is_sorted(uint32_t rank, uint64_t nnz, const uint32_t* coords,
                 const uint32_t* order);

#ifdef __cplusplus
}
#endif
#endif
