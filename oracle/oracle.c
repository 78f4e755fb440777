/* TEST INFRASTRUCTURE ONLY — see oracle.h.  Plain-C restatement of the
 * reference's serial transpose path; each function cites the reference
 * file:line (relative to /root/reference/proj) it restates. */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---- planner ----------------------------------------------------------- */

/* follow_set(ord, p): bitmask of modes after p in ord (planner.cpp:12-17). */
static uint64_t follow_set(const uint32_t* ord, uint32_t r, uint32_t p) {
  uint32_t pos = 0;
  while (pos < r && ord[pos] != p) ++pos;
  uint64_t s = 0;
  for (uint32_t i = pos + 1; i < r; ++i) s |= (uint64_t)1 << ord[i];
  return s;
}

static int valid_ordering(const uint32_t* ord, uint32_t r) {
  /* Ordering ctor, ordering.cpp:13-31 */
  if (r == 0 || r > 64) return 0;
  uint64_t seen = 0;
  for (uint32_t i = 0; i < r; ++i) {
    if (ord[i] >= r) return 0;
    if (seen & ((uint64_t)1 << ord[i])) return 0;
    seen |= (uint64_t)1 << ord[i];
  }
  return 1;
}

/* plan_to_prefix, planner.cpp:37-56; prefix_plan bounds check 64-69. */
int qo_plan(const uint32_t* target, uint32_t rank, uint32_t want,
            uint32_t* steps, uint32_t max_steps, uint32_t* nsteps) {
  if (!valid_ordering(target, rank)) return 1;
  if (want == 0) want = rank;
  else if (want > rank) return 1;
  uint32_t simple[64];
  for (uint32_t i = 0; i < rank; ++i) simple[i] = i;
  uint32_t n = 0, l = 0;
  while (l < want) {
    uint32_t k = l;
    while (k + 1 < rank) {
      uint64_t ft = follow_set(target, rank, target[k]);
      uint64_t fs = follow_set(simple, rank, target[k]);
      if ((ft & ~fs) == 0) break; /* subset: this mode is settled */
      ++k;
    }
    uint32_t hi = k < want ? k : want;
    for (uint32_t j = hi; j > l; --j) {
      if (n < max_steps) {
        steps[2 * n] = l;
        steps[2 * n + 1] = target[j - 1];
      }
      ++n;
    }
    l = k + 1;
  }
  *nsteps = n;
  return 0;
}

/* ---- partial sorts ------------------------------------------------------ */

/* rows_equal_on, sort.cpp:13-22 */
static int rows_equal_on(const uint32_t* c, uint32_t r, uint64_t a, uint64_t b,
                         const uint32_t* modes, uint32_t nm) {
  for (uint32_t i = 0; i < nm; ++i)
    if (c[a * r + modes[i]] != c[b * r + modes[i]]) return 0;
  return 1;
}

/* validate_sort_args, sort.cpp:153-166 */
static int validate(uint32_t r, const uint32_t* prefix, uint32_t plen,
                    uint32_t mode) {
  if (mode >= r) return 1;
  if (plen >= r) return 1;
  for (uint32_t i = 0; i < plen; ++i) {
    if (prefix[i] >= r) return 1;
    if (prefix[i] == mode) return 1;
  }
  return 0;
}

int qo_partial_sort(uint32_t r, const uint32_t* dims, uint64_t nnz,
                    uint32_t* crd, double* val, const uint32_t* prefix,
                    uint32_t plen, uint32_t mode) {
  if (validate(r, prefix, plen, mode)) return 1;
  if (nnz == 0) return 0;
  const uint32_t n = dims[mode];
  uint32_t* count = (uint32_t*)calloc((size_t)n + 1, sizeof(uint32_t));
  uint32_t* oc = (uint32_t*)malloc(nnz * r * sizeof(uint32_t));
  double* ov = (double*)malloc(nnz * sizeof(double));
  int status = 0;
  if (plen == 0) {
    /* Alg. 1: count_keys (sort.cpp:54-64), prefix sum (184),
     * scatter_rows (66-78). */
    for (uint64_t j = 0; j < nnz; ++j) {
      uint32_t key = crd[j * r + mode];
      if (key >= n) { status = 2; goto done; }
      ++count[key + 1];
    }
    for (uint32_t i = 1; i <= n; ++i) count[i] += count[i - 1];
    for (uint64_t j = 0; j < nnz; ++j) {
      uint32_t p = count[crd[j * r + mode]]++;
      memcpy(oc + (uint64_t)p * r, crd + j * r, r * sizeof(uint32_t));
      ov[p] = val[j];
    }
  } else {
    /* Alg. 2: bucketed_sort_range (sort.cpp:80-134) over [0, nnz). */
    uint32_t* bucket = (uint32_t*)malloc(nnz * sizeof(uint32_t));
    uint32_t* pos = (uint32_t*)malloc(nnz * sizeof(uint32_t));
    uint32_t* perm = (uint32_t*)malloc(nnz * sizeof(uint32_t));
    uint32_t nb = 0;
    bucket[0] = 0;
    pos[0] = 0;
    for (uint64_t j = 0; j < nnz; ++j) {
      if (j > 0 && !rows_equal_on(crd, r, j - 1, j, prefix, plen)) {
        ++nb;
        pos[nb] = (uint32_t)j;
      }
      bucket[j] = nb;
      uint32_t key = crd[j * r + mode];
      if (key >= n) { status = 2; break; }
      ++count[key + 1];
    }
    if (status == 0) {
      for (uint32_t i = 1; i <= n; ++i) count[i] += count[i - 1];
      for (uint64_t j = 0; j < nnz; ++j)
        perm[count[crd[j * r + mode]]++] = (uint32_t)j;
      for (uint64_t p = 0; p < nnz; ++p) {
        uint32_t j = perm[p];
        uint32_t dst = pos[bucket[j]]++;
        memcpy(oc + (uint64_t)dst * r, crd + (uint64_t)j * r,
               r * sizeof(uint32_t));
        ov[dst] = val[j];
      }
    }
    free(bucket);
    free(pos);
    free(perm);
    if (status) goto done;
  }
  /* swap with the workspace (sort.cpp:199-200): copy back. */
  memcpy(crd, oc, nnz * r * sizeof(uint32_t));
  memcpy(val, ov, nnz * sizeof(double));
done:
  free(count);
  free(oc);
  free(ov);
  return status;
}

/* ---- comparison sort (sort_rows_by, sort.cpp:203-235) ------------------- */

typedef struct {
  const uint32_t* crd;
  uint32_t r;
  const uint32_t* keys;
  uint32_t nk;
} cmp_ctx;

static int row_less(const cmp_ctx* c, uint32_t a, uint32_t b) {
  for (uint32_t i = 0; i < c->nk; ++i) {
    uint32_t x = c->crd[(uint64_t)a * c->r + c->keys[i]];
    uint32_t y = c->crd[(uint64_t)b * c->r + c->keys[i]];
    if (x != y) return x < y;
  }
  return 0;
}

/* Stable bottom-up merge sort of idx[0..m) (std::stable_sort semantics). */
static void stable_sort_idx(const cmp_ctx* c, uint32_t* idx, uint32_t* tmp,
                            uint64_t m) {
  for (uint64_t w = 1; w < m; w *= 2) {
    for (uint64_t lo = 0; lo < m; lo += 2 * w) {
      uint64_t mid = lo + w < m ? lo + w : m;
      uint64_t hi = lo + 2 * w < m ? lo + 2 * w : m;
      uint64_t i = lo, j = mid, o = lo;
      while (i < mid && j < hi) tmp[o++] = row_less(c, idx[j], idx[i]) ? idx[j++] : idx[i++];
      while (i < mid) tmp[o++] = idx[i++];
      while (j < hi) tmp[o++] = idx[j++];
    }
    memcpy(idx, tmp, m * sizeof(uint32_t));
  }
}

static void sort_rows_by(uint32_t r, uint32_t* crd, double* val, uint64_t b,
                         uint64_t e, const uint32_t* keys, uint32_t nk) {
  uint64_t m = e - b;
  if (m < 2) return;
  uint32_t* idx = (uint32_t*)malloc(m * sizeof(uint32_t));
  uint32_t* tmp = (uint32_t*)malloc(m * sizeof(uint32_t));
  for (uint64_t i = 0; i < m; ++i) idx[i] = (uint32_t)i;
  cmp_ctx c = {crd + b * r, r, keys, nk};
  stable_sort_idx(&c, idx, tmp, m);
  uint32_t* tc = (uint32_t*)malloc(m * r * sizeof(uint32_t));
  double* tv = (double*)malloc(m * sizeof(double));
  for (uint64_t p = 0; p < m; ++p) {
    memcpy(tc + p * r, crd + (b + idx[p]) * r, r * sizeof(uint32_t));
    tv[p] = val[b + idx[p]];
  }
  memcpy(crd + b * r, tc, m * r * sizeof(uint32_t));
  memcpy(val + b, tv, m * sizeof(double));
  free(idx);
  free(tmp);
  free(tc);
  free(tv);
}

/* sort_rows_by as a public entry (sort.cpp:203-211 validates the key modes,
 * then stable-sorts rows [b, e)). */
int qo_sort_rows_by(uint32_t r, uint64_t nnz, uint32_t* crd, double* val, uint64_t b,
                    uint64_t e, const uint32_t* keys, uint32_t nk) {
  for (uint32_t i = 0; i < nk; ++i)
    if (keys[i] >= r) return 1;
  if (b > e || e > nnz) return 1;
  sort_rows_by(r, crd, val, b, e, keys, nk);
  return 0;
}

/* relabel_target, planner.cpp:148-158: position of each target mode within
 * source. */
int qo_relabel_target(const uint32_t* source, const uint32_t* target, uint32_t r, uint32_t* out) {
  if (!valid_ordering(source, r) || !valid_ordering(target, r)) return 1;
  for (uint32_t i = 0; i < r; ++i)
    for (uint32_t j = 0; j < r; ++j)
      if (source[j] == target[i]) out[i] = j;
  return 0;
}

/* ---- transpose driver (transpose.cpp:59-112) ----------------------------- */

int qo_is_sorted(uint32_t r, uint64_t nnz, const uint32_t* crd,
                 const uint32_t* order) {
  for (uint64_t j = 1; j < nnz; ++j) {
    for (uint32_t i = 0; i < r; ++i) {
      uint32_t a = crd[(j - 1) * r + order[i]], b = crd[j * r + order[i]];
      if (a != b) {
        if (a > b) return 0;
        break;
      }
    }
  }
  return 1;
}

uint64_t qo_bucket_starts(uint32_t r, uint64_t nnz, const uint32_t* crd,
                          const uint32_t* modes, uint32_t nm,
                          uint64_t* starts) {
  if (nnz == 0) return 0;
  uint64_t n = 0;
  starts[n++] = 0;
  for (uint64_t j = 1; j < nnz; ++j)
    if (!rows_equal_on(crd, r, j - 1, j, modes, nm)) starts[n++] = j;
  return n;
}

static int run_step(uint32_t r, const uint32_t* dims, uint64_t nnz,
                    uint32_t* crd, double* val, const uint32_t* target,
                    uint32_t l, uint32_t mode, uint32_t* steps_out,
                    uint32_t max_steps, uint32_t* n_log) {
  int s = qo_partial_sort(r, dims, nnz, crd, val, target, l, mode);
  if (s) return s;
  if (*n_log < max_steps) {
    steps_out[2 * *n_log] = l;
    steps_out[2 * *n_log + 1] = mode;
  }
  ++*n_log;
  return 0;
}

int qo_transpose(uint32_t r, const uint32_t* dims, uint64_t nnz,
                 uint32_t* crd, double* val, const uint32_t* target, int kind,
                 uint32_t k, int verify_input, uint32_t* steps_out,
                 uint32_t max_steps, uint32_t* nsteps_out) {
  uint32_t nlog = 0, dummy[2];
  if (!steps_out) { steps_out = dummy; max_steps = 0; }
  if (!valid_ordering(target, r)) return 1;
  if (verify_input) {
    uint32_t simple[64];
    for (uint32_t i = 0; i < r; ++i) simple[i] = i;
    if (!qo_is_sorted(r, nnz, crd, simple)) return 1;
  }
  int s = 0;
  uint32_t plan[128], np = 0;
  switch (kind) {
    case QO_QUESADILLA:
      qo_plan(target, r, 0, plan, 64, &np);
      for (uint32_t i = 0; i < np && !s; ++i)
        s = run_step(r, dims, nnz, crd, val, target, plan[2 * i], plan[2 * i + 1],
                     steps_out, max_steps, &nlog);
      break;
    case QO_RADIX:
      for (uint32_t j = r; j > 0 && !s; --j)
        s = run_step(r, dims, nnz, crd, val, target, 0, target[j - 1], steps_out,
                     max_steps, &nlog);
      break;
    case QO_TOPK:
      if (k < 1 || k > r) return 1;
      qo_plan(target, r, k, plan, 64, &np);
      for (uint32_t i = 0; i < np && !s; ++i)
        s = run_step(r, dims, nnz, crd, val, target, plan[2 * i], plan[2 * i + 1],
                     steps_out, max_steps, &nlog);
      /* parallel_topk_bucket_sort serial branch, parallel.cpp:190-218 */
      if (!s && k < r && nnz >= 2) {
        uint64_t* st = (uint64_t*)malloc(nnz * sizeof(uint64_t));
        uint64_t nb = qo_bucket_starts(r, nnz, crd, target, k, st);
        for (uint64_t b = 0; b < nb; ++b) {
          uint64_t e = b + 1 < nb ? st[b + 1] : nnz;
          sort_rows_by(r, crd, val, st[b], e, target + k, r - k);
        }
        free(st);
      }
      break;
    case QO_COMPARISON:
      sort_rows_by(r, crd, val, 0, nnz, target, r);
      break;
    default:
      return 1;
  }
  if (nsteps_out) *nsteps_out = nlog;
  return s;
}
