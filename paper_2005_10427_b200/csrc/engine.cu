// B200 (sm_100a) device engine of the Quesadilla COO transpose.
//
// Every logical plan group (internal.hpp: a run of same-prefix plan steps)
// is one SEGMENTED STABLE SORT: rows are cut into maximal runs agreeing on
// the group's prefix modes (Alg. 2's "buckets", sort.cpp:80-134), and each
// run is stably sorted by the group's combined key (Alg. 1 when the prefix is
// empty, sort.cpp:54-78; consecutive same-prefix steps compose LSD-wise into
// one combined key).  Device work per group:
//
//   k_heads / scan / k_compact     run discovery (bucket_starts, sort.cpp:136)
//   k_classify_chunks/k_gen_chunks small runs -> local CTA sorts, large runs ->
//                                  chunks of contiguous rows
//   per radix digit (LSD, <= 8 bits):
//     k_chunk_hist                 digit histogram of every chunk (+ range
//                                  check on the first digit: count_keys);
//                                  later digits from a 1-byte side channel
//     scan                         (run, bin, chunk) exclusive scan = every
//                                  chunk's output cursor per bin: the
//                                  (key, worker) order of parallel.cpp:88-100
//     k_scatter                    chunk-ordered stable scatter of whole rows:
//                                  TMA bulk-copy double buffering, MATCH.ANY
//                                  warp ranking in shared memory, coalesced
//                                  stores; intermediates as packed 16-byte
//                                  rows (bit fields / mixed radix / run prefix)
//   k_local3                       the small runs: merged items staged by TMA,
//                                  block-wide LSD over (run, key), written once
//   k_small                        latency regime (single-group plans, <= 2^22
//                                  rows): the whole call in one cooperative
//                                  kernel over {key, row} elements in L2
//
// Rows are always moved whole (the reference's scatter_rows) or gathered once
// by k_small, so there is no separate gather pass.  No CPU fallback exists:
// every path here is a kernel.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <deque>
#include <exception>
#include <map>
#include <mutex>
#include <string>
#include <thread>

#include <nvtx3/nvToolsExt.h>

#include "internal.hpp"

namespace qb200 {

#define QD_CUDA(x)                                                              \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess)                                                      \
      throw Error(QD_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// NVTX ranges (nsys / ncu --nvtx filters): the call, each plan group, each
// digit pass, run discovery and the small-run sort.  Header-only NVTX v3:
// without an attached tool a range is a null-pointer check.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  explicit NvtxRange(const std::string& name) { nvtxRangePushA(name.c_str()); }
  ~NvtxRange() { nvtxRangePop(); }
};

constexpr int kThreads = 256;       // utility kernels
constexpr int kWarps = kThreads / 32;
#ifndef QD_SORT_THREADS
#define QD_SORT_THREADS 512
#endif
constexpr int kSortThreads = QD_SORT_THREADS;  // k_scatter / k_local
constexpr int kSortWarps = kSortThreads / 32;
#ifndef QD_LOCAL_THREADS
#define QD_LOCAL_THREADS 512
#endif
constexpr int kLocalThreads = QD_LOCAL_THREADS;  // k_local
constexpr int kLocalWarps = kLocalThreads / 32;
constexpr int kRadixLog = 8;
constexpr int kBins = 1 << kRadixLog;
constexpr int kMaxTerms = 12;
constexpr int kMaxKeys = QD_MAX_RANK;
constexpr uint32_t kChunkTiles = 16;  // tiles per scatter chunk
constexpr double kRunSortMinAvg = 2.5;       // mean run length that pays for a run sort
constexpr uint64_t kRunSortMinRows = 1u << 20;  // below this, not worth a probe
#ifndef QD_MAX_TILE
#define QD_MAX_TILE 4096
#endif
#ifndef QD_SCATTER_CTAS
#define QD_SCATTER_CTAS 2  // resident k_scatter CTAs per SM (register / shared-memory split)
#endif
constexpr int kMaxRounds = QD_MAX_TILE / kSortThreads;  // 32-row rounds per warp per tile
#ifndef QD_LOCAL_BALLOT
#define QD_LOCAL_BALLOT 1
#endif
#ifndef QD_EARLY_ADVANCE
#define QD_EARLY_ADVANCE 1
#endif
#ifndef QD_DYNAMIC_CHUNKS
#define QD_DYNAMIC_CHUNKS 1
#endif
#ifndef QD_ASYNC_SLOTS
#define QD_ASYNC_SLOTS 2
#endif
#ifndef QD_FULL_ROUNDS
#define QD_FULL_ROUNDS 1
#endif
#ifndef QD_RANK_BCAST
#define QD_RANK_BCAST 1
#endif

// ---------------------------------------------------------------------------
// kernel parameter blocks
// ---------------------------------------------------------------------------

// Digit of one pass: bits [lo, lo+b) of the combined key, gathered from at
// most kMaxTerms mode fields.
struct DigitSpec {
  uint32_t n;
  uint8_t mode[kMaxTerms], rsh[kMaxTerms], bits[kMaxTerms], lsh[kMaxTerms];
  // lookup digit (stable partition): digit = lookup[row[lookup_mode]]
  const uint32_t* lookup;
  uint32_t lookup_mode, lookup_dim;
};

// Combined key of a group: keys[0] most significant; field i occupies
// [off[i], off[i] + width[i]).
struct KeySpec {
  uint32_t n;
  uint32_t total_bits;
  int check;  // range-check key coordinates against dim
  uint8_t mode[kMaxKeys], width[kMaxKeys];
  uint16_t off[kMaxKeys];
  uint32_t dim[kMaxKeys];
};

constexpr int kMaxGroups = 64;

struct ErrBlock {
  unsigned int flags;  // bit0 out_of_range, bit1 not simply sorted
  unsigned int pad;
  unsigned long long rowmode;  // min over (row << 6 | mode)
  unsigned long long rows[kMaxGroups];  // rows of large runs, per group (profiling)
};

struct LocalArgs {
  const uint32_t* in_c;
  const double* in_v;
  uint32_t* out_c;
  double* out_v;
  uint32_t rank;
  uint64_t nnz;
  uint32_t TL;  // chunk span; runs with len <= TL are "small"
  uint32_t cap; // rows per chunk buffer (>= 2*TL, or nnz for a single run)
  const unsigned long long* seg_start;  // S+1 entries; nullptr: one run [0,nnz)
  uint64_t nseg;
  KeySpec key;
  ErrBlock* err;
  const uint32_t* chunk_list;  // chunk ids holding small runs (blockIdx.x -> chunk)
  const uint32_t* first_run;   // per chunk: first run starting in it (k_classify_chunks)
};

// A chunk: a contiguous row range inside one run, processed by one CTA in
// input order; the (bin, chunk) exclusive scan gives every chunk its own
// output cursor per bin (parallel.cpp:88-100's (key, worker) order, with CTA
// chunks as the workers), so no inter-CTA waiting is needed.
struct ChunkDesc {
  unsigned long long row_begin;
  unsigned int len;
  unsigned int li;          // large-run index
  unsigned int cidx;        // chunk index inside its run
  unsigned int nchunks;     // chunks in its run
  unsigned long long coff;  // global index of the run's first chunk
};

// Row storage: AoS = coords[N*R] (row-major, the API layout) + values[N];
// SoA = column m at coords + m*N (intermediate passes) + values[N].
// Row formats.  AoS: coords[N*R] + values[N] (the API layout).  SoA: column m
// at coords + m*N, values[N].  PK: 16-byte rows {u64 packed coordinates, f64
// value} where the packed word holds the group's combined key in its low
// bits (digit q = shift + mask) and the other modes above it.
enum { kAoS = 0, kSoA = 1, kPK = 2 };
struct Rows {
  const uint32_t* c;  // PK: the 16-byte rows
  const double* v;
  int fmt;
};
struct RowsOut {
  uint32_t* c;
  double* v;
  int fmt;
};

// Packed coordinate layout: mode m at bits [off[m], off[m] + width[m]).
// Packed coordinate layout: key mode m at bits [off[m], off[m] + width[m])
// (the group's combined key in the low key_bits), the other modes above it
// either as bit fields too or, when those would overflow 64 bits
// (`mixed`), as one mixed-radix number hi = ((c_a * d_b + c_b) * d_c + c_c)
// ... over their dimensions, stored at bit key_bits.  lim[m] is the bound
// a coordinate must respect to pack losslessly (2^width or the dimension).
struct PackSpec {
  uint32_t rank;
  uint8_t off[kMaxKeys], width[kMaxKeys];
  uint32_t lim[kMaxKeys];
  uint32_t mixed, key_bits, nk_n;
  uint8_t nk_mode[kMaxKeys];
  uint32_t nk_dim[kMaxKeys];
  double nk_rcp[kMaxKeys];  // 1 / nk_dim
  // prefix modes left out of the packed word: constant within a run, so the
  // last pass restores them from the run (run_prefix[li * n_imp + k])
  uint32_t n_imp;
  uint8_t imp_mode[kMaxKeys];
  uint8_t kind[kMaxKeys];  // per mode: 0 bit field (width may be 0), 1 mixed radix, 2 implicit
};

// x / d for d < 2^32: a double multiply by the precomputed reciprocal when
// x < 2^53 (then exact after a short fix-up), else the 64-bit hardware path
__device__ __forceinline__ unsigned long long div_u64_u32(unsigned long long x, uint32_t d,
                                                          double rcp) {
  if (x < (1ull << 53)) {
    // |x * rcp - x / d| < 1 for x < 2^53: one correction either way
    unsigned long long q = (unsigned long long)((double)x * rcp);
    if (q * d > x) --q;
    else if ((q + 1) * d <= x) ++q;
    return q;
  }
  return x / d;
}
template <class F>
__device__ __forceinline__ unsigned long long pack_coords(const PackSpec& p, uint32_t R, F coord) {
  unsigned long long pk = 0;
  for (uint32_t m = 0; m < R; ++m)
    if (p.width[m]) pk |= (unsigned long long)coord(m) << p.off[m];
  if (p.mixed) {
    unsigned long long hi = 0;
    for (uint32_t j = 0; j < p.nk_n; ++j) hi = hi * p.nk_dim[j] + coord(p.nk_mode[j]);
    pk |= hi << p.key_bits;
  }
  return pk;
}
// writes the R coordinates of packed word x through put(m, value)
template <class P>
__device__ __forceinline__ void unpack_coords(const PackSpec& p, uint32_t R, unsigned long long x,
                                              P put) {
  for (uint32_t m = 0; m < R; ++m)  // every bit field, including 0-bit ones (extent 1)
    if (p.kind[m] == 0) put(m, (uint32_t)(x >> p.off[m]) & (uint32_t)((1ull << p.width[m]) - 1ull));
  if (p.mixed) {
    unsigned long long hi = p.key_bits < 64 ? x >> p.key_bits : 0ull;
    for (int j = (int)p.nk_n - 1; j >= 0; --j) {
      const unsigned long long q = div_u64_u32(hi, p.nk_dim[j], p.nk_rcp[j]);
      put(p.nk_mode[j], (uint32_t)(hi - q * p.nk_dim[j]));
      hi = q;
    }
  }
}

// PackSpec decoded on the host for the static-rank (RT = 3, 4) scatter paths:
// per-mode u32/u64 words at fixed offsets, which the compiler reads as
// constant-bank operands (the byte arrays of PackSpec indexed per row cost
// extracts and loads: the round-1 c5 profile had the pack and mixed-radix
// unpack at ~45 % of the unpacking pass's instructions).
struct PackFast {
  uint32_t fsh[4], fmask[4];        // bit field of the mode (mask 0: not a field)
  unsigned long long mul[4];        // mixed-radix weight of the mode (0: not mixed)
  uint32_t mpos[4];                 // mixed-radix position of the mode (0xFF: none)
  uint32_t dimj[4];                 // mixed-radix dimension by position
  unsigned long long magic[4];      // floor((2^64 - 1) / dimj)
  uint32_t impk[4];                 // implicit prefix mode: its index in run_prefix (0xFF: none)
  uint32_t key_bits, mixed, nk_n;
};

// q = x / d, r = x % d for x < 2^63 and d >= 1 with mg = floor((2^64-1)/d):
// umulhi(x, mg) is q or q - 1 (its error is below x (1 + 1/d) / 2^64 < 1),
// one correction step
__device__ __forceinline__ unsigned long long div_magic(unsigned long long x, uint32_t d,
                                                        unsigned long long mg, uint32_t& r) {
  unsigned long long q = __umul64hi(x, mg);
  unsigned long long rem = x - q * d;
  if (rem >= d) {
    ++q;
    rem -= d;
  }
  r = (uint32_t)rem;
  return q;
}

struct ChunkHistArgs {
  Rows in;
  uint32_t rank;
  uint64_t nnz;
  const ChunkDesc* chunks;
  uint32_t num_chunks;
  const unsigned long long* nc_dev;  // device chunk count (latency mode; num_chunks = its bound)
  uint32_t* flat;  // [(coff + c) * kBins layout: coff*kBins + b*nchunks + cidx]
  DigitSpec dig;
  KeySpec key;
  int do_check;
  ErrBlock* err;
  unsigned long long* rows_counter;
  uint32_t pk_shift, pk_mask;  // digit of a PK row
  int check_pack;              // flag bit2 if a coordinate would not pack losslessly
  uint32_t lim[4];             // rank <= 4: per mode, min(key dimension if checked, pack limit), host-folded
  PackSpec pack;
  const uint8_t* digits;       // this pass's digit per row, written by the previous scatter
};

// One destination of a peer-writing partition pass: part p's rows go to
// (c, v) (device addresses, typically NVLink peer mappings of another rank's
// receive buffer) starting at row `off`.
struct PeerDest {
  unsigned long long c, v, off;
};

struct ScatterArgs {
  int dbg;  // experiment switches (QD_SCATTER_DBG): 1 = skip global stores
  unsigned long long* dbg_t;  // QD_SCATTER_DBG & 2: per-phase clock totals
  Rows in;
  RowsOut out;
  uint32_t rank;
  uint64_t nnz;
  uint32_t T;  // rows per tile
  const ChunkDesc* chunks;
  uint32_t num_chunks;
  const unsigned long long* nc_dev;     // device chunk count (latency mode; num_chunks = its bound)
  const unsigned long long* offs;       // exclusive scan of the chunk-hist flat array
  const unsigned long long* run_start;  // [li]; nullptr: 0
  uint32_t* chunk_counter;
  DigitSpec dig;
  uint32_t pk_shift, pk_mask;  // digit of a PK row
  PackSpec pack;
  uint8_t* next_dig;           // next pass's digit per row (side channel for its histogram)
  uint32_t nd_shift, nd_mask;  // PK output: next digit = (packed >> nd_shift) & nd_mask
  DigitSpec ndig;              // unpacked output: next digit of the coordinates
  const uint32_t* run_prefix;  // implicit prefix modes per large run (PackSpec::n_imp)
  const PeerDest* peers;       // AoS output per bin (partition straight into peer buffers)
  int vec_out;                 // AoS output rows may use 16-byte stores (rank 4, aligned base)
  PackFast pf;                 // pack decoded for the RT = 3, 4 paths
  uint32_t dbits;              // bits of this pass's digit (ballot ranking)
  int rank_mode;               // adaptive_peers mode (QD_RANK_MODE)
  uint32_t match_max;          // mode 1: MATCH.ANY when a round has <= this many digit runs
};

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------

// One AoS row of RT coordinates: rank 4 as one 16-byte access (the caller
// guarantees 16-byte alignment), other ranks word by word.  (Rank 3 as an
// 8-byte + 4-byte pair chosen by the row's word parity measured 1.5 % slower
// on c2: the selects cost more than the saved shared-memory wavefronts.)
template <int RT>
__device__ __forceinline__ void load_row_words(const uint32_t* w, uint32_t (&cv)[RT]) {
  if constexpr (RT == 4) {
    const uint4 x = *reinterpret_cast<const uint4*>(w);
    cv[0] = x.x; cv[1] = x.y; cv[2] = x.z; cv[3] = x.w;
  } else {
#pragma unroll
    for (int m = 0; m < RT; ++m) cv[m] = w[m];
  }
}
template <int RT>
__device__ __forceinline__ void store_row_words(uint32_t* w, const uint32_t (&cv)[RT]) {
  if constexpr (RT == 4) {
    __stcs(reinterpret_cast<uint4*>(w), make_uint4(cv[0], cv[1], cv[2], cv[3]));
  } else {
#pragma unroll
    for (int m = 0; m < RT; ++m) __stcs(w + m, cv[m]);
  }
}

__device__ __forceinline__ uint32_t digit_of(const uint32_t* row, const DigitSpec& d) {
  if (d.lookup) {
    uint32_t c = row[d.lookup_mode];
    return c < d.lookup_dim ? __ldg(d.lookup + c) : 0u;
  }
  uint32_t v = ((row[d.mode[0]] >> d.rsh[0]) & ((1u << d.bits[0]) - 1u)) << d.lsh[0];
#pragma unroll 1
  for (uint32_t i = 1; i < d.n; ++i)
    v |= ((row[d.mode[i]] >> d.rsh[i]) & ((1u << d.bits[i]) - 1u)) << d.lsh[i];
  return v;
}

__device__ __forceinline__ uint64_t full_key(const uint32_t* row, const KeySpec& k) {
  uint64_t v = 0;
#pragma unroll 1
  for (uint32_t i = 0; i < k.n; ++i) {
    const uint32_t w = k.width[i];
    if (w) v |= (uint64_t)(row[k.mode[i]] & (uint32_t)((1ull << w) - 1ull)) << k.off[i];
  }
  return v;
}

__device__ __forceinline__ void check_row(const uint32_t* row, const KeySpec& k,
                                          uint64_t grow, ErrBlock* e) {
#pragma unroll 1
  for (uint32_t i = 0; i < k.n; ++i) {
    if (row[k.mode[i]] >= k.dim[i]) {
      atomicOr(&e->flags, 1u);
      atomicMin(&e->rowmode, (unsigned long long)((grow << 6) | k.mode[i]));
    }
  }
}

// Exclusive scan across the block of one value per thread (NT threads).
template <int NT = kThreads>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_tmp,
                                                    uint32_t* total = nullptr) {
  constexpr int kWarps = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_tmp[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < kWarps ? s_tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xFFFFFFFFu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kWarps) s_tmp[lane] = t;  // inclusive warp totals
  }
  __syncthreads();
  const uint32_t before = w ? s_tmp[w - 1] : 0;
  const uint32_t tot = s_tmp[kWarps - 1];
  __syncthreads();
  if (total) *total = tot;
  return before + x - v;
}

// Same for 64-bit values.
template <int NT = kThreads>
__device__ __forceinline__ unsigned long long block_excl_scan64(unsigned long long v,
                                                                unsigned long long* s_tmp) {
  constexpr int kWarps = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_tmp[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned long long t = lane < kWarps ? s_tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kWarps) s_tmp[lane] = t;
  }
  __syncthreads();
  const unsigned long long before = w ? s_tmp[w - 1] : 0;
  __syncthreads();
  return before + x - v;
}

// Lanes of the warp whose digit equals this lane's (digits < 2^BITS), by
// BITS ballots; cheaper than MATCH.ANY on sm_100.  Only lanes in `valid` count.
template <int BITS = kRadixLog>
__device__ __forceinline__ unsigned warp_peers(uint32_t d, unsigned valid) {
#ifndef QD_BALLOT_MATCH
  return __match_any_sync(0xFFFFFFFFu, d) & valid;  // MATCH.ANY: one instruction
#endif
  unsigned m = valid;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const unsigned bit = (d >> b) & 1u;
    const unsigned v = __ballot_sync(0xFFFFFFFFu, bit);
    m &= bit ? v : ~v;
  }
  return m;
}

// Peers of d among the lanes in `valid` for a digit of `nbits` bits (<= 8):
// MATCH.ANY costs ~2 SM cycles per DISTINCT digit in the warp (61 for 32
// random 8-bit digits), nbits ballots a flat ~3.2 each
// (profiles/microbench/match_any_vs_ballot.*).  mode 1 picks per 32-row
// round from the number of runs of equal digits among the lanes (an upper
// bound on the distinct count): MATCH for clustered digits, ballots for
// high-entropy ones; mode 0 = MATCH only, 2 = ballots only.  Measured
// (B200, c5/c2/c3 steps): MATCH only 104.8 / 11.59 / 21.42 ms, adaptive
// 109.6 / 12.15 / 21.89, ballots only 112.6 / 12.10 / 21.81: the kernel is
// issue-bound enough that 7-8 VOTE + LOP pairs per round cost more than the
// MATCH.ANY they replace, so mode 0 is the default (QD_RANK_MODE).
__device__ __forceinline__ unsigned ballot_peers(uint32_t d, unsigned valid, uint32_t nbits) {
  unsigned m = valid;
#pragma unroll
  for (uint32_t b = 0; b < 8; ++b) {
    if (b < nbits) {  // warp-uniform
      const unsigned bit = (d >> b) & 1u;
      const unsigned v = __ballot_sync(0xFFFFFFFFu, bit);
      m &= bit ? v : ~v;
    }
  }
  return m;
}
// the same for digits of up to MAXB bits (k_local3's 9-bit digits)
template <int MAXB>
__device__ __forceinline__ unsigned ballot_peers_n(uint32_t d, unsigned valid, uint32_t nbits) {
  unsigned m = valid;
#pragma unroll
  for (uint32_t b = 0; b < (uint32_t)MAXB; ++b) {
    if (b < nbits) {  // warp-uniform
      const unsigned bit = (d >> b) & 1u;
      const unsigned v = __ballot_sync(0xFFFFFFFFu, bit);
      m &= bit ? v : ~v;
    }
  }
  return m;
}
__device__ __forceinline__ unsigned adaptive_peers(uint32_t d, unsigned valid, uint32_t nbits,
                                                   int mode, uint32_t match_max) {
  if (mode == 0) return __match_any_sync(0xFFFFFFFFu, d) & valid;
  if (mode == 2) return ballot_peers(d, valid, nbits);
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, d, 1);
  const unsigned heads = __ballot_sync(0xFFFFFFFFu, lane == 0u || prev != d);
  if ((uint32_t)__popc(heads) <= match_max) return __match_any_sync(0xFFFFFFFFu, d) & valid;
  return ballot_peers(d, valid, nbits);
}

// Stable per-warp ranking of positions [0, n): positions are cut into NW
// contiguous stripes of `ipw`; warp w walks its stripe in rounds of 32, so
// rank order = position order.  s_rank[p] = rank of p among equal digits
// earlier in its stripe; s_whist[w][d] = count of digit d in stripe w.
template <bool kBallot = false, class F>
__device__ __forceinline__ void warp_rank(F get_digit, uint32_t n, uint32_t ipw,
                                          uint16_t* s_rank, uint16_t* s_whist) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint16_t* wh = s_whist + w * kBins;
  const uint32_t lo = w * ipw;
  const uint32_t hi = min(n, lo + ipw);
  const unsigned below = (1u << lane) - 1u;
  for (uint32_t base = lo; base < hi; base += 32) {
    const uint32_t p = base + lane;
    const bool valid = p < hi;
    const uint32_t d = valid ? get_digit(p) : 0u;
    unsigned peers;
    if (kBallot) {  // flat cost: 8 ballots
      peers = __ballot_sync(0xFFFFFFFFu, valid);
#pragma unroll
      for (int bb = 0; bb < kRadixLog; ++bb) {
        const unsigned bit = (d >> bb) & 1u;
        const unsigned v = __ballot_sync(0xFFFFFFFFu, bit);
        peers &= bit ? v : ~v;
      }
    } else {
      peers = warp_peers(d, __ballot_sync(0xFFFFFFFFu, valid));
    }
    if (!valid) peers = 1u << lane;
    const int leader = __ffs(peers) - 1;
    uint32_t b = 0;
    if (valid && lane == leader) {
      b = wh[d];
      wh[d] = (uint16_t)(b + __popc(peers));
    }
    b = __shfl_sync(0xFFFFFFFFu, b, leader);  // leader's old count
    if (valid) s_rank[p] = (uint16_t)(b + __popc(peers & below));
  }
}

// Turn per-warp counts into per-bin warp-exclusive offsets; s_cnt[b] = total.
template <int NT = kThreads>
__device__ __forceinline__ void bin_totals(uint16_t* s_whist, uint32_t* s_cnt) {
  constexpr int kWarps = NT / 32;
  for (int b = threadIdx.x; b < kBins; b += NT) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = s_whist[w * kBins + b];
      s_whist[w * kBins + b] = (uint16_t)run;
      run += c;
    }
    s_cnt[b] = run;
  }
}

// Per-warp bin counts -> warp-exclusive offsets (in place) and each bin's
// exclusive start in the tile, with two barriers: thread b < kBins walks its
// bin's column, the first kBins/32 warps scan their 32 bins with shuffles and
// combine the warp sums.  Returns (for threads < kBins) the bin's count.
template <int NT>
__device__ __forceinline__ uint32_t bin_offsets(uint16_t* s_whist, uint32_t* s_wsum,
                                                uint32_t* s_start) {
  constexpr int kW = NT / 32;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t cnt = 0, incl = 0;
  if (threadIdx.x < kBins) {
#pragma unroll
    for (int x = 0; x < kW; ++x) {
      const uint32_t c = s_whist[x * kBins + threadIdx.x];
      s_whist[x * kBins + threadIdx.x] = (uint16_t)cnt;
      cnt += c;
    }
    incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    if (lane == 31) s_wsum[w] = incl;
  }
  __syncthreads();
  if (threadIdx.x < kBins) {
    uint32_t base = 0;
    for (uint32_t x = 0; x < w; ++x) base += s_wsum[x];
    s_start[threadIdx.x] = base + incl - cnt;
  }
  return cnt;
}

// Word offset of g + a inside its 16-byte line (any caller pointer: device
// buffers need only be 4-byte aligned), and the same for doubles.
__device__ __forceinline__ uint32_t words_head(const uint32_t* g, unsigned long long a) {
  return (uint32_t)((reinterpret_cast<uintptr_t>(g + a) >> 2) & 3u);
}
__device__ __forceinline__ uint32_t doubles_head(const double* g, unsigned long long a) {
  return (uint32_t)((reinterpret_cast<uintptr_t>(g + a) >> 3) & 1u);
}

// Load words [a, a+nw) of g into s_raw so that word a+k lands at
// s_raw[words_head(g, a) + k]; 16-byte vector loads for the aligned body.
template <int NT = kThreads>
__device__ __forceinline__ void load_words(uint32_t* s_raw, const uint32_t* g,
                                           unsigned long long a, uint32_t nw) {
  const uint32_t h = words_head(g, a);
  const uint32_t* gb = g + (a - h);
  const uint32_t total = h + nw;
  const uint32_t nvec = total >> 2;
  const uint4* gv = reinterpret_cast<const uint4*>(gb);
  uint4* sv = reinterpret_cast<uint4*>(s_raw);
#pragma unroll 4
  for (uint32_t v = threadIdx.x; v < nvec; v += NT) sv[v] = __ldcs(gv + v);
  for (uint32_t w = (nvec << 2) + threadIdx.x; w < total; w += NT) s_raw[w] = __ldcs(gb + w);
}

// Same for doubles: element a+k lands at s_raw[doubles_head(g, a) + k].
template <int NT = kThreads>
__device__ __forceinline__ void load_doubles(double* s_raw, const double* g,
                                             unsigned long long a, uint32_t n) {
  const uint32_t h = doubles_head(g, a);
  const double* gb = g + (a - h);
  const uint32_t total = h + n;
  const uint32_t nvec = total >> 1;
  const double2* gv = reinterpret_cast<const double2*>(gb);
  double2* sv = reinterpret_cast<double2*>(s_raw);
#pragma unroll 4
  for (uint32_t v = threadIdx.x; v < nvec; v += NT) sv[v] = __ldcs(gv + v);
  for (uint32_t w = (nvec << 1) + threadIdx.x; w < total; w += NT) s_raw[w] = __ldcs(gb + w);
}

__device__ __forceinline__ void store_row(uint32_t* out_c, double* out_v, uint32_t rank,
                                          unsigned long long dst, const uint32_t* srow,
                                          double v) {
  uint32_t* o = out_c + dst * rank;
#pragma unroll 4
  for (uint32_t m = 0; m < rank; ++m) __stcs(o + m, srow[m]);
  __stcs(out_v + dst, v);
}

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// ---- TMA bulk copies (cp.async.bulk) completing on an mbarrier ----------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "QD_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra QD_WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// A byte span [g, g+len) of global memory staged at dst so that byte g+k
// lands at dst[head + k]: the enclosing 16-byte-aligned blocks are copied
// whole (a 16-byte block holding a valid byte never crosses a page, so the
// few extra bytes are always readable; they are never used).
struct Stage {
  const char* gal;  // 16-byte aligned start
  uint32_t head;    // g - gal
  uint32_t bulk;    // bytes moved by TMA from gal (multiple of 16)
};
__device__ __forceinline__ Stage make_stage(const void* g, uint32_t len) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(g);
  Stage s;
  s.gal = reinterpret_cast<const char*>(a & ~uintptr_t(15));
  s.head = (uint32_t)(a & 15);
  s.bulk = (s.head + len + 15u) & ~15u;
  return s;
}

// Digit of the row whose coordinate of mode m is get(m).
template <class G>
__device__ __forceinline__ uint32_t digit_by(G get, const DigitSpec& d) {
  if (d.lookup) {
    const uint32_t c = get(d.lookup_mode);
    return c < d.lookup_dim ? __ldg(d.lookup + c) : 0u;
  }
  uint32_t v = ((get(d.mode[0]) >> d.rsh[0]) & ((1u << d.bits[0]) - 1u)) << d.lsh[0];
#pragma unroll 1
  for (uint32_t i = 1; i < d.n; ++i)
    v |= ((get(d.mode[i]) >> d.rsh[i]) & ((1u << d.bits[i]) - 1u)) << d.lsh[i];
  return v;
}

// Register copy of a digit with at most two mode fields (the common case:
// 8-bit digits rarely straddle more than one field boundary).
struct Dig2 {
  uint32_t two, m0, r0, k0, l0, m1, r1, k1, l1;
};
__device__ __forceinline__ Dig2 dig2_of(const DigitSpec& d) {
  Dig2 f;
  f.two = d.n > 1;
  f.m0 = d.mode[0];
  f.r0 = d.rsh[0];
  f.k0 = (1u << d.bits[0]) - 1u;
  f.l0 = d.lsh[0];
  f.m1 = d.n > 1 ? d.mode[1] : d.mode[0];
  f.r1 = d.n > 1 ? d.rsh[1] : 0u;
  f.k1 = d.n > 1 ? (1u << d.bits[1]) - 1u : 0u;
  f.l1 = d.n > 1 ? d.lsh[1] : 0u;
  return f;
}
template <class G>
__device__ __forceinline__ uint32_t digit2(G get, const Dig2& f) {
  uint32_t v = ((get(f.m0) >> f.r0) & f.k0) << f.l0;
  if (f.two) v |= ((get(f.m1) >> f.r1) & f.k1) << f.l1;
  return v;
}

// Warp-aggregated counting of 32 consecutive rows' digits into a per-warp
// histogram: each run of equal digits is added once by its head lane (sorted
// inputs make long runs common).
__device__ __forceinline__ void add_runs(uint32_t* h, uint32_t d, bool valid, uint32_t nvalid) {
  const int lane = threadIdx.x & 31;
  const uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, d, 1);
  const bool head = valid && (lane == 0 || prev != d);
  const unsigned heads = __ballot_sync(0xFFFFFFFFu, head);
  if (head) {
    const unsigned after = heads & ~((2u << lane) - 1u);
    const uint32_t end = after ? (uint32_t)(__ffs(after) - 1) : nvalid;
    atomicAdd(h + d, end - lane);
  }
}

// ---------------------------------------------------------------------------
// k_chunk_hist: digit histogram of every chunk (one pass), written into the
// (run, bin, chunk) flat array that the scan turns into output cursors.
// Pass 0 also range-checks the key coordinates (count_keys, sort.cpp:54-64).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_chunk_hist(ChunkHistArgs a) {
  __shared__ uint32_t s_h[kWarps * kBins];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t R = a.rank;
  const uint64_t N = a.nnz;
  const bool fast_dig = a.dig.lookup == nullptr && a.dig.n <= 2;
  const Dig2 dg = dig2_of(a.dig);
  const uint32_t NCH = a.nc_dev ? (uint32_t)min(*a.nc_dev, (unsigned long long)a.num_chunks)
                                : a.num_chunks;
  for (uint32_t ci = blockIdx.x; ci < NCH; ci += gridDim.x) {
    for (int k = threadIdx.x; k < kWarps * kBins; k += kThreads) s_h[k] = 0;
    __syncthreads();
    const ChunkDesc cd = a.chunks[ci];
    if (threadIdx.x == 0 && a.rows_counter) atomicAdd(a.rows_counter, (unsigned long long)cd.len);
    if (a.digits) {
      // digit bytes left by the previous pass's scatter: 16 rows per load
      const uint8_t* dg8 = a.digits + cd.row_begin;
      uint32_t* wh = s_h + w * kBins;
      const uint32_t head = (uint32_t)min((unsigned long long)cd.len,
                                          (unsigned long long)((16u - ((uintptr_t)dg8 & 15u)) & 15u));
      if (threadIdx.x < head) atomicAdd(wh + dg8[threadIdx.x], 1u);
      const uint32_t nv = (cd.len - head) >> 4;
      const uint4* v4 = reinterpret_cast<const uint4*>(dg8 + head);
#pragma unroll 2
      for (uint32_t v = threadIdx.x; v < nv; v += kThreads) {
        const uint4 x = __ldcs(v4 + v);
        const uint32_t wd[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          atomicAdd(wh + (wd[q] & 0xFFu), 1u);
          atomicAdd(wh + ((wd[q] >> 8) & 0xFFu), 1u);
          atomicAdd(wh + ((wd[q] >> 16) & 0xFFu), 1u);
          atomicAdd(wh + (wd[q] >> 24), 1u);
        }
      }
      for (uint32_t k = head + nv * 16 + threadIdx.x; k < cd.len; k += kThreads)
        atomicAdd(wh + dg8[k], 1u);
      __syncthreads();
      goto flush;
    }
    if (a.in.fmt == kPK) {
      // 16-byte rows: digit from the packed word
      const ulonglong2* rows = reinterpret_cast<const ulonglong2*>(a.in.c) + cd.row_begin;
      uint32_t* wh = s_h + w * kBins;
#pragma unroll 4
      for (uint32_t k = threadIdx.x; k < cd.len; k += kThreads)
        atomicAdd(wh + ((uint32_t)(__ldcs(rows + k).x >> a.pk_shift) & a.pk_mask), 1u);
      __syncthreads();
      goto flush;
    }
    if (a.in.fmt == kSoA && fast_dig && !dg.two) {
      // SoA column, one-field digit: 16-byte loads of 4 rows per thread and
      // per-warp shared-memory atomics (intermediate order has few runs)
      const uint32_t* col = a.in.c + (size_t)dg.m0 * N + cd.row_begin;
      const uint32_t head = (uint32_t)min((unsigned long long)cd.len,
                                          (unsigned long long)((4u - ((uintptr_t)col >> 2)) & 3u));
      uint32_t* wh = s_h + w * kBins;
      if (threadIdx.x < head) atomicAdd(wh + ((col[threadIdx.x] >> dg.r0) & dg.k0), 1u);
      const uint32_t nv = (cd.len - head) >> 2;
      const uint4* vcol = reinterpret_cast<const uint4*>(col + head);
#pragma unroll 2
      for (uint32_t v = threadIdx.x; v < nv; v += kThreads) {
        const uint4 x = __ldcs(vcol + v);
        atomicAdd(wh + ((x.x >> dg.r0) & dg.k0), 1u);
        atomicAdd(wh + ((x.y >> dg.r0) & dg.k0), 1u);
        atomicAdd(wh + ((x.z >> dg.r0) & dg.k0), 1u);
        atomicAdd(wh + ((x.w >> dg.r0) & dg.k0), 1u);
      }
      for (uint32_t k = head + nv * 4 + threadIdx.x; k < cd.len; k += kThreads)
        atomicAdd(wh + ((col[k] >> dg.r0) & dg.k0), 1u);
      __syncthreads();
      goto flush;
    }
    if (a.in.fmt == kAoS && R == 4 && fast_dig && ((uintptr_t)a.in.c & 15u) == 0) {
      // AoS rank-4 rows are aligned 16-byte vectors: one load per row, two
      // rows in flight per thread, range + pack checks from the registers
      const uint32_t lim[4] = {a.lim[0], a.lim[1], a.lim[2], a.lim[3]};
      uint32_t* wh = s_h + w * kBins;
      const uint4* rows4 = reinterpret_cast<const uint4*>(a.in.c) + cd.row_begin;
      auto sel = [&](const uint4& x, uint32_t m) {
        return m == 0 ? x.x : (m == 1 ? x.y : (m == 2 ? x.z : x.w));
      };
      for (uint32_t i0 = threadIdx.x; i0 < cd.len; i0 += 2 * kThreads) {
        uint4 x[2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (i0 + u * kThreads < cd.len) x[u] = __ldcs(rows4 + i0 + u * kThreads);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t i = i0 + u * kThreads;
          if (i >= cd.len) break;
          if (x[u].x >= lim[0] || x[u].y >= lim[1] || x[u].z >= lim[2] || x[u].w >= lim[3]) {
            const unsigned long long gr = cd.row_begin + i;
            if (a.do_check) check_row(a.in.c + gr * 4, a.key, gr, a.err);
            if (a.check_pack && (x[u].x >= a.pack.lim[0] || x[u].y >= a.pack.lim[1] ||
                                 x[u].z >= a.pack.lim[2] || x[u].w >= a.pack.lim[3]))
              atomicOr(&a.err->flags, 4u);
          }
          uint32_t d = ((sel(x[u], dg.m0) >> dg.r0) & dg.k0) << dg.l0;
          if (dg.two) d |= ((sel(x[u], dg.m1) >> dg.r1) & dg.k1) << dg.l1;
          atomicAdd(wh + d, 1u);
        }
      }
      __syncthreads();
      goto flush;
    }
    if (a.in.fmt == kAoS && R == 3 && fast_dig) {
      // AoS rank-3 rows (the common first pass): coordinates in registers,
      // range + pack checks from them
      const uint32_t dm0 = dg.m0, dm1 = dg.m1;
      // per-mode limits: range check (dim for key modes) and pack check
      // (2^width) folded into one compare per coordinate
      const uint32_t lim[3] = {a.lim[0], a.lim[1], a.lim[2]};
      uint32_t* wh = s_h + w * kBins;
      auto digit3 = [&](uint32_t c0, uint32_t c1, uint32_t c2) {
        const uint32_t x0 = dm0 == 0 ? c0 : (dm0 == 1 ? c1 : c2);
        uint32_t d = ((x0 >> dg.r0) & dg.k0) << dg.l0;
        if (dg.two) {
          const uint32_t x1 = dm1 == 0 ? c0 : (dm1 == 1 ? c1 : c2);
          d |= ((x1 >> dg.r1) & dg.k1) << dg.l1;
        }
        return d;
      };
      auto check3 = [&](unsigned long long grow, uint32_t c0, uint32_t c1, uint32_t c2) {
        if (c0 >= lim[0] || c1 >= lim[1] || c2 >= lim[2]) {
          // rare: the exact checks (range: first (row, mode); pack: flag)
          if (a.do_check) check_row(a.in.c + grow * 3, a.key, grow, a.err);
          if (a.check_pack &&
              (c0 >= a.pack.lim[0] || c1 >= a.pack.lim[1] || c2 >= a.pack.lim[2]))
            atomicOr(&a.err->flags, 4u);
        }
      };
      auto scalar_rows = [&](uint32_t from, uint32_t to) {  // rows [from, to) of the chunk
        for (uint32_t i = from + threadIdx.x; i < to; i += kThreads) {
          const unsigned long long gr = cd.row_begin + i;
          const uint32_t* row = a.in.c + gr * 3;
          const uint32_t c0 = __ldcs(row), c1 = __ldcs(row + 1), c2 = __ldcs(row + 2);
          check3(gr, c0, c1, c2);
          atomicAdd(wh + digit3(c0, c1, c2), 1u);
        }
      };
      // Four rows (48 bytes = three 16-byte loads) per thread and two such
      // quads in flight; equal neighbouring digits add once.
      const uint32_t head = (uint32_t)min((unsigned long long)cd.len, (4ull - (cd.row_begin & 3ull)) & 3ull);
      const bool vec = ((uintptr_t)a.in.c & 15u) == 0;
      const uint32_t nquad = vec ? (cd.len - head) >> 2 : 0u;
      scalar_rows(0, vec ? head : cd.len);
      const uint4* q4 = reinterpret_cast<const uint4*>(a.in.c + (cd.row_begin + head) * 3);
      for (uint32_t q0 = threadIdx.x; q0 < nquad; q0 += 2 * kThreads) {
        uint4 x[2][3];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t q = q0 + u * kThreads;
          if (q < nquad) {
            x[u][0] = __ldcs(q4 + 3 * q);
            x[u][1] = __ldcs(q4 + 3 * q + 1);
            x[u][2] = __ldcs(q4 + 3 * q + 2);
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t q = q0 + u * kThreads;
          if (q >= nquad) break;
          const uint32_t wv[12] = {x[u][0].x, x[u][0].y, x[u][0].z, x[u][0].w,
                                   x[u][1].x, x[u][1].y, x[u][1].z, x[u][1].w,
                                   x[u][2].x, x[u][2].y, x[u][2].z, x[u][2].w};
          const unsigned long long gr = cd.row_begin + head + 4ull * q;
          uint32_t d[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            check3(gr + k, wv[3 * k], wv[3 * k + 1], wv[3 * k + 2]);
            d[k] = digit3(wv[3 * k], wv[3 * k + 1], wv[3 * k + 2]);
          }
          uint32_t run = 1;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (k < 3 && d[k] == d[k + 1]) {
              ++run;
            } else {
              atomicAdd(wh + d[k], run);
              run = 1;
            }
          }
        }
      }
      if (vec) scalar_rows(head + 4 * nquad, cd.len);
      __syncthreads();
      goto flush;
    }
    for (uint32_t g = w * 32; g < cd.len; g += kThreads) {  // warp-uniform
      const uint32_t i = g + lane;
      const bool valid = i < cd.len;
      const uint32_t nvalid = min(32u, cd.len - g);
      const unsigned long long r = cd.row_begin + (valid ? i : 0u);
      uint32_t d = 0;
      if (a.in.fmt == kSoA) {
        if (valid) {
          auto get = [&](uint32_t m) { return __ldcs(a.in.c + m * N + r); };
          d = fast_dig ? digit2(get, dg) : digit_by(get, a.dig);
        }
      } else {
        const uint32_t* row = a.in.c + r * R;
        if (valid) {
          if (a.do_check) check_row(row, a.key, r, a.err);
          if (a.check_pack) {
            uint32_t bad = 0;
            for (uint32_t m = 0; m < R; ++m) bad |= row[m] >= a.pack.lim[m];
            if (bad) atomicOr(&a.err->flags, 4u);
          }
          auto get = [&](uint32_t m) { return __ldg(row + m); };
          d = fast_dig ? digit2(get, dg) : digit_by(get, a.dig);
        }
      }
      add_runs(s_h + w * kBins, d, valid, nvalid);
    }
    __syncthreads();
    flush:
    uint32_t* f = a.flat + cd.coff * kBins + cd.cidx;
    for (int b = threadIdx.x; b < kBins; b += kThreads) {
      uint32_t v = 0;
#pragma unroll
      for (int x = 0; x < kWarps; ++x) v += s_h[x * kBins + b];
      f[(size_t)b * cd.nchunks] = v;
    }
    __syncthreads();
  }
}

// Shared-memory layout of k_scatter: two staging buffers (TMA double
// buffering) of T rows, plus ranking scratch and per-bin cursors.
struct ScatterLayout {
  size_t cspan, cbuf, vbuf, c0, v0, dig, rnk, sorted, whist, cnt, start, run, gbase, tmp, ofs,
      bar, total;
  __host__ __device__ ScatterLayout(uint32_t T, uint32_t rank, int fmt) {
    size_t o = 0;
    cspan = align16(size_t(T) * 4 + 32);  // one SoA column span
    if (fmt == kPK) {
      cbuf = align16(size_t(T) * 16 + 32);
      vbuf = 0;
    } else {
      cbuf = fmt == kSoA ? cspan * rank : align16(size_t(T) * rank * 4 + 32);
      vbuf = align16(size_t(T) * 8 + 32);
    }
    c0 = o; o += 2 * cbuf;
    v0 = o; o += 2 * vbuf;
    dig = o; o += 0;  // digits travel with the sorted index (s_sorted)
    rnk = o; o += 0;  // ranks live in registers
    sorted = o; o += align16(size_t(T) * 4);  // (row << 8) | digit by sorted slot
    whist = o; o += align16(size_t(kSortWarps) * kBins * 2);
    cnt = o; o += align16(kBins * 4);
    start = o; o += align16(kBins * 4);
    run = o; o += align16(kBins * 8);
    gbase = o; o += align16(kBins * 8);
    tmp = o; o += align16(64 * 8);
    ofs = o; o += align16(2 * 66 * 4);  // per buffer: R column heads + value head
    bar = o; o += 16;
    total = o;
  }
};

// ---------------------------------------------------------------------------
// k_scatter: one stable counting pass over one radix digit, chunk-ordered.
// Persistent CTAs take chunks (statically dealt); inside a chunk, tiles are
// processed in order and the advancer warp prefetches the next tile with TMA
// bulk copies (cp.async.bulk, mbarrier completion) into the other buffer
// while the CTA ranks the current tile (MATCH.ANY per 32-row round) and
// scatters it coalesced through shared memory.
// RT: compile-time rank (0 = runtime); IN/OUT: row formats (kAoS/kSoA/kPK);
// DM: digit of an AoS/SoA row inside 1 or 2 key fields (0 = general).
// ---------------------------------------------------------------------------
template <int RT, int IN, int OUT, int DM, int MX = 0>
#ifndef QD_SCATTER_MINB
#define QD_SCATTER_MINB (QD_SCATTER_CTAS * 512 / kSortThreads)
#endif
__global__ void __launch_bounds__(kSortThreads, QD_SCATTER_MINB) k_scatter(ScatterArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t R = RT ? RT : a.rank;
  const uint64_t N = a.nnz;
  const ScatterLayout L(a.T, R, IN);
  const uint32_t NCH = a.nc_dev ? (uint32_t)min(*a.nc_dev, (unsigned long long)a.num_chunks)
                                : a.num_chunks;
  uint32_t* s_sorted = reinterpret_cast<uint32_t*>(smem + L.sorted);
  uint16_t* s_whist = reinterpret_cast<uint16_t*>(smem + L.whist);
  uint32_t* s_start = reinterpret_cast<uint32_t*>(smem + L.start);
  unsigned long long* s_run = reinterpret_cast<unsigned long long*>(smem + L.run);
  long long* s_gbase = reinterpret_cast<long long*>(smem + L.gbase);
  unsigned long long* s_tmp = reinterpret_cast<unsigned long long*>(smem + L.tmp);
  uint32_t* s_ofs = reinterpret_cast<uint32_t*>(smem + L.ofs);  // [2][66] byte offsets
  unsigned long long* s_bar = reinterpret_cast<unsigned long long*>(smem + L.bar);
  // (chunk, tile-in-chunk) of iteration it, double-buffered by it & 1: the
  // advancer publishes iteration it+1's during iteration it, and the barrier
  // ending iteration it orders that before every thread's read
  __shared__ uint32_t s_chunk[2], s_tile[2];
  __shared__ ChunkDesc s_cd[2];          // descriptor of the chunk staged in buffer b

  // spans of a tile: AoS {coords, values}, SoA {column 0..R-1, values},
  // PK {rows}.  Span index R always means "values".
  constexpr bool kSoAIn = IN == kSoA;
  auto nspans = [&]() { return IN == kPK ? 1u : (kSoAIn ? R + 1 : 2u); };
  auto span_index = [&](uint32_t j) { return (IN == kAoS && j == 1) ? R : j; };
  auto span = [&](uint32_t k, unsigned long long rb, uint32_t n, const void*& g, uint32_t& len) {
    if (IN == kPK) {
      g = reinterpret_cast<const ulonglong2*>(a.in.c) + rb;
      len = n * 16;
    } else if (k == R) {
      g = a.in.v + rb;
      len = n * 8;
    } else if (kSoAIn) {
      g = a.in.c + (size_t)k * N + rb;
      len = n * 4;
    } else {
      g = a.in.c + rb * R;
      len = n * R * 4;
    }
  };
  auto span_dst = [&](uint32_t b, uint32_t k) -> unsigned char* {
    if (IN != kPK && k == R) return smem + L.v0 + b * L.vbuf;
    return smem + L.c0 + b * L.cbuf + (kSoAIn ? k * L.cspan : 0);
  };

  // The advancer warp (the last one, idle while the first kBins threads fold
  // the bin counts) issues the bulk loads of the next tile.  Chunks are
  // assigned statically (blockIdx.x + k*gridDim.x): no atomics, and the next
  // chunk's descriptor is loaded one chunk ahead.
  constexpr uint32_t kAdv = kSortThreads - 32;
  ChunkDesc pre{};  // advancer only: descriptor of this CTA's next chunk
  uint32_t pre_idx = 0;  // advancer only: index of that chunk
  // the chunk after the current one: dynamic (a per-launch atomic counter
  // deals chunks gridDim.x.. in completion order, so CTAs that drew easy
  // tiles take more) or static round robin; whole advancer warp
  auto next_chunk = [&](uint32_t cur) -> uint32_t {
#if QD_DYNAMIC_CHUNKS
    uint32_t x = 0;
    if ((threadIdx.x & 31) == 0) x = gridDim.x + atomicAdd(a.chunk_counter, 1u);
    (void)cur;
    return __shfl_sync(0xFFFFFFFFu, x, 0);
#else
    return cur + gridDim.x;
#endif
  };
  // called by the whole advancer warp: lane j issues span j's bulk copy
  auto load_tile = [&](uint32_t b, const ChunkDesc& cd, uint32_t ti) {
    const uint32_t lane = threadIdx.x & 31;
    if (lane == 0) s_cd[b] = cd;
    const unsigned long long rb = cd.row_begin + (unsigned long long)ti * a.T;
    const uint32_t n = (uint32_t)min((unsigned long long)a.T, cd.row_begin + cd.len - rb);
    const uint32_t ns = nspans();
    uint32_t bulk = 0;
    Stage st{};
    if (lane < ns) {
      const void* g;
      uint32_t len;
      span(span_index(lane), rb, n, g, len);
      st = make_stage(g, len);
      bulk = st.bulk;
      s_ofs[b * 66 + span_index(lane)] = st.head;
    }
    uint32_t total = bulk;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xFFFFFFFFu, total, o);
    // No proxy fence: the buffer was only READ by the generic proxy, and the
    // CTA barrier that ended its last use orders those reads before this.
    if (lane == 0) mbar_expect_tx(&s_bar[b], total);
    __syncwarp();
    if (lane < ns && st.bulk) bulk_g2s(span_dst(b, span_index(lane)), st.gal, st.bulk, &s_bar[b]);
  };
  // advancer warp: pick the tile after (ci, ti) (whose chunk is in slot b^1),
  // publish it in s_chunk/s_tile and start loading it into buffer b
  auto advance = [&](uint32_t b, uint32_t ci, uint32_t ti, uint32_t pslot) {
    uint32_t nc = ci, nt = ti + 1;
    ChunkDesc cd = s_cd[b ^ 1u];
    if (nt * (unsigned long long)a.T >= cd.len) {
      nc = pre_idx;
      nt = 0;
      cd = pre;
      if (nc < NCH) {
        pre_idx = next_chunk(nc);
        if (pre_idx < NCH) pre = a.chunks[pre_idx];
      }
    }
    if ((threadIdx.x & 31) == 0) {
      s_chunk[pslot] = nc;
      s_tile[pslot] = nt;
    }
    if (nc < NCH) load_tile(b, cd, nt);
  };

  if (threadIdx.x == kAdv) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= kAdv) {  // the advancer warp
    const uint32_t c0 = blockIdx.x;
    if (threadIdx.x == kAdv) {
      s_chunk[0] = c0;
      s_tile[0] = 0;
    }
    pre_idx = c0 < NCH ? next_chunk(c0) : NCH;
    if (c0 < NCH) {
      if (pre_idx < NCH) pre = a.chunks[pre_idx];
      load_tile(0, a.chunks[c0], 0);
    }
  }
  __syncthreads();

  const Dig2 dg = dig2_of(a.dig);
  uint32_t phases = 0u;
  long long peer_shift = 0;  // peers: destination row of this bin's first row minus its part start
  long long t_last = clock64();
#define QD_TMARK(ph)                                           \
  if (a.dbg_t && threadIdx.x == 0) {                           \
    const long long t_now = clock64();                         \
    atomicAdd(a.dbg_t + (ph), (unsigned long long)(t_now - t_last)); \
    t_last = t_now;                                            \
  }
  for (uint32_t it = 0;; ++it) {
    const uint32_t b = it & 1u;
    const uint32_t ci = s_chunk[it & 1u], ti = s_tile[it & 1u];
    if (ci >= NCH) break;
    QD_TMARK(1);
    const ChunkDesc cd = s_cd[b];  // the advancer only refills the other slot
    const unsigned long long rb = cd.row_begin + (unsigned long long)ti * a.T;
    const uint32_t n = (uint32_t)min((unsigned long long)a.T, cd.row_begin + cd.len - rb);
    if (ti == 0 && threadIdx.x < kBins) {
      // this chunk's cursor per bin: scanned (run, bin, chunk) offset
      const unsigned long long base0 = a.offs[cd.coff * kBins];
      const unsigned long long rs = a.run_start ? a.run_start[cd.li] : 0ull;
      s_run[threadIdx.x] =
          a.offs[cd.coff * kBins + (size_t)threadIdx.x * cd.nchunks + cd.cidx] - base0 + rs;
      if (a.peers)  // part start = the bin's cursor in the run's first chunk
        peer_shift = (long long)a.peers[threadIdx.x].off -
                     (long long)(a.offs[cd.coff * kBins + (size_t)threadIdx.x * cd.nchunks] - base0 + rs);
    }
    {  // each warp clears its own histogram (no block barrier before ranking)
      uint16_t* whz = s_whist + (threadIdx.x >> 5) * kBins;
      for (int k = threadIdx.x & 31; k < kBins; k += 32) whz[k] = 0;
      __syncwarp();
    }
#if QD_EARLY_ADVANCE
    // buffer b^1 was released by the previous tile's closing barrier: start
    // the next tile's bulk copies before this tile's work
    if (threadIdx.x >= kAdv) advance(b ^ 1u, ci, ti, (it + 1) & 1u);
#endif
    mbar_wait(&s_bar[b], (phases >> b) & 1u);  // each thread observes the TMA completion
    QD_TMARK(2);
    phases ^= 1u << b;
    const unsigned char* scb = smem + L.c0 + b * L.cbuf;
    const uint32_t* s_ofsb = s_ofs + b * 66;
    const ulonglong2* s_pk = reinterpret_cast<const ulonglong2*>(scb);  // PK rows
    // byte offset of (row 0, mode m) in the staged tile, and the row stride
    const uint32_t rstride = kSoAIn ? 4u : R * 4u;
    auto mbase = [&](uint32_t m) -> uint32_t {
      return kSoAIn ? m * (uint32_t)L.cspan + s_ofsb[m] : s_ofsb[0] + m * 4u;
    };
    auto coord = [&](uint32_t i, uint32_t m) -> uint32_t {
      return *reinterpret_cast<const uint32_t*>(scb + mbase(m) + i * rstride);
    };
    // the digit's (at most two) fields, resolved once per tile
    const uint32_t dbase0 = (IN != kPK && DM) ? mbase(dg.m0) : 0u;
    const uint32_t dbase1 = (IN != kPK && DM == 2) ? mbase(dg.m1) : 0u;
    auto digit_at = [&](uint32_t i) -> uint32_t {
      if (IN == kPK) return (uint32_t)(s_pk[i].x >> a.pk_shift) & a.pk_mask;
      if (DM == 0) return digit_by([&](uint32_t m) { return coord(i, m); }, a.dig);
      const uint32_t x0 = *reinterpret_cast<const uint32_t*>(scb + dbase0 + i * rstride);
      uint32_t v = (x0 >> dg.r0) & dg.k0;
      if (DM == 2) {
        const uint32_t x1 = *reinterpret_cast<const uint32_t*>(scb + dbase1 + i * rstride);
        v = (v << dg.l0) | (((x1 >> dg.r1) & dg.k1) << dg.l1);
      }
      return v;
    };

    // Digits and stable warp ranks, kept in registers: warp w owns rows
    // [w*ipw, (w+1)*ipw) and walks them in rounds of 32 (rank order = row
    // order); packed[r] = (rank within the warp's equal digits << 8) | digit.
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // rows per warp rounded up to whole 32-row rounds: every round but the
    // tile's last is full (trailing warps may get fewer rows or none)
#if QD_FULL_ROUNDS
    const uint32_t ipw = (((n + kSortWarps - 1) / kSortWarps) + 31u) & ~31u;
#else
    const uint32_t ipw = (n + kSortWarps - 1) / kSortWarps;
#endif
    const uint32_t lo = w * ipw, hi = min(n, lo + ipw);
    uint16_t* wh = s_whist + w * kBins;
    const unsigned below = (1u << lane) - 1u;
    uint32_t packed[kMaxRounds];
    // full rounds (every lane valid: no ballot, no predicates), then at most
    // one partial round
    const uint32_t nrow = hi > lo ? hi - lo : 0u;
    const uint32_t nfull = nrow >> 5;
#pragma unroll
    for (int r = 0; r < kMaxRounds; ++r) {
      if ((uint32_t)r >= nfull) break;  // warp-uniform
      const uint32_t p = lo + r * 32 + lane;
      const uint32_t d = digit_at(p);
      const unsigned peers = adaptive_peers(d, 0xFFFFFFFFu, a.dbits, a.rank_mode, a.match_max);
#if QD_RANK_BCAST
      // every lane reads its digit's count (equal digits: one broadcast
      // wavefront), the lowest peer writes it back: no shuffle
      const uint32_t bcount = wh[d];
      if ((peers & below) == 0u) wh[d] = (uint16_t)(bcount + __popc(peers));
      __syncwarp();
#else
      const int leader = __ffs(peers) - 1;
      uint32_t bcount = 0;
      if (lane == leader) {
        bcount = wh[d];
        wh[d] = (uint16_t)(bcount + __popc(peers));
      }
      bcount = __shfl_sync(0xFFFFFFFFu, bcount, leader);
#endif
      packed[r] = ((bcount + __popc(peers & below)) << 8) | d;
    }
    if (nrow & 31u) {  // warp-uniform
      const uint32_t r = nfull;
      const uint32_t p = lo + r * 32 + lane;
      const bool valid = lane < (nrow & 31u);
      uint32_t d = 0;
      if (valid) d = digit_at(p);
      unsigned peers = adaptive_peers(d, (1u << (nrow & 31u)) - 1u, a.dbits, a.rank_mode, a.match_max);
      if (!valid) peers = 1u << lane;
#if QD_RANK_BCAST
      const uint32_t bcount = valid ? wh[d] : 0u;
      if (valid && (peers & below) == 0u) wh[d] = (uint16_t)(bcount + __popc(peers));
      __syncwarp();
#else
      const int leader = __ffs(peers) - 1;
      uint32_t bcount = 0;
      if (valid && lane == leader) {
        bcount = wh[d];
        wh[d] = (uint16_t)(bcount + __popc(peers));
      }
      bcount = __shfl_sync(0xFFFFFFFFu, bcount, leader);
#endif
      const uint32_t v = ((bcount + __popc(peers & below)) << 8) | d;
#pragma unroll
      for (int q = 0; q < kMaxRounds; ++q)
        if ((uint32_t)q == r) packed[q] = v;  // static register index
    }
    __syncthreads();
    QD_TMARK(3);
#if !QD_EARLY_ADVANCE
    if (threadIdx.x >= kAdv) advance(b ^ 1u, ci, ti, (it + 1) & 1u);  // overlaps bin_totals
#endif
    // bin totals + bin scan with two barriers: thread b (< kBins) turns the
    // column of warp counts into warp-exclusive offsets, the first kBins/32
    // warps scan their 32 bins with shuffles, then combine the warp sums
    {
      uint32_t* s_wsum = reinterpret_cast<uint32_t*>(s_tmp);
      uint32_t cnt = 0, incl = 0;
      if (threadIdx.x < kBins) {
#pragma unroll
        for (int x = 0; x < kSortWarps; ++x) {
          const uint32_t c = s_whist[x * kBins + threadIdx.x];
          s_whist[x * kBins + threadIdx.x] = (uint16_t)cnt;
          cnt += c;
        }
        incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= (uint32_t)o) incl += y;
        }
        if (lane == 31) s_wsum[w] = incl;
      }
      __syncthreads();
      QD_TMARK(4);
      if (threadIdx.x < kBins) {
        uint32_t base = 0;
        for (uint32_t x = 0; x < w; ++x) base += s_wsum[x];
        const uint32_t start = base + incl - cnt;
        s_start[threadIdx.x] = start;
        const unsigned long long r0 = s_run[threadIdx.x];
        s_gbase[threadIdx.x] = (long long)r0 - (long long)start + peer_shift;
        s_run[threadIdx.x] = r0 + cnt;
      }
    }
    __syncthreads();
    QD_TMARK(5);
    // sorted position of every row: all lookups first, then the stores (the
    // compiler cannot hoist a lookup above a possibly aliasing store); the
    // row's digit travels with its index, so the store loop reads both
    // sequentially by sorted slot (no random digit gather)
#pragma unroll
    for (int r = 0; r < kMaxRounds; ++r) {
      if (lo + r * 32 >= hi) break;
      const uint32_t d = packed[r] & 0xFFu;
      packed[r] = ((s_start[d] + wh[d] + (packed[r] >> 8)) << 8) | d;
    }
#pragma unroll
    for (int r = 0; r < kMaxRounds; ++r) {
      const uint32_t p = lo + r * 32 + lane;
      if (lo + r * 32 >= hi) break;
      if (p < hi) s_sorted[packed[r] >> 8] = (p << 8) | (packed[r] & 0xFFu);
    }
    __syncthreads();
    QD_TMARK(6);
    // ---- scatter, in sorted order so consecutive threads write consecutive rows
    uint32_t cb[RT > 0 ? RT : 1];
    if (IN != kPK && RT) {
#pragma unroll
      for (int m = 0; m < (RT > 0 ? RT : 1); ++m) cb[m] = mbase(m);
    }
    // AoS tiles: a row's coordinates with vector shared loads (rank 4 needs a
    // 16-byte aligned staging head; tile-uniform)
    const bool vec_in = IN == kAoS && RT && (RT != 4 || (s_ofsb[0] & 15u) == 0);
    auto load_cv = [&](uint32_t i, uint32_t (&cv)[RT > 0 ? RT : 1]) {
      if (vec_in) {
        load_row_words<(RT > 0 ? RT : 1)>(
            reinterpret_cast<const uint32_t*>(scb + cb[0] + i * rstride), cv);
      } else {
#pragma unroll
        for (int m = 0; m < (RT > 0 ? RT : 1); ++m)
          cv[m] = *reinterpret_cast<const uint32_t*>(scb + cb[m] + i * rstride);
      }
    };
    const uint32_t vbase = IN == kPK ? 0u : (uint32_t)(span_dst(b, R) - scb) + s_ofsb[R];
    // prefix modes left out of the packed rows: constant within the tile's run
    uint32_t impv[RT > 0 ? RT : 1];
#pragma unroll
    for (int m = 0; m < (RT > 0 ? RT : 1); ++m) {
      impv[m] = 0u;
      if (MX && IN == kPK && OUT != kPK && a.pf.impk[m] != 0xFFu)
        impv[m] = __ldg(a.run_prefix + (size_t)cd.li * a.pack.n_imp + a.pf.impk[m]);
    }
    for (uint32_t j = threadIdx.x; j < n; j += kSortThreads) {
      const uint32_t sj = s_sorted[j];
      const uint32_t i = sj >> 8;
      const unsigned long long dst = (unsigned long long)(s_gbase[sj & 0xFFu] + j);
      if (a.dbg & 1) continue;
      if (IN == kPK) {
        const ulonglong2 row = s_pk[i];
        if (OUT == kPK) {
          __stcs(reinterpret_cast<ulonglong2*>(a.out.c) + dst, row);
          if (a.next_dig) __stcs(a.next_dig + dst, (uint8_t)((row.x >> a.nd_shift) & a.nd_mask));
        } else {  // unpack into AoS
          uint32_t* o = a.out.c + dst * R;
          if (MX && RT) {
            // bit fields, then the mixed-radix part from its last position
            // down (nk_n - 1 divisions); static indices keep cv in registers
            constexpr int kR = RT > 0 ? RT : 1;
            uint32_t cv[kR];
#pragma unroll
            for (int m = 0; m < kR; ++m) cv[m] = (uint32_t)(row.x >> a.pf.fsh[m]) & a.pf.fmask[m];
            if (a.pf.mixed) {
              unsigned long long hi = row.x >> a.pf.key_bits;
              uint32_t v[kR];
#pragma unroll
              for (int jj = kR - 1; jj >= 1; --jj) {
                v[jj] = 0u;
                if ((uint32_t)jj < a.pf.nk_n) hi = div_magic(hi, a.pf.dimj[jj], a.pf.magic[jj], v[jj]);
              }
              v[0] = (uint32_t)hi;
#pragma unroll
              for (int m = 0; m < kR; ++m) {
                const uint32_t pos = a.pf.mpos[m];
                uint32_t x = v[0];
#pragma unroll
                for (int jj = 1; jj < kR; ++jj) x = pos == (uint32_t)jj ? v[jj] : x;
                if (pos < (uint32_t)kR) cv[m] = x;
              }
            }
#pragma unroll
            for (int m = 0; m < (RT > 0 ? RT : 1); ++m)
              if (a.pf.impk[m] != 0xFFu) cv[m] = impv[m];
            if (RT != 4 || a.vec_out) {
              store_row_words<(RT > 0 ? RT : 1)>(o, cv);
            } else {
#pragma unroll
              for (int m = 0; m < (RT > 0 ? RT : 1); ++m) __stcs(o + m, cv[m]);
            }
          } else if (MX) {
            unpack_coords(a.pack, R, row.x, [&](uint32_t m, uint32_t v) { __stcs(o + m, v); });
            for (uint32_t k = 0; k < a.pack.n_imp; ++k)
              __stcs(o + a.pack.imp_mode[k],
                     __ldg(a.run_prefix + (size_t)s_cd[b].li * a.pack.n_imp + k));
          } else if (RT) {
            uint32_t cv[RT > 0 ? RT : 1];
#pragma unroll
            for (int m = 0; m < (RT > 0 ? RT : 1); ++m)
              cv[m] = (uint32_t)(row.x >> a.pf.fsh[m]) & a.pf.fmask[m];
            if (RT != 4 || a.vec_out) {
              store_row_words<(RT > 0 ? RT : 1)>(o, cv);
            } else {
#pragma unroll
              for (int m = 0; m < (RT > 0 ? RT : 1); ++m) __stcs(o + m, cv[m]);
            }
          } else {
            for (uint32_t m = 0; m < R; ++m)
              __stcs(o + m, (uint32_t)(row.x >> a.pack.off[m]) &
                                (uint32_t)((1ull << a.pack.width[m]) - 1ull));
          }
          __stcs(a.out.v + dst, __longlong_as_double((long long)row.y));
        }
        continue;
      }
      const double v = *reinterpret_cast<const double*>(scb + vbase + i * 8u);
      // AoS output arrays: the bin's peer destination when partitioning into peers
      uint32_t* const oc = (OUT == kAoS && a.peers)
                               ? reinterpret_cast<uint32_t*>(a.peers[sj & 0xFFu].c) : a.out.c;
      double* const ov = (OUT == kAoS && a.peers)
                             ? reinterpret_cast<double*>(a.peers[sj & 0xFFu].v) : a.out.v;
      if (OUT == kPK) {  // pack (first pass)
        unsigned long long pk = 0;
        if (MX && RT) {
          uint32_t cv[RT > 0 ? RT : 1];
          load_cv(i, cv);
          unsigned long long hi = 0;
#pragma unroll
          for (int m = 0; m < (RT > 0 ? RT : 1); ++m) {
            pk |= (unsigned long long)(cv[m] & a.pf.fmask[m]) << a.pf.fsh[m];
            hi += (unsigned long long)cv[m] * a.pf.mul[m];
          }
          if (a.pf.mixed) pk |= hi << a.pf.key_bits;
        } else if (MX) {
          pk = pack_coords(a.pack, R, [&](uint32_t m) { return coord(i, m); });
        } else if (RT) {
          uint32_t cv[RT > 0 ? RT : 1];
          load_cv(i, cv);
#pragma unroll
          for (int m = 0; m < (RT > 0 ? RT : 1); ++m)
            pk |= (unsigned long long)(cv[m] & a.pf.fmask[m]) << a.pf.fsh[m];
        } else {
          for (uint32_t m = 0; m < R; ++m)
            pk |= (unsigned long long)coord(i, m) << a.pack.off[m];
        }
        __stcs(reinterpret_cast<ulonglong2*>(a.out.c) + dst,
               make_ulonglong2(pk, (unsigned long long)__double_as_longlong(v)));
        if (a.next_dig) __stcs(a.next_dig + dst, (uint8_t)((pk >> a.nd_shift) & a.nd_mask));
        continue;
      }
      if (RT && OUT == kAoS && IN == kAoS) {
        uint32_t cv[RT > 0 ? RT : 1];
        load_cv(i, cv);
        uint32_t* o = oc + dst * (RT > 0 ? RT : 1);
        if (RT != 4 || a.vec_out) {
          store_row_words<(RT > 0 ? RT : 1)>(o, cv);
        } else {
#pragma unroll
          for (int m = 0; m < (RT > 0 ? RT : 1); ++m) __stcs(o + m, cv[m]);
        }
      } else if (RT) {
#pragma unroll
        for (int m = 0; m < (RT > 0 ? RT : 1); ++m) {
          const uint32_t x = *reinterpret_cast<const uint32_t*>(scb + cb[m] + i * rstride);
          __stcs(OUT == kSoA ? a.out.c + (size_t)m * N + dst : oc + dst * RT + m, x);
        }
      } else {
        for (uint32_t m = 0; m < R; ++m)
          __stcs(OUT == kSoA ? a.out.c + (size_t)m * N + dst : oc + dst * R + m, coord(i, m));
      }
      __stcs(ov + dst, v);
      if (a.next_dig)  // next pass's digit (unpacked rows: from the coordinates)
        __stcs(a.next_dig + dst, (uint8_t)digit_by([&](uint32_t m) { return coord(i, m); }, a.ndig));
    }
    __syncthreads();  // buffer b and the scratch are free again
    QD_TMARK(7);
  }
}

// ---------------------------------------------------------------------------
// k_small: the latency regime in ONE cooperative kernel.  A single-group plan
// (prefix P, keys K; every plan of configs 1 and 4) on a tensor of at most
// kSmallRows rows is a stable sort by the composite key (P, K) whenever the
// rows are non-decreasing in P — the group's runs of equal P are then
// contiguous and in P order, so sorting within them (Alg. 2, sort.cpp:80-134)
// equals sorting by (P, K).  The kernel checks exactly that (and that every
// composite coordinate is below its dimension); if either fails it raises a
// flag and the host reruns the call on the general path, which reproduces the
// reference's semantics (and errors) for any input.
//
// Elements {composite key, source row} (16 bytes) go through ceil(bits/8)
// stable LSD counting passes, L2-resident at these sizes; grid-wide barriers
// replace kernel boundaries.  Per pass: (1) one CTA per bin scans that bin's
// per-CTA counts (the (bin, CTA) order = parallel.cpp:88-100's (key, worker)
// order), (2) every CTA scatters its own contiguous chunk tile by tile (warp
// MATCH.ANY ranking, per-warp counts, bin offsets in shared memory), (3) every
// CTA counts the next digit over its chunk of the output.  The last step
// gathers the AoS rows by source row (random reads hit L2).
// ---------------------------------------------------------------------------
constexpr int kSmallThreads = 512;
constexpr int kSmallWarps = kSmallThreads / 32;
constexpr uint32_t kSmallTile = 4096;                      // elements per ranked tile (dynamic smem)
constexpr int kSmallRounds = kSmallTile / kSmallThreads;  // 32-row rounds per warp
constexpr uint64_t kSmallRows = 1ull << 22;
constexpr int kSmallMaxPasses = 8;

constexpr size_t kSmallSmem = kSmallTile * 20 + kSmallWarps * kBins * 2 + 3 * kBins * 4 + 64 * 4 + 16;

struct SmallArgs {
  const uint32_t* in_c;
  const double* in_v;
  uint32_t* out_c;
  double* out_v;
  uint32_t rank;
  uint64_t nnz;
  uint32_t nc, npre;  // composite modes (prefix first), number of prefix modes
  uint8_t cmode[kMaxKeys], csh[kMaxKeys];
  uint32_t cdim[kMaxKeys];
  uint32_t P;
  uint32_t dlo[kSmallMaxPasses], dmask[kSmallMaxPasses];
  ulonglong2* ea;
  ulonglong2* eb;
  uint32_t* hist;   // [kBins][gridDim.x]
  uint32_t* offs;   // [kBins][gridDim.x]
  uint32_t* total;  // [kBins]
  ErrBlock* err;
  unsigned long long* dbg;  // QD_SMALL_DBG: %globaltimer at phase ends (CTA 0, thread 0)
  int rank_mode;            // 0: MATCH.ANY peers, 1: ballots (QD_SMALL_RANK)
  uint32_t dbits[kSmallMaxPasses];
};

__device__ __forceinline__ void small_mark(const SmallArgs& a, int k) {
  if (a.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg[k] = t;
  }
}

__global__ void __launch_bounds__(kSmallThreads, 2) k_small(SmallArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem[];
  ulonglong2* s_el = reinterpret_cast<ulonglong2*>(smem);                    // [kSmallTile]
  uint32_t* s_srt = reinterpret_cast<uint32_t*>(s_el + kSmallTile);         // [kSmallTile]
  uint16_t* s_wh = reinterpret_cast<uint16_t*>(s_srt + kSmallTile);         // [warps][kBins]
  uint32_t* s_cur = reinterpret_cast<uint32_t*>(s_wh + kSmallWarps * kBins);
  uint32_t* s_tstart = s_cur + kBins;
  uint32_t* s_h = s_tstart + kBins;
  uint32_t* s_tmp = s_h + kBins;  // [64]

  const uint32_t G = gridDim.x, cta = blockIdx.x, t = threadIdx.x;
  const uint32_t lane = t & 31, w = t >> 5;
  const uint64_t N = a.nnz;
  const uint64_t lo = N * cta / G, hi = N * (cta + 1) / G;
  const uint32_t R = a.rank;
  small_mark(a, 0);
  unsigned long long* s_bar = reinterpret_cast<unsigned long long*>(s_tmp + 64);
  uint32_t phase = 0;
  // the first tile of this CTA's chunk of `src`, by TMA (issued as soon as
  // the data is final, so the copy overlaps the barriers and scans after it)
  auto issue_first = [&](const ulonglong2* src) {
    if (threadIdx.x == 0 && lo < hi) {
      const uint32_t n0 = (uint32_t)min((unsigned long long)kSmallTile, (unsigned long long)(hi - lo));
      mbar_expect_tx(s_bar, n0 * 16u);
      bulk_g2s(s_el, src + lo, n0 * 16u, s_bar);
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }

  // elements in input order + the first digit's counts of this chunk
  for (uint32_t b = t; b < kBins; b += kSmallThreads) s_h[b] = 0u;
  __syncthreads();
  for (uint64_t i = lo + t; i < hi; i += kSmallThreads) {
    const uint32_t* row = a.in_c + i * R;
    unsigned long long key = 0;
    bool bad = false;
    for (uint32_t j = 0; j < a.nc; ++j) {
      const uint32_t x = row[a.cmode[j]];
      bad |= x >= a.cdim[j];
      key |= (unsigned long long)x << a.csh[j];
    }
    if (a.npre && i > 0) {  // rows non-decreasing in the prefix
      const uint32_t* pr = row - R;
      for (uint32_t j = 0; j < a.npre; ++j) {
        const uint32_t x = row[a.cmode[j]], y = pr[a.cmode[j]];
        if (x != y) {
          bad |= x < y;
          break;
        }
      }
    }
    if (bad) atomicOr(&a.err->flags, 8u);
    // the final gather reads the values at random: bring them into L2 now
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a.in_v + i));
    a.ea[i] = make_ulonglong2(key, i);
    atomicAdd(&s_h[(uint32_t)(key >> a.dlo[0]) & a.dmask[0]], 1u);
  }
  __syncthreads();
  for (uint32_t b = t; b < kBins; b += kSmallThreads) a.hist[(size_t)b * G + cta] = s_h[b];
  small_mark(a, 1);
  grid.sync();
  small_mark(a, 2);
  // (generic-proxy writes of ea by other CTAs, ordered by the grid barrier,
  // before this CTA's async-proxy reads)
  asm volatile("fence.proxy.async.global;" ::: "memory");
  issue_first(a.ea);

  const unsigned below = (1u << lane) - 1u;
  for (uint32_t q = 0; q < a.P; ++q) {
    const ulonglong2* src = (q & 1u) ? a.eb : a.ea;
    ulonglong2* dst = (q & 1u) ? a.ea : a.eb;
    const uint32_t dlo = a.dlo[q], dmask = a.dmask[q];
    // (1) one CTA per bin: exclusive scan of the bin's counts over the CTAs
    for (uint32_t b = cta; b < kBins; b += G) {
      const uint32_t v = t < G ? a.hist[(size_t)b * G + t] : 0u;
      uint32_t tot = 0;
      const uint32_t ex = block_excl_scan<kSmallThreads>(v, s_tmp, &tot);
      if (t < G) a.offs[(size_t)b * G + t] = ex;
      if (t == 0) a.total[b] = tot;
    }
    small_mark(a, 3 + 6 * q);
    grid.sync();
    small_mark(a, 4 + 6 * q);
    // (2) this CTA's cursor per bin, then its chunk tile by tile
    {
      const uint32_t v = t < kBins ? a.total[t] : 0u;
      const uint32_t ex = block_excl_scan<kSmallThreads>(v, s_tmp);
      if (t < kBins) s_cur[t] = ex + a.offs[(size_t)t * G + cta];
    }
    for (uint64_t base = lo; base < hi; base += kSmallTile) {
      const uint32_t n = (uint32_t)min((unsigned long long)kSmallTile, (unsigned long long)(hi - base));
      if (base == lo) {  // issued after the previous pass's barrier
        mbar_wait(s_bar, phase);
        phase ^= 1u;
        if (q == 0) small_mark(a, 50);
      } else {
        for (uint32_t k = t; k < n; k += kSmallThreads) s_el[k] = src[base + k];
      }
      uint16_t* wh = s_wh + w * kBins;
      for (uint32_t k = lane; k < kBins / 8; k += 32)
        reinterpret_cast<uint4*>(wh)[k] = make_uint4(0u, 0u, 0u, 0u);
      __syncthreads();
      const uint32_t ipw = (((n + kSmallWarps - 1) / kSmallWarps) + 31u) & ~31u;
      const uint32_t rlo = w * ipw, rhi = min(n, rlo + ipw);
      uint32_t packed[kSmallRounds];
#pragma unroll
      for (int r = 0; r < kSmallRounds; ++r) {
        const uint32_t p = rlo + r * 32 + lane;
        if (rlo + r * 32 >= rhi) break;  // warp-uniform
        const bool valid = p < rhi;
        const uint32_t d = valid ? (uint32_t)(s_el[p].x >> dlo) & dmask : 0xFFFFFFFFu;
        const unsigned vm = __ballot_sync(0xFFFFFFFFu, valid);
        const unsigned peers = a.rank_mode ? (ballot_peers(d, vm, a.dbits[q]) | (valid ? 0u : 1u << lane))
                                           : __match_any_sync(0xFFFFFFFFu, d);
        const uint32_t c0 = valid ? wh[d] : 0u;
        __syncwarp();
        if (valid && (peers & below) == 0u) wh[d] = (uint16_t)(c0 + __popc(peers));
        __syncwarp();
        packed[r] = ((c0 + __popc(peers & below)) << 8) | (d & 0xFFu);
      }
      __syncthreads();
      if (q == 0 && base == lo) small_mark(a, 51);
      // warp-exclusive offsets per bin and the bins' starts in the tile
      uint32_t cnt = 0;
      {
        uint32_t incl = 0;
        if (t < kBins) {
#pragma unroll
          for (int x = 0; x < kSmallWarps; ++x) {
            const uint32_t cx = s_wh[x * kBins + t];
            s_wh[x * kBins + t] = (uint16_t)cnt;
            cnt += cx;
          }
        }
        const uint32_t ex = block_excl_scan<kSmallThreads>(t < kBins ? cnt : 0u, s_tmp);
        (void)incl;
        if (t < kBins) s_tstart[t] = ex;
      }
      __syncthreads();
      if (q == 0 && base == lo) small_mark(a, 52);
#pragma unroll
      for (int r = 0; r < kSmallRounds; ++r) {
        const uint32_t p = rlo + r * 32 + lane;
        if (rlo + r * 32 >= rhi) break;
        if (p < rhi) {
          const uint32_t d = packed[r] & 0xFFu;
          s_srt[s_tstart[d] + wh[d] + (packed[r] >> 8)] = (p << 8) | d;
        }
      }
      __syncthreads();
      if (q == 0 && base == lo) small_mark(a, 53);
      if (q + 1 < a.P) {
        for (uint32_t j = t; j < n; j += kSmallThreads) {
          const uint32_t x = s_srt[j];
          const uint32_t d = x & 0xFFu;
          dst[s_cur[d] + (j - s_tstart[d])] = s_el[x >> 8];
        }
      } else {
        // the last pass writes the rows themselves, gathered by source row
        // (random reads hit L2), four per thread in flight
        constexpr int kG = 4;
        for (uint32_t j0 = t; j0 < n; j0 += kG * kSmallThreads) {
          unsigned long long pos[kG], src[kG];
#pragma unroll
          for (int u = 0; u < kG; ++u) {
            const uint32_t j = j0 + u * kSmallThreads;
            pos[u] = ~0ull;
            src[u] = 0ull;
            if (j < n) {
              const uint32_t x = s_srt[j];
              const uint32_t d = x & 0xFFu;
              pos[u] = s_cur[d] + (j - s_tstart[d]);
              src[u] = s_el[x >> 8].y;
            }
          }
          double v[kG];
#pragma unroll
          for (int u = 0; u < kG; ++u) v[u] = __ldg(a.in_v + src[u]);
          if (R == 3) {
            uint32_t cx[kG][3];
#pragma unroll
            for (int u = 0; u < kG; ++u)
#pragma unroll
              for (int m = 0; m < 3; ++m) cx[u][m] = __ldg(a.in_c + src[u] * 3 + m);
#pragma unroll
            for (int u = 0; u < kG; ++u) {
              if (pos[u] == ~0ull) continue;
#pragma unroll
              for (int m = 0; m < 3; ++m) a.out_c[pos[u] * 3 + m] = cx[u][m];
              a.out_v[pos[u]] = v[u];
            }
          } else {
#pragma unroll
            for (int u = 0; u < kG; ++u) {
              if (pos[u] == ~0ull) continue;
              const uint32_t* sr = a.in_c + src[u] * R;
              uint32_t* o = a.out_c + pos[u] * R;
              for (uint32_t m = 0; m < R; ++m) o[m] = __ldg(sr + m);
              a.out_v[pos[u]] = v[u];
            }
          }
        }
      }
      __syncthreads();
      if (q == 0 && base == lo) small_mark(a, 54);
      if (t < kBins) s_cur[t] += cnt;
      // (the next tile's first barrier orders this before any s_cur read)
    }
    small_mark(a, 5 + 6 * q);
    if (q + 1 == a.P) break;  // the last pass wrote the output rows
    grid.sync();
    small_mark(a, 6 + 6 * q);
    if (q + 1 < a.P) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      issue_first(dst);
    }
    // (3) the next digit's counts over this CTA's chunk of the output
    if (q + 1 < a.P) {
      const uint32_t nlo = a.dlo[q + 1], nmask = a.dmask[q + 1];
      for (uint32_t b = t; b < kBins; b += kSmallThreads) s_h[b] = 0u;
      __syncthreads();
      for (uint64_t i = lo + t; i < hi; i += kSmallThreads)
        atomicAdd(&s_h[(uint32_t)(dst[i].x >> nlo) & nmask], 1u);
      __syncthreads();
      for (uint32_t b = t; b < kBins; b += kSmallThreads) a.hist[(size_t)b * G + cta] = s_h[b];
      small_mark(a, 7 + 6 * q);
      grid.sync();
      small_mark(a, 8 + 6 * q);
    }
  }
  small_mark(a, 63);
}

// ---------------------------------------------------------------------------
// k_local: small runs, fully sorted inside one CTA
// ---------------------------------------------------------------------------
struct LocalLayout {
  size_t c, v, key, perm0, perm1, rnk, whist, cnt, start, seg, tmp, total;
  __host__ __device__ LocalLayout(uint32_t cap, uint32_t rank, uint32_t TL) {
    size_t o = 0;
    c = o; o += align16((size_t(cap) * rank + 4) * 4);
    v = o; o += align16((size_t(cap) + 2) * 8);
    key = o; o += align16(size_t(cap) * 8);
    perm0 = o; o += align16(size_t(cap) * 2);
    perm1 = o; o += align16(size_t(cap) * 2);
    rnk = o; o += align16(size_t(cap) * 2);
    whist = o; o += align16(size_t(kLocalWarps) * kBins * 2);
    cnt = o; o += align16(kBins * 4);
    start = o; o += align16(kBins * 4);
    seg = o; o += align16((size_t(TL) + 2) * 8);
    tmp = o; o += align16(64 * 8);
    total = o;
  }
};

__device__ __forceinline__ uint32_t ceil_log2_dev(uint64_t x) {
  return x <= 1 ? 0u : 64u - (uint32_t)__clzll((long long)(x - 1));
}

__global__ void __launch_bounds__(kLocalThreads) k_local(LocalArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const LocalLayout L(a.cap, a.rank, a.TL);
  uint32_t* s_craw = reinterpret_cast<uint32_t*>(smem + L.c);
  double* s_vraw = reinterpret_cast<double*>(smem + L.v);
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(smem + L.key);
  uint16_t* s_p0 = reinterpret_cast<uint16_t*>(smem + L.perm0);
  uint16_t* s_p1 = reinterpret_cast<uint16_t*>(smem + L.perm1);
  uint16_t* s_rank = reinterpret_cast<uint16_t*>(smem + L.rnk);
  uint16_t* s_whist = reinterpret_cast<uint16_t*>(smem + L.whist);
  uint32_t* s_start = reinterpret_cast<uint32_t*>(smem + L.start);
  unsigned long long* s_seg = reinterpret_cast<unsigned long long*>(smem + L.seg);
  uint32_t* s_tmp = reinterpret_cast<uint32_t*>(smem + L.tmp);
  __shared__ unsigned long long s_sa;
  __shared__ uint32_t s_nsl;

  unsigned long long r0, r1;
  uint32_t nsl;
  if (a.seg_start == nullptr) {
    r0 = 0;
    r1 = a.nnz;
    nsl = 1;
    if (threadIdx.x == 0) {
      s_seg[0] = 0;
      s_seg[1] = a.nnz;
    }
  } else {
    const uint32_t chunk = a.chunk_list ? a.chunk_list[blockIdx.x] : blockIdx.x;
    const unsigned long long lo = (unsigned long long)chunk * a.TL;
    const unsigned long long hi = min((unsigned long long)a.nnz, lo + (unsigned long long)a.TL);
    const uint64_t S = a.nseg;  // seg_start has S+1 entries
    if (threadIdx.x == 0) {
      // first run starting at or after lo (precomputed per chunk; a binary
      // search here would be a chain of dependent global loads per CTA)
      uint64_t l;
      if (a.first_run) {
        l = a.first_run[chunk];
      } else {
        l = 0;
        uint64_t h = S;
        while (l < h) {
          const uint64_t m = (l + h) >> 1;
          if (a.seg_start[m] < lo) l = m + 1; else h = m;
        }
      }
      s_sa = l;
      s_nsl = 0xFFFFFFFFu;
    }
    __syncthreads();
    const uint64_t sa = s_sa;
    // runs sa .. sa+k starting in [lo, hi) and small; at most TL of them.
    // Read in batches that stop at the first batch holding the end: 64
    // entries first (chunks of a few hundred-row runs end there), then
    // kLocalThreads at a time (chunks of tiny runs)
    for (uint32_t base = 0, width = 64; base <= a.TL; base += width, width = kLocalThreads) {
      const uint32_t k = base + threadIdx.x;
      if (threadIdx.x < width && k <= a.TL) {
        const uint64_t s = sa + k;
        bool stop = true;
        if (s < S) {
          const unsigned long long b = a.seg_start[s], e = a.seg_start[s + 1];
          s_seg[k] = b;
          stop = b >= hi || (e - b) > a.TL;
          if (!stop) s_seg[k + 1] = e;
        }
        if (stop) atomicMin(&s_nsl, k);
      }
      __syncthreads();
      const bool done = s_nsl != 0xFFFFFFFFu;
      __syncthreads();  // every thread has read s_nsl before the next batch updates it
      if (done) break;
    }
    nsl = min(s_nsl, a.TL + 1);
    if (nsl == 0) return;
    r0 = s_seg[0];
    r1 = s_seg[nsl];
  }
  __syncthreads();
  const uint32_t n = (uint32_t)(r1 - r0);
  const uint32_t R = a.rank;
  load_words<kLocalThreads>(s_craw, a.in_c, r0 * R, n * R);
  load_doubles<kLocalThreads>(s_vraw, a.in_v, r0, n);
  __syncthreads();
  const uint32_t* s_c = s_craw + words_head(a.in_c, r0 * R);
  const double* s_v = s_vraw + doubles_head(a.in_v, r0);

  const uint32_t kb = a.key.total_bits;
  // the key's first (up to) four fields in registers, hoisted out of the row
  // loop (the general KeySpec walk reloads every field per row)
  constexpr int kF = 4;
  const bool few = a.key.n <= (uint32_t)kF;
  uint32_t fm[kF], fw[kF], fo[kF], fd[kF];
#pragma unroll
  for (int f = 0; f < kF; ++f) {
    const bool on = (uint32_t)f < a.key.n;
    fm[f] = on ? a.key.mode[f] : 0u;
    fw[f] = on ? a.key.width[f] : 0u;
    fo[f] = on ? a.key.off[f] : 0u;
    fd[f] = on ? a.key.dim[f] : 0xFFFFFFFFu;
  }
  // each thread walks its rows in order, so the run index only moves forward
  uint32_t run = 0;
  for (uint32_t i = threadIdx.x; i < n; i += kLocalThreads) {
    const uint32_t* row = s_c + (size_t)i * R;
    unsigned long long k = 0;
    if (few) {
      bool bad = false;
#pragma unroll
      for (int f = 0; f < kF; ++f) {
        if ((uint32_t)f < a.key.n) {
          const uint32_t x = row[fm[f]];
          bad |= x >= fd[f];
          if (fw[f]) k |= (unsigned long long)(x & (uint32_t)((1ull << fw[f]) - 1ull)) << fo[f];
        }
      }
      if (a.key.check && bad) check_row(row, a.key, r0 + i, a.err);
    } else {
      if (a.key.check) check_row(row, a.key, r0 + i, a.err);
      k = full_key(row, a.key);
    }
    if (nsl > 1) {
      // local run index: last run start <= row (this thread's rows only move
      // forward, so the search starts at the previous answer)
      const unsigned long long g = r0 + i;
      uint32_t h = nsl;
      while (h - run > 1) {
        const uint32_t m = (run + h) >> 1;
        if (s_seg[m] <= g) run = m; else h = m;
      }
      k |= (unsigned long long)run << kb;
    }
    s_key[i] = k;
    s_p0[i] = (uint16_t)i;
  }
  const uint32_t nbits = kb + ceil_log2_dev(nsl);
  const uint32_t passes = (nbits + kRadixLog - 1) / kRadixLog;
#if QD_FULL_ROUNDS
  const uint32_t ipw = (((n + kLocalWarps - 1) / kLocalWarps) + 31u) & ~31u;  // whole rounds
#else
  const uint32_t ipw = (n + kLocalWarps - 1) / kLocalWarps;
#endif
  uint16_t* cur = s_p0;
  uint16_t* nxt = s_p1;
  for (uint32_t q = 0; q < passes; ++q) {
    const uint32_t sh = q * kRadixLog;
    for (int k = threadIdx.x; k < kLocalWarps * kBins; k += kLocalThreads) s_whist[k] = 0;
    __syncthreads();
    // the local sort's digits are key bits in arbitrary order (high entropy):
    // ballot peers beat MATCH.ANY there (~25 vs ~61 SM cycles per warp round)
    warp_rank<QD_LOCAL_BALLOT>([&](uint32_t p) { return (uint32_t)((s_key[cur[p]] >> sh) & (kBins - 1)); },
                               n, ipw, s_rank, s_whist);
    __syncthreads();
    bin_offsets<kLocalThreads>(s_whist, s_tmp, s_start);
    __syncthreads();
    {
      const uint32_t w = threadIdx.x >> 5;
      const uint32_t hi = min(n, (w + 1) * ipw);
      const uint16_t* wh = s_whist + w * kBins;
      for (uint32_t p = w * ipw + (threadIdx.x & 31); p < hi; p += 32) {
        const uint32_t it = cur[p];
        const uint32_t d = (uint32_t)((s_key[it] >> sh) & (kBins - 1));
        nxt[s_start[d] + wh[d] + s_rank[p]] = (uint16_t)it;
      }
    }
    __syncthreads();
    uint16_t* t = cur;
    cur = nxt;
    nxt = t;
  }
  for (uint32_t j = threadIdx.x; j < n; j += kLocalThreads) {
    const uint32_t i = cur[j];
    store_row(a.out_c, a.out_v, R, r0 + j, s_c + (size_t)i * R, s_v[i]);
  }
}

// ---------------------------------------------------------------------------
// k_local2: the small runs of a bucketed group (Alg. 2 buckets of <= TL
// rows), streamed.  Persistent CTAs take items (one item = the small runs
// starting in one TL-row chunk, a contiguous span of < 2*TL rows) from a
// per-launch counter; the advancer warp loads the NEXT item's span into the
// other shared-memory buffer with TMA bulk copies (cp.async.bulk + mbarrier)
// while the CTA sorts the current one.  Inside an item every warp takes whole
// runs (a shared counter; no block barrier between runs) and sorts each one
// by the group's key: runs of <= 32 rows by an all-pairs rank of the full key
// in registers, longer runs by a warp-private LSD radix sort (<= 8-bit
// digits, MATCH.ANY ranking) over an index array; then the warp writes the
// run's rows to the output in sorted order (coalesced by output row).  Reads
// of a span complete (into shared memory) before any row of it is written, so
// in == out is safe.  sort.cpp:80-134 (Alg. 2) on small buckets.
// ---------------------------------------------------------------------------
constexpr int kLocal2Threads = 512;
constexpr int kLocal2Warps = kLocal2Threads / 32;
constexpr int kMaxLocalPasses = 8;

struct LocalItem {
  unsigned long long r0;  // first row of the span
  uint32_t n;             // rows in the span
  uint32_t run_first;     // index of its first run in seg_start
  uint32_t nruns;         // runs in the span (all small)
  uint32_t maxrun;        // longest of them (<= 32: k_local3 sorts every run within a warp)
};

struct Local2Args {
  const uint32_t* in_c;
  const double* in_v;
  uint32_t* out_c;
  double* out_v;
  uint32_t rank;
  uint32_t cap;  // rows per staging buffer (>= the longest span)
  const unsigned long long* seg_start;
  const LocalItem* items;
  uint32_t n_items;                        // (bound, when n_items_dev is set)
  const unsigned long long* n_items_dev;   // device item count (latency mode)
  uint32_t* item_counter;
  KeySpec key;
  uint32_t npasses;
  DigitSpec dig[kMaxLocalPasses];
  uint32_t dig_bits[kMaxLocalPasses];
  ErrBlock* err;
  uint32_t ballot_passes;  // k_local3: bit q = pass q ranks with ballots instead of MATCH.ANY
};

struct Local2Layout {
  size_t cbuf, vbuf, c0, v0, idx0, idx1, rnk, whist, total;
  __host__ __device__ Local2Layout(uint32_t cap, uint32_t rank) {
    size_t o = 0;
    cbuf = align16(size_t(cap) * rank * 4 + 32);
    vbuf = align16(size_t(cap) * 8 + 32);
    c0 = o; o += 2 * cbuf;
    v0 = o; o += 2 * vbuf;
    idx0 = o; o += align16(size_t(cap) * 2);
    idx1 = o; o += align16(size_t(cap) * 2);
    rnk = o; o += align16(size_t(cap) * 2);
    whist = o; o += align16(size_t(kLocal2Warps) * kBins * 2);
    total = o;
  }
};

// items: for each listed chunk c, its small runs [first_run[c], first run
// that starts at/after (c+1)*TL or is large) and their row span
__global__ void k_local_items(const uint32_t* list, const uint32_t* first_run,
                              const unsigned long long* seg_start, const unsigned long long* S_ptr,
                              uint64_t nnz, uint32_t TL, uint32_t n_items,
                              const unsigned long long* n_dev, const uint32_t* maxrun,
                              LocalItem* items) {
  const unsigned long long S = *S_ptr;
  if (n_dev) n_items = (uint32_t)min(*n_dev, (unsigned long long)n_items);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_items; i += gridDim.x * blockDim.x) {
    const uint32_t c = list[i];
    const unsigned long long hi = min((unsigned long long)nnz, ((unsigned long long)c + 1) * TL);
    const uint32_t f = first_run[c];
    // the runs starting in [c*TL, hi): binary search for the first run
    // starting at or after hi; a large run can only be the last of them
    // (it reaches past hi), and is left out
    unsigned long long l = f, h = S;
    while (l < h) {
      const unsigned long long m = (l + h) >> 1;
      if (seg_start[m] < hi) l = m + 1; else h = m;
    }
    uint32_t k = (uint32_t)l;
    if (k > f && seg_start[k] - seg_start[k - 1] > TL) --k;
    LocalItem it;
    it.r0 = seg_start[f];
    it.n = (uint32_t)(seg_start[k] - seg_start[f]);
    it.run_first = f;
    it.nruns = k - f;
    it.maxrun = maxrun ? maxrun[c] : TL;
    items[i] = it;
  }
}

// Adjacent items (one per TL-row window of run starts) whose spans touch —
// no large run between them — are merged while the span fits the staging
// capacity: kMergeGroup consecutive items per thread, greedily, the merged
// item written at its first slot and the absorbed ones emptied (n = 0; the
// sorter skips them).  Items average a few hundred rows otherwise (c5's
// (0,2,1): runs of ~66-900 rows), and k_local3's per-item cost (histogram
// clears, bin offsets, barriers per digit pass) dominated its time.
constexpr uint32_t kMergeGroup = 16;
__global__ void k_merge_items(LocalItem* items, uint32_t n_items, const unsigned long long* n_dev,
                              uint32_t cap) {
  if (n_dev) n_items = (uint32_t)min(*n_dev, (unsigned long long)n_items);
  const uint32_t ng = (n_items + kMergeGroup - 1) / kMergeGroup;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
    const uint32_t b = g * kMergeGroup, e = min(n_items, b + kMergeGroup);
    uint32_t head = b;
    LocalItem cur = items[b];
    for (uint32_t i = b + 1; i < e; ++i) {
      const LocalItem nx = items[i];
      if (cur.r0 + cur.n == nx.r0 && cur.run_first + cur.nruns == nx.run_first &&
          cur.n + nx.n <= cap) {
        cur.n += nx.n;
        cur.nruns += nx.nruns;
        cur.maxrun = max(cur.maxrun, nx.maxrun);
        items[i].n = 0u;
      } else {
        items[head] = cur;
        head = i;
        cur = nx;
      }
    }
    items[head] = cur;
  }
}

__global__ void __launch_bounds__(kLocal2Threads, 2) k_local2(Local2Args a) {
  const uint32_t NI = a.n_items_dev ? (uint32_t)min(*a.n_items_dev, (unsigned long long)a.n_items)
                                    : a.n_items;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t R = a.rank;
  const Local2Layout L(a.cap, R);
  uint16_t* s_idx0 = reinterpret_cast<uint16_t*>(smem + L.idx0);
  uint16_t* s_idx1 = reinterpret_cast<uint16_t*>(smem + L.idx1);
  uint16_t* s_rank = reinterpret_cast<uint16_t*>(smem + L.rnk);
  uint16_t* s_whist = reinterpret_cast<uint16_t*>(smem + L.whist);
  __shared__ unsigned long long s_bar[2];
  __shared__ uint32_t s_item[2];       // item index staged in buffer b
  __shared__ uint32_t s_ofs[2][2];     // staging heads (bytes) of coords / values
  __shared__ uint32_t s_next_run;      // next run of the current item (warps take runs)
  // key and digit specs in shared memory (dynamically indexed below; kernel
  // parameters indexed at run time would go through local memory)
  __shared__ KeySpec s_key;
  __shared__ DigitSpec s_dig[kMaxLocalPasses];
  __shared__ uint32_t s_dbits[kMaxLocalPasses];
  constexpr uint32_t kAdv = kLocal2Threads - 32;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;

  // advancer warp: draw the next item and start its bulk copies into buffer b
  auto advance = [&](uint32_t b) {
    uint32_t it = 0;
    LocalItem item{};
    for (;;) {  // merged-away items are empty: skip them
      if (lane == 0) it = atomicAdd(a.item_counter, 1u);
      it = __shfl_sync(0xFFFFFFFFu, it, 0);
      if (it >= NI) break;
      item = a.items[it];
      if (item.n) break;
    }
    if (lane == 0) s_item[b] = it;
    if (it >= NI) return;
    const Stage sc = make_stage(a.in_c + item.r0 * R, item.n * R * 4);
    const Stage sv = make_stage(a.in_v + item.r0, item.n * 8);
    if (lane == 0) {
      s_ofs[b][0] = sc.head;
      s_ofs[b][1] = sv.head;
      mbar_expect_tx(&s_bar[b], sc.bulk + sv.bulk);
    }
    __syncwarp();
    if (lane == 0 && sc.bulk) bulk_g2s(smem + L.c0 + b * L.cbuf, sc.gal, sc.bulk, &s_bar[b]);
    if (lane == 1 && sv.bulk) bulk_g2s(smem + L.v0 + b * L.vbuf, sv.gal, sv.bulk, &s_bar[b]);
  };

  if (threadIdx.x == kAdv) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    s_key = a.key;
    for (uint32_t q = 0; q < a.npasses; ++q) {
      s_dig[q] = a.dig[q];
      s_dbits[q] = a.dig_bits[q];
    }
  }
  __syncthreads();
  if (threadIdx.x >= kAdv) advance(0);
  __syncthreads();
  const KeySpec& key = s_key;
  const uint32_t nk = key.n;
  uint32_t phases = 0;
  for (uint32_t iter = 0;; ++iter) {
    const uint32_t b = iter & 1u;
    const uint32_t it = s_item[b];
    if (it >= NI) break;
    if (threadIdx.x == 0) s_next_run = 0;
    // the other buffer was released by the previous item's closing barrier
    if (threadIdx.x >= kAdv) advance(b ^ 1u);
    mbar_wait(&s_bar[b], (phases >> b) & 1u);
    phases ^= 1u << b;
    __syncthreads();  // s_next_run reset visible; s_item[b^1] written
    const LocalItem item = a.items[it];
    const uint32_t* s_c =
        reinterpret_cast<const uint32_t*>(smem + L.c0 + b * L.cbuf + s_ofs[b][0]);
    const double* s_v = reinterpret_cast<const double*>(smem + L.v0 + b * L.vbuf + s_ofs[b][1]);
    auto coord = [&](uint32_t i, uint32_t m) { return s_c[i * R + m]; };
    auto full_key_at = [&](uint32_t i) -> unsigned long long {
      unsigned long long k = 0;
      for (uint32_t f = 0; f < nk; ++f) {
        const uint32_t wd = key.width[f];
        if (wd) k |= (unsigned long long)(coord(i, key.mode[f]) & (uint32_t)((1ull << wd) - 1ull))
                     << key.off[f];
      }
      return k;
    };
    auto check_at = [&](uint32_t i) {
      if (!key.check) return;
      bool bad = false;
      for (uint32_t f = 0; f < nk; ++f) bad |= coord(i, key.mode[f]) >= key.dim[f];
      if (bad) check_row(s_c + (size_t)i * R, key, item.r0 + i, a.err);
    };
    auto store = [&](uint32_t j, uint32_t i) {  // output row j of the span <- staged row i
      const unsigned long long dst = item.r0 + j;
      uint32_t* o = a.out_c + dst * R;
      for (uint32_t m = 0; m < R; ++m) __stcs(o + m, s_c[i * R + m]);
      __stcs(a.out_v + dst, s_v[i]);
    };
    for (;;) {
      uint32_t run = 0;
      if (lane == 0) run = atomicAdd(&s_next_run, 1u);
      run = __shfl_sync(0xFFFFFFFFu, run, 0);
      if (run >= item.nruns) break;
      const uint32_t rb = (uint32_t)(a.seg_start[item.run_first + run] - item.r0);
      const uint32_t re = (uint32_t)(a.seg_start[item.run_first + run + 1] - item.r0);
      const uint32_t n = re - rb;
      if (n <= 32) {
        // all-pairs stable rank of the full key: position = #smaller keys
        // + #equal keys earlier in the run
        const bool valid = lane < n;
        const uint32_t i = rb + (valid ? lane : 0u);
        if (valid) check_at(i);
        const unsigned long long k = valid ? full_key_at(i) : ~0ull;
        uint32_t pos = 0;
        for (uint32_t j = 0; j < n; ++j) {
          const unsigned long long kj = __shfl_sync(0xFFFFFFFFu, k, j);
          pos += (kj < k) || (kj == k && j < lane);
        }
        if (valid) store(rb + pos, i);
        continue;
      }
      // warp-private LSD radix sort of positions [rb, re) by the key digits
      uint16_t* wh = s_whist + w * kBins;
      uint16_t* cur = s_idx0;
      uint16_t* nxt = s_idx1;
      for (uint32_t p = rb + lane; p < re; p += 32) {
        check_at(p);
        cur[p] = (uint16_t)p;
      }
      const unsigned below = (1u << lane) - 1u;
      for (uint32_t q = 0; q < a.npasses; ++q) {
        const uint32_t nb = 1u << s_dbits[q];
        for (uint32_t k = lane; k < nb; k += 32) wh[k] = 0;
        __syncwarp();
        const DigitSpec& dg = s_dig[q];
        for (uint32_t base = rb; base < re; base += 32) {  // ranking rounds
          const uint32_t p = base + lane;
          const bool valid = p < re;
          const uint32_t d = valid ? digit_by([&](uint32_t m) { return coord(cur[p], m); }, dg) : nb;
          const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
          uint32_t c = 0;
          if (valid) c = wh[d];
          __syncwarp();
          if (valid && (peers & below) == 0u) wh[d] = (uint16_t)(c + __popc(peers));
          if (valid) s_rank[p] = (uint16_t)(c + __popc(peers & below));
          __syncwarp();
        }
        // exclusive scan of the warp's bin counts (lane owns nb/32 bins)
        {
          const uint32_t per = (nb + 31) / 32;
          uint32_t loc[8];
          uint32_t sum = 0;
#pragma unroll
          for (uint32_t t = 0; t < 8; ++t) {
            const uint32_t k = lane * per + t;
            loc[t] = (t < per && k < nb) ? wh[k] : 0u;
            sum += loc[t];
          }
          uint32_t incl = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
          }
          uint32_t run_sum = incl - sum;
          __syncwarp();
#pragma unroll
          for (uint32_t t = 0; t < 8; ++t) {
            const uint32_t k = lane * per + t;
            if (t < per && k < nb) {
              wh[k] = (uint16_t)run_sum;
              run_sum += loc[t];
            }
          }
          __syncwarp();
        }
        for (uint32_t p = rb + lane; p < re; p += 32) {  // scatter of the indices
          const uint32_t i = cur[p];
          const uint32_t d = digit_by([&](uint32_t m) { return coord(i, m); }, dg);
          nxt[rb + wh[d] + s_rank[p]] = (uint16_t)i;
        }
        __syncwarp();
        uint16_t* t = cur;
        cur = nxt;
        nxt = t;
      }
      for (uint32_t j = rb + lane; j < re; j += 32) store(j, cur[j]);
      __syncwarp();
    }
    __syncthreads();  // buffer b and the index arrays are free again
  }
}

// ---------------------------------------------------------------------------
// k_local3: the small runs of a bucketed group, streamed through shared
// memory with one block-wide LSD radix sort per item.  Persistent CTAs take
// items (the small runs starting in one TL-row chunk: a contiguous span of
// < 2*TL rows) from a per-launch counter; the advancer warp loads the NEXT
// item's span (TMA bulk copies + mbarrier) and its run starts into the other
// buffer while the CTA sorts the current one.  Every row gets the composite
// key (local run index, group key) — rows are already grouped by run, so the
// run index keeps the runs apart through the LSD passes — and the item is
// sorted by <= 8-bit digits of it (MATCH.ANY ranking per warp stripe, ranks
// in registers, (key, row) pairs ping-ponged in shared memory), then written
// out in sorted order.  A span is read completely (into shared memory)
// before any row of it is written, so in == out is safe.  sort.cpp:80-134
// (Alg. 2) on small buckets.
// ---------------------------------------------------------------------------
// k_local3 digits: up to 9 bits, so composite keys of up to 27 bits (21-bit
// key + 64 runs) take 3 passes instead of 4
constexpr int kLocalBitsMax = 9;
constexpr int kLocalBins = 1 << kLocalBitsMax;

struct Local3Layout {
  size_t cbuf, vbuf, c0, v0, k0, k1, i0, i1, seg, whist, start, wsum, total;
  __host__ __device__ Local3Layout(uint32_t cap, uint32_t rank, uint32_t key_bytes,
                                   uint32_t warps = kLocal2Warps) {
    size_t o = 0;
    cbuf = align16(size_t(cap) * rank * 4 + 32);
    vbuf = align16(size_t(cap) * 8 + 32);
    c0 = o; o += 2 * cbuf;
    v0 = o; o += 2 * vbuf;
    k0 = o; o += align16(size_t(cap) * key_bytes);
    k1 = o; o += align16(size_t(cap) * key_bytes);
    i0 = o; o += align16(size_t(cap) * 2);
    i1 = o; o += align16(size_t(cap) * 2);
    seg = o; o += 2 * align16(size_t(cap + 2) * 2);
    whist = o; o += align16(size_t(warps) * kLocalBins * 2);
    start = o; o += align16(kLocalBins * 4);
    wsum = o; o += align16(64 * 4);
    total = o;
  }
};

template <class K, int NT, int RT = 0>
__global__ void __launch_bounds__(NT, 1024 / NT) k_local3(Local2Args a) {
  const uint32_t NI = a.n_items_dev ? (uint32_t)min(*a.n_items_dev, (unsigned long long)a.n_items)
                                    : a.n_items;
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int NW = NT / 32;
  const uint32_t R = RT ? (uint32_t)RT : a.rank;
  const Local3Layout L(a.cap, R, sizeof(K), NW);
  K* s_k0 = reinterpret_cast<K*>(smem + L.k0);
  K* s_k1 = reinterpret_cast<K*>(smem + L.k1);
  uint16_t* s_i0 = reinterpret_cast<uint16_t*>(smem + L.i0);
  uint16_t* s_i1 = reinterpret_cast<uint16_t*>(smem + L.i1);
  uint16_t* s_whist = reinterpret_cast<uint16_t*>(smem + L.whist);
  uint32_t* s_start = reinterpret_cast<uint32_t*>(smem + L.start);
  uint32_t* s_wsum = reinterpret_cast<uint32_t*>(smem + L.wsum);
  const size_t seg_stride = align16(size_t(a.cap + 2) * 2);
  __shared__ unsigned long long s_bar[2];
  __shared__ uint32_t s_item[2];
  __shared__ LocalItem s_desc[2];  // descriptor of the item staged in buffer b
  __shared__ uint32_t s_ofs[2][2];
  __shared__ KeySpec s_key;
  __shared__ uint32_t s_next_run;  // warp path: next run of the item
  constexpr uint32_t kAdv = NT - 32;
  constexpr uint32_t kR = 8;  // ranking rounds per warp stripe (cap <= 16 * 32 * kR)
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;

  // advancer warp: draw the next item, start its bulk copies into buffer b
  // and copy its run starts (local u16 offsets) into the buffer's seg array
  auto advance = [&](uint32_t b) {
    uint32_t it = 0;
    LocalItem item{};
    for (;;) {  // merged-away items are empty: skip them
      if (lane == 0) it = atomicAdd(a.item_counter, 1u);
      it = __shfl_sync(0xFFFFFFFFu, it, 0);
      if (it >= NI) break;
      item = a.items[it];
      if (item.n) break;
    }
    if (lane == 0) s_item[b] = it;
    if (it >= NI) return;
    const Stage sc = make_stage(a.in_c + item.r0 * R, item.n * R * 4);
    const Stage sv = make_stage(a.in_v + item.r0, item.n * 8);
    if (lane == 0) {
      s_desc[b] = item;
      s_ofs[b][0] = sc.head;
      s_ofs[b][1] = sv.head;
      mbar_expect_tx(&s_bar[b], sc.bulk + sv.bulk);
    }
    __syncwarp();
    if (lane == 0 && sc.bulk) bulk_g2s(smem + L.c0 + b * L.cbuf, sc.gal, sc.bulk, &s_bar[b]);
    if (lane == 1 && sv.bulk) bulk_g2s(smem + L.v0 + b * L.vbuf, sv.gal, sv.bulk, &s_bar[b]);
    uint16_t* sg = reinterpret_cast<uint16_t*>(smem + L.seg + b * seg_stride);
    for (uint32_t k = lane; k <= item.nruns; k += 32)
      sg[k] = (uint16_t)(a.seg_start[item.run_first + k] - item.r0);
  };

  if (threadIdx.x == kAdv) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    s_key = a.key;
    s_next_run = 0;
  }
  __syncthreads();
  if (threadIdx.x >= kAdv) advance(0);
  __syncthreads();
  const KeySpec& key = s_key;
  const uint32_t nk = key.n;
  const uint32_t kb = key.total_bits;
  // the key's first (up to) four fields in registers (the general KeySpec
  // walk reloads every field from shared memory per row)
  constexpr int kF = 4;
  const bool few = nk <= (uint32_t)kF;
  uint32_t fm[kF], fmask[kF], fo[kF], fd[kF];
#pragma unroll
  for (int f = 0; f < kF; ++f) {
    const bool on = (uint32_t)f < nk;
    fm[f] = on ? key.mode[f] : 0u;
    fmask[f] = on ? (uint32_t)((1ull << key.width[f]) - 1ull) : 0u;
    fo[f] = on ? key.off[f] : 0u;
    fd[f] = on ? key.dim[f] : 0xFFFFFFFFu;
  }
  const bool check = key.check;
  const unsigned below = (1u << lane) - 1u;
  uint32_t phases = 0;
  for (uint32_t iter = 0;; ++iter) {
    const uint32_t b = iter & 1u;
    const uint32_t it = s_item[b];
    if (it >= NI) break;
    // buffer b^1 was released by the previous item's closing barrier
    if (threadIdx.x >= kAdv) advance(b ^ 1u);
    mbar_wait(&s_bar[b], (phases >> b) & 1u);
    phases ^= 1u << b;
    const LocalItem item = s_desc[b];
    const uint32_t n = item.n, nsl = item.nruns;
    const uint32_t* s_c =
        reinterpret_cast<const uint32_t*>(smem + L.c0 + b * L.cbuf + s_ofs[b][0]);
    const double* s_v = reinterpret_cast<const double*>(smem + L.v0 + b * L.vbuf + s_ofs[b][1]);
    const uint16_t* sg = reinterpret_cast<const uint16_t*>(smem + L.seg + b * seg_stride);
    // (the advancer's seg writes for buffer b happened before the barrier
    // that closed the previous item)
    if (item.maxrun <= 32) {
      // every run is at most 32 rows: row-parallel.  Keys go to shared
      // memory; then each row finds its run (binary search over the run
      // starts) and its place in it = #rows of the run with a smaller key +
      // #equal keys before it (stable), and is written there directly.
      unsigned long long* s_kk = reinterpret_cast<unsigned long long*>(
          smem + L.k0);  // k0 and k1 together hold cap u64 keys
      for (uint32_t p = threadIdx.x; p < n; p += NT) {
        const uint32_t* row = s_c + (size_t)p * R;
        unsigned long long k = 0;
        bool bad = false;
        if (few) {
#pragma unroll
          for (int f = 0; f < kF; ++f) {
            if ((uint32_t)f < nk) {
              const uint32_t x = row[fm[f]];
              bad |= x >= fd[f];
              k |= (unsigned long long)(x & fmask[f]) << fo[f];
            }
          }
        } else {
          for (uint32_t f = 0; f < nk; ++f) {
            const uint32_t x = row[key.mode[f]];
            bad |= x >= key.dim[f];
            const uint32_t wd = key.width[f];
            if (wd) k |= (unsigned long long)(x & (uint32_t)((1ull << wd) - 1ull)) << key.off[f];
          }
        }
        if (check && bad) check_row(row, key, item.r0 + p, a.err);
        s_kk[p] = k;
      }
      __syncthreads();
      for (uint32_t p = threadIdx.x; p < n; p += NT) {
        uint32_t l = 0, h = nsl;  // run of p: last start <= p
        while (h - l > 1) {
          const uint32_t m = (l + h) >> 1;
          if (sg[m] <= p) l = m; else h = m;
        }
        const uint32_t rb = sg[l], re = sg[l + 1];
        const unsigned long long k = s_kk[p];
        uint32_t pos = rb;
        for (uint32_t j = rb; j < re; ++j) {
          const unsigned long long kj = s_kk[j];
          pos += (kj < k) || (kj == k && j < p);
        }
        const unsigned long long dst = item.r0 + pos;
        const uint32_t* row = s_c + (size_t)p * R;
        uint32_t* o = a.out_c + dst * R;
        for (uint32_t q = 0; q < R; ++q) __stcs(o + q, row[q]);
        __stcs(a.out_v + dst, s_v[p]);
      }
      __syncthreads();  // buffer b and the key scratch are free again
      continue;
    }
    const uint32_t rbits = nsl > 1 ? 32u - __clz(nsl - 1) : 0u;
    const uint32_t tb = kb + rbits;
    const uint32_t P = (tb + kLocalBitsMax - 1) / kLocalBitsMax;
    const uint32_t per = P ? (tb + P - 1) / P : 0u;
    // warp stripes of whole 32-row rounds
    const uint32_t ipw = (((n + NW - 1) / NW) + 31u) & ~31u;
    const uint32_t lo = w * ipw, hi = min(n, lo + ipw);
    // composite keys: (local run index << kb) | key; range check of the key
    {
      uint32_t run = 0;
      for (uint32_t p = lo + lane; p < hi; p += 32) {
        if (nsl > 1) {
          if (p == lo + lane) {  // first row of this lane: binary search
            uint32_t l = 0, h = nsl;
            while (h - l > 1) {
              const uint32_t m = (l + h) >> 1;
              if (sg[m] <= p) l = m; else h = m;
            }
            run = l;
          }
          while (run + 1 < nsl && sg[run + 1] <= p) ++run;
        }
        const uint32_t* row = s_c + (size_t)p * R;
        K k = 0;
        bool bad = false;
        if (few) {
#pragma unroll
          for (int f = 0; f < kF; ++f) {
            if ((uint32_t)f < nk) {
              const uint32_t x = row[fm[f]];
              bad |= x >= fd[f];
              k |= (K)(x & fmask[f]) << fo[f];
            }
          }
        } else {
          for (uint32_t f = 0; f < nk; ++f) {
            const uint32_t x = row[key.mode[f]];
            bad |= x >= key.dim[f];
            const uint32_t wd = key.width[f];
            if (wd) k |= (K)(x & (uint32_t)((1ull << wd) - 1ull)) << key.off[f];
          }
        }
        if (check && bad) check_row(row, key, item.r0 + p, a.err);
        if (rbits) k |= (K)run << kb;
        s_k0[p] = k;
        s_i0[p] = (uint16_t)p;
      }
    }
    K* kc = s_k0;
    K* kn = s_k1;
    uint16_t* ic = s_i0;
    uint16_t* in_ = s_i1;
    uint16_t* wh = s_whist + w * kLocalBins;
    __syncwarp();
    for (uint32_t q = 0; q < P; ++q) {
      const uint32_t sh = q * per;
      const uint32_t dbits = min(per, tb - sh);
      const uint32_t mask = (1u << dbits) - 1u;
      const uint32_t nb = 1u << dbits;  // bins of this digit (<= kLocalBins)
      if (lo < n) {  // warps past the item's rows keep no counts
        // 16-byte clears (8 bins each); whist rows are 16-byte aligned
        uint4* wz = reinterpret_cast<uint4*>(wh);
        for (uint32_t k = lane; k < (nb + 7) / 8; k += 32) wz[k] = make_uint4(0u, 0u, 0u, 0u);
      }
      __syncwarp();
      uint32_t packed[kR];
#pragma unroll
      for (uint32_t r = 0; r < kR; ++r) {
        const uint32_t p = lo + r * 32 + lane;
        if (lo + r * 32 >= hi) break;  // warp-uniform
        const bool valid = p < hi;
        const uint32_t d = valid ? (uint32_t)(kc[p] >> sh) & mask : 0xFFFFFFFFu;
        unsigned peers;
        if ((a.ballot_passes >> q) & 1u) {  // warp-uniform
          const unsigned vm = __ballot_sync(0xFFFFFFFFu, valid);
          peers = ballot_peers_n<kLocalBitsMax>(d, vm, dbits);
        } else {
          peers = __match_any_sync(0xFFFFFFFFu, d);
        }
        const uint32_t c = valid ? wh[d] : 0u;
        __syncwarp();
        if (valid && (peers & below) == 0u) wh[d] = (uint16_t)(c + __popc(peers));
        __syncwarp();
        packed[r] = ((c + __popc(peers & below)) << kLocalBitsMax) | (d & (kLocalBins - 1u));
      }
      __syncthreads();
      // bin pairs (2t, 2t+1): warp-exclusive offsets with 16-bit SIMD adds,
      // then the bins' starts by a scan over the pair totals
      {
        const uint32_t npair = (nb + 1) / 2;
        uint32_t lo_cnt = 0, hi_cnt = 0, pair_excl = 0;
        if (threadIdx.x < npair) {
          uint32_t* wp = reinterpret_cast<uint32_t*>(s_whist) + threadIdx.x;
          uint32_t run2 = 0;
          const uint32_t nwa = (n + ipw - 1) / ipw;  // warps holding rows
#pragma unroll
          for (int x = 0; x < NW; ++x) {
            if ((uint32_t)x >= nwa) break;
            const uint32_t c = wp[x * (kLocalBins / 2)];
            wp[x * (kLocalBins / 2)] = run2;
            run2 = __vadd2(run2, c);
          }
          lo_cnt = run2 & 0xFFFFu;
          hi_cnt = run2 >> 16;
        }
        const uint32_t tot = lo_cnt + hi_cnt;
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= (uint32_t)o) incl += y;
        }
        if (threadIdx.x < npair && lane == 31) s_wsum[w] = incl;
        if (npair > 32) __syncthreads();
        if (threadIdx.x < npair) {
          uint32_t base = 0;
          for (uint32_t x = 0; x < w; ++x) base += s_wsum[x];
          pair_excl = base + incl - tot;
          s_start[2 * threadIdx.x] = pair_excl;
          s_start[2 * threadIdx.x + 1] = pair_excl + lo_cnt;
        }
      }
      __syncthreads();
#pragma unroll
      for (uint32_t r = 0; r < kR; ++r) {
        const uint32_t p = lo + r * 32 + lane;
        if (lo + r * 32 >= hi) break;
        if (p < hi) {
          const uint32_t d = packed[r] & (kLocalBins - 1u);
          const uint32_t slot = s_start[d] + wh[d] + (packed[r] >> kLocalBitsMax);
          kn[slot] = kc[p];
          in_[slot] = ic[p];
        }
      }
      __syncthreads();
      K* tk = kc; kc = kn; kn = tk;
      uint16_t* ti = ic; ic = in_; in_ = ti;
    }
    if (P == 0) __syncthreads();
    if (RT) {
      // the item's output rows are contiguous: coordinate WORDS one per
      // thread (coalesced 128-byte warp stores), word w = row w / RT, mode
      // w % RT of the sorted order
      uint32_t* oc = a.out_c + item.r0 * RT;
      for (uint32_t wd = threadIdx.x; wd < n * RT; wd += NT) {
        const uint32_t j = wd / RT, m = wd - j * RT;
        __stcs(oc + wd, s_c[(uint32_t)ic[j] * RT + m]);
      }
      for (uint32_t j = threadIdx.x; j < n; j += NT) __stcs(a.out_v + item.r0 + j, s_v[ic[j]]);
    } else {
      for (uint32_t j = threadIdx.x; j < n; j += NT) {
        const uint32_t i = ic[j];
        const unsigned long long dst = item.r0 + j;
        uint32_t* o = a.out_c + dst * R;
        for (uint32_t m = 0; m < R; ++m) __stcs(o + m, s_c[i * R + m]);
        __stcs(a.out_v + dst, s_v[i]);
      }
    }
    __syncthreads();  // buffer b, its seg array and the scratch are free again
  }
}

// ---------------------------------------------------------------------------
// segment discovery
// ---------------------------------------------------------------------------
#ifndef QD_HEAD_ROWS
#define QD_HEAD_ROWS 4096
#endif
constexpr uint32_t kHeadRows = QD_HEAD_ROWS;  // rows per k_heads CTA (words = rows / 32 <= kThreads)
static_assert(kHeadRows / 32 <= (uint32_t)kThreads && (kHeadRows / kThreads) % 8 == 0, "k_heads/k_compact block shape");

struct ModeList {
  uint32_t n;
  uint8_t m[kMaxKeys];
};

// head bit of row i = 1 iff i == 0 or row i differs from row i-1 on `modes`.
// Optional second job of k_heads for a bucketed group's first digit pass: the
// rows stream through this kernel anyway (the prefix column's sectors hold the
// whole AoS row), so it also range-checks the key coordinates (count_keys,
// sort.cpp:54-64), checks that the row packs, and leaves the first digit of
// every row as a byte — the first k_chunk_hist then reads 1 byte per row
// instead of the coordinates again (c5 (0,2,1): 20.9 GB less to read).
struct HeadsExtra {
  uint8_t* digits;  // nullptr: run discovery only
  int quad;         // k_heads_quad (rank 3/4, one prefix mode, aligned rows, <= 2 digit fields)
  uint32_t lim[4];  // k_heads_quad: per mode, min(key dimension if range-checked, pack limit)
  ErrBlock* err;
  int do_check, check_pack;
  uint32_t pack_lim[kMaxKeys];
  DigitSpec dig;
  KeySpec key;
};

__device__ __forceinline__ void heads_extra_row(const HeadsExtra& x, const Dig2& dg, bool fast,
                                                const uint32_t* c, uint32_t rank,
                                                unsigned long long i) {
  const uint32_t* row = c + i * rank;
  if (x.do_check) {
    bool bad = false;
#pragma unroll 1
    for (uint32_t k = 0; k < x.key.n; ++k) bad |= __ldg(row + x.key.mode[k]) >= x.key.dim[k];
    if (bad) check_row(row, x.key, i, x.err);
  }
  if (x.check_pack) {
    uint32_t bad = 0;
#pragma unroll 1
    for (uint32_t m = 0; m < rank; ++m) bad |= __ldg(row + m) >= x.pack_lim[m];
    if (bad) atomicOr(&x.err->flags, 4u);
  }
  auto get = [&](uint32_t m) { return __ldg(row + m); };
  x.digits[i] = (uint8_t)(fast ? digit2(get, dg) : digit_by(get, x.dig));
}

__global__ void __launch_bounds__(kThreads) k_heads(const uint32_t* c, uint32_t rank,
                                                    uint64_t nnz, ModeList modes,
                                                    uint32_t* words, uint32_t* block_cnt,
                                                    HeadsExtra ex) {
  const unsigned long long r0 = (unsigned long long)blockIdx.x * kHeadRows;
  uint32_t cnt = 0;
  const bool ex_fast = ex.dig.lookup == nullptr && ex.dig.n <= 2;
  const Dig2 ex_dg = dig2_of(ex.dig);
  if (modes.n == 1) {
    // one prefix mode: each row's coordinate is loaded once (all rounds'
    // loads in flight together); the previous row's comes from lane - 1
    constexpr int kQ = 8;
    const uint32_t m = modes.m[0];
    const int lane = threadIdx.x & 31;
#pragma unroll 1
    for (uint32_t k0 = 0; k0 < kHeadRows / kThreads; k0 += kQ) {
      uint32_t x[kQ], y0[kQ];
#pragma unroll
      for (int k = 0; k < kQ; ++k) {
        const unsigned long long i = r0 + (k0 + k) * kThreads + threadIdx.x;
        x[k] = i < nnz ? __ldcs(c + i * rank + m) : 0u;
        y0[k] = (lane == 0 && i > 0 && i < nnz) ? __ldg(c + (i - 1) * rank + m) : 0u;
      }
#pragma unroll
      for (int k = 0; k < kQ; ++k) {
        const unsigned long long i = r0 + (k0 + k) * kThreads + threadIdx.x;
        const uint32_t up = __shfl_up_sync(0xFFFFFFFFu, x[k], 1);
        const uint32_t y = lane == 0 ? y0[k] : up;
        const bool head = i < nnz && (i == 0 || x[k] != y);
        const unsigned bits = __ballot_sync(0xFFFFFFFFu, head);
        if (lane == 0 && i < nnz) words[i >> 5] = bits;
        cnt += head;
        if (ex.digits && i < nnz) heads_extra_row(ex, ex_dg, ex_fast, c, rank, i);
      }
    }
  } else
  for (uint32_t k = 0; k < kHeadRows / kThreads; ++k) {
    const unsigned long long i = r0 + k * kThreads + threadIdx.x;
    bool head = false;
    if (i < nnz) {
      if (i == 0) {
        head = true;
      } else {
        const uint32_t* x = c + i * rank;
        const uint32_t* y = x - rank;
        for (uint32_t j = 0; j < modes.n; ++j)
          if (x[modes.m[j]] != y[modes.m[j]]) { head = true; break; }
      }
    }
    const unsigned bits = __ballot_sync(0xFFFFFFFFu, head);
    if ((threadIdx.x & 31) == 0 && r0 + k * kThreads + threadIdx.x < nnz)
      words[(r0 + k * kThreads + threadIdx.x) >> 5] = bits;
    cnt += head;
    if (ex.digits && i < nnz) heads_extra_row(ex, ex_dg, ex_fast, c, rank, i);
  }
  __shared__ uint32_t s_tmp[64];
  uint32_t tot;
  block_excl_scan(cnt, s_tmp, &tot);
  if (threadIdx.x == 0) block_cnt[blockIdx.x] = tot;
}

// k_heads + HeadsExtra for rank-3 / rank-4 AoS rows with ONE prefix mode, four
// consecutive rows per thread from 16-byte loads (rank 3: three loads hold four
// rows; rank 4: one load per row): head flags, range/pack checks and the first
// digit all come from the registers, the four digit bytes leave as one word and
// the head bits of a 32-row word are assembled from eight lanes' nibbles.
// `c` must be 16-byte aligned.
template <int RT>
struct QuadRows {
  uint32_t w[4][RT];
};
template <int RT>
__device__ __forceinline__ QuadRows<RT> load_quad(const uint32_t* __restrict__ c, uint64_t nnz,
                                                  unsigned long long i0) {
  QuadRows<RT> r;
  if (i0 + 3 < nnz) {
    if constexpr (RT == 3) {
      const uint4* q = reinterpret_cast<const uint4*>(c + i0 * 3);
      const uint4 a = __ldcs(q), b = __ldcs(q + 1), d = __ldcs(q + 2);
      r.w[0][0] = a.x; r.w[0][1] = a.y; r.w[0][2] = a.z;
      r.w[1][0] = a.w; r.w[1][1] = b.x; r.w[1][2] = b.y;
      r.w[2][0] = b.z; r.w[2][1] = b.w; r.w[2][2] = d.x;
      r.w[3][0] = d.y; r.w[3][1] = d.z; r.w[3][2] = d.w;
    } else {
      const uint4* q = reinterpret_cast<const uint4*>(c + i0 * 4);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint4 a = __ldcs(q + k);
        r.w[k][0] = a.x; r.w[k][1] = a.y; r.w[k][2] = a.z; r.w[k][3] = a.w;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int m = 0; m < RT; ++m) r.w[k][m] = i0 + k < nnz ? __ldg(c + (i0 + k) * RT + m) : 0u;
  }
  return r;
}

template <int RT>
__global__ void __launch_bounds__(kThreads) k_heads_quad(const uint32_t* __restrict__ c, uint64_t nnz,
                                                         uint32_t pm, uint32_t* words,
                                                         uint32_t* block_cnt, HeadsExtra ex) {
  static_assert(RT == 3 || RT == 4, "rank 3 or 4");
  const unsigned long long r0 = (unsigned long long)blockIdx.x * kHeadRows;
  const int lane = threadIdx.x & 31;
  const Dig2 dg = dig2_of(ex.dig);
  // (per-mode limits folded on the host: building them here from the key
  // spec cost ~600 instructions per thread, 37 per row at 16 rows per thread)
  uint32_t lim[RT];
#pragma unroll
  for (int m = 0; m < RT; ++m) lim[m] = ex.lim[m];
#define QD_SEL(k, m) \
  ((m) == 0u ? row.w[k][0] : ((m) == 1u ? row.w[k][1] : ((RT == 3 || (m) == 2u) ? row.w[k][2] : row.w[k][RT - 1])))
  uint32_t cnt = 0;
  auto process = [&](const QuadRows<RT> row, const unsigned long long i0) {
    const bool full = i0 + 3 < nnz;
    uint32_t pv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) pv[k] = QD_SEL(k, pm);
    uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, pv[3], 1);
    if (lane == 0) prev = (i0 > 0 && i0 < nnz) ? __ldg(c + (i0 - 1) * RT + pm) : 0u;
    uint32_t nib = 0, dword = 0;
    const bool first = i0 == 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const unsigned long long i = i0 + k;
      const bool valid = full || i < nnz;  // (one test per quad on the common path)
      const bool head = valid && ((k == 0 && first) || pv[k] != (k ? pv[k - 1] : prev));
      nib |= (uint32_t)head << k;
      cnt += head;
      if (valid) {
        bool over = false;
#pragma unroll
        for (int m = 0; m < RT; ++m) over |= row.w[k][m] >= lim[m];
        if (over) {  // rare: the exact checks (range: first (row, mode); pack: flag)
          if (ex.do_check) check_row(c + i * RT, ex.key, i, ex.err);
          if (ex.check_pack) {
            bool bad = false;
#pragma unroll
            for (int m = 0; m < RT; ++m) bad |= row.w[k][m] >= ex.pack_lim[m];
            if (bad) atomicOr(&ex.err->flags, 4u);
          }
        }
        uint32_t d = ((QD_SEL(k, dg.m0) >> dg.r0) & dg.k0) << dg.l0;
        if (dg.two) d |= ((QD_SEL(k, dg.m1) >> dg.r1) & dg.k1) << dg.l1;
        dword |= (d & 0xFFu) << (8 * k);
      }
    }
    // the 32-row head word = the nibbles of eight consecutive lanes
    uint32_t x = nib << (4 * (lane & 7));
    x |= __shfl_xor_sync(0xFFFFFFFFu, x, 1);
    x |= __shfl_xor_sync(0xFFFFFFFFu, x, 2);
    x |= __shfl_xor_sync(0xFFFFFFFFu, x, 4);
    if ((lane & 7) == 0 && i0 < nnz) words[i0 >> 5] = x;
    if (full) {
      *reinterpret_cast<uint32_t*>(ex.digits + i0) = dword;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (i0 + k < nnz) ex.digits[i0 + k] = (uint8_t)(dword >> (8 * k));
    }
  };
  // one quad at a time (two in flight: 63 registers, 0.99 -> 1.15 ms per 400 M rows)
#pragma unroll 1
  for (uint32_t it = 0; it < kHeadRows / (4 * kThreads); ++it) {
    const unsigned long long ia = r0 + 4ull * (it * kThreads + threadIdx.x);
    process(load_quad<RT>(c, nnz, ia), ia);
  }
#undef QD_SEL
  __shared__ uint32_t s_tmp[64];
  uint32_t tot;
  block_excl_scan(cnt, s_tmp, &tot);
  if (threadIdx.x == 0) block_cnt[blockIdx.x] = tot;
}

// Write seg_start[off + rank] = row for every head; the last CTA also writes
// seg_start[S] = nnz.
__global__ void __launch_bounds__(kThreads) k_compact(const uint32_t* words, uint64_t nnz,
                                                      const unsigned long long* block_off,
                                                      uint32_t nblocks,
                                                      unsigned long long* seg_start,
                                                      const unsigned long long* total) {
  const unsigned long long w0 = (unsigned long long)blockIdx.x * (kHeadRows / 32);
  const unsigned long long nwords = (nnz + 31) / 32;
  // a block without heads (most blocks inside long runs) has nothing to write
  const bool last = blockIdx.x == nblocks - 1;
  if (!last && block_off[blockIdx.x + 1] == block_off[blockIdx.x]) return;
  __shared__ uint32_t s_tmp[64];
  // kHeadRows/32 = 128 words per CTA; threads 0..127 own one word each
  const unsigned long long wi = w0 + threadIdx.x;
  uint32_t word = 0;
  if (threadIdx.x < kHeadRows / 32 && wi < nwords) word = words[wi];
  const uint32_t pre = block_excl_scan(__popc(word), s_tmp);
  unsigned long long out = block_off[blockIdx.x] + pre;
  while (word) {
    const int b = __ffs(word) - 1;
    word &= word - 1;
    seg_start[out++] = wi * 32 + b;
  }
  if (blockIdx.x == nblocks - 1 && threadIdx.x == 0) seg_start[*total] = nnz;
}

// Per run: large flag and its chunk count (CH rows per chunk).
__global__ void k_classify_chunks(const unsigned long long* seg_start,
                                  const unsigned long long* S_ptr, uint32_t TL, uint32_t CH,
                                  uint32_t* is_large, uint32_t* nchunks, uint32_t* local_flag,
                                  uint32_t* first_run, uint32_t* local_maxrun) {
  const unsigned long long S = *S_ptr;
  for (unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; s < S;
       s += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long len = seg_start[s + 1] - seg_start[s];
    const bool large = len > TL;
    is_large[s] = large;
    nchunks[s] = large ? (uint32_t)((len + CH - 1) / CH) : 0u;
    if (TL) {
      const unsigned long long cl = seg_start[s] / TL;
      if (!large) local_flag[cl] = 1u;  // a local chunk has work
      // the first run starting in a chunk records itself (one writer per
      // chunk; a flagged chunk always starts with a small run)
      if (s == 0 || seg_start[s - 1] / TL != cl) first_run[cl] = (uint32_t)s;
    }
    if (TL && local_maxrun) {
      // longest small run per local chunk; consecutive runs share a chunk,
      // so lanes of one chunk reduce first and one of them updates it
      const unsigned long long cl = seg_start[s] / TL;
      const uint32_t v = large ? 0u : (uint32_t)len;
      const unsigned act = __activemask();
      const unsigned peers = __match_any_sync(act, cl);
      const uint32_t mx = __reduce_max_sync(peers, v);
      if ((peers & ((1u << (threadIdx.x & 31)) - 1u)) == 0u && mx) atomicMax(local_maxrun + cl, mx);
    }
  }
}

// list[pos[c]] = c for every flagged c
__global__ void k_compact_flags(const uint32_t* flag, const unsigned long long* pos, uint64_t n,
                                uint32_t* list) {
  for (unsigned long long c = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; c < n;
       c += (unsigned long long)gridDim.x * blockDim.x)
    if (flag[c]) list[pos[c]] = (uint32_t)c;
}

__global__ void k_gen_chunks(const unsigned long long* seg_start, const unsigned long long* S_ptr,
                             uint32_t CH, const uint32_t* is_large,
                             const unsigned long long* large_off,
                             const unsigned long long* chunk_off, ChunkDesc* chunks,
                             unsigned long long* run_start) {
  const unsigned long long S = *S_ptr;
  for (unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; s < S;
       s += (unsigned long long)gridDim.x * blockDim.x) {
    if (!is_large[s]) continue;
    const unsigned long long b = seg_start[s], e = seg_start[s + 1];
    const uint32_t li = (uint32_t)large_off[s];
    run_start[li] = b;
    const unsigned long long c0 = chunk_off[s];
    const uint32_t nc = (uint32_t)((e - b + CH - 1) / CH);
    for (uint32_t k = 0; k < nc; ++k) {
      ChunkDesc d;
      d.row_begin = b + (unsigned long long)k * CH;
      d.len = (uint32_t)min((unsigned long long)CH, e - d.row_begin);
      d.li = li;
      d.cidx = k;
      d.nchunks = nc;
      d.coff = c0;
      chunks[c0 + k] = d;
    }
  }
}

// One run [0, nnz) cut into chunks of CH rows.
__global__ void k_uniform_chunks(uint64_t nnz, uint32_t CH, uint32_t nc, ChunkDesc* chunks) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nc; k += gridDim.x * blockDim.x) {
    ChunkDesc d;
    d.row_begin = (unsigned long long)k * CH;
    d.len = (uint32_t)min((unsigned long long)CH, nnz - d.row_begin);
    d.li = 0;
    d.cidx = k;
    d.nchunks = nc;
    d.coff = 0;
    chunks[k] = d;
  }
}

// out[i] = in[i * stride] for i < n (reads a column of the scanned offsets)
__global__ void k_gather_stride(const unsigned long long* in, uint64_t stride, uint32_t n,
                                unsigned long long* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = in[i * stride];
}

// ---------------------------------------------------------------------------
// generic exclusive scan (u32 in -> u64 out), 3 phases
// ---------------------------------------------------------------------------
constexpr uint32_t kScanItems = 8;
constexpr uint32_t kScanTile = kThreads * kScanItems;

__global__ void k_scan_reduce(const uint32_t* in, unsigned long long n, unsigned long long* part,
                              const unsigned long long* n_dev, uint32_t n_mul) {
  if (n_dev) n = min(n, *n_dev * n_mul);
  const unsigned long long b = (unsigned long long)blockIdx.x * kScanTile;
  unsigned long long s = 0;
  for (uint32_t k = 0; k < kScanItems; ++k) {
    const unsigned long long i = b + k * kThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  __shared__ unsigned long long s_tmp[64];
  const unsigned long long ex = block_excl_scan64(s, s_tmp);
  if (threadIdx.x == kThreads - 1) part[blockIdx.x] = ex + s;
}

// single CTA: exclusive scan of part[0..np) in place, total to *total
__global__ void k_scan_parts(unsigned long long* part, uint32_t np, unsigned long long* total) {
  __shared__ unsigned long long s_tmp[64];
  unsigned long long carry = 0;
  for (uint32_t b = 0; b < np; b += kThreads) {
    const uint32_t i = b + threadIdx.x;
    const unsigned long long v = i < np ? part[i] : 0;
    const unsigned long long ex = block_excl_scan64(v, s_tmp);
    if (i < np) part[i] = carry + ex;
    __shared__ unsigned long long s_last;
    if (threadIdx.x == kThreads - 1) s_last = ex + v;
    __syncthreads();
    carry += s_last;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void k_scan_down(const uint32_t* in, unsigned long long n, const unsigned long long* part,
                            unsigned long long* out, const unsigned long long* n_dev,
                            uint32_t n_mul) {
  if (n_dev) n = min(n, *n_dev * n_mul);
  const unsigned long long b = (unsigned long long)blockIdx.x * kScanTile;
  // each thread owns kScanItems consecutive elements
  unsigned long long v[kScanItems];
  unsigned long long s = 0;
  for (uint32_t k = 0; k < kScanItems; ++k) {
    const unsigned long long i = b + threadIdx.x * kScanItems + k;
    v[k] = i < n ? in[i] : 0;
    s += v[k];
  }
  __shared__ unsigned long long s_tmp[64];
  unsigned long long run = part[blockIdx.x] + block_excl_scan64(s, s_tmp);
  for (uint32_t k = 0; k < kScanItems; ++k) {
    const unsigned long long i = b + threadIdx.x * kScanItems + k;
    if (i < n) out[i] = run;
    run += v[k];
  }
}

// Single-pass exclusive scan with decoupled look-back (one launch instead of
// reduce / parts / down).  Tiles are taken in ticket order (a monotone
// counter, so a tile only ever waits on tiles that are already running);
// each tile publishes its aggregate, then its inclusive prefix, in a status
// word {tag:24 | flag:2 | value:38} whose tag is the tile's global ticket, so
// the status array never needs clearing between calls.
constexpr unsigned long long kLbValBits = 38, kLbValMask = (1ull << kLbValBits) - 1;
__global__ void __launch_bounds__(kThreads) k_scan_lookback(
    const uint32_t* in, unsigned long long n, unsigned long long* out, unsigned long long* total,
    unsigned long long* status, uint32_t nstat, unsigned long long* ticket,
    unsigned long long ticket_base, const unsigned long long* n_dev, uint32_t n_mul) {
  if (n_dev) n = min(n, *n_dev * n_mul);  // latency mode: the count is on the device
  __shared__ unsigned long long s_tile, s_prefix;
  __shared__ unsigned long long s_tmp[64];
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1ull) - ticket_base;
  __syncthreads();
  const unsigned long long t = s_tile;
  const unsigned long long tag = (ticket_base + t) & 0xFFFFFFull;
  const unsigned long long b = t * kScanTile;
  unsigned long long v[kScanItems];
  unsigned long long sum = 0;
#pragma unroll
  for (uint32_t k = 0; k < kScanItems; ++k) {
    const unsigned long long i = b + threadIdx.x * kScanItems + k;
    v[k] = i < n ? __ldcs(in + i) : 0ull;
    sum += v[k];
  }
  unsigned long long agg;
  {
    // block scan (inclusive total via the last thread)
    const unsigned long long ex = block_excl_scan64<kThreads>(sum, s_tmp);
    if (threadIdx.x == kThreads - 1) s_prefix = ex + sum;  // tile aggregate
    __syncthreads();
    agg = s_prefix;
    __syncthreads();
    sum = ex;  // this thread's exclusive offset inside the tile
  }
  volatile unsigned long long* st = status;
  if (threadIdx.x < 32) {
    const unsigned long long kA = 1ull << kLbValBits, kP = 2ull << kLbValBits;
    if (t == 0) {
      if (threadIdx.x == 0) {
        st[0] = (tag << 40) | kP | (agg & kLbValMask);
        s_prefix = 0;
      }
    } else {
      if (threadIdx.x == 0) st[t] = (tag << 40) | kA | (agg & kLbValMask);
      // lane l inspects tile base - l; stop at the nearest inclusive prefix
      unsigned long long prefix = 0;
      long long base = (long long)t - 1;
      while (true) {
        const long long j = base - (long long)threadIdx.x;
        unsigned long long w = 0, f = 2;  // before tile 0: inclusive prefix 0
        if (j >= 0) {
          const unsigned long long want = (ticket_base + (unsigned long long)j) & 0xFFFFFFull;
          do {
            w = st[j];
            f = (w >> 40) == want ? ((w >> kLbValBits) & 3ull) : 0ull;
          } while (f == 0);
        }
        const unsigned full = __ballot_sync(0xFFFFFFFFu, f == 2);
        const unsigned stop = full ? (unsigned)(__ffs(full) - 1) : 31u;
        unsigned long long val = (j >= 0 && threadIdx.x <= stop) ? (w & kLbValMask) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xFFFFFFFFu, val, o);
        prefix += val;
        if (full) break;
        base -= 32;
      }
      if (threadIdx.x == 0) {
        st[t] = (tag << 40) | kP | ((prefix + agg) & kLbValMask);
        s_prefix = prefix;
      }
    }
  }
  __syncthreads();
  unsigned long long run = s_prefix + sum;
  if (b + kScanTile >= n && b < n + kScanTile && threadIdx.x == kThreads - 1)
    *total = s_prefix + agg;
#pragma unroll
  for (uint32_t k = 0; k < kScanItems; ++k) {
    const unsigned long long i = b + threadIdx.x * kScanItems + k;
    if (i < n) out[i] = run;
    run += v[k];
  }
}

// ---------------------------------------------------------------------------
// small utility kernels
// ---------------------------------------------------------------------------
__global__ void k_copy_check(const uint32_t* in_c, const double* in_v, uint32_t* out_c,
                             double* out_v, uint32_t rank, uint64_t nnz, KeySpec key,
                             ErrBlock* err) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t* row = in_c + i * rank;
    if (key.check) check_row(row, key, i, err);
    for (uint32_t m = 0; m < rank; ++m) out_c[i * rank + m] = row[m];
    out_v[i] = in_v[i];
  }
}

// flags bit1 unless rows are non-decreasing under `order` (coo.cpp:32-49)
__global__ void k_is_sorted(const uint32_t* c, uint32_t rank, uint64_t nnz, ModeList order,
                            ErrBlock* err) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x + 1;
       i < nnz; i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t* x = c + i * rank;
    const uint32_t* y = x - rank;
    for (uint32_t j = 0; j < order.n; ++j) {
      const uint32_t a = y[order.m[j]], b = x[order.m[j]];
      if (a != b) {
        if (a > b) atomicOr(&err->flags, 2u);
        break;
      }
    }
  }
}

__global__ void k_mode_max(const uint32_t* c, uint32_t rank, uint64_t nnz, ModeList modes,
                           uint32_t* mx) {
  __shared__ uint32_t s_mx[kMaxKeys];
  for (uint32_t j = threadIdx.x; j < modes.n; j += blockDim.x) s_mx[j] = 0;
  __syncthreads();
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (unsigned long long)gridDim.x * blockDim.x)
    for (uint32_t j = 0; j < modes.n; ++j) atomicMax(&s_mx[j], c[i * rank + modes.m[j]]);
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < modes.n; j += blockDim.x) atomicMax(&mx[j], s_mx[j]);
}

// Warp-aggregated: lanes holding the same value add once (MATCH.ANY), so a
// Zipf head value (~9 % of config 5's rows) does not serialise on one address.
__global__ void k_mode_hist(const uint32_t* c, uint32_t rank, uint64_t nnz, uint32_t mode,
                            uint32_t dim, unsigned long long* hist) {
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i0 = (unsigned long long)blockIdx.x * blockDim.x; i0 < nnz; i0 += stride) {
    const unsigned long long i = i0 + threadIdx.x;  // warp-uniform loop bound
    const uint32_t k = i < nnz ? c[i * rank + mode] : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, k);
    if (k < dim && (peers & ((1u << (threadIdx.x & 31)) - 1u)) == 0u)
      atomicAdd(hist + k, (unsigned long long)__popc(peers));
  }
}

// ---------------------------------------------------------------------------
// run-level sort: when the rows to sort by key k come in long runs of equal
// (prefix, key) — the input's existing order (e.g. (i0,i1) fibers when sorting
// by i1) — a stable sort moves each run as a block.  Runs become records
// {key, start << 32 | len}, the records are sorted with the same engine, and
// k_move_runs2 copies every run to its place.
// ---------------------------------------------------------------------------
// Run-length probe for the run-sort decision: heads of mode-`mode` runs in
// 256 evenly spaced blocks of 1024 consecutive rows.
constexpr uint32_t kProbeBlocks = 256, kProbeRows = 1024;
__global__ void __launch_bounds__(kThreads) k_probe_runs(const uint32_t* c, uint32_t rank,
                                                         uint64_t nnz, uint32_t mode,
                                                         unsigned long long* heads) {
  const unsigned long long span = nnz / kProbeBlocks;
  const unsigned long long b0 = blockIdx.x * span;
  uint32_t h = 0;
  for (uint32_t i = 1 + threadIdx.x; i < kProbeRows; i += kThreads) {
    const unsigned long long r = b0 + i;
    if (r < nnz && c[r * rank + mode] != c[(r - 1) * rank + mode]) ++h;
  }
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xFFFFFFFFu, h, o);
  if ((threadIdx.x & 31) == 0 && h) atomicAdd(heads, (unsigned long long)h);
}

// implicit prefix coordinates of every large run (PackSpec::n_imp)
__global__ void k_run_prefix(const uint32_t* c, uint32_t rank, const unsigned long long* run_start,
                             uint64_t nruns, const unsigned long long* n_dev, ModeList modes,
                             uint32_t* out) {
  if (n_dev) nruns = min((unsigned long long)nruns, *n_dev);
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nruns;
       r += (uint64_t)gridDim.x * blockDim.x)
    for (uint32_t k = 0; k < modes.n; ++k) out[r * modes.n + k] = c[run_start[r] * rank + modes.m[k]];
}

__global__ void k_run_records(const uint32_t* c, uint32_t rank, uint32_t mode, uint32_t dim,
                              const unsigned long long* seg, uint64_t S, uint32_t* rkey,
                              double* rval, ErrBlock* err) {
  for (unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; s < S;
       s += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long b = seg[s], e = seg[s + 1];
    const uint32_t key = c[b * rank + mode];
    if (key >= dim) {  // every row of the run has this key (count_keys check)
      atomicOr(&err->flags, 1u);
      atomicMin(&err->rowmode, (b << 6) | mode);
    }
    rkey[s] = key;
    rval[s] = __longlong_as_double((long long)((b << 32) | (e - b)));
  }
}

// CSF levels: crd[f] = coordinate `mode` of fiber f's first row
__global__ void k_fiber_crd(const uint32_t* c, uint32_t rank, uint32_t mode,
                            const unsigned long long* starts, uint64_t nf, uint32_t* crd) {
  for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < nf;
       f += (uint64_t)gridDim.x * blockDim.x)
    crd[f] = c[starts[f] * rank + mode];
}
// pos[j] = index of parent fiber j's first row among the child fiber starts
// (parents' starts are a subset of the children's, both sorted), j <= np
__global__ void k_fiber_pos(const unsigned long long* child, uint64_t nc,
                            const unsigned long long* parent, uint64_t np, uint64_t nnz,
                            unsigned long long* pos) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j <= np;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long x = j < np ? parent[j] : nnz;
    uint64_t l = 0, h = nc;  // first child start >= x
    while (l < h) {
      const uint64_t m = (l + h) >> 1;
      if (child[m] < x) l = m + 1; else h = m;
    }
    pos[j] = l;
  }
}

__global__ void k_run_lens(const double* rval, uint64_t S, uint32_t* lens) {
  for (unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; s < S;
       s += (unsigned long long)gridDim.x * blockDim.x)
    lens[s] = (uint32_t)((unsigned long long)__double_as_longlong(rval[s]) & 0xFFFFFFFFull);
}

// Run move v2: output tiles of kMoveTile rows; thread t resolves the source
// row of the tile's rows [8t, 8t+8) (one binary search, then a forward walk
// over the sorted run starts), then the tile's coordinate WORDS and values are
// copied word-per-thread, so every warp access is 128 contiguous bytes on
// the write side and contiguous within each run on the read side.
constexpr uint32_t kMoveTile = 2048;
constexpr int kMoveThreads = 256;
constexpr int kMoveRowsPerThread = kMoveTile / kMoveThreads;

// first run of every output tile (upper_bound(dsto, tile * kMoveTile) - 1)
__global__ void k_tile_first_run(const unsigned long long* dsto, uint64_t S, uint64_t ntiles,
                                 uint32_t* first) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t <= ntiles;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long p = t * kMoveTile;
    uint64_t l = 0, h = S;  // first run with dsto > p
    while (l < h) {
      const uint64_t m = (l + h) >> 1;
      if (dsto[m] <= p) l = m + 1; else h = m;
    }
    first[t] = (uint32_t)(l ? l - 1 : 0);
  }
}

template <int RT>
__global__ void __launch_bounds__(kMoveThreads) k_move_runs2(
    const uint32_t* __restrict__ in_c, const double* __restrict__ in_v, uint32_t* __restrict__ out_c,
    double* __restrict__ out_v, uint32_t rank, uint64_t N, const double* rval,
    const unsigned long long* dsto, uint64_t S, const uint32_t* first) {
  __shared__ unsigned long long s_rdst[kMoveTile + 2];
  __shared__ uint32_t s_rsrc[kMoveTile + 2];
  __shared__ uint32_t s_rowsrc[kMoveTile];
  const uint32_t R = RT ? RT : rank;
  const unsigned long long p0 = (unsigned long long)blockIdx.x * kMoveTile;
  const uint32_t n = (uint32_t)min((unsigned long long)kMoveTile, N - p0);
  const uint32_t j0 = first[blockIdx.x];
  const uint32_t nr = min((uint32_t)(first[blockIdx.x + 1] - j0 + 1), (uint32_t)(S - j0));
  for (uint32_t k = threadIdx.x; k < nr; k += kMoveThreads) {
    s_rdst[k] = dsto[j0 + k];
    s_rsrc[k] = (uint32_t)((unsigned long long)__double_as_longlong(rval[j0 + k]) >> 32);
  }
  __syncthreads();
  {
    const uint32_t i0 = threadIdx.x * kMoveRowsPerThread;
    if (i0 < n) {
      const unsigned long long row0 = p0 + i0;
      uint32_t l = 0, h = nr;  // last run start <= row0
      while (h - l > 1) {
        const uint32_t m = (l + h) >> 1;
        if (s_rdst[m] <= row0) l = m; else h = m;
      }
#pragma unroll
      for (int q = 0; q < kMoveRowsPerThread; ++q) {
        const unsigned long long row = row0 + q;
        while (l + 1 < nr && s_rdst[l + 1] <= row) ++l;
        if (i0 + q < n) s_rowsrc[i0 + q] = s_rsrc[l] + (uint32_t)(row - s_rdst[l]);
      }
    }
  }
  __syncthreads();
  constexpr int kB = 8;
  if (RT == 4) {
    // rank 4: a row's coordinates are one aligned 16-byte vector
    const uint4* ic4 = reinterpret_cast<const uint4*>(in_c);
    uint4* oc4 = reinterpret_cast<uint4*>(out_c) + p0;
    for (uint32_t ib = threadIdx.x; ib < n; ib += kB * kMoveThreads) {
      uint4 x[kB];
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const uint32_t i = ib + q * kMoveThreads;
        if (i < n) x[q] = __ldg(ic4 + s_rowsrc[i]);
      }
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const uint32_t i = ib + q * kMoveThreads;
        if (i < n) __stcs(oc4 + i, x[q]);
      }
    }
  }
  // coordinates: the tile's words, several per thread in flight
  const uint32_t nw = RT == 4 ? 0u : n * R;
  const unsigned long long w0 = p0 * R;
  for (uint32_t wb = threadIdx.x; wb < nw; wb += kB * kMoveThreads) {
    uint32_t x[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const uint32_t w = wb + q * kMoveThreads;
      if (w < nw) {
        const uint32_t i = w / R, m = w - i * R;
        x[q] = __ldg(in_c + (unsigned long long)s_rowsrc[i] * R + m);
      }
    }
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const uint32_t w = wb + q * kMoveThreads;
      if (w < nw) __stcs(out_c + w0 + w, x[q]);
    }
  }
  // values
  for (uint32_t ib = threadIdx.x; ib < n; ib += kB * kMoveThreads) {
    double v[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const uint32_t i = ib + q * kMoveThreads;
      if (i < n) v[q] = __ldg(in_v + s_rowsrc[i]);
    }
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const uint32_t i = ib + q * kMoveThreads;
      if (i < n) __stcs(out_v + p0 + i, v[q]);
    }
  }
}


// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {
void preload_kernels();  // (defined after the kernels it names)
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Workspace {
  int device = 0;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
  std::map<std::string, DevBuf> bufs;
  uint64_t launches = 0;
  ErrBlock* h_err = nullptr;  // pinned
  ErrBlock* h_err_init = nullptr;  // pinned, the reset value (flags 0, rowmode ~0)
  uint64_t* h_small = nullptr;  // pinned scratch for small D2H reads
  bool allow_pack = true;  // packed intermediates (cleared for a lossy-pack redo)
  bool allow_small = true;  // k_small for latency-mode single-group calls (cleared for a redo)
  // asynchronous host-buffer transposes (qd_transpose_inplace_async): the
  // caller's thread enqueues each call's host->device copy (s_in) into one of
  // two device slots and hands the device work to a worker thread, which runs
  // it on s_comp and enqueues the device->host copy (s_out).  Input copies of
  // consecutive calls run back to back, overlapping the previous calls'
  // device work and output copies (PCIe is full duplex).
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
  cudaStream_t s_host = nullptr;  // synchronous host-buffer calls (capturable, unlike stream 0)
  // sliced host-buffer calls (run_groups_host): the input and output copy
  // streams of the slice pipeline, and one "slice arrived" event per slice
  cudaStream_t s_sl_in = nullptr, s_sl_out = nullptr;
  std::vector<cudaEvent_t> ev_slices;
  bool allow_latency = true;  // cleared while a sliced call runs its slices (no per-slice graphs)
  uint64_t last_slices = 1;
  bool sliced_warm = false;  // a sliced call has completed (its kernels are loaded)
  static constexpr int kSlots = QD_ASYNC_SLOTS;  // device in/out buffer pairs in flight
  cudaEvent_t ev_in[kSlots] = {}, ev_comp[kSlots] = {}, ev_out[kSlots] = {};
  struct SlotBuf {
    uint32_t* ic = nullptr;
    double* iv = nullptr;
    uint32_t* oc = nullptr;
    double* ov = nullptr;
    size_t rows = 0, rank = 0;
  } slots[kSlots];
  bool slot_busy[kSlots] = {};  // job queued / running, output copy not yet issued
  int slot = 0;
  struct HostSpan {
    const void* c = nullptr;
    size_t nc = 0;
    const void* v = nullptr;
    size_t nv = 0;
  };
  // every async call whose device->host copy may still be pending: the host
  // bytes it writes back, and an event recorded after that copy (by the
  // worker, once it has issued it: issued_seq >= seq)
  struct Pending {
    HostSpan span;
    cudaEvent_t done = nullptr;
    uint64_t seq = 0;
  };
  std::deque<Pending> pending;
  std::vector<cudaEvent_t> done_pool;  // recycled Pending::done events (under mu)
  uint64_t next_seq = 0, issued_seq = 0;
  struct AsyncJob {
    std::vector<uint32_t> dims;
    uint64_t nnz = 0;
    uint32_t* coords = nullptr;
    double* values = nullptr;
    std::vector<Group> groups;
    bool verify_input = false;
    int slot = 0;
    cudaEvent_t done = nullptr;  // recorded after the output copy
    uint64_t seq = 0;
  };
  std::thread worker;
  std::mutex mu;
  std::condition_variable cv;
  std::deque<AsyncJob> jobs;
  int running = 0;  // jobs popped and not yet finished by the worker
  bool stop = false;
  bool async_failed = false;  // first error of a device job, reported at synchronize
  qd_status async_code = QD_OK;
  std::string async_msg;
  uint64_t async_row = 0;
  uint32_t async_mode = 0;
  // single-pass scan (k_scan_lookback): tile status words and the ticket
  // counter; lb_base = tickets issued so far (the device counter's value)
  unsigned long long* lb_status = nullptr;
  unsigned long long* lb_ticket = nullptr;
  size_t lb_cap = 0;
  unsigned long long lb_base = 0, lb_cleared_epoch = ~0ull;
  // CUDA graphs of latency-mode calls, keyed by the call's shape and buffers;
  // a reallocated workspace buffer (buf_epoch) invalidates them all
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    uint64_t launches = 0;
    uint64_t epoch = 0;
    int seen = 0;
  };
  std::map<std::string, GraphEntry> graphs;
  uint64_t buf_epoch = 0;
  // live per-kernel-class timing (CUDA events on the launch stream)
  bool prof = false;
  struct ProfStat {
    uint64_t launches = 0;
    double ms = 0, bytes = 0;
  } prof_stats[5];
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t event() {
    if (ev_pool.empty()) {
      cudaEvent_t e;
      QD_CUDA(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }

  template <class T>
  T* get(const std::string& name, size_t count) {
    const size_t bytes = std::max<size_t>(count * sizeof(T), 256);
    DevBuf& b = bufs[name];
    if (b.bytes < bytes) {
      ++buf_epoch;
      if (b.p) QD_CUDA(cudaFree(b.p));
      b.p = nullptr;
      b.bytes = 0;
      const size_t want = bytes + bytes / 8;  // headroom against regrowth
      QD_CUDA(cudaMalloc(&b.p, want));
      b.bytes = want;
      static const int poison = [] {
        const char* e = getenv("QD_POISON");
        return e ? atoi(e) : 0;
      }();
      static const char* only = getenv("QD_POISON_ONLY");
      static const char* except = getenv("QD_POISON_EXCEPT");
      if (poison && (!only || name.find(only) != std::string::npos) &&
          (!except || name.find(except) == std::string::npos))
        QD_CUDA(cudaMemset(b.p, poison & 0xFF, want));  // debug: expose reads of unwritten scratch
    }
    return static_cast<T*>(b.p);
  }
};

using ScatterFn = void (*)(ScatterArgs);
// (in, out) format pairs used: AoS->AoS, AoS->SoA, SoA->SoA, SoA->AoS (any
// group), AoS->PK, PK->PK, PK->AoS (packed groups)
template <int RT, int DM>
ScatterFn scatter_kernel_fmt(int in, int out, int mx) {
  if (in == kAoS && out == kAoS) return k_scatter<RT, kAoS, kAoS, DM>;
  if (in == kAoS && out == kSoA) return k_scatter<RT, kAoS, kSoA, DM>;
  if (in == kSoA && out == kSoA) return k_scatter<RT, kSoA, kSoA, DM>;
  if (in == kSoA && out == kAoS) return k_scatter<RT, kSoA, kAoS, DM>;
  if (in == kAoS && out == kPK)
    return mx ? k_scatter<RT, kAoS, kPK, DM, 1> : k_scatter<RT, kAoS, kPK, DM>;
  return nullptr;
}
template <int RT>
ScatterFn scatter_kernel_rt(int dm, int in, int out, int mx) {
  if (in == kPK) {
    if (out == kPK) return k_scatter<RT, kPK, kPK, 0>;
    return mx ? k_scatter<RT, kPK, kAoS, 0, 1> : k_scatter<RT, kPK, kAoS, 0>;
  }
  switch (dm) {
    case 1: return scatter_kernel_fmt<RT, 1>(in, out, mx);
    case 2: return scatter_kernel_fmt<RT, 2>(in, out, mx);
    default: return scatter_kernel_fmt<RT, 0>(in, out, mx);
  }
}
// rt: compile-time rank (3, 4 or 0 = runtime); dm: digit mode; in/out
// formats; mx: mixed-radix packed rows (PackSpec::mixed)
ScatterFn scatter_kernel(int rt, int dm, int in, int out, int mx = 0) {
  switch (rt) {
    case 3: return scatter_kernel_rt<3>(dm, in, out, mx);
    case 4: return scatter_kernel_rt<4>(dm, in, out, mx);
    default: return scatter_kernel_rt<0>(dm, in, out, mx);
  }
}

Workspace* workspace_create(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw Error(QD_NO_DEVICE, "no CUDA device visible (this library has no CPU path)");
  if (device < 0 || device >= n) invalid("device index out of range");
  QD_CUDA(cudaSetDevice(device));
  auto* ws = new Workspace;
  ws->device = device;
  QD_CUDA(cudaDeviceGetAttribute(&ws->num_sms, cudaDevAttrMultiProcessorCount, device));
  int optin = 0;
  QD_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  ws->smem_optin = optin;
  preload_kernels();
  QD_CUDA(cudaMallocHost(&ws->h_err, sizeof(ErrBlock)));
  QD_CUDA(cudaMallocHost(&ws->h_err_init, sizeof(ErrBlock)));
  std::memset(ws->h_err_init, 0, sizeof(ErrBlock));
  ws->h_err_init->rowmode = ~0ull;
  QD_CUDA(cudaMallocHost(&ws->h_small, 512 * sizeof(uint64_t)));
  auto allow_smem = [&](const void* fn) {
    cudaFuncAttributes fa{};
    QD_CUDA(cudaFuncGetAttributes(&fa, fn));
    QD_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 optin - (int)fa.sharedSizeBytes));
  };
  for (int rt : {0, 3, 4})
    for (int dm = 0; dm < 3; ++dm)
      for (int in = 0; in < 3; ++in)
        for (int out = 0; out < 3; ++out)
          for (int mx = 0; mx < 2; ++mx)
            if (ScatterFn f = scatter_kernel(rt, dm, in, out, mx))
              allow_smem(reinterpret_cast<const void*>(f));
  allow_smem(reinterpret_cast<const void*>(k_local));
  allow_smem(reinterpret_cast<const void*>(k_local2));
  allow_smem(reinterpret_cast<const void*>(k_local3<uint32_t, 512>));
  allow_smem(reinterpret_cast<const void*>(k_local3<unsigned long long, 512>));
  allow_smem(reinterpret_cast<const void*>(k_small));
  allow_smem(reinterpret_cast<const void*>(k_local3<uint32_t, 512, 3>));
  allow_smem(reinterpret_cast<const void*>(k_local3<unsigned long long, 512, 3>));
  allow_smem(reinterpret_cast<const void*>(k_local3<uint32_t, 512, 4>));
  allow_smem(reinterpret_cast<const void*>(k_local3<unsigned long long, 512, 4>));
  allow_smem(reinterpret_cast<const void*>(k_local3<uint32_t, 256>));
  allow_smem(reinterpret_cast<const void*>(k_local3<unsigned long long, 256>));
  ws->smem_optin = optin - 1024;  // dynamic budget below the static usage
  return ws;
}

void workspace_destroy(Workspace* ws) {
  if (!ws) return;
  if (ws->worker.joinable()) {
    {
      std::lock_guard<std::mutex> lk(ws->mu);
      ws->stop = true;
    }
    ws->cv.notify_all();
    ws->worker.join();
  }
  cudaSetDevice(ws->device);
  for (auto& sb : ws->slots)
    for (void* p : {(void*)sb.ic, (void*)sb.iv, (void*)sb.oc, (void*)sb.ov})
      if (p) cudaFree(p);
  for (cudaEvent_t e : ws->ev_slices) cudaEventDestroy(e);
  for (cudaStream_t st : {ws->s_in, ws->s_comp, ws->s_out, ws->s_host, ws->s_sl_in, ws->s_sl_out})
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  for (int i = 0; i < Workspace::kSlots; ++i)
    for (cudaEvent_t e : {ws->ev_in[i], ws->ev_comp[i], ws->ev_out[i]})
      if (e) cudaEventDestroy(e);
  for (auto& kv : ws->bufs)
    if (kv.second.p) cudaFree(kv.second.p);
  if (ws->h_err) cudaFreeHost(ws->h_err);
  if (ws->h_err_init) cudaFreeHost(ws->h_err_init);
  if (ws->h_small) cudaFreeHost(ws->h_small);
  for (auto e : ws->ev_pool) cudaEventDestroy(e);
  for (auto& g : ws->graphs)
    if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
  for (auto e : ws->done_pool) cudaEventDestroy(e);
  for (auto& p : ws->pending) cudaEventDestroy(p.done);
  delete ws;
}

uint64_t workspace_bytes(const Workspace* ws) {
  uint64_t b = 0;
  for (auto& kv : ws->bufs) b += kv.second.bytes;
  return b;
}
uint64_t workspace_launches(const Workspace* ws) { return ws->launches; }
uint64_t workspace_slices(const Workspace* ws) { return ws->last_slices; }
void* workspace_buffer(Workspace& ws, const char* name, size_t bytes) {
  return ws.get<unsigned char>(name, bytes);
}
int workspace_device(const Workspace& ws) { return ws.device; }
int workspace_sms(const Workspace& ws) { return ws.num_sms; }
void workspace_count_launch(Workspace& ws) { ++ws.launches; }

void workspace_profile(Workspace* ws, int enable) {
  ws->prof = enable != 0;
}
void workspace_profile_reset(Workspace* ws) {
  for (auto& p : ws->prof_stats) p = Workspace::ProfStat{};
}
bool workspace_profile_get(const Workspace* ws, int cls, uint64_t* launches, double* ms,
                           double* bytes) {
  if (cls < 0 || cls >= 5) return false;
  const auto& p = ws->prof_stats[cls];
  *launches = p.launches;
  *ms = p.ms;
  *bytes = p.bytes;
  return true;
}

namespace {

uint32_t ceil_log2(uint64_t x) {
  uint32_t b = 0;
  while ((uint64_t{1} << b) < x && b < 64) ++b;
  return b;
}

// kernel classes for profiling
enum { kSweep = 0, kHistK = 1, kLocalK = 2, kSegK = 3, kOtherK = 4 };

struct Ctx {
  Workspace& ws;
  cudaStream_t st;
  ErrBlock* err;       // device
  uint32_t* counters;  // device, tile counters
  uint32_t next_counter = 0;
  // profiling records, resolved after the call's final synchronisation
  struct Rec {
    int cls;
    cudaEvent_t a, b;
    int group;
    int all_rows;  // local: 1 = every row of the group, 0 = rows outside large runs
    // rows and rank of the arrays a digit pass ran over (0: the call's): the
    // passes over run RECORDS of a run-level sort move far fewer rows than
    // the tensor has, and must not be credited with the tensor's bytes
    unsigned long long pass_rows;
    uint32_t pass_rank;
  };
  std::vector<Rec> recs;
  cudaEvent_t pending = nullptr;
  int group = 0;
  uint64_t nnz = 0;
  uint32_t rank = 0;
  // latency mode (small tensors): no host synchronisation inside the call —
  // run counts, chunk counts and item counts stay on the device and the
  // kernels bound their grid-stride loops by them; buffers are sized for the
  // worst case; the launch sequence is then capturable as a CUDA graph
  bool lat = false;
  bool small = false;  // the whole call is one k_small launch (latency mode)
  SmallArgs sa{};
  void pre() {
    if (ws.prof) {
      pending = ws.event();
      QD_CUDA(cudaEventRecord(pending, st));
    }
  }
  void launched(int cls = kOtherK, int all_rows = 0, unsigned long long pass_rows = 0,
                uint32_t pass_rank = 0) {
    ++ws.launches;
    QD_CUDA(cudaGetLastError());
    if (ws.prof && pending) {
      cudaEvent_t b = ws.event();
      QD_CUDA(cudaEventRecord(b, st));
      recs.push_back({cls, pending, b, std::min(group, kMaxGroups - 1), all_rows, pass_rows, pass_rank});
      pending = nullptr;
    }
  }
  // after the final stream sync: fold the records into ws.prof_stats
  void resolve(const ErrBlock& e) {
    const double row_bytes = 4.0 * rank + 8.0;
    for (auto& r : recs) {
      float ms = 0;
      QD_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      double large = (double)e.rows[r.group];
      double rb = row_bytes, rk = rank;
      if (r.pass_rows) {
        large = std::min(large, (double)r.pass_rows);
        rb = 4.0 * r.pass_rank + 8.0;
        rk = r.pass_rank;
      }
      double bytes = 0;
      if (r.cls == kSweep) bytes = large * 2 * rb;
      else if (r.cls == kHistK) bytes = large * 4.0 * rk;
      else if (r.cls == kLocalK) bytes = (r.all_rows ? (double)nnz : (double)nnz - large) * 2 * row_bytes;
      auto& p = ws.prof_stats[r.cls];
      ++p.launches;
      p.ms += ms;
      p.bytes += bytes;
      ws.ev_pool.push_back(r.a);
      ws.ev_pool.push_back(r.b);
    }
    recs.clear();
  }
};

// Small device->host reads of counts and of the error block (h: pinned).  A
// sliced host-buffer call keeps the device->host copy engine busy with the
// previous slice's rows, and a cudaMemcpyAsync of 8 bytes would queue behind
// gigabytes of them (measured: every slice's passes started only when the
// previous slice's output copy had drained); there a one-warp kernel stores
// the words through the pinned buffer's device mapping instead.
__global__ void k_readback(uint32_t* __restrict__ h, const uint32_t* __restrict__ d, uint32_t words) {
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) h[i] = d[i];
  __threadfence_system();
}
// load the readback kernel at workspace creation: its first launch happens
// inside a sliced call, where a lazy module load would wait for the copies in flight
void preload_kernels() {
  cudaFuncAttributes fa{};
  QD_CUDA(cudaFuncGetAttributes(&fa, k_readback));
}
static void readback(Ctx& c, void* h, const void* d, size_t bytes) {
  if (!c.ws.allow_latency && bytes % 4 == 0) {  // inside a sliced call
    k_readback<<<1, 32, 0, c.st>>>(static_cast<uint32_t*>(h), static_cast<const uint32_t*>(d),
                                   (uint32_t)(bytes / 4));
    ++c.ws.launches;
    QD_CUDA(cudaGetLastError());
    return;
  }
  QD_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, c.st));
}


constexpr uint32_t kCounters = 4096;

// Rows per onesweep tile / local chunk for a given rank, from the smem budget.
// fmt < 0: the largest tile every input format fits; else that format's
uint32_t sweep_tile_rows(const Workspace& ws, uint32_t rank, int fmt = -1) {
  if (const char* e = getenv("QD_TILE_ROWS")) return (uint32_t)atoi(e);
  size_t budget = std::min<size_t>(ws.smem_optin, (226 / QD_SCATTER_CTAS) * 1024);
  if (const char* e = getenv("QD_SMEM_BUDGET")) budget = (size_t)atoi(e) * 1024;
  auto need = [&](uint32_t T) {
    if (fmt >= 0) return ScatterLayout(T, rank, fmt).total;
    return std::max({ScatterLayout(T, rank, kAoS).total, ScatterLayout(T, rank, kSoA).total,
                     ScatterLayout(T, rank, kPK).total});
  };
  uint32_t T = QD_MAX_TILE;
  while (T > 512 && need(T) > budget) T -= 512;
  while (T > 32 && need(T) > budget) T -= 32;
  return T;
}
uint32_t local_span(const Workspace& ws, uint32_t rank) {
  size_t budget = std::min<size_t>(ws.smem_optin, 112 * 1024);
  if (const char* e = getenv("QD_LOCAL_KB")) budget = (size_t)atoi(e) * 1024;
  uint32_t TL = 2048;
  while (TL > 32 && LocalLayout(2 * TL, rank, TL).total > budget) TL -= 32;
  return TL;
}

// small-run span of k_local2: runs of <= TL rows, spans < 2*TL rows, two
// staging buffers; two CTAs per SM
uint32_t local2_span(const Workspace& ws, uint32_t rank) {
  size_t budget = std::min<size_t>(ws.smem_optin, 110 * 1024);
  if (const char* e = getenv("QD_LOCAL_KB")) budget = (size_t)atoi(e) * 1024;
  uint32_t TL = 2048;
  while (TL > 32 && Local2Layout(2 * TL, rank).total > budget) TL -= 32;
  return TL;
}

uint32_t local3_span(const Workspace& ws, uint32_t rank, uint32_t key_bytes, uint32_t warps) {
  size_t budget = std::min<size_t>(ws.smem_optin, 110 * 1024);
  if (const char* e = getenv("QD_LOCAL3_KB")) budget = (size_t)atoi(e) * 1024;
  uint32_t TL = std::min<uint32_t>(2048, warps * 32 * 8 / 2);  // k_local3's kR rounds per stripe
  while (TL > 32 && Local3Layout(2 * TL, rank, key_bytes, warps).total > budget) TL -= 32;
  return TL;
}

// n_dev (latency mode): the element count is *n_dev * n_mul on the device
// and n is its bound; tiles past the count see zeros.  (A latency-mode call
// resets the look-back ticket and status words first, so its launches
// replay identically from a CUDA graph.)
void scan_exclusive(Ctx& c, const uint32_t* in, uint64_t n, unsigned long long* out,
                    unsigned long long* d_total, const unsigned long long* n_dev = nullptr,
                    uint32_t n_mul = 1) {
  const uint32_t nb = (uint32_t)((n + kScanTile - 1) / kScanTile);
  auto* part = c.ws.get<unsigned long long>("scan_part", nb + 1);
  if (n == 0) {
    QD_CUDA(cudaMemsetAsync(d_total, 0, sizeof(unsigned long long), c.st));
    return;
  }
  Workspace& ws = c.ws;
  static const bool three_kernel = [] {
    const char* e = getenv("QD_SCAN3");
    return e && atoi(e) == 1;
  }();
  if (three_kernel) {
    c.pre();
    k_scan_reduce<<<nb, kThreads, 0, c.st>>>(in, n, part, n_dev, n_mul);
    c.launched(kSegK);
    c.pre();
    k_scan_parts<<<1, kThreads, 0, c.st>>>(part, nb, d_total);
    c.launched(kSegK);
    c.pre();
    k_scan_down<<<nb, kThreads, 0, c.st>>>(in, n, part, out, n_dev, n_mul);
    c.launched(kSegK);
    return;
  }
  if (!ws.lb_ticket) {
    ws.lb_ticket = ws.get<unsigned long long>("lb_ticket", 1);
    QD_CUDA(cudaMemsetAsync(ws.lb_ticket, 0, 8, c.st));
    ws.lb_base = 0;
  }
  // status words: cleared when (re)allocated and whenever the ticket count
  // enters a new 2^23 window, so live tags (ticket mod 2^24) never repeat
  if (nb > ws.lb_cap || (ws.lb_base >> 23) != ws.lb_cleared_epoch ||
      ((ws.lb_base + nb) >> 23) != (ws.lb_base >> 23)) {
    if (nb > ws.lb_cap) {
      ws.lb_cap = std::max<size_t>(nb, 1024);
      ws.lb_status = ws.get<unsigned long long>("lb_status", ws.lb_cap);
    }
    QD_CUDA(cudaMemsetAsync(ws.lb_status, 0, ws.lb_cap * 8, c.st));
    ws.lb_cleared_epoch = (ws.lb_base + nb) >> 23;
  }
  c.pre();
  k_scan_lookback<<<nb, kThreads, 0, c.st>>>(in, n, out, d_total, ws.lb_status,
                                             (uint32_t)ws.lb_cap, ws.lb_ticket, ws.lb_base,
                                             n_dev, n_mul);
  c.launched(kSegK);
  ws.lb_base += nb;
}

// Segment discovery on `coords` with respect to `modes`: fills seg_start[0..S]
// (device, seg_start[S] = nnz) and returns S (host sync).
uint64_t find_runs(Ctx& c, const uint32_t* coords, uint32_t rank, uint64_t nnz,
                   const std::vector<uint32_t>& modes, unsigned long long** seg_out,
                   unsigned long long** S_dev_out = nullptr, const HeadsExtra* extra = nullptr) {
  NvtxRange r_runs("run discovery");
  ModeList ml{};
  ml.n = (uint32_t)modes.size();
  for (uint32_t i = 0; i < ml.n; ++i) ml.m[i] = (uint8_t)modes[i];
  const uint32_t nb = (uint32_t)((nnz + kHeadRows - 1) / kHeadRows);
  auto* words = c.ws.get<uint32_t>("head_words", (nnz + 31) / 32 + 1);
  auto* bcnt = c.ws.get<uint32_t>("head_bcnt", nb + 1);
  auto* boff = c.ws.get<unsigned long long>("head_boff", nb + 1);
  auto* tot = c.ws.get<unsigned long long>("head_total", 1);
  c.pre();
  if (extra && extra->quad && rank == 3)
    k_heads_quad<3><<<nb, kThreads, 0, c.st>>>(coords, nnz, ml.m[0], words, bcnt, *extra);
  else if (extra && extra->quad && rank == 4)
    k_heads_quad<4><<<nb, kThreads, 0, c.st>>>(coords, nnz, ml.m[0], words, bcnt, *extra);
  else
    k_heads<<<nb, kThreads, 0, c.st>>>(coords, rank, nnz, ml, words, bcnt, extra ? *extra : HeadsExtra{});
  c.launched(kSegK);
  scan_exclusive(c, bcnt, nb, boff, tot);
  if (S_dev_out) *S_dev_out = tot;
  uint64_t S = nnz;  // latency mode: the run count stays on the device (bound: nnz)
  if (!c.lat) {
    readback(c, c.ws.h_small, tot, 8);
    QD_CUDA(cudaStreamSynchronize(c.st));
    S = c.ws.h_small[0];
  }
  auto* seg = c.ws.get<unsigned long long>("seg_start", S + 1);
  c.pre();
  k_compact<<<nb, kThreads, 0, c.st>>>(words, nnz, boff, nb, seg, tot);
  c.launched(kSegK);
  *seg_out = seg;
  return S;
}

KeySpec make_keyspec(const std::vector<uint32_t>& keys, const std::vector<uint32_t>& widths,
                     const uint32_t* dims, bool check) {
  KeySpec k{};
  k.n = (uint32_t)keys.size();
  k.check = check;
  uint32_t off = 0;
  for (int i = (int)k.n - 1; i >= 0; --i) {
    k.mode[i] = (uint8_t)keys[i];
    k.width[i] = (uint8_t)widths[i];
    k.off[i] = (uint16_t)off;
    k.dim[i] = dims[keys[i]];
    off += widths[i];
  }
  k.total_bits = off;
  return k;
}

DigitSpec make_digit(const KeySpec& k, uint32_t lo, uint32_t hi) {
  DigitSpec d{};
  for (uint32_t i = 0; i < k.n; ++i) {
    const uint32_t fb = k.off[i], fe = k.off[i] + k.width[i];
    const uint32_t b = std::max(fb, lo), e = std::min(fe, hi);
    if (b >= e) continue;
    if (d.n == kMaxTerms) throw Error(QD_INVALID_ARGUMENT, "digit spans too many modes");
    d.mode[d.n] = k.mode[i];
    d.rsh[d.n] = (uint8_t)(b - fb);
    d.bits[d.n] = (uint8_t)(e - b);
    d.lsh[d.n] = (uint8_t)(b - lo);
    ++d.n;
  }
  return d;
}

// Packed row layout of a group (PackSpec): key fields at their key offsets,
// the other modes as bit fields above when everything fits 64 bits, else as
// one mixed-radix number when THAT fits; false if neither does.
bool make_pack(const KeySpec& key, uint32_t R, const uint32_t* dims, PackSpec* out,
               const std::vector<uint32_t>& implicit = {}, bool allow_mixed = true) {
  PackSpec p{};
  p.rank = R;
  p.key_bits = key.total_bits;
  for (uint32_t m = 0; m < R; ++m) p.lim[m] = 0xFFFFFFFFu;
  std::vector<uint32_t> nonkey;
  for (uint32_t m = 0; m < R; ++m) {
    bool is_key = false;
    for (uint32_t k = 0; k < key.n; ++k) is_key |= key.mode[k] == m;
    for (uint32_t q : implicit) is_key |= q == m;  // not stored at all
    if (!is_key) nonkey.push_back(m);
  }
  p.n_imp = (uint32_t)implicit.size();
  for (uint32_t k = 0; k < p.n_imp; ++k) {
    p.imp_mode[k] = (uint8_t)implicit[k];
    p.kind[implicit[k]] = 2;
  }
  for (uint32_t k = 0; k < key.n; ++k) {
    p.off[key.mode[k]] = (uint8_t)key.off[k];
    p.width[key.mode[k]] = key.width[k];
    if (key.width[k] < 32) p.lim[key.mode[k]] = 1u << key.width[k];
  }
  uint32_t bits = key.total_bits;
  for (uint32_t m : nonkey) bits += ceil_log2(dims[m]);
  if (bits <= 64) {
    uint32_t o = key.total_bits;
    for (uint32_t m : nonkey) {
      const uint32_t w = ceil_log2(dims[m]);
      p.off[m] = (uint8_t)o;
      p.width[m] = (uint8_t)w;
      p.lim[m] = w < 32 ? (1u << w) : 0xFFFFFFFFu;
      o += w;
    }
    *out = p;
    return true;
  }
  // mixed radix: the product of the non-key dimensions must fit the bits
  // left above the key
  if (key.total_bits >= 64 || !allow_mixed) return false;
  const unsigned __int128 room = (unsigned __int128)1 << (64 - key.total_bits);
  unsigned __int128 prod = 1;
  for (uint32_t m : nonkey) {
    prod *= dims[m];
    if (prod > room) return false;
  }
  p.mixed = 1;
  p.nk_n = (uint32_t)nonkey.size();
  for (uint32_t j = 0; j < p.nk_n; ++j) {
    p.nk_mode[j] = (uint8_t)nonkey[j];
    p.nk_dim[j] = dims[nonkey[j]];
    p.nk_rcp[j] = 1.0 / (double)dims[nonkey[j]];
    p.lim[nonkey[j]] = dims[nonkey[j]];
    p.width[nonkey[j]] = 0;
    p.kind[nonkey[j]] = 1;
  }
  *out = p;
  return true;
}

// Tiles per chunk: ~11 chunks per resident CTA (chunks are dealt dynamically;
// measured on c2: 8 tiles 658 us/pass, 11 665, 16 674, 4 654 but with more
// histogram/scan work), at most kChunkTiles tiles each.
uint32_t chunk_tiles(const Workspace& ws, uint64_t rows, uint32_t T) {
  if (const char* e = getenv("QD_CHUNK_TILES")) return (uint32_t)atoi(e);
  const uint64_t ctas = (uint64_t)ws.num_sms * 2;
  const uint64_t tiles = (rows + T - 1) / T;
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(kChunkTiles, tiles / (11 * ctas)));
}

// QD_VEC_ROWS=0: scalar rank-4 row stores in k_scatter's store loop (A/B switch)
static bool vec_rows_enabled() {
  static const bool on = [] {
    const char* e = getenv("QD_VEC_ROWS");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// One stable counting pass of digit `dig` over the chunks: chunk histograms,
// (run, bin, chunk) exclusive scan, chunk-ordered scatter.
void run_pass(Ctx& c, uint32_t R, uint64_t N, uint32_t T, Rows in, RowsOut out,
              const ChunkDesc* chunks, uint64_t num_chunks,
              const unsigned long long* run_start, const DigitSpec& dig, const KeySpec& key,
              bool check, unsigned long long** offs_out = nullptr, const PackSpec* pack = nullptr,
              uint32_t pk_shift = 0, uint32_t pk_mask = 0, const uint8_t* digits_in = nullptr,
              uint8_t* digits_out = nullptr, uint32_t nd_shift = 0, uint32_t nd_mask = 0,
              const DigitSpec* next_dig = nullptr, const uint32_t* run_prefix = nullptr,
              const PeerDest* peers = nullptr, bool peers_aligned = false,
              const unsigned long long* nc_dev = nullptr, bool scattered_digits = false) {
  Workspace& ws = c.ws;
  const uint64_t nflat = num_chunks * kBins;
  auto* flat = ws.get<uint32_t>("chunk_flat", nflat);
  auto* offs = ws.get<unsigned long long>("chunk_offs", nflat);
  auto* tot = ws.get<unsigned long long>("chunk_total", 1);
  ChunkHistArgs h{};
  h.in = in;
  h.rank = R;
  h.nnz = N;
  h.chunks = chunks;
  h.num_chunks = (uint32_t)num_chunks;
  h.nc_dev = nc_dev;
  h.flat = flat;
  h.dig = dig;
  h.key = key;
  h.do_check = check;
  h.err = c.err;
  h.rows_counter = check ? &c.err->rows[std::min(c.group, kMaxGroups - 1)] : nullptr;
  h.pk_shift = pk_shift;
  h.pk_mask = pk_mask;
  h.digits = digits_in;
  if (pack) {
    h.pack = *pack;
    h.check_pack = in.fmt == kAoS && out.fmt == kPK;
  }
  for (uint32_t m = 0; m < 4; ++m) {
    h.lim[m] = 0xFFFFFFFFu;
    if (m >= R) continue;
    if (h.do_check)
      for (uint32_t k = 0; k < key.n; ++k)
        if (key.mode[k] == m) h.lim[m] = key.dim[k];
    if (h.check_pack) h.lim[m] = std::min(h.lim[m], h.pack.lim[m]);
  }
  c.pre();
  k_chunk_hist<<<(uint32_t)std::min<uint64_t>(num_chunks, (uint64_t)ws.num_sms * 8), kThreads, 0,
                 c.st>>>(h);
  c.launched(kHistK, 0, N, R);
  scan_exclusive(c, flat, nflat, offs, tot, nc_dev, kBins);

  ScatterArgs a{};
  a.in = in;
  a.out = out;
  a.rank = R;
  a.nnz = N;
  a.T = T;
  a.chunks = chunks;
  a.num_chunks = (uint32_t)num_chunks;
  a.nc_dev = nc_dev;
  a.offs = offs;
  a.run_start = run_start;
  a.dig = dig;
  a.pk_shift = pk_shift;
  a.pk_mask = pk_mask;
  if (pack) {
    a.pack = *pack;
    PackFast& f = a.pf;
    for (uint32_t m = 0; m < 4; ++m) f.mpos[m] = f.impk[m] = 0xFFu;
    for (uint32_t k = 0; k < pack->n_imp; ++k)
      if (pack->imp_mode[k] < 4) f.impk[pack->imp_mode[k]] = k;
    for (uint32_t m = 0; m < R && m < 4; ++m) {
      if (pack->kind[m] == 0 && pack->width[m]) {
        f.fsh[m] = pack->off[m];
        f.fmask[m] = (uint32_t)((1ull << pack->width[m]) - 1ull);
      }
    }
    f.mixed = pack->mixed;
    f.key_bits = pack->key_bits;
    f.nk_n = pack->nk_n;
    if (pack->mixed) {
      unsigned long long w = 1;
      for (int j = (int)pack->nk_n - 1; j >= 0; --j) {
        const uint32_t m = pack->nk_mode[j];
        if (j < 4) {
          f.dimj[j] = pack->nk_dim[j];
          f.magic[j] = ~0ull / pack->nk_dim[j];
        }
        if (m < 4) {
          f.mul[m] = w;
          f.mpos[m] = (uint32_t)j;
        }
        w *= pack->nk_dim[j];
      }
    }
  }
  a.next_dig = digits_out;
  a.nd_shift = nd_shift;
  a.nd_mask = nd_mask;
  if (next_dig) a.ndig = *next_dig;
  a.run_prefix = run_prefix;
  a.peers = peers;
  a.vec_out = out.fmt == kAoS && vec_rows_enabled() &&
              (peers ? peers_aligned : (reinterpret_cast<uintptr_t>(out.c) & 15u) == 0);
  if (const char* e = getenv("QD_SCATTER_DBG")) a.dbg = atoi(e);
  {
    static const int rank_mode = [] {
      const char* e = getenv("QD_RANK_MODE");
      return e ? atoi(e) : 3;  // 0 MATCH.ANY, 1 adaptive, 2 ballots, 3 (default) by pass
    }();
    static const uint32_t match_max = [] {
      const char* e = getenv("QD_MATCH_MAX");
      return e ? (uint32_t)atoi(e) : 8u;
    }();
    uint32_t nb = 0;
    if (dig.lookup) {
      nb = 8;
    } else {
      for (uint32_t i = 0; i < dig.n; ++i) nb += dig.bits[i];
    }
    if (in.fmt == kPK) nb = (uint32_t)__builtin_popcount(pk_mask);
    a.dbits = std::min<uint32_t>(8, std::max<uint32_t>(1, nb));
    // by pass: ballots where the planner expects nearly random digits within
    // a tile (the first digit of a group whose least significant key mode is
    // the fastest-varying mode of the rows' order: a warp's 32 digits are then
    // nearly all distinct and MATCH.ANY costs ~2 cycles per distinct value);
    // every other pass sees digit runs, where MATCH.ANY wins.  400 M rows of
    // c5 (0,2,1): first pass 3.05 -> 2.89 ms with ballots, later passes
    // +3-14 %; c2 (2,0,1) 1.83 -> 1.76 ms, (1,2,0) 3.17 -> 3.11 ms, while
    // (1,0,2) and (2,1,0) (key mode 1 first) lose 4-9 % with ballots.
    a.rank_mode = rank_mode == 3 ? (scattered_digits && !dig.lookup ? 2 : 0)
                  : rank_mode == 4 ? ((pk_shift == 0 && !dig.lookup) ? 2 : 0)  // experiment: every first pass
                                   : rank_mode;
    a.match_max = match_max;
  }
  if (a.dbg & 2) {
    a.dbg_t = ws.get<unsigned long long>("dbg_t", 16);
    QD_CUDA(cudaMemsetAsync(a.dbg_t, 0, 128, c.st));
  }
  if (c.next_counter >= kCounters) {
    QD_CUDA(cudaMemsetAsync(c.counters, 0, kCounters * 4, c.st));
    c.next_counter = 0;
  }
  a.chunk_counter = c.counters + c.next_counter++;
  const size_t smem = ScatterLayout(T, R, in.fmt).total;
  const int rt = (R == 3 || R == 4) ? (int)R : 0;
  const int dm = dig.lookup ? 0 : (dig.n == 1 ? 1 : (dig.n == 2 ? 2 : 0));
  ScatterFn fn = scatter_kernel(rt, dm, in.fmt, out.fmt, pack && (pack->mixed || pack->n_imp) ? 1 : 0);
  if (!fn) throw Error(QD_CUDA_ERROR, "no scatter kernel for this row format pair");
  int per_sm = 0;
  QD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kSortThreads, smem));
  const uint32_t grid =
      (uint32_t)std::min<uint64_t>(num_chunks, (uint64_t)std::max(1, per_sm) * ws.num_sms);
  c.pre();
  fn<<<grid, kSortThreads, smem, c.st>>>(a);
  c.launched(kSweep, 0, N, R);
  if (a.dbg & 2) {
    unsigned long long h[16];
    QD_CUDA(cudaMemcpyAsync(h, a.dbg_t, 128, cudaMemcpyDeviceToHost, c.st));
    QD_CUDA(cudaStreamSynchronize(c.st));
    fprintf(stderr, "scatter phases (Mcycles, thread0 sum over CTAs): grid %u", grid);
    for (int i = 1; i < 9; ++i) fprintf(stderr, " p%d=%.2f", i, h[i] / 1e6);
    fprintf(stderr, "\n");
  }
  if (offs_out) *offs_out = offs;
}

// One segmented stable sort (a plan group), src -> dst, with tmp scratch.
void segmented_sort(Ctx& c, const TensorView& t, const uint32_t* src_c, const double* src_v,
                    uint32_t* dst_c, double* dst_v, uint32_t* tmp_c, double* tmp_v,
                    const Group& g) {
  Workspace& ws = c.ws;
  const uint64_t N = t.nnz;
  const uint32_t R = t.rank;
  if (N == 0) return;

  // key field widths
  std::vector<uint32_t> widths(g.keys.size());
  if (g.check_range) {
    for (size_t i = 0; i < g.keys.size(); ++i) widths[i] = ceil_log2(t.dims[g.keys[i]]);
  } else {
    ModeList ml{};
    ml.n = (uint32_t)g.keys.size();
    for (uint32_t i = 0; i < ml.n; ++i) ml.m[i] = (uint8_t)g.keys[i];
    auto* mx = ws.get<uint32_t>("mode_max", kMaxKeys);
    QD_CUDA(cudaMemsetAsync(mx, 0, kMaxKeys * 4, c.st));
    const uint32_t grid = (uint32_t)std::min<uint64_t>((N + kThreads - 1) / kThreads, ws.num_sms * 8);
    c.pre();
    k_mode_max<<<grid, kThreads, 0, c.st>>>(src_c, R, N, ml, mx);
    c.launched(kOtherK);
    uint32_t* h = reinterpret_cast<uint32_t*>(ws.h_small);
    readback(c, h, mx, kMaxKeys * 4);
    QD_CUDA(cudaStreamSynchronize(c.st));
    for (size_t i = 0; i < g.keys.size(); ++i) widths[i] = ceil_log2((uint64_t)h[i] + 1);
  }
  const KeySpec key = make_keyspec(g.keys, widths, t.dims, g.check_range);
  const uint32_t bits = key.total_bits;

  if (bits == 0 || N == 1) {
    // nothing to reorder; still the histogram pass's range check
    const uint32_t grid = (uint32_t)std::min<uint64_t>((N + kThreads - 1) / kThreads, ws.num_sms * 8);
    c.pre();
    k_copy_check<<<grid, kThreads, 0, c.st>>>(src_c, src_v, dst_c, dst_v, R, N, key, c.err);
    c.launched(kOtherK);
    return;
  }

  const uint32_t D = (bits + kRadixLog - 1) / kRadixLog;
  const uint32_t per = (bits + D - 1) / D;
  std::vector<DigitSpec> digs(D);
  // digit q = key bits [cut[q], cut[q+1]): `per` bits each from the bottom,
  // the last one narrower (the narrower digit FIRST for groups whose first
  // digit is scattered measured slower: c2 (0,2,1) 2.04 -> 2.12, (2,0,1)
  // 1.77 -> 1.88, (1,2,0) 3.10 -> 3.29 ms)
  std::vector<uint32_t> cut(D + 1);
  for (uint32_t q = 0; q <= D; ++q) cut[q] = std::min(bits, q * per);
  if (const char* e = getenv("QD_CUTS")) {  // experiment: explicit upper cuts "8,15,21" for keys of that width
    std::vector<uint32_t> v;
    for (const char* p = e; *p;) {
      v.push_back((uint32_t)strtoul(p, const_cast<char**>(&p), 10));
      if (*p == ',') ++p;
    }
    bool ok = v.size() == D && v.back() == bits;
    for (size_t i = 0; ok && i < v.size(); ++i)
      ok = v[i] > (i ? v[i - 1] : 0u) && v[i] - (i ? v[i - 1] : 0u) <= (uint32_t)kRadixLog;
    if (ok)
      for (uint32_t q = 0; q < D; ++q) cut[q + 1] = v[q];
  }
  for (uint32_t q = 0; q < D; ++q) digs[q] = make_digit(key, cut[q], cut[q + 1]);

  const uint32_t T = sweep_tile_rows(ws, R);
  static const bool per_fmt_tiles = [] {
    const char* e = getenv("QD_PK_TILES");
    return !(e && atoi(e) == 0);
  }();
  // small runs: k_local2 (bucketed groups; keys up to 64 bits, no run bits)
  // or, for a whole tensor that fits one CTA, k_local (run bits in its key)
  // QD_LOCAL_V: 3 (default) = k_local3 (streamed block LSD over (run, key)),
  // 2 = k_local2 (warp per run), 1 = k_local (round-1 kernel)
  static const int local_v = [] {
    const char* e = getenv("QD_LOCAL_V");
    return e ? atoi(e) : 3;
  }();
  const bool local2 = !g.prefix.empty() && local_v >= 2;
  uint32_t TL = 0;
  uint32_t kbytes = 4;
  static const int l3_threads = [] {
    const char* e = getenv("QD_LOCAL3_THREADS");
    return e && atoi(e) == 256 ? 256 : 512;
  }();
  if (local2 && local_v == 3) {
    TL = local3_span(ws, R, 4, l3_threads / 32);
    if (bits + ceil_log2(2 * TL) > 32) {
      kbytes = 8;
      TL = local3_span(ws, R, 8, l3_threads / 32);
    }
    if (bits + ceil_log2(2 * TL) > 64) TL = 0;  // composite key would not fit 64 bits
  } else if (local2) {
    TL = local2_span(ws, R);
    if (bits > 64) TL = 0;
  } else {
    TL = local_span(ws, R);
    if (bits + ceil_log2(TL) + 1 > 64) TL = 0;  // local key would not fit 64 bits
  }

  // chunks hold whole tiles of the passes that dominate: the packed-row
  // tile when the rows will pack (the first, AoS, pass then ends each chunk
  // with a partial tile)
  uint32_t Tch = T;
  if (per_fmt_tiles && ws.allow_pack && g.check_range && D > 1) {
    PackSpec probe{};
    if (make_pack(key, R, t.dims, &probe)) Tch = sweep_tile_rows(ws, R, kPK);
  }
  const uint32_t CH = Tch * chunk_tiles(ws, N, Tch);
  ChunkDesc* chunks = ws.get<ChunkDesc>("chunks", 1);
  const unsigned long long* run_start = nullptr;
  uint64_t num_chunks = 0;
  unsigned long long* seg = nullptr;
  uint64_t S = 0, num_large = 0, local_chunks = 0;
  const uint32_t* local_list = nullptr;
  const uint32_t* local_first = nullptr;
  bool small_runs = false;
  const unsigned long long* lat_counts = nullptr;  // latency mode: {large runs, chunks, items}
  const uint32_t* local_maxrun = nullptr;            // per local chunk: its longest small run

  // Intermediate rows: packed 16-byte rows when every coordinate packs into
  // one u64 (key fields at their key offsets, so a digit is shift + mask),
  // else AoS rows.  A coordinate that would not pack losslessly (only
  // possible for modes the plan never range-checks) is flagged by the first
  // pass over the rows and the whole call is redone unpacked (run_groups).
  // (Decided before run discovery, which does that first pass's checks for a
  // bucketed group; a bucketed group's passes always have their runs' table.)
  PackSpec pack{};
  bool packed = ws.allow_pack && g.check_range && D > 1;
  const bool have_runs = !g.prefix.empty();
  if (packed) {
    // prefix modes are constant within a run: when the row does not pack
    // otherwise, leave them out and restore them from the run
    // QD_PACK_ORDER=1 (default): plain bit fields with the prefix restored
    // from the run before a mixed-radix word (no division in the
    // unpacking pass; c5 (0,2,1) 59.3 -> 58.6 ms); 0: mixed radix first
    static const int pack_order = [] {
      const char* e = getenv("QD_PACK_ORDER");
      return e ? atoi(e) : 1;
    }();
    if (pack_order == 1)
      packed = make_pack(key, R, t.dims, &pack, {}, false) ||
               (have_runs && make_pack(key, R, t.dims, &pack, g.prefix, false)) ||
               make_pack(key, R, t.dims, &pack) ||
               (have_runs && make_pack(key, R, t.dims, &pack, g.prefix));
    else
      packed = make_pack(key, R, t.dims, &pack) ||
               (have_runs && make_pack(key, R, t.dims, &pack, g.prefix));
  }
  // unpacked intermediates: AoS rows (two streams) and the digit side
  // channel, or (QD_SOA_INTERMEDIATES=1) SoA columns whose histogram reads
  // the key column
  static const bool unpacked_soa = [] {
    const char* e = getenv("QD_SOA_INTERMEDIATES");
    return e && atoi(e) == 1;
  }();
  const bool side = packed || !unpacked_soa;
  bool fused_first = false;  // the first digit bytes were written by run discovery

  if (g.prefix.empty()) {
    if (TL && N <= TL) {
      LocalArgs la{src_c, src_v, dst_c, dst_v, R, N, TL, (uint32_t)N, nullptr, 1, key, c.err,
                   nullptr, nullptr};
      const size_t smem = LocalLayout((uint32_t)N, R, TL).total;
      c.pre();
      k_local<<<1, kLocalThreads, smem, c.st>>>(la);
      c.launched(kLocalK, 1);
      return;
    }
    num_chunks = (N + CH - 1) / CH;
    chunks = ws.get<ChunkDesc>("chunks", num_chunks);
    c.pre();
    k_uniform_chunks<<<(uint32_t)((num_chunks + kThreads - 1) / kThreads), kThreads, 0, c.st>>>(
        N, CH, (uint32_t)num_chunks, chunks);
    c.launched(kSegK);
  } else {
    unsigned long long* S_found = nullptr;
    // Run discovery also does the first pass's range and pack checks and
    // leaves every row's first digit as a byte, so the first histogram reads
    // 1 byte per row instead of the coordinates again (HeadsExtra): for
    // rank-3/4 rows with one prefix mode through k_heads_quad.  The generic
    // per-row form (QD_FUSE_HEADS=2: any rank / prefix) measured SLOWER — its
    // strided loads and byte stores cost k_heads more than the histogram
    // saves (c5 (0,2,1) 58.4 -> 62.3 ms).  QD_FUSE_HEADS=0: off.
    static const int fuse_mode = [] {
      const char* e = getenv("QD_FUSE_HEADS");
      return e ? atoi(e) : 1;
    }();
    const bool quad_ok = (R == 3 || R == 4) && g.prefix.size() == 1 && digs[0].lookup == nullptr &&
                         digs[0].n <= 2 && (reinterpret_cast<uintptr_t>(src_c) & 15u) == 0;
    const bool fuse_heads = fuse_mode == 2 || (fuse_mode == 1 && quad_ok);
    HeadsExtra hx{};
    if (fuse_heads && side) {
      hx.digits = ws.get<uint8_t>("digits", N + 16);
      hx.quad = fuse_mode == 1;
      for (uint32_t m = 0; m < 4; ++m) {
        hx.lim[m] = 0xFFFFFFFFu;
        if (m >= R) continue;
        if (key.check)
          for (uint32_t k = 0; k < key.n; ++k)
            if (key.mode[k] == m) hx.lim[m] = key.dim[k];
        if (packed) hx.lim[m] = std::min(hx.lim[m], pack.lim[m]);
      }
      hx.err = c.err;
      hx.do_check = key.check;
      hx.check_pack = packed;
      for (uint32_t m = 0; m < R; ++m) hx.pack_lim[m] = packed ? pack.lim[m] : 0xFFFFFFFFu;
      hx.dig = digs[0];
      hx.key = key;
      fused_first = true;
    }
    S = find_runs(c, src_c, R, N, g.prefix, &seg, &S_found, hx.digits ? &hx : nullptr);  // latency mode: a bound (N)
    auto* is_large = ws.get<uint32_t>("run_large", S + 1);
    auto* nch = ws.get<uint32_t>("run_nchunks", S + 1);
    auto* loff = ws.get<unsigned long long>("run_loff", S + 1);
    auto* coff = ws.get<unsigned long long>("run_coff", S + 1);
    auto* totals = ws.get<unsigned long long>("run_totals", 3);
    auto* S_dev = ws.get<unsigned long long>("run_S", 1);
    const uint64_t nloc = TL ? (N + TL - 1) / TL : 0;
    auto* lflag = ws.get<uint32_t>("local_flag", nloc + 1);
    auto* lpos = ws.get<unsigned long long>("local_pos", nloc + 1);
    auto* llist = ws.get<uint32_t>("local_list", nloc + 1);
    auto* lfirst = ws.get<uint32_t>("local_first", nloc + 1);
    auto* lmax = ws.get<uint32_t>("local_maxrun", nloc + 1);
    if (nloc) QD_CUDA(cudaMemsetAsync(lflag, 0, nloc * 4, c.st));
    if (nloc) QD_CUDA(cudaMemsetAsync(lmax, 0, nloc * 4, c.st));
    local_maxrun = lmax;
    if (c.lat) {  // the device's run count; no host round trip
      QD_CUDA(cudaMemcpyAsync(S_dev, S_found, 8, cudaMemcpyDeviceToDevice, c.st));
    } else {
      ws.h_small[0] = S;
      QD_CUDA(cudaMemcpyAsync(S_dev, ws.h_small, 8, cudaMemcpyHostToDevice, c.st));
    }
    const uint32_t grid = (uint32_t)std::min<uint64_t>((S + kThreads - 1) / kThreads, ws.num_sms * 8);
    c.pre();
    k_classify_chunks<<<grid, kThreads, 0, c.st>>>(seg, S_dev, TL, CH, is_large, nch, lflag,
                                                   lfirst, lmax);
    c.launched(kSegK);
    scan_exclusive(c, is_large, S, loff, totals, c.lat ? S_found : nullptr);
    scan_exclusive(c, nch, S, coff, totals + 1, c.lat ? S_found : nullptr);
    if (nloc) {
      scan_exclusive(c, lflag, nloc, lpos, totals + 2);
      c.pre();
      k_compact_flags<<<(uint32_t)std::min<uint64_t>((nloc + kThreads - 1) / kThreads, ws.num_sms * 8),
                        kThreads, 0, c.st>>>(lflag, lpos, nloc, llist);
      c.launched(kSegK);
    } else {
      QD_CUDA(cudaMemsetAsync(totals + 2, 0, 8, c.st));
    }
    if (c.lat) {
      // bounds only; the counts stay on the device (totals[0..2])
      num_large = N / (TL + 1) + 1;
      num_chunks = N / CH + num_large + 1;
      local_chunks = nloc;
      small_runs = TL != 0;
      lat_counts = totals;
    } else {
      readback(c, ws.h_small + 1, totals, 24);
      QD_CUDA(cudaStreamSynchronize(c.st));
      num_large = ws.h_small[1];
      num_chunks = ws.h_small[2];
      local_chunks = ws.h_small[3];
      small_runs = S > num_large;
    }
    local_list = llist;
    local_first = lfirst;
    if (num_chunks) {
      chunks = ws.get<ChunkDesc>("chunks", num_chunks);
      auto* rs = ws.get<unsigned long long>("run_start", num_large);
      c.pre();
      k_gen_chunks<<<grid, kThreads, 0, c.st>>>(seg, S_dev, CH, is_large, loff, coff, chunks, rs);
      c.launched(kSegK);
      run_start = rs;
    }
  }

  if (num_chunks) {
    uint32_t* run_prefix = nullptr;
    if (packed && pack.n_imp) {
      run_prefix = ws.get<uint32_t>("run_prefix", num_large * pack.n_imp + 1);
      ModeList pm{};
      pm.n = pack.n_imp;
      for (uint32_t k = 0; k < pack.n_imp; ++k) pm.m[k] = pack.imp_mode[k];
      c.pre();
      k_run_prefix<<<(uint32_t)std::min<uint64_t>((num_large + kThreads - 1) / kThreads + 1,
                                                   ws.num_sms * 8),
                     kThreads, 0, c.st>>>(src_c, R, run_start, num_large,
                                          lat_counts ? lat_counts : nullptr, pm, run_prefix);
      c.launched(kSegK);
    }
    if (!packed && D > 1 && !tmp_c) {
      tmp_c = ws.get<uint32_t>("rowsA_c", N * R);
      tmp_v = ws.get<double>("rowsA_v", N);
    }
    // packed intermediates ping-pong in workspace buffers of 16 bytes/row
    uint32_t* pk[2] = {nullptr, nullptr};
    if (packed) {
      pk[0] = ws.get<uint32_t>("pkA", N * 4);
      if (D > 2) pk[1] = ws.get<uint32_t>("pkB", N * 4);
    }
    uint8_t* digbuf = (side && D > 1) || fused_first ? ws.get<uint8_t>("digits", N + 16) : nullptr;
    Rows in{src_c, src_v, kAoS};
    for (uint32_t q = 0; q < D; ++q) {
      const bool last = q + 1 == D;
      const bool to_dst = ((D - 1 - q) % 2) == 0;
      const int ofmt = last ? kAoS : (packed ? kPK : (unpacked_soa ? kSoA : kAoS));
      RowsOut out{to_dst ? dst_c : tmp_c, to_dst ? dst_v : tmp_v, ofmt};
      if (ofmt == kPK) out = RowsOut{pk[q % 2], nullptr, kPK};
      const uint32_t lo = cut[q], hi = cut[q + 1];
      // packed passes hand the next pass its digit bytes (1 B/row instead of
      // re-reading 16 B rows for the next histogram)
      const uint8_t* dig_in = (side && (q > 0 || fused_first)) ? digbuf : nullptr;
      uint8_t* dig_out = (side && !last) ? digbuf : nullptr;
      const uint32_t nlo = cut[std::min(q + 1, D)], nhi = cut[std::min(q + 2, D)];
      // packed-row passes afford a larger tile (16-byte staged rows)
      const uint32_t Tq = (per_fmt_tiles && in.fmt == kPK) ? sweep_tile_rows(ws, R, kPK) : T;
      NvtxRange r_pass("pass " + std::to_string(q) + " bits [" + std::to_string(lo) + "," +
                       std::to_string(hi) + ")");
      run_pass(c, R, N, Tq, in, out, chunks, num_chunks, run_start, digs[q], key,
               q == 0 && key.check, nullptr, packed ? &pack : nullptr, lo,
               (1u << (hi - lo)) - 1u, dig_in, dig_out, nlo, last ? 0u : (1u << (nhi - nlo)) - 1u,
               last ? nullptr : &digs[q + 1], run_prefix, nullptr, false,
               lat_counts ? lat_counts + 1 : nullptr, q == 0 && g.first_digit_scattered);
      in = Rows{out.c, out.v, out.fmt};
    }
  }
  if (small_runs && local_chunks && local2) {
    NvtxRange r_local("small runs (k_local3)");
    // small runs: items = the runs starting in [c*TL, (c+1)*TL) of every
    // chunk that holds some (compact list); after the passes, whose
    // intermediates may use dst's storage
    auto* items = ws.get<LocalItem>("local_items", local_chunks);
    auto* S_dev = ws.get<unsigned long long>("run_S", 1);
    c.pre();
    k_local_items<<<(uint32_t)std::min<uint64_t>((local_chunks + kThreads - 1) / kThreads,
                                                 ws.num_sms * 8),
                    kThreads, 0, c.st>>>(local_list, local_first, seg, S_dev, N, TL,
                                         (uint32_t)local_chunks,
                                         lat_counts ? lat_counts + 2 : nullptr, local_maxrun,
                                         items);
    c.launched(kSegK);
    static const bool merge_items = [] {
      const char* e = getenv("QD_MERGE_ITEMS");
      return !(e && atoi(e) == 0);
    }();
    if (local_v == 3 && merge_items) {
      const uint32_t ng = (uint32_t)((local_chunks + kMergeGroup - 1) / kMergeGroup);
      c.pre();
      k_merge_items<<<(uint32_t)std::min<uint64_t>((ng + kThreads - 1) / kThreads + 1, ws.num_sms * 8),
                      kThreads, 0, c.st>>>(items, (uint32_t)local_chunks,
                                           lat_counts ? lat_counts + 2 : nullptr, 2 * TL);
      c.launched(kSegK);
    }
    Local2Args la{};
    la.in_c = src_c;
    la.in_v = src_v;
    la.out_c = dst_c;
    la.out_v = dst_v;
    la.rank = R;
    la.cap = 2 * TL;
    la.seg_start = seg;
    la.items = items;
    la.n_items = (uint32_t)local_chunks;
    la.n_items_dev = lat_counts ? lat_counts + 2 : nullptr;
    if (c.next_counter >= kCounters) {
      QD_CUDA(cudaMemsetAsync(c.counters, 0, kCounters * 4, c.st));
      c.next_counter = 0;
    }
    la.item_counter = c.counters + c.next_counter++;
    la.key = key;
    la.npasses = (bits + kRadixLog - 1) / kRadixLog;
    const uint32_t lper = (bits + la.npasses - 1) / la.npasses;
    for (uint32_t q = 0; q < la.npasses; ++q) {
      const uint32_t lo = q * lper, hi = std::min(bits, lo + lper);
      la.dig[q] = make_digit(key, lo, hi);
      la.dig_bits[q] = hi - lo;
    }
    la.err = c.err;
    {
      // QD_LOCAL3_BALLOT: bit q = pass q of k_local3 ranks with ballots
      static const int bp = [] {
        const char* e = getenv("QD_LOCAL3_BALLOT");
        return e ? atoi(e) : 0;
      }();
      la.ballot_passes = (uint32_t)bp;
    }
    using LocalFn = void (*)(Local2Args);
    const int nt = local_v == 3 ? l3_threads : kLocal2Threads;
    const LocalFn fn =
        local_v != 3 ? k_local2
        : nt == 256 ? (kbytes == 4 ? k_local3<uint32_t, 256> : k_local3<unsigned long long, 256>)
        : R == 3    ? (kbytes == 4 ? k_local3<uint32_t, 512, 3> : k_local3<unsigned long long, 512, 3>)
        : R == 4    ? (kbytes == 4 ? k_local3<uint32_t, 512, 4> : k_local3<unsigned long long, 512, 4>)
                    : (kbytes == 4 ? k_local3<uint32_t, 512> : k_local3<unsigned long long, 512>);
    const size_t smem = local_v == 3 ? Local3Layout(2 * TL, R, kbytes, nt / 32).total
                                     : Local2Layout(2 * TL, R).total;
    int per_sm = 0;
    QD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nt, smem));
    const uint32_t grid = (uint32_t)std::min<uint64_t>(local_chunks,
                                                       (uint64_t)std::max(1, per_sm) * ws.num_sms);
    c.pre();
    fn<<<grid, nt, smem, c.st>>>(la);
    c.launched(kLocalK);
    if (getenv("QD_LOCAL_STATS") && !c.lat) {  // debug: the small-run items of this call
      std::vector<LocalItem> h(local_chunks);
      QD_CUDA(cudaMemcpyAsync(h.data(), items, local_chunks * sizeof(LocalItem),
                              cudaMemcpyDeviceToHost, c.st));
      QD_CUDA(cudaStreamSynchronize(c.st));
      uint64_t ne = 0, rows = 0, runs = 0, pcnt[8] = {0}, prow[8] = {0}, small32 = 0;
      for (const LocalItem& it : h) {
        if (!it.n) continue;
        ++ne;
        rows += it.n;
        runs += it.nruns;
        const uint32_t rb = it.nruns > 1 ? 32 - __builtin_clz(it.nruns - 1) : 0;
        const uint32_t P = (bits + rb + kLocalBitsMax - 1) / kLocalBitsMax;
        if (it.maxrun <= 32) {
          ++small32;
        } else {
          ++pcnt[std::min<uint32_t>(P, 7)];
          prow[std::min<uint32_t>(P, 7)] += it.n;
        }
      }
      fprintf(stderr, "local: TL %u items %llu non-empty %llu rows %llu runs %llu (avg item %.0f rows, "
              "%.1f runs) row-parallel items %llu; P:", TL, (unsigned long long)local_chunks,
              (unsigned long long)ne, (unsigned long long)rows, (unsigned long long)runs,
              ne ? (double)rows / ne : 0.0, ne ? (double)runs / ne : 0.0,
              (unsigned long long)small32);
      for (int q = 0; q < 8; ++q)
        if (pcnt[q]) fprintf(stderr, " %d:%llu items/%llu rows", q, (unsigned long long)pcnt[q],
                             (unsigned long long)prow[q]);
      fprintf(stderr, "\n");
    }
  } else if (small_runs && local_chunks) {
    // small runs: chunks of runs starting in [c*TL, (c+1)*TL), only the
    // chunks that hold some (compact list); after the passes, whose
    // intermediates may use dst's storage
    LocalArgs la{src_c, src_v, dst_c, dst_v, R, N, TL, 2 * TL, seg, S, key, c.err, local_list,
                 local_first};
    const size_t smem = LocalLayout(2 * TL, R, TL).total;
    c.pre();
    k_local<<<(uint32_t)local_chunks, kLocalThreads, smem, c.st>>>(la);
    c.launched(kLocalK);
  }
}


// Run-level stable sort by mode k (empty prefix): see k_run_records.  Returns
// false (nothing written) when the runs are too short to pay off.
template <class Pays>
bool try_run_sort(Ctx& c, const TensorView& t, const uint32_t* src_c, const double* src_v,
                  uint32_t* dst_c, double* dst_v, uint32_t k, Pays pays) {
  Workspace& ws = c.ws;
  const uint64_t N = t.nnz;
  const uint32_t R = t.rank;
  unsigned long long* seg = nullptr;
  const uint64_t S = find_runs(c, src_c, R, N, {k}, &seg);
  if (S == 0 || (double)N / (double)S < kRunSortMinAvg || !pays(S)) return false;
  auto* rk0 = ws.get<uint32_t>("run_rk0", S);
  auto* rv0 = ws.get<double>("run_rv0", S);
  auto* rk1 = ws.get<uint32_t>("run_rk1", S);
  auto* rv1 = ws.get<double>("run_rv1", S);
  auto* rkt = ws.get<uint32_t>("run_rkt", S);
  auto* rvt = ws.get<double>("run_rvt", S);
  const uint32_t grid = (uint32_t)std::min<uint64_t>((S + kThreads - 1) / kThreads, ws.num_sms * 8);
  c.pre();
  k_run_records<<<grid, kThreads, 0, c.st>>>(src_c, R, k, t.dims[k], seg, S, rk0, rv0, c.err);
  c.launched(kSegK);
  // the records are a rank-1 tensor: sort them by their key with the engine
  const uint32_t rdim = t.dims[k];
  TensorView rt{1, &rdim, S};
  Group rg;
  rg.keys = {0};
  segmented_sort(c, rt, rk0, rv0, rk1, rv1, rkt, rvt, rg);
  auto* lens = ws.get<uint32_t>("run_lens", S);
  auto* dsto = ws.get<unsigned long long>("run_dsto", S + 1);
  auto* tot = ws.get<unsigned long long>("run_tot", 1);
  c.pre();
  k_run_lens<<<grid, kThreads, 0, c.st>>>(rv1, S, lens);
  c.launched(kSegK);
  scan_exclusive(c, lens, S, dsto, tot);
  const uint64_t ntiles = (N + kMoveTile - 1) / kMoveTile;
  auto* first = ws.get<uint32_t>("run_tile_first", ntiles + 1);
  c.pre();
  k_tile_first_run<<<(uint32_t)std::min<uint64_t>((ntiles + kThreads) / kThreads, ws.num_sms * 8),
                     kThreads, 0, c.st>>>(dsto, S, ntiles, first);
  c.launched(kSegK);
  c.pre();
  if (R == 3)
    k_move_runs2<3><<<(uint32_t)ntiles, kMoveThreads, 0, c.st>>>(src_c, src_v, dst_c, dst_v, R, N,
                                                                 rv1, dsto, S, first);
  else if (R == 4 && ((reinterpret_cast<uintptr_t>(src_c) | reinterpret_cast<uintptr_t>(dst_c)) & 15u) == 0)
    k_move_runs2<4><<<(uint32_t)ntiles, kMoveThreads, 0, c.st>>>(src_c, src_v, dst_c, dst_v, R, N,
                                                                 rv1, dsto, S, first);
  else
    k_move_runs2<0><<<(uint32_t)ntiles, kMoveThreads, 0, c.st>>>(src_c, src_v, dst_c, dst_v, R, N,
                                                                 rv1, dsto, S, first);
  c.launched(kSweep);
  return true;
}

// One plan group, possibly decomposed: a stable sort by keys (k1..km) within
// prefix runs equals [sort by k1, then by (k2..km) within (prefix, k1) runs]
// (MSD) and [sort by km, then by (k1..km-1)] (LSD).  When the first such step
// can be a run-level sort (its key's runs are long), use that chain.
void exec_group(Ctx& c, const TensorView& t, const uint32_t* src_c, const double* src_v,
                uint32_t* dst_c, double* dst_v, uint32_t* tmp_c, double* tmp_v, const Group& g) {
  Workspace& ws = c.ws;
  const uint64_t N = t.nnz;
  const uint32_t R = t.rank;
  // QD_RUN_SORT: unset = decide by the cost model below, 0 = never, 1 = always
  // (when a candidate's runs are long enough)
  const char* rs_env = getenv("QD_RUN_SORT");
  const int rs_mode = rs_env ? atoi(rs_env) : -1;
  const bool disabled = rs_mode == 0;
  uint64_t min_rows = kRunSortMinRows;
  if (const char* e = getenv("QD_RUN_SORT_MIN_ROWS")) min_rows = strtoull(e, nullptr, 10);
  // candidates: the key mode is not the last mode (its runs would be single
  // rows of a duplicate-free tensor) and every prefix mode precedes it
  auto candidate = [&](uint32_t k) {
    if (k + 1 >= R) return false;
    for (uint32_t p : g.prefix)
      if (p > k) return false;
    return true;
  };
  const size_t m = g.keys.size();
  // Cost model (per row / per run, measured on B200 with c2/c3 data): a
  // chunked digit pass (histogram, scan, scatter) costs ~10.5 ps per row when
  // the coordinates pack into 64 bits (16-byte rows), ~14.5 ps for wider
  // rank-3 rows and ~16 ps for wider rank >= 4 rows; a run sort pays ~2.3 ps
  // per row for run discovery plus ~13.5 ps (rank 3) / 17 ps (rank >= 4)
  // per row for the run move, and ~(20 + 10 x its digit passes) ps per run.
  // the chunked passes' per-row cost: 16-byte packed rows whenever the
  // group's rows pack (plain or mixed-radix, as segmented_sort decides)
  bool packs = false;
  if (ws.allow_pack && g.check_range) {
    std::vector<uint32_t> wd(m);
    for (size_t i = 0; i < m; ++i) wd[i] = ceil_log2(t.dims[g.keys[i]]);
    PackSpec probe{};
    packs = make_pack(make_keyspec(g.keys, wd, t.dims, true), R, t.dims, &probe);
  }
  const double c_row = packs ? 10.5 : (R <= 3 ? 14.5 : 16.0);
  const double c_move = (R <= 3 ? 13.5 : 17.0) + 2.3;
  // run-sort vs chunked cost (ps) for S runs
  auto costs = [&](uint32_t k, const std::vector<uint32_t>& rest_keys, double S) {
    uint32_t key_bits = ceil_log2(t.dims[k]), rest_bits = 0;
    for (uint32_t q : rest_keys) rest_bits += ceil_log2(t.dims[q]);
    const double chunked = (double)((key_bits + rest_bits + 7) / 8) * N * c_row;
    const double rest = rest_keys.empty() ? 0.0 : (double)((rest_bits + 7) / 8) * N * c_row;
    const double run = N * c_move + S * (20.0 + 10.0 * ((key_bits + 7) / 8)) + rest;
    return std::make_pair(run, chunked);
  };
  auto worth_it = [&](uint32_t k, const std::vector<uint32_t>& rest_keys) -> bool {
    if (rs_mode == 1) return true;
    // expected runs from a probe of 256 x 1024 rows
    auto* heads = ws.get<unsigned long long>("probe_heads", 1);
    QD_CUDA(cudaMemsetAsync(heads, 0, 8, c.st));
    c.pre();
    k_probe_runs<<<kProbeBlocks, kThreads, 0, c.st>>>(src_c, R, N, k, heads);
    c.launched(kSegK);
    readback(c, ws.h_small, heads, 8);
    QD_CUDA(cudaStreamSynchronize(c.st));
    const double frac = ((double)ws.h_small[0] + kProbeBlocks) / ((double)kProbeBlocks * kProbeRows);
    const double S_est = std::min(1.0, frac) * (double)N;
    const auto rc = costs(k, rest_keys, S_est);
    return rc.first < 0.9 * rc.second;
  };
  // after run discovery: the actual run count must still pay (the probe's
  // evenly spaced blocks can over-sample a skewed head)
  auto still_worth = [&](uint32_t k, const std::vector<uint32_t>& rest_keys, uint64_t S) -> bool {
    if (rs_mode == 1) return true;
    const auto rc = costs(k, rest_keys, (double)S);
    return rc.first < rc.second;
  };
  // MSD split: sort by the first key, then by the rest within its runs, when
  // those runs come out short enough for the in-shared-memory small-run sort
  // (expected length N / dim(k1) at most half its span) and the rest of the
  // key would otherwise cost at least two more chunked passes — e.g. config
  // 4's (4,3,2,1,0): 57 key bits = 8 chunked passes become 3 (mode 4) plus
  // one small-run pass over its ~2-row runs.  QD_MSD=0 disables it.
  static const bool msd_on = [] {
    const char* e = getenv("QD_MSD");
    return !(e && atoi(e) == 0);
  }();
  if (msd_on && g.check_range && m >= 2) {
    uint32_t rest_bits = 0;
    for (size_t i = 1; i < m; ++i) rest_bits += ceil_log2(t.dims[g.keys[i]]);
    const uint32_t TLs = local3_span(ws, R, 8, kLocal2Warps);
    const double avg_run = (double)N / (double)std::max<uint32_t>(1, t.dims[g.keys[0]]);
    uint32_t first_bits = ceil_log2(t.dims[g.keys[0]]);
    if (rest_bits >= 9 && avg_run * 2.0 <= (double)TLs && first_bits > 0 &&
        (first_bits + rest_bits + 7) / 8 > (first_bits + 7) / 8 + 1) {
      auto* xc = ws.get<uint32_t>("rowsC_c", N * R);
      auto* xv = ws.get<double>("rowsC_v", N);
      Group first;
      first.prefix = g.prefix;
      first.keys = {g.keys[0]};
      segmented_sort(c, t, src_c, src_v, xc, xv, tmp_c, tmp_v, first);
      Group rest;
      rest.prefix = g.prefix;
      rest.prefix.push_back(g.keys[0]);
      rest.keys.assign(g.keys.begin() + 1, g.keys.end());
      segmented_sort(c, t, xc, xv, dst_c, dst_v, tmp_c, tmp_v, rest);
      return;
    }
  }
  // run records hold a run's start row in 32 bits (k_run_records)
  if (!disabled && !c.lat && g.check_range && g.prefix.empty() && m >= 1 && N >= min_rows &&
      N <= 0xFFFFFFFFull) {
    auto* xc = m >= 2 ? ws.get<uint32_t>("rowsC_c", N * R) : nullptr;
    auto* xv = m >= 2 ? ws.get<double>("rowsC_v", N) : nullptr;
    const uint32_t k1 = g.keys[0], km = g.keys[m - 1];
    const std::vector<uint32_t> rest1(g.keys.begin() + 1, g.keys.end());
    const std::vector<uint32_t> restm(g.keys.begin(), g.keys.end() - 1);
    if (candidate(k1) && worth_it(k1, rest1)) {
      if (try_run_sort(c, t, src_c, src_v, m == 1 ? dst_c : xc, m == 1 ? dst_v : xv, k1,
                       [&](uint64_t S) { return still_worth(k1, rest1, S); })) {
        if (m >= 2) {
          Group rest;
          rest.prefix = g.prefix;
          rest.prefix.push_back(k1);
          rest.keys.assign(g.keys.begin() + 1, g.keys.end());
          segmented_sort(c, t, xc, xv, dst_c, dst_v, tmp_c, tmp_v, rest);
        }
        return;
      }
    } else if (m >= 2 && candidate(km) && worth_it(km, restm)) {
      if (try_run_sort(c, t, src_c, src_v, xc, xv, km,
                       [&](uint64_t S) { return still_worth(km, restm, S); })) {
        Group rest;
        rest.prefix = g.prefix;
        rest.keys.assign(g.keys.begin(), g.keys.end() - 1);
        segmented_sort(c, t, xc, xv, dst_c, dst_v, tmp_c, tmp_v, rest);
        return;
      }
    }
  }
  segmented_sort(c, t, src_c, src_v, dst_c, dst_v, tmp_c, tmp_v, g);
}
}  // namespace

// Synchronise, fold profiling records, and throw the first error found.
// Returns the error flags (bit2 = a coordinate did not pack losslessly).
// copy = false: the error block's device->host copy is already enqueued
// (it is the last node of a latency-mode graph)
static unsigned check_errors(Ctx& c, bool copy = true) {
  if (copy) readback(c, c.ws.h_err, c.err, sizeof(ErrBlock));
  QD_CUDA(cudaStreamSynchronize(c.st));
  const ErrBlock e = *c.ws.h_err;
  c.resolve(e);
  if (e.flags & 2u) invalid("input tensor is not sorted under the simple ordering");
  if (e.flags & 1u) {
    Error err(QD_OUT_OF_RANGE, "coordinate in row " + std::to_string(e.rowmode >> 6) +
                                   " exceeds the dimension of mode " +
                                   std::to_string(e.rowmode & 63));
    err.row = e.rowmode >> 6;
    err.mode = (uint32_t)(e.rowmode & 63);
    throw err;
  }
  return e.flags;
}

// the call's error block and chunk counters back to their initial values
// (stream-ordered; part of a latency-mode graph when captured)
static void reset_ctx(Ctx& c, bool counters = true) {
  QD_CUDA(cudaMemcpyAsync(c.err, c.ws.h_err_init, sizeof(ErrBlock), cudaMemcpyHostToDevice, c.st));
  if (counters) QD_CUDA(cudaMemsetAsync(c.counters, 0, kCounters * 4, c.st));
}

static Ctx make_ctx(Workspace& ws, void* stream, bool reset = true) {
  QD_CUDA(cudaSetDevice(ws.device));
  Ctx c{ws, static_cast<cudaStream_t>(stream), nullptr, nullptr};
  c.err = ws.get<ErrBlock>("err", 1);
  c.counters = ws.get<uint32_t>("counters", kCounters);
  if (reset) reset_ctx(c);
  return c;
}

// k_small's plan for a call, or false: one range-checked group whose
// composite key (prefix modes, then keys; widths from the dimensions) fits
// 64 bits in at most kSmallMaxPasses 8-bit digits.
static bool small_plan(const TensorView& t, const std::vector<Group>& groups, SmallArgs* a) {
  if (groups.size() != 1 || !groups[0].check_range) return false;
  const Group& g = groups[0];
  std::vector<uint32_t> C(g.prefix);
  C.insert(C.end(), g.keys.begin(), g.keys.end());
  if (C.empty() || C.size() > (size_t)kMaxKeys) return false;
  uint32_t bits = 0;
  for (uint32_t m : C) bits += ceil_log2(t.dims[m]);
  if (bits == 0 || bits > 64) return false;
  SmallArgs x{};
  x.rank = t.rank;
  x.nnz = t.nnz;
  x.nc = (uint32_t)C.size();
  x.npre = (uint32_t)g.prefix.size();
  uint32_t sh = bits;
  for (size_t j = 0; j < C.size(); ++j) {
    sh -= ceil_log2(t.dims[C[j]]);
    x.cmode[j] = (uint8_t)C[j];
    x.csh[j] = (uint8_t)sh;
    x.cdim[j] = t.dims[C[j]];
  }
  x.P = (bits + kRadixLog - 1) / kRadixLog;
  if (x.P > (uint32_t)kSmallMaxPasses) return false;
  const uint32_t per = (bits + x.P - 1) / x.P;
  for (uint32_t q = 0; q < x.P; ++q) {
    x.dlo[q] = q * per;
    x.dmask[q] = (1u << std::min(per, bits - q * per)) - 1u;
    x.dbits[q] = std::min(per, bits - q * per);
  }
  static const int rank_mode = [] {
    const char* e = getenv("QD_SMALL_RANK");
    return e ? atoi(e) : 1;
  }();
  x.rank_mode = rank_mode;
  *a = x;
  return true;
}

static void launch_small(Ctx& c, const TensorView& t, const uint32_t* d_c_in, const double* d_v_in,
                         uint32_t* d_c_out, double* d_v_out) {
  Workspace& ws = c.ws;
  const uint64_t N = t.nnz;
  int per_sm = 0;
  QD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_small, kSmallThreads, kSmallSmem));
  uint64_t gmax = (uint64_t)std::max(1, per_sm) * ws.num_sms;
  if (const char* e = getenv("QD_SMALL_G")) gmax = std::min<uint64_t>(gmax, strtoull(e, nullptr, 10));
  const uint32_t G = (uint32_t)std::max<uint64_t>(
      1, std::min<uint64_t>({gmax, (N + 1023) / 1024, (uint64_t)kSmallThreads}));
  SmallArgs a = c.sa;
  a.in_c = d_c_in;
  a.in_v = d_v_in;
  a.out_c = d_c_out;
  a.out_v = d_v_out;
  a.ea = ws.get<ulonglong2>("small_ea", N);
  a.eb = ws.get<ulonglong2>("small_eb", N);
  a.hist = ws.get<uint32_t>("small_hist", (size_t)kBins * G);
  a.offs = ws.get<uint32_t>("small_offs", (size_t)kBins * G);
  a.total = ws.get<uint32_t>("small_total", kBins);
  a.err = c.err;
  static const bool dbg = getenv("QD_SMALL_DBG") != nullptr;
  if (dbg) {
    a.dbg = ws.get<unsigned long long>("small_dbg", 64);
    QD_CUDA(cudaMemsetAsync(a.dbg, 0, 64 * 8, c.st));
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kSmallThreads);
  cfg.dynamicSmemBytes = kSmallSmem;
  cfg.stream = c.st;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeCooperative;
  attr.val.cooperative = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  c.pre();
  QD_CUDA(cudaLaunchKernelEx(&cfg, k_small, a));
  c.launched(kSweep);
  if (dbg) {
    unsigned long long h[64];
    QD_CUDA(cudaMemcpyAsync(h, a.dbg, sizeof(h), cudaMemcpyDeviceToHost, c.st));
    QD_CUDA(cudaStreamSynchronize(c.st));
    fprintf(stderr, "k_small G=%u P=%u N=%llu (us from start):", G, a.P, (unsigned long long)N);
    for (int k = 1; k < 64; ++k)
      if (h[k]) fprintf(stderr, " %d:%.1f", k, (h[k] - h[0]) / 1e3);
    fprintf(stderr, "\n");
  }
}

// Every launch of a call (no final synchronisation): the part a latency-mode
// call captures into a CUDA graph.
static void launch_groups(Ctx& c, const TensorView& t, const uint32_t* d_c_in,
                          const double* d_v_in, uint32_t* d_c_out, double* d_v_out,
                          const std::vector<Group>& groups, bool verify_input,
                          uint64_t* d_boundaries, uint64_t* n_boundaries,
                          uint32_t boundary_mode) {
  NvtxRange r_call(c.small ? "qd call (k_small)" : "qd call");
  Workspace& ws = c.ws;
  const uint64_t N = t.nnz;
  const uint32_t R = t.rank;
  if (c.lat && !c.small) {
    // look-back scan state from tile 0 each call (graph-replayable)
    if (!ws.lb_ticket) ws.lb_ticket = ws.get<unsigned long long>("lb_ticket", 1);
    QD_CUDA(cudaMemsetAsync(ws.lb_ticket, 0, 8, c.st));
    if (ws.lb_status) QD_CUDA(cudaMemsetAsync(ws.lb_status, 0, ws.lb_cap * 8, c.st));
    ws.lb_base = 0;
    ws.lb_cleared_epoch = 0;
  }
  if (verify_input && N > 1) {
    ModeList ml{};
    ml.n = R;
    for (uint32_t i = 0; i < R; ++i) ml.m[i] = (uint8_t)i;
    const uint32_t grid = (uint32_t)std::min<uint64_t>((N + kThreads - 1) / kThreads, ws.num_sms * 8);
    c.pre();
    k_is_sorted<<<grid, kThreads, 0, c.st>>>(d_c_in, R, N, ml, c.err);
    c.launched(kOtherK);
  }
  const size_t G = groups.size();
  if (c.small) {
    launch_small(c, t, d_c_in, d_v_in, d_c_out, d_v_out);
  } else if (G == 0 || N == 0) {
    if (N && d_c_out != d_c_in) {
      QD_CUDA(cudaMemcpyAsync(d_c_out, d_c_in, N * R * 4, cudaMemcpyDeviceToDevice, c.st));
      QD_CUDA(cudaMemcpyAsync(d_v_out, d_v_in, N * 8, cudaMemcpyDeviceToDevice, c.st));
    }
  } else {
    // one group: its scratch rows are allocated by segmented_sort only if an
    // unpacked multi-pass sort needs them (packed passes use pkA/pkB)
    uint32_t* Ac = G >= 2 ? ws.get<uint32_t>("rowsA_c", N * R) : nullptr;
    double* Av = G >= 2 ? ws.get<double>("rowsA_v", N) : nullptr;
    uint32_t* Bc = G >= 2 ? ws.get<uint32_t>("rowsB_c", N * R) : nullptr;
    double* Bv = G >= 2 ? ws.get<double>("rowsB_v", N) : nullptr;
    const uint32_t* sc = d_c_in;
    const double* sv = d_v_in;
    for (size_t gi = 0; gi < G; ++gi) {
      const bool last = gi + 1 == G;
      uint32_t *dc, *tc;
      double *dv, *tv;
      // chain: in -> A -> B -> A ... -> out
      uint32_t* Xc = (gi % 2 == 0) ? Ac : Bc;
      double* Xv = (gi % 2 == 0) ? Av : Bv;
      if (last) {
        dc = d_c_out;
        dv = d_v_out;
        if (sc == Ac) { tc = Bc; tv = Bv; } else { tc = Ac; tv = Av; }
      } else {
        dc = Xc;
        dv = Xv;
        tc = d_c_out;  // not yet written by anyone
        tv = d_v_out;
      }
      c.group = (int)gi;
      std::string gname = "group prefix=";
      for (uint32_t m : groups[gi].prefix) gname += std::to_string(m);
      gname += " keys=";
      for (uint32_t m : groups[gi].keys) gname += std::to_string(m);
      NvtxRange r_group(gname);
      exec_group(c, t, sc, sv, dc, dv, tc, tv, groups[gi]);
      sc = dc;
      sv = dv;
    }
  }
  if (d_boundaries && N > 0) {
    unsigned long long* seg = nullptr;
    const uint64_t S = find_runs(c, d_c_out, R, N, {boundary_mode}, &seg);
    QD_CUDA(cudaMemcpyAsync(d_boundaries, seg, (S + 1) * 8, cudaMemcpyDeviceToDevice, c.st));
    if (n_boundaries) *n_boundaries = S + 1;
  } else if (n_boundaries) {
    *n_boundaries = 0;
  }
}

// Latency mode applies to tensors up to kLatRows rows whose groups all use
// range-checked keys (widths known without a device read), without
// boundary output; QD_LATENCY=0 disables it, QD_GRAPHS=0 keeps it eager.
constexpr uint64_t kLatRows = 1ull << 24;

static std::string graph_key(const Workspace& ws, const TensorView& t, const void* a,
                             const void* b, const void* cc, const void* d,
                             const std::vector<Group>& groups, bool verify) {
  std::string k;
  auto put = [&](uint64_t x) { k.append(reinterpret_cast<const char*>(&x), 8); };
  put(t.nnz);
  put(t.rank);
  for (uint32_t m = 0; m < t.rank; ++m) put(t.dims[m]);
  put(reinterpret_cast<uintptr_t>(a));
  put(reinterpret_cast<uintptr_t>(b));
  put(reinterpret_cast<uintptr_t>(cc));
  put(reinterpret_cast<uintptr_t>(d));
  put(verify);
  put(ws.allow_pack);
  put(ws.allow_small);
  for (const Group& g : groups) {
    put(0xFFFF0000ull | g.prefix.size());
    for (uint32_t m : g.prefix) put(m);
    put(0xEEEE0000ull | g.keys.size());
    for (uint32_t m : g.keys) put(m);
    put(g.check_range);
  }
  return k;
}

static void run_groups_once(Workspace& ws, const TensorView& t, const uint32_t* d_c_in,
                            const double* d_v_in, uint32_t* d_c_out, double* d_v_out,
                            const std::vector<Group>& groups, bool verify_input,
                            uint64_t* d_boundaries, uint64_t* n_boundaries,
                            uint32_t boundary_mode, void* stream, unsigned* flags) {
  Ctx c = make_ctx(ws, stream, false);  // reset below: eagerly, or inside the graph
  const uint64_t N = t.nnz;
  c.nnz = N;
  c.rank = t.rank;
  static const bool lat_on = [] {
    const char* e = getenv("QD_LATENCY");
    return !(e && atoi(e) == 0);
  }();
  static const bool graphs_on = [] {
    const char* e = getenv("QD_GRAPHS");
    return !(e && atoi(e) == 0);
  }();
  static const bool local_v1 = [] {
    const char* e = getenv("QD_LOCAL_V");
    return e && atoi(e) == 1;
  }();
  bool lat = lat_on && ws.allow_latency && !local_v1 && N > 0 && N <= kLatRows && !d_boundaries;
  for (const Group& g : groups) lat &= g.check_range;
  c.lat = lat;
  // one cooperative kernel for the whole call (QD_SMALL=0 disables it)
  static const bool small_on = [] {
    const char* e = getenv("QD_SMALL");
    return !(e && atoi(e) == 0);
  }();
  if (lat && small_on && ws.allow_small && N >= 2 && N <= kSmallRows && small_plan(t, groups, &c.sa)) {
    const uintptr_t ib = reinterpret_cast<uintptr_t>(d_c_in), ob = reinterpret_cast<uintptr_t>(d_c_out);
    const uintptr_t vb = reinterpret_cast<uintptr_t>(d_v_in), wb = reinterpret_cast<uintptr_t>(d_v_out);
    const uint64_t cb = N * t.rank * 4, db = N * 8;
    // the gather reads the input while writing the output: no overlap
    c.small = (ib + cb <= ob || ob + cb <= ib) && (vb + db <= wb || wb + db <= vb);
  }
  auto eager = [&] {
    launch_groups(c, t, d_c_in, d_v_in, d_c_out, d_v_out, groups, verify_input, d_boundaries,
                  n_boundaries, boundary_mode);
  };
  // k_small alone: no graph and no copy nodes around the kernel — the error
  // block lives in the pinned host block (reset by a host store; the kernel
  // only ever raises its redo flag there, through the device mapping), so the
  // call is one cooperative launch and one stream synchronisation
  static const bool small_direct = [] {
    const char* e = getenv("QD_SMALL_DIRECT");
    return !(e && atoi(e) == 0);
  }();
  if (c.small && small_direct && !verify_input && !ws.prof && !getenv("QD_SMALL_DBG")) {
    *ws.h_err = *ws.h_err_init;
    c.err = ws.h_err;
    eager();
    *flags = check_errors(c, false);
    return;
  }
  // the legacy / per-thread default streams cannot be captured
  const bool capturable = c.st != nullptr && c.st != cudaStreamLegacy && c.st != cudaStreamPerThread;
  if (lat && graphs_on && !ws.prof && capturable) {
    const std::string key = graph_key(ws, t, d_c_in, d_v_in, d_c_out, d_v_out, groups, verify_input);
    Workspace::GraphEntry& e = ws.graphs[key];
    if (e.exec && e.epoch != ws.buf_epoch) {  // a buffer it uses was reallocated
      cudaGraphExecDestroy(e.exec);
      e = Workspace::GraphEntry{};
    }
    // a graph holds the whole call: error-block reset, launches, and the
    // error block's copy back to the host (then only a stream sync remains)
    if (e.exec) {
      QD_CUDA(cudaGraphLaunch(e.exec, c.st));
      ws.launches += e.launches;
      *flags = check_errors(c, false);
      return;
    }
    if (e.seen == 0) {
      // first call of this shape: eager (sizes every workspace buffer)
      e.seen = 1;
      reset_ctx(c);
      eager();
      e.epoch = ws.buf_epoch;
      *flags = check_errors(c);
      return;
    }
    // second call: capture (no allocation happens: the buffers were sized by
    // the first call) and replay from now on
    const uint64_t epoch0 = ws.buf_epoch, l0 = ws.launches;
    QD_CUDA(cudaStreamBeginCapture(c.st, cudaStreamCaptureModeThreadLocal));
    cudaGraph_t g = nullptr;
    try {
      reset_ctx(c, !c.small);
      eager();
      QD_CUDA(cudaMemcpyAsync(ws.h_err, c.err, sizeof(ErrBlock), cudaMemcpyDeviceToHost, c.st));
    } catch (...) {
      cudaStreamEndCapture(c.st, &g);
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      throw;
    }
    QD_CUDA(cudaStreamEndCapture(c.st, &g));
    if (ws.buf_epoch != epoch0) {
      // a buffer grew during capture (should not happen): run eagerly
      cudaGraphDestroy(g);
      e = Workspace::GraphEntry{};
      reset_ctx(c);
      eager();
      *flags = check_errors(c);
      return;
    }
    QD_CUDA(cudaGraphInstantiate(&e.exec, g, 0));
    QD_CUDA(cudaGraphDestroy(g));
    e.launches = ws.launches - l0;
    e.epoch = ws.buf_epoch;
    QD_CUDA(cudaGraphLaunch(e.exec, c.st));
    *flags = check_errors(c, false);
    return;
  }
  reset_ctx(c);
  eager();
  *flags = check_errors(c);
}

void run_groups(Workspace& ws, const TensorView& t, const uint32_t* d_c_in, const double* d_v_in,
                uint32_t* d_c_out, double* d_v_out, const std::vector<Group>& groups,
                bool verify_input, uint64_t* d_boundaries, uint64_t* n_boundaries,
                uint32_t boundary_mode, void* stream) {
  unsigned flags = 0;
  run_groups_once(ws, t, d_c_in, d_v_in, d_c_out, d_v_out, groups, verify_input, d_boundaries,
                  n_boundaries, boundary_mode, stream, &flags);
  // both switches are restored on every exit; a call whose k_small attempt
  // failed keeps k_small off for its unpacked redo too (the second redo used
  // to try k_small again and ignore its flag)
  struct Restore {
    Workspace& ws;
    ~Restore() {
      ws.allow_small = true;
      ws.allow_pack = true;
    }
  } restore{ws};
  if (flags & 8u) {
    // k_small's preconditions failed (rows not ordered by the group prefix,
    // or a composite coordinate out of range): the general path
    ws.allow_small = false;
    run_groups_once(ws, t, d_c_in, d_v_in, d_c_out, d_v_out, groups, verify_input, d_boundaries,
                    n_boundaries, boundary_mode, stream, &flags);
  }
  if (flags & 4u) {
    // a coordinate of a mode the plan never range-checks does not fit its
    // packed field: redo the call with unpacked intermediates
    ws.allow_pack = false;
    run_groups_once(ws, t, d_c_in, d_v_in, d_c_out, d_v_out, groups, verify_input, d_boundaries,
                    n_boundaries, boundary_mode, stream, &flags);
  }
}

// ---- sliced host-buffer calls ------------------------------------------------
// When every group of the call sorts within runs of a prefix that contains
// one common mode m (a target that keeps the leading mode: Alg. 2 all the way,
// sort.cpp:80-134), rows on different sides of a change of m never meet, so
// the tensor can be cut at such changes and each slice transposed on its own:
// slice k's input copy, slice k-1's passes and slice k-2's output copy then
// overlap (PCIe is full duplex), and the call costs about one direction's
// copy time instead of both.  The cuts come from the host rows (a gallop and
// a bisection per cut: any row whose m differs from its predecessor's is a
// run boundary whether or not the rows are ordered).
static bool common_prefix_mode(const std::vector<Group>& groups, uint32_t* mode) {
  if (groups.empty()) return false;
  for (uint32_t m : groups[0].prefix) {
    bool all = true;
    for (const Group& g : groups)
      all &= std::find(g.prefix.begin(), g.prefix.end(), m) != g.prefix.end();
    if (all) {
      *mode = m;
      return true;
    }
  }
  return false;
}

// a row index b in [from, N] with coords[b][m] != coords[b-1][m] (N: none found)
static uint64_t next_cut(const uint32_t* c, uint32_t R, uint32_t m, uint64_t N, uint64_t from) {
  if (from >= N) return N;
  const uint32_t a = c[(from - 1) * R + m];
  if (c[from * R + m] != a) return from;
  uint64_t lo = from, hi, step = 4096;
  for (;;) {
    hi = lo + step;
    if (hi >= N) {
      hi = N - 1;
      if (c[hi * R + m] == a) return N;
      break;
    }
    if (c[hi * R + m] != a) break;
    lo = hi;
    step *= 2;
  }
  while (hi - lo > 1) {  // c[lo][m] == a, c[hi][m] != a
    const uint64_t mid = lo + (hi - lo) / 2;
    if (c[mid * R + m] == a) lo = mid; else hi = mid;
  }
  return hi;
}

constexpr uint64_t kSliceMinRows = 1ull << 25;  // calls below this stay whole
constexpr uint64_t kSliceRows = (1ull << 24) + 1;  // smallest slice (above the latency regime)

static std::vector<uint64_t> slice_cuts(const TensorView& t, const uint32_t* coords, uint32_t m) {
  const char* env = getenv("QD_SLICE_ROWS");  // 0: never slice (read per call: tests set it)
  const int64_t env_rows = env ? atoll(env) : -1;
  const uint64_t N = t.nnz;
  std::vector<uint64_t> cuts{0};
  if (env_rows == 0 || N < (env_rows > 0 ? 2 * (uint64_t)env_rows : kSliceMinRows)) {
    cuts.push_back(N);
    return cuts;
  }
  const uint64_t S = env_rows > 0 ? (uint64_t)env_rows : std::max<uint64_t>(kSliceRows, N / 24);
  while (cuts.back() < N) {
    const uint64_t want = cuts.back() + S;
    if (want >= N || N - want < S / 2) {
      cuts.push_back(N);
      break;
    }
    const uint64_t b = next_cut(coords, t.rank, m, N, want);
    cuts.push_back(N - b < S / 2 ? N : b);
  }
  return cuts;
}

// cuts.size() > 2.  Pinned host buffers (stage = false): every slice's input
// copy is enqueued up front and each output copy as soon as its slice is
// sorted.  Pageable buffers (stage = true): a feeder thread stages the input
// slices through its pinned chunk ring (tns.cu) while this thread runs each
// arrived slice's passes and stages its rows out.  Returns false when a slice
// raised an error: the caller's rows are then as they were (the slices already
// copied out are restored from the device's input copy) and the whole-tensor
// call is redone for the canonical error (the first bad row in PASS order).
static bool run_slices(Workspace& ws, const TensorView& t, uint32_t* coords, double* values,
                       uint32_t* ic, double* iv, uint32_t* oc, double* ov,
                       const std::vector<Group>& groups, const std::vector<uint64_t>& cuts,
                       cudaStream_t st, bool stage) {
  const uint32_t R = t.rank;
  const size_t ns = cuts.size() - 1;
  if (!ws.s_sl_in) {
    QD_CUDA(cudaStreamCreateWithFlags(&ws.s_sl_in, cudaStreamNonBlocking));
    QD_CUDA(cudaStreamCreateWithFlags(&ws.s_sl_out, cudaStreamNonBlocking));
  }
  while (ws.ev_slices.size() < ns) {
    cudaEvent_t e;
    QD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ws.ev_slices.push_back(e);
  }
  static const bool dbg = getenv("QD_HOST_DBG") != nullptr;
  std::vector<cudaEvent_t> tev;  // QD_HOST_DBG: t0, then per slice {arrived, sorted, out begin, out end}
  if (dbg) {
    tev.resize(1 + 4 * ns);
    for (cudaEvent_t& e : tev) QD_CUDA(cudaEventCreate(&e));
    QD_CUDA(cudaEventRecord(tev[0], ws.s_sl_in));
  }
  // slices whose input copy has been enqueued (staged: by the feeder thread)
  std::mutex fmu;
  std::condition_variable fcv;
  size_t fed = 0;
  std::exception_ptr feed_err;
  auto feed = [&](size_t k) {
    const uint64_t a = cuts[k], n = cuts[k + 1] - a;
    if (stage) {
      staged_h2d(ic + a * R, coords + a * R, n * R * 4, ws.s_sl_in);
      staged_h2d(iv + a, values + a, n * 8, ws.s_sl_in);
    } else {
      QD_CUDA(cudaMemcpyAsync(ic + a * R, coords + a * R, n * R * 4, cudaMemcpyHostToDevice, ws.s_sl_in));
      QD_CUDA(cudaMemcpyAsync(iv + a, values + a, n * 8, cudaMemcpyHostToDevice, ws.s_sl_in));
    }
    QD_CUDA(cudaEventRecord(ws.ev_slices[k], ws.s_sl_in));
    if (dbg) QD_CUDA(cudaEventRecord(tev[1 + 4 * k], ws.s_sl_in));
  };
  std::thread feeder;
  if (stage) {
    feeder = std::thread([&] {
      try {
        QD_CUDA(cudaSetDevice(ws.device));
        for (size_t k = 0; k < ns; ++k) {
          feed(k);
          {
            std::lock_guard<std::mutex> lk(fmu);
            fed = k + 1;
          }
          fcv.notify_all();
        }
      } catch (...) {
        std::lock_guard<std::mutex> lk(fmu);
        feed_err = std::current_exception();
        fcv.notify_all();
      }
    });
  } else {
    // The first sliced call of a workspace enqueues only two slices before
    // slice 0's passes: a kernel launched for the first time is loaded then
    // (lazy module loading), and a load waits for every copy in flight —
    // measured: slice 0 sorted after the LAST input slice had arrived.
    fed = ws.sliced_warm ? ns : std::min<size_t>(ns, 2);
    for (size_t k = 0; k < fed; ++k) feed(k);
  }
  // every exit joins the feeder (it always feeds all slices: the whole-tensor
  // redo after an error needs the full input on the device)
  struct Join {
    std::thread& t;
    ~Join() {
      if (t.joinable()) t.join();
    }
  } join_feeder{feeder};
  size_t done = 0;  // slices whose output copy was issued
  bool ok = true;
  ws.allow_latency = false;
  try {
    for (size_t k = 0; k < ns; ++k) {
      const uint64_t a = cuts[k], n = cuts[k + 1] - a;
      const TensorView tv{R, t.dims, n};
      if (stage) {
        std::unique_lock<std::mutex> lk(fmu);
        fcv.wait(lk, [&] { return fed > k || feed_err; });
        if (feed_err) std::rethrow_exception(feed_err);
      }
      QD_CUDA(cudaStreamWaitEvent(st, ws.ev_slices[k], 0));
      // returns with the stream synchronised: the slice's rows are sorted
      run_groups(ws, tv, ic + a * R, iv + a, oc + a * R, ov + a, groups, false, nullptr, nullptr, 0, st);
      if (dbg) {
        QD_CUDA(cudaEventRecord(tev[2 + 4 * k], st));
        QD_CUDA(cudaEventRecord(tev[3 + 4 * k], ws.s_sl_out));
      }
      done = k + 1;  // (a staged copy-out that fails part-way is restored too)
      if (!stage && fed < ns) {
        for (size_t j = fed; j < ns; ++j) feed(j);
        fed = ns;
      }
      if (stage) {
        const StageSeg segs[2] = {{coords + a * R, oc + a * R, n * R * 4}, {values + a, ov + a, n * 8}};
        staged_d2h_multi(segs, 2, ws.s_sl_out);
      } else {
        QD_CUDA(cudaMemcpyAsync(coords + a * R, oc + a * R, n * R * 4, cudaMemcpyDeviceToHost, ws.s_sl_out));
        QD_CUDA(cudaMemcpyAsync(values + a, ov + a, n * 8, cudaMemcpyDeviceToHost, ws.s_sl_out));
      }
      if (dbg) QD_CUDA(cudaEventRecord(tev[4 + 4 * k], ws.s_sl_out));
    }
  } catch (const Error& e) {
    if (feeder.joinable()) feeder.join();
    if (e.code != QD_OUT_OF_RANGE && e.code != QD_INVALID_ARGUMENT) {
      ws.allow_latency = true;
      cudaStreamSynchronize(ws.s_sl_in);
      cudaStreamSynchronize(ws.s_sl_out);
      throw;
    }
    ok = false;
  } catch (...) {
    if (feeder.joinable()) feeder.join();
    ws.allow_latency = true;
    cudaStreamSynchronize(ws.s_sl_in);
    cudaStreamSynchronize(ws.s_sl_out);
    throw;
  }
  if (feeder.joinable()) feeder.join();
  if (feed_err) {
    ws.allow_latency = true;
    std::rethrow_exception(feed_err);
  }
  if (!stage && fed < ns) {  // (an error in slice 0 of a first call: the redo needs every row)
    for (size_t j = fed; j < ns; ++j) feed(j);
    fed = ns;
  }
  ws.sliced_warm = ok;
  ws.allow_latency = true;
  QD_CUDA(cudaStreamSynchronize(ws.s_sl_in));
  QD_CUDA(cudaStreamSynchronize(ws.s_sl_out));
  if (dbg) {
    if (ok)
      for (size_t k = 0; k < ns; ++k) {
        float t[4];
        for (int j = 0; j < 4; ++j) cudaEventElapsedTime(&t[j], tev[0], tev[1 + 4 * k + j]);
        fprintf(stderr, "  slice %2zu: %10llu rows  arrived %7.1f  sorted %7.1f  out %7.1f .. %7.1f ms\n", k,
                (unsigned long long)(cuts[k + 1] - cuts[k]), t[0], t[1], t[2], t[3]);
      }
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
  }
  if (!ok && done) {
    const uint64_t n = cuts[done];
    if (stage) {
      const StageSeg segs[2] = {{coords, ic, n * R * 4}, {values, iv, n * 8}};
      staged_d2h_multi(segs, 2, st);
    } else {
      QD_CUDA(cudaMemcpyAsync(coords, ic, n * R * 4, cudaMemcpyDeviceToHost, st));
      QD_CUDA(cudaMemcpyAsync(values, iv, n * 8, cudaMemcpyDeviceToHost, st));
    }
    QD_CUDA(cudaStreamSynchronize(st));
  }
  return ok;
}

void run_groups_host(Workspace& ws, const TensorView& t, uint32_t* coords, double* values,
                     const std::vector<Group>& groups, bool verify_input, uint64_t* h_boundaries,
                     uint64_t* n_boundaries, uint32_t boundary_mode) {
  QD_CUDA(cudaSetDevice(ws.device));
  const uint64_t N = t.nnz;
  const uint32_t R = t.rank;
  uint32_t* ic = ws.get<uint32_t>("host_in_c", N * R);
  double* iv = ws.get<double>("host_in_v", N);
  uint32_t* oc = ws.get<uint32_t>("host_out_c", N * R);
  double* ov = ws.get<double>("host_out_v", N);
  uint64_t* db = h_boundaries ? ws.get<uint64_t>("host_bounds", N + 1) : nullptr;
  if (!ws.s_host) QD_CUDA(cudaStreamCreateWithFlags(&ws.s_host, cudaStreamNonBlocking));
  cudaStream_t st = ws.s_host;
  // Pageable caller buffers (a std::vector in the C++ drop-in) go through the
  // pinned chunk ring with a parallel host memcpy (tns.cu): the driver's own
  // pageable path runs at ~11 GB/s.  Pinned buffers are copied directly.
  auto pinned = [](const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return a.type == cudaMemoryTypeHost;
  };
  static const bool no_stage = getenv("QD_NO_STAGE") != nullptr;
  static const bool dbg = getenv("QD_HOST_DBG") != nullptr;
  const bool stage = N && !no_stage && !(pinned(coords) && pinned(values));
  auto now = [] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  double tm[4] = {now(), 0, 0, 0};
  ws.last_slices = 1;
  bool input_on_device = false;
  uint32_t cut_mode = 0;
  // (pageable buffers: measured no gain — the staged copies are bound by the
  // host's copy threads, 1598 vs 1548 ms on c5 (0,2,1) — so QD_SLICE_PAGEABLE=1 only)
  const char* sp_env = getenv("QD_SLICE_PAGEABLE");
  const bool slice_ok = !stage || (sp_env && atoi(sp_env) != 0);
  if (N && slice_ok && !verify_input && !h_boundaries && common_prefix_mode(groups, &cut_mode)) {
    const std::vector<uint64_t> cuts = slice_cuts(t, coords, cut_mode);
    if (cuts.size() > 2) {
      ws.last_slices = cuts.size() - 1;
      if (run_slices(ws, t, coords, values, ic, iv, oc, ov, groups, cuts, st, stage)) {
        if (dbg) fprintf(stderr, "host call: %zu slices, %.2f ms\n", cuts.size() - 1, (now() - tm[0]) * 1e3);
        if (n_boundaries) *n_boundaries = 0;
        return;
      }
      input_on_device = true;  // the whole-tensor call below raises the canonical error
    }
  }
  if (input_on_device) {
  } else if (N && stage) {
    staged_h2d(ic, coords, N * R * 4, st);
    staged_h2d(iv, values, N * 8, st);
  } else if (N) {
    QD_CUDA(cudaMemcpyAsync(ic, coords, N * R * 4, cudaMemcpyHostToDevice, st));
    QD_CUDA(cudaMemcpyAsync(iv, values, N * 8, cudaMemcpyHostToDevice, st));
  }
  if (dbg) {
    QD_CUDA(cudaStreamSynchronize(st));
    tm[1] = now();
  }
  uint64_t nb = 0;
  run_groups(ws, t, ic, iv, oc, ov, groups, verify_input, db, &nb, boundary_mode, st);
  if (dbg) tm[2] = now();
  if (N && stage) {
    const StageSeg segs[2] = {{coords, oc, N * R * 4}, {values, ov, N * 8}};
    staged_d2h_multi(segs, 2, st);
  } else if (N) {
    QD_CUDA(cudaMemcpyAsync(coords, oc, N * R * 4, cudaMemcpyDeviceToHost, st));
    QD_CUDA(cudaMemcpyAsync(values, ov, N * 8, cudaMemcpyDeviceToHost, st));
  }
  if (N) {
    if (db && nb) QD_CUDA(cudaMemcpyAsync(h_boundaries, db, nb * 8, cudaMemcpyDeviceToHost, st));
    QD_CUDA(cudaStreamSynchronize(st));
    if (dbg) {
      tm[3] = now();
      fprintf(stderr, "host call (%s): h2d %.2f ms, device %.2f ms, d2h %.2f ms\n",
              stage ? "staged" : "pinned", (tm[1] - tm[0]) * 1e3, (tm[2] - tm[1]) * 1e3,
              (tm[3] - tm[2]) * 1e3);
    }
  }
  if (n_boundaries) *n_boundaries = nb;
}

namespace {
// the worker: device work of each queued call, then its output copy
void async_worker(Workspace* ws) {
  cudaSetDevice(ws->device);
  for (;;) {
    Workspace::AsyncJob job;
    {
      std::unique_lock<std::mutex> lk(ws->mu);
      ws->cv.wait(lk, [&] { return ws->stop || !ws->jobs.empty(); });
      if (ws->jobs.empty()) return;  // stop requested, nothing left
      job = std::move(ws->jobs.front());
      ws->jobs.pop_front();
      ++ws->running;
    }
    const int sl = job.slot;
    Workspace::SlotBuf& sb = ws->slots[sl];
    const uint32_t R = (uint32_t)job.dims.size();
    const uint64_t N = job.nnz;
    try {
      TensorView t{R, job.dims.data(), N};
      QD_CUDA(cudaStreamWaitEvent(ws->s_comp, ws->ev_in[sl], 0));
      // the slot's OUTPUT buffers are rewritten only after the previous
      // job's output copy from them has drained (its input buffers were
      // refilled as soon as that job's sort had read them)
      QD_CUDA(cudaStreamWaitEvent(ws->s_comp, ws->ev_out[sl], 0));
      // its internal host syncs return once this call's rows are sorted (an
      // out_of_range is found before any host byte is written)
      run_groups(*ws, t, sb.ic, sb.iv, sb.oc, sb.ov, job.groups, job.verify_input, nullptr,
                 nullptr, 0, ws->s_comp);
      QD_CUDA(cudaEventRecord(ws->ev_comp[sl], ws->s_comp));
      QD_CUDA(cudaStreamWaitEvent(ws->s_out, ws->ev_comp[sl], 0));
      QD_CUDA(cudaMemcpyAsync(job.coords, sb.oc, N * R * 4, cudaMemcpyDeviceToHost, ws->s_out));
      QD_CUDA(cudaMemcpyAsync(job.values, sb.ov, N * 8, cudaMemcpyDeviceToHost, ws->s_out));
      QD_CUDA(cudaEventRecord(ws->ev_out[sl], ws->s_out));
      QD_CUDA(cudaEventRecord(job.done, ws->s_out));
    } catch (const Error& e) {
      std::lock_guard<std::mutex> lk(ws->mu);
      if (!ws->async_failed) {
        ws->async_failed = true;
        ws->async_code = e.code;
        ws->async_msg = e.what();
        ws->async_row = e.row;
        ws->async_mode = e.mode;
      }
      cudaEventRecord(ws->ev_comp[sl], ws->s_comp);  // slot reusable after the failed work
      cudaEventRecord(ws->ev_out[sl], ws->s_comp);
      cudaEventRecord(job.done, ws->s_comp);
    } catch (const std::exception& e) {
      std::lock_guard<std::mutex> lk(ws->mu);
      if (!ws->async_failed) {
        ws->async_failed = true;
        ws->async_code = QD_CUDA_ERROR;
        ws->async_msg = e.what();
      }
      cudaEventRecord(ws->ev_comp[sl], ws->s_comp);
      cudaEventRecord(ws->ev_out[sl], ws->s_comp);
      cudaEventRecord(job.done, ws->s_comp);
    }
    {
      std::lock_guard<std::mutex> lk(ws->mu);
      ws->issued_seq = job.seq;  // jobs run in FIFO order
      ws->slot_busy[sl] = false;
      --ws->running;
    }
    ws->cv.notify_all();
  }
}
}  // namespace

void run_groups_host_async(Workspace& ws, const TensorView& t, uint32_t* coords, double* values,
                           const std::vector<Group>& groups, bool verify_input) {
  QD_CUDA(cudaSetDevice(ws.device));
  if (!ws.s_in) {
    for (cudaStream_t* st : {&ws.s_in, &ws.s_comp, &ws.s_out})
      QD_CUDA(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
    for (int i = 0; i < Workspace::kSlots; ++i)
      for (cudaEvent_t* e : {&ws.ev_in[i], &ws.ev_comp[i], &ws.ev_out[i]}) {
        QD_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        QD_CUDA(cudaEventRecord(*e, ws.s_in));  // "done" until first use
      }
    ws.worker = std::thread(async_worker, &ws);
  }
  const uint64_t N = t.nnz;
  const uint32_t R = t.rank;
  const int sl = ws.slot;
  auto overlaps = [](const void* a, size_t na, const void* b, size_t nb) {
    const char *x = static_cast<const char*>(a), *y = static_cast<const char*>(b);
    return na && nb && x < y + nb && y < x + na;
  };
  const Workspace::HostSpan cur{coords, N * R * 4, values, N * 8};
  // every earlier call (any slot, not only the previous one: A, B, A
  // interleavings) whose output copy writes host bytes this call reads must
  // finish that copy before this call's input copy starts.  Calls whose copy
  // has completed leave the pending list.
  std::vector<cudaEvent_t> waits;
  {
    std::unique_lock<std::mutex> lk(ws.mu);
    while (!ws.pending.empty() && ws.pending.front().seq <= ws.issued_seq &&
           cudaEventQuery(ws.pending.front().done) == cudaSuccess) {
      ws.done_pool.push_back(ws.pending.front().done);
      ws.pending.pop_front();
    }
    cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error
    uint64_t need = 0;
    for (const Workspace::Pending& p : ws.pending) {
      const Workspace::HostSpan& h = p.span;
      if (overlaps(cur.c, cur.nc, h.c, h.nc) || overlaps(cur.c, cur.nc, h.v, h.nv) ||
          overlaps(cur.v, cur.nv, h.c, h.nc) || overlaps(cur.v, cur.nv, h.v, h.nv)) {
        need = std::max(need, p.seq);
        waits.push_back(p.done);
      }
    }
    // this slot's previous job must have issued its output copy (so ev_out
    // is its final record), and so must every overlapping one (so its done
    // event is recorded)
    ws.cv.wait(lk, [&] { return !ws.slot_busy[sl] && ws.issued_seq >= need; });
  }
  Workspace::SlotBuf& sb = ws.slots[sl];
  if (sb.rows < N || sb.rank < R) {
    QD_CUDA(cudaEventSynchronize(ws.ev_out[sl]));  // its buffers are no longer read
    for (void* p : {(void*)sb.ic, (void*)sb.iv, (void*)sb.oc, (void*)sb.ov})
      if (p) QD_CUDA(cudaFree(p));
    sb = Workspace::SlotBuf{};
    const size_t rows = std::max<size_t>(N + N / 8, 1024), rk = std::max<size_t>(R, 4);
    QD_CUDA(cudaMalloc(&sb.ic, rows * rk * 4));
    QD_CUDA(cudaMalloc(&sb.iv, rows * 8));
    QD_CUDA(cudaMalloc(&sb.oc, rows * rk * 4));
    QD_CUDA(cudaMalloc(&sb.ov, rows * 8));
    sb.rows = rows;
    sb.rank = rk;
  }
  // the slot's input buffers are free once its previous job's sort has read
  // them (ev_comp; the output buffers wait for their copy-out in the worker),
  // so input copies run back to back while earlier outputs drain; a chained
  // call reads host bytes the previous call's output copy writes
  QD_CUDA(cudaStreamWaitEvent(ws.s_in, ws.ev_comp[sl], 0));
  for (cudaEvent_t e : waits) QD_CUDA(cudaStreamWaitEvent(ws.s_in, e, 0));
  QD_CUDA(cudaMemcpyAsync(sb.ic, coords, N * R * 4, cudaMemcpyHostToDevice, ws.s_in));
  QD_CUDA(cudaMemcpyAsync(sb.iv, values, N * 8, cudaMemcpyHostToDevice, ws.s_in));
  QD_CUDA(cudaEventRecord(ws.ev_in[sl], ws.s_in));
  Workspace::AsyncJob job;
  job.dims.assign(t.dims, t.dims + R);
  job.nnz = N;
  job.coords = coords;
  job.values = values;
  job.groups = groups;
  job.verify_input = verify_input;
  job.slot = sl;
  job.seq = ++ws.next_seq;
  {
    std::lock_guard<std::mutex> lk(ws.mu);
    if (ws.done_pool.empty()) {
      QD_CUDA(cudaEventCreateWithFlags(&job.done, cudaEventDisableTiming));
    } else {
      job.done = ws.done_pool.back();
      ws.done_pool.pop_back();
    }
    ws.pending.push_back({cur, job.done, job.seq});
    ws.slot_busy[sl] = true;
    ws.jobs.push_back(std::move(job));
  }
  ws.cv.notify_all();
  ws.slot = (sl + 1) % Workspace::kSlots;
}

// Wait until the worker has no queued or running job (the calling thread may
// then use the workspace's buffers).
void async_drain(Workspace* ws) {
  if (!ws->worker.joinable()) return;
  std::unique_lock<std::mutex> lk(ws->mu);
  ws->cv.wait(lk, [&] { return ws->jobs.empty() && ws->running == 0; });
}

void workspace_synchronize(Workspace* ws) {
  async_drain(ws);
  QD_CUDA(cudaSetDevice(ws->device));
  for (cudaStream_t st : {ws->s_in, ws->s_comp, ws->s_out})
    if (st) QD_CUDA(cudaStreamSynchronize(st));
  std::lock_guard<std::mutex> lk(ws->mu);
  if (ws->async_failed) {
    ws->async_failed = false;
    Error e(ws->async_code, ws->async_msg);
    e.row = ws->async_row;
    e.mode = ws->async_mode;
    throw e;
  }
}

void copy_rows_device(Workspace& ws, uint32_t rank, uint64_t nnz, const uint32_t* c_in,
                      const double* v_in, uint32_t* c_out, double* v_out, uint64_t row_begin,
                      uint64_t row_end, bool whole, void* stream) {
  QD_CUDA(cudaSetDevice(ws.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto cp = [&](uint64_t a, uint64_t b) {
    if (b <= a) return;
    QD_CUDA(cudaMemcpyAsync(c_out + a * rank, c_in + a * rank, (b - a) * rank * 4,
                            cudaMemcpyDeviceToDevice, st));
    QD_CUDA(cudaMemcpyAsync(v_out + a, v_in + a, (b - a) * 8, cudaMemcpyDeviceToDevice, st));
  };
  if (whole) {
    cp(0, nnz);
  } else {
    cp(0, row_begin);
    cp(row_end, nnz);
  }
}

bool is_sorted_device(Workspace& ws, uint32_t rank, uint64_t nnz, const uint32_t* d_coords,
                      const uint32_t* order, void* stream) {
  Ctx c = make_ctx(ws, stream);
  ModeList ml{};
  ml.n = rank;
  for (uint32_t i = 0; i < rank; ++i) ml.m[i] = (uint8_t)order[i];
  if (nnz > 1) {
    const uint32_t grid = (uint32_t)std::min<uint64_t>((nnz + kThreads - 1) / kThreads, ws.num_sms * 8);
    c.pre();
    k_is_sorted<<<grid, kThreads, 0, c.st>>>(d_coords, rank, nnz, ml, c.err);
    c.launched(kOtherK);
  }
  QD_CUDA(cudaMemcpyAsync(ws.h_err, c.err, sizeof(ErrBlock), cudaMemcpyDeviceToHost, c.st));
  QD_CUDA(cudaStreamSynchronize(c.st));
  return (ws.h_err->flags & 2u) == 0;
}

uint64_t bucket_starts_device(Workspace& ws, uint32_t rank, uint64_t nnz, const uint32_t* d_coords,
                              const uint32_t* modes, uint32_t n_modes, uint64_t* d_starts,
                              void* stream) {
  Ctx c = make_ctx(ws, stream);
  if (nnz == 0) return 0;
  unsigned long long* seg = nullptr;
  const uint64_t S = find_runs(c, d_coords, rank, nnz,
                               std::vector<uint32_t>(modes, modes + n_modes), &seg);
  QD_CUDA(cudaMemcpyAsync(d_starts, seg, (S + 1) * 8, cudaMemcpyDeviceToDevice, c.st));
  QD_CUDA(cudaStreamSynchronize(c.st));
  return S + 1;
}

void csf_device(Workspace& ws, uint32_t rank, uint64_t nnz, const uint32_t* d_coords,
                const uint32_t* order, uint64_t* const* d_pos, uint32_t* const* d_crd,
                uint64_t* n_fibers, void* stream) {
  Ctx c = make_ctx(ws, stream);
  uint64_t prev_n = 0;
  for (uint32_t k = 0; k < rank; ++k) {
    unsigned long long* seg = nullptr;
    uint64_t S = 0;
    if (nnz) S = find_runs(c, d_coords, rank, nnz, std::vector<uint32_t>(order, order + k + 1), &seg);
    n_fibers[k] = S;
    // keep this level's starts for the next level's pos (find_runs reuses its buffer)
    auto* cur = c.ws.get<unsigned long long>(k & 1 ? "csf_starts1" : "csf_starts0", S + 1);
    const auto* prev = c.ws.get<unsigned long long>(k & 1 ? "csf_starts0" : "csf_starts1", 1);
    const uint32_t grid = (uint32_t)std::min<uint64_t>((S + kThreads) / kThreads, ws.num_sms * 8);
    if (S) {
      QD_CUDA(cudaMemcpyAsync(cur, seg, S * 8, cudaMemcpyDeviceToDevice, c.st));
      c.pre();
      k_fiber_crd<<<grid, kThreads, 0, c.st>>>(d_coords, rank, order[k], cur, S, d_crd[k]);
      c.launched(kOtherK);
    }
    if (k == 0) {
      const unsigned long long h[2] = {0ull, (unsigned long long)S};
      QD_CUDA(cudaMemcpyAsync(d_pos[0], h, 16, cudaMemcpyHostToDevice, c.st));
      QD_CUDA(cudaStreamSynchronize(c.st));  // h is on the stack
    } else {
      const uint32_t g2 = (uint32_t)std::min<uint64_t>((prev_n + kThreads) / kThreads, ws.num_sms * 8);
      c.pre();
      k_fiber_pos<<<g2, kThreads, 0, c.st>>>(cur, S, prev, prev_n, nnz,
                                              reinterpret_cast<unsigned long long*>(d_pos[k]));
      c.launched(kOtherK);
    }
    prev_n = S;
  }
  QD_CUDA(cudaStreamSynchronize(c.st));
}

void mode_histogram_device(Workspace& ws, uint32_t rank, uint64_t nnz, const uint32_t* d_coords,
                           uint32_t mode, uint32_t dim, uint64_t* d_hist, void* stream) {
  Ctx c = make_ctx(ws, stream);
  if (nnz) {
    const uint32_t grid = (uint32_t)std::min<uint64_t>((nnz + kThreads - 1) / kThreads, ws.num_sms * 8);
    c.pre();
    k_mode_hist<<<grid, kThreads, 0, c.st>>>(d_coords, rank, nnz, mode, dim,
                                              reinterpret_cast<unsigned long long*>(d_hist));
    c.launched(kOtherK);
  }
  QD_CUDA(cudaStreamSynchronize(c.st));
}

void partition_rows_device(Workspace& ws, uint32_t rank, uint64_t nnz, const uint32_t* d_c_in,
                           const double* d_v_in, uint32_t mode, uint32_t dim,
                           const uint32_t* d_lookup, uint32_t n_parts, uint32_t* d_c_out,
                           double* d_v_out, uint64_t* part_counts, void* stream,
                           const uint64_t* peer_c, const uint64_t* peer_v,
                           const uint64_t* peer_off) {
  if (n_parts == 0 || n_parts > (uint32_t)kBins) invalid("n_parts must be in 1..256");
  if (mode >= rank) invalid("partition mode out of range");
  Ctx c = make_ctx(ws, stream);
  for (uint32_t p = 0; p < n_parts; ++p) part_counts[p] = 0;
  if (nnz == 0) return;
  const uint32_t T = sweep_tile_rows(ws, rank);
  const uint32_t CH = T * chunk_tiles(ws, nnz, T);
  const uint64_t nc = (nnz + CH - 1) / CH;
  ChunkDesc* chunks = ws.get<ChunkDesc>("chunks", nc);
  c.pre();
  k_uniform_chunks<<<(uint32_t)((nc + kThreads - 1) / kThreads), kThreads, 0, c.st>>>(
      nnz, CH, (uint32_t)nc, chunks);
  c.launched(kSegK);
  DigitSpec dig{};
  dig.lookup = d_lookup;
  dig.lookup_mode = mode;
  dig.lookup_dim = dim;
  KeySpec key{};
  unsigned long long* offs = nullptr;
  // peer destinations: a kBins-entry table on the device (unused bins zero)
  PeerDest* d_peers = nullptr;
  bool aligned = true;
  if (peer_c) {
    std::vector<PeerDest> hp(kBins, PeerDest{0, 0, 0});
    for (uint32_t p = 0; p < n_parts; ++p) {
      hp[p] = PeerDest{peer_c[p], peer_v[p], peer_off[p]};
      aligned &= ((peer_c[p] + peer_off[p] * 4ull * rank) & 15ull) == 0;
    }
    d_peers = ws.get<PeerDest>("peer_table", kBins);
    QD_CUDA(cudaMemcpyAsync(d_peers, hp.data(), kBins * sizeof(PeerDest), cudaMemcpyHostToDevice,
                            c.st));
    QD_CUDA(cudaStreamSynchronize(c.st));  // hp is pageable and goes out of scope
  }
  run_pass(c, rank, nnz, T, Rows{d_c_in, d_v_in, 0}, RowsOut{d_c_out, d_v_out, 0}, chunks, nc,
           nullptr, dig, key, false, &offs, nullptr, 0, 0, nullptr, nullptr, 0, 0, nullptr, nullptr,
           d_peers, aligned);
  // part p starts at offs[p * nc] (bin-major flat layout of one run)
  const uint32_t nb = std::min<uint32_t>(n_parts + 1, kBins);
  auto* starts = ws.get<unsigned long long>("part_starts", kBins + 1);
  c.pre();
  k_gather_stride<<<1, kThreads, 0, c.st>>>(offs, nc, nb, starts);
  c.launched(kOtherK);
  QD_CUDA(cudaMemcpyAsync(ws.h_small, starts, nb * 8, cudaMemcpyDeviceToHost, c.st));
  QD_CUDA(cudaStreamSynchronize(c.st));
  for (uint32_t p = 0; p < n_parts; ++p) {
    const uint64_t b = ws.h_small[p];
    const uint64_t e = p + 1 < nb ? ws.h_small[p + 1] : nnz;
    part_counts[p] = e - b;
  }
  check_errors(c);
}

}  // namespace qb200
