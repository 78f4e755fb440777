// GPU .tns reader: the reference's read_tns (io.cpp:42-126) as device passes
// over the file's bytes ("on-disk format and
// canonicalisation").  Canonicalisation itself (io.cpp:36-38, sort_rows_by)
// reuses the transpose engine (capi.cpp, qd_read_tns).
//
// Passes (text resident in HBM, padded to 16 bytes):
//   k_nl_count      per 4 KB tile: newline count (16-byte loads)
//   k_scan_excl     one-CTA exclusive scan of the tile counts
//   k_nl_positions  per tile: line starts at the scanned offsets
//   k_line_classify thread per line: field count, data/blank/comment
//                   (io.cpp:56-57), per-CTA data-line count, first data line
//   k_scan_excl     row offsets of the CTAs
//   k_line_parse    thread per line: std::from_chars of every field
//                   (tns_parse.cuh), 0-based AoS coords + f64 values at the
//                   line's row, per-mode maxima (dims, io.cpp:117-124),
//                   first failing line (atomicMin)
//   k_line_error    one thread re-parses the first failing line and reports
//                   what failed, so the host can build the reference's exact
//                   ParseError text (io.cpp:16-18)
// All byte work is HBM-bound: ~1 read of the text per pass, plus the row write.
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <sys/mman.h>

#include <algorithm>
#include <cstring>
#include <condition_variable>
#include <map>
#include <mutex>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "internal.hpp"
#include "tns_format.cuh"
#include "tns_parse.cuh"

namespace qb200 {

namespace {

constexpr int kTileThreads = 256;
constexpr uint64_t kTileBytes = kTileThreads * 16;
constexpr int kLineThreads = 256;

#define TNS_CUDA(x)                                                                  \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess)                                                           \
      throw Error(QD_CUDA_ERROR, std::string("CUDA error in .tns reader: ") +       \
                                     cudaGetErrorString(e_));                        \
  } while (0)

__device__ __forceinline__ int count_nl16(uint4 v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  int c = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    // bytes equal to '\n' (0x0A): zero-byte test on w ^ 0x0A0A0A0A
    const uint32_t x = w[k] ^ 0x0A0A0A0Au;
    c += __popc(((x - 0x01010101u) & ~x & 0x80808080u));
  }
  return c;
}

__global__ void k_nl_count(const uint4* __restrict__ text, uint64_t n16,
                           uint32_t* __restrict__ tile_counts) {
  const uint64_t i = (uint64_t)blockIdx.x * kTileThreads + threadIdx.x;
  int c = 0;
  if (i < n16) c = count_nl16(text[i]);
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ int ws[kTileThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int k = 0; k < kTileThreads / 32; ++k) t += ws[k];
    tile_counts[blockIdx.x] = (uint32_t)t;
  }
}

// Exclusive scan of n u32 counts into u64 offsets (out[n] = total); one CTA.
__global__ void k_scan_excl(const uint32_t* __restrict__ in, uint64_t n,
                            uint64_t* __restrict__ out) {
  __shared__ uint64_t wsum[32];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t base = 0; base < n; base += blockDim.x) {
    const uint64_t i = base + threadIdx.x;
    const uint64_t v = i < n ? in[i] : 0;
    uint64_t s = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t t = __shfl_up_sync(0xffffffffu, s, d);
      if (lane >= d) s += t;
    }
    if (lane == 31) wsum[warp] = s;
    __syncthreads();
    if (warp == 0) {
      const int nw = blockDim.x >> 5;
      uint64_t x = lane < nw ? wsum[lane] : 0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t t = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += t;
      }
      if (lane < nw) wsum[lane] = x;
    }
    __syncthreads();
    const uint64_t before = carry + (warp ? wsum[warp - 1] : 0) + s - v;
    if (i < n) out[i] = before;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = before + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
}

// line_start[0] = 0; the line after the j-th newline starts at its byte + 1.
__global__ void k_nl_positions(const uint4* __restrict__ text, uint64_t n16,
                               const uint64_t* __restrict__ tile_off,
                               uint64_t* __restrict__ line_start) {
  const uint64_t i = (uint64_t)blockIdx.x * kTileThreads + threadIdx.x;
  uint4 v = make_uint4(0, 0, 0, 0);
  if (i < n16) v = text[i];
  const int c = count_nl16(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int s = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, s, d);
    if (lane >= d) s += t;
  }
  __shared__ int ws[kTileThreads / 32];
  if (lane == 31) ws[warp] = s;
  __syncthreads();
  int before = s - c;
  for (int k = 0; k < warp; ++k) before += ws[k];
  uint64_t out = tile_off[blockIdx.x] + before + 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) line_start[0] = 0;
  if (c) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      if (((w[b >> 2] >> ((b & 3) * 8)) & 0xFF) == '\n') line_start[out++] = i * 16 + b + 1;
    }
  }
}

// Bytes [begin, end) of line k (the newline excluded).
__device__ __forceinline__ void line_span(const uint64_t* line_start, uint64_t n_nl, uint64_t n,
                                          uint64_t k, uint64_t* b, uint64_t* e) {
  *b = line_start[k];
  *e = k < n_nl ? line_start[k + 1] - 1 : n;
}

// Field count of a line (split_fields, io.cpp:24-34); 0 for blank and
// comment lines (io.cpp:57).
__device__ uint32_t line_fields(const char* t, uint64_t b, uint64_t e) {
  uint32_t nf = 0;
  bool in = false, comment = false;
  for (uint64_t p = b; p < e; ++p) {
    const bool sp = tns::is_space(t[p]);
    if (!sp && !in) {
      if (nf == 0 && t[p] == '#') comment = true;
      ++nf;
    }
    in = !sp;
  }
  return comment ? 0 : nf;
}

__global__ void k_line_classify(const char* __restrict__ text, uint64_t n,
                                const uint64_t* __restrict__ line_start, uint64_t n_nl,
                                uint64_t n_lines, uint32_t* __restrict__ nf_out,
                                uint32_t* __restrict__ cta_rows,
                                unsigned long long* __restrict__ first_data) {
  const uint64_t k = (uint64_t)blockIdx.x * kLineThreads + threadIdx.x;
  uint32_t nf = 0;
  if (k < n_lines) {
    uint64_t b, e;
    line_span(line_start, n_nl, n, k, &b, &e);
    nf = line_fields(text, b, e);
    nf_out[k] = nf;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, nf != 0);  // one atomic per warp
  if (bal && (threadIdx.x & 31) == __ffs(bal) - 1) atomicMin(first_data, (unsigned long long)k);
  const int c = __syncthreads_count(nf != 0);
  if (threadIdx.x == 0) cta_rows[blockIdx.x] = (uint32_t)c;
}

struct ParseArgs {
  const char* text;
  uint64_t n;
  const uint64_t* line_start;
  uint64_t n_nl, n_lines;
  const uint32_t* nf;
  const uint64_t* cta_row_off;
  uint32_t fields;           // rank + 1 (from the first data line)
  const uint32_t* declared;  // device, or null
  uint32_t* coords;
  double* values;
  uint32_t* max_index;       // [rank]
  unsigned long long* err_line;
  // lines whose value needs the big-integer slow path (k_line_slow)
  unsigned long long* slow_count;
  uint64_t* slow_line;  // pairs {line, row}
  uint64_t slow_cap;
};

// Error kinds (the reference's ParseError texts, io.cpp:60-113).
enum : uint32_t {
  kErrNone = 0,
  kErrFieldCount = 3,
  kErrIndex = 4,
  kErrZeroIndex = 5,
  kErrExceeds = 6,
  kErrValue = 7,
};

struct LineError {
  uint32_t kind, field, got;
  uint64_t tok_begin, tok_len;
};

// Parses line [b, e) with nf fields; writes the row when row_out is set.
// Returns the first failure in the reference's check order.
template <bool kSlow>
__device__ LineError parse_line(const ParseArgs& a, uint64_t b, uint64_t e, uint32_t nf,
                                uint64_t row, bool write, uint32_t* smax, uint64_t line) {
  LineError err{kErrNone, 0, nf, 0, 0};
  if (nf != a.fields) {
    err.kind = kErrFieldCount;
    return err;
  }
  const uint32_t rank = a.fields - 1;
  uint64_t p = b;
  for (uint32_t m = 0; m < a.fields; ++m) {
    while (p < e && tns::is_space(a.text[p])) ++p;
    const uint64_t tb = p;
    while (p < e && !tns::is_space(a.text[p])) ++p;
    const uint32_t tl = (uint32_t)(p - tb);
    if (m < rank) {
      uint32_t idx = 0;
      if (!tns::parse_u32(a.text + tb, tl, &idx)) return LineError{kErrIndex, m, nf, tb, tl};
      if (idx < 1) return LineError{kErrZeroIndex, m, nf, tb, tl};
      if (a.declared && idx > a.declared[m]) return LineError{kErrExceeds, m, nf, tb, tl};
      if (write) {
        a.coords[row * rank + m] = idx - 1;
        if (smax) atomicMax(&smax[m], idx);
      }
    } else {
      double v = 0;
      const int r = tns::parse_f64_impl<kSlow>(a.text + tb, tl, &v);
      if (r == 2) {  // rare: finished by k_line_slow (or a full slow re-run)
        const unsigned long long i = atomicAdd(a.slow_count, 1ull);
        if (i < a.slow_cap) {
          a.slow_line[2 * i] = line;
          a.slow_line[2 * i + 1] = row;
        }
        return err;
      }
      if (!r) return LineError{kErrValue, m, nf, tb, tl};
      if (write) a.values[row] = v;
    }
  }
  return err;
}

template <bool kSlow>
__global__ void __launch_bounds__(kLineThreads) k_line_parse(ParseArgs a) {
  __shared__ uint32_t smax[QD_MAX_RANK];
  __shared__ int wcount[kLineThreads / 32];
  const uint32_t rank = a.fields - 1;
  for (uint32_t m = threadIdx.x; m < rank; m += blockDim.x) smax[m] = 0;
  const uint64_t k = (uint64_t)blockIdx.x * kLineThreads + threadIdx.x;
  const uint32_t nf = k < a.n_lines ? a.nf[k] : 0;
  // row = the CTA's offset + data lines before this one in the CTA
  const unsigned bal = __ballot_sync(0xffffffffu, nf != 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wcount[warp] = __popc(bal);
  __syncthreads();
  uint64_t row = a.cta_row_off[blockIdx.x] + __popc(bal & ((1u << lane) - 1));
  for (int w = 0; w < warp; ++w) row += wcount[w];
  if (nf) {
    uint64_t b, e;
    line_span(a.line_start, a.n_nl, a.n, k, &b, &e);
    const LineError err = parse_line<kSlow>(a, b, e, nf, row, true, smax, k);
    if (err.kind != kErrNone) atomicMin(a.err_line, (unsigned long long)k);
  }
  __syncthreads();
  for (uint32_t m = threadIdx.x; m < rank; m += blockDim.x)
    if (smax[m]) atomicMax(&a.max_index[m], smax[m]);
}

__global__ void k_line_error(ParseArgs a, uint64_t k, LineError* out) {
  uint64_t b, e;
  line_span(a.line_start, a.n_nl, a.n, k, &b, &e);
  *out = parse_line<true>(a, b, e, a.nf[k], 0, false, nullptr, k);
}

// The listed lines' values through the exact slow path (their indices were
// written by k_line_parse).
__global__ void k_line_slow(ParseArgs a, uint64_t count) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint64_t k = a.slow_line[2 * i], row = a.slow_line[2 * i + 1];
  uint64_t b, e;
  line_span(a.line_start, a.n_nl, a.n, k, &b, &e);
  // the value is the last field: skip trailing blanks, then back to its start
  while (e > b && tns::is_space(a.text[e - 1])) --e;
  uint64_t tb = e;
  while (tb > b && !tns::is_space(a.text[tb - 1])) --tb;
  double v = 0;
  if (tns::parse_f64_impl<true>(a.text + tb, (uint32_t)(e - tb), &v) == 1) a.values[row] = v;
  else atomicMin(a.err_line, (unsigned long long)k);
}


// ---- host <-> device copies of the large buffers ---------------------------
// Pageable cudaMemcpy runs at ~11 GB/s here (driver staging, one thread).
// Instead: a ring of pinned chunks; host threads fill (or drain) a chunk with
// a parallel memcpy while the copy engine moves the previous one.
// staging chunk (QD_STAGE_MB overrides; experiments)
uint64_t stage_chunk() {
  static const uint64_t c = [] {
    if (const char* e = getenv("QD_STAGE_MB")) return (uint64_t)std::max(1, atoi(e)) << 20;
    return (uint64_t)16 << 20;  // 16 MB x 8 slots: 30M-row pageable call 28.4 -> 27.6 ms
  }();
  return c;
}
constexpr int kMaxStageSlots = 16;
// slots of the ring (QD_STAGE_SLOTS overrides; experiments)
int stage_slots() {
  static const int n = [] {
    if (const char* e = getenv("QD_STAGE_SLOTS")) return std::max(2, std::min(kMaxStageSlots, atoi(e)));
    return 8;
  }();
  return n;
}
constexpr int kMaxCopyThreads = 16;

int copy_threads() {
  static const int n = [] {
    if (const char* e = getenv("QD_COPY_THREADS")) return std::max(1, std::min(kMaxCopyThreads, atoi(e)));
    // 8 (streaming-store) threads saturate this host's DRAM next to the DMA
    // engine; more only contend (profiles/microbench/host_staging.*)
    const unsigned hc = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min<unsigned>(8, hc ? hc : 4));
  }();
  return n;
}

struct StageRing {
  char* buf[kMaxStageSlots] = {};
  cudaEvent_t ev[kMaxStageSlots] = {};
  int device = -1;
  ~StageRing() {
    for (int i = 0; i < kMaxStageSlots; ++i) {
      if (buf[i]) cudaFreeHost(buf[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
  }
  void init() {
    int dev = 0;
    TNS_CUDA(cudaGetDevice(&dev));
    if (device == dev) return;
    for (int i = 0; i < stage_slots(); ++i) {
      if (buf[i]) cudaFreeHost(buf[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
      TNS_CUDA(cudaMallocHost(&buf[i], stage_chunk()));
      TNS_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    device = dev;
  }
};

// Host copy with non-temporal (streaming) stores: a regular store first reads
// the destination line (read-for-ownership), so a staged copy would move 4
// bytes of host DRAM traffic per byte next to the DMA engine's own; with
// streaming stores it moves 3 (profiles/microbench/host_staging.*: the
// staged pageable path is host-memory-bandwidth bound).  QD_COPY_NT=0: memcpy.
void copy_nt(char* dst, const char* src, uint64_t n) {
  static const bool nt = [] {
    const char* e = getenv("QD_COPY_NT");
    return !(e && atoi(e) == 0);
  }();
  if (!nt || n < 4096) {
    std::memcpy(dst, src, n);
    return;
  }
  const uint64_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  const uint64_t body = n & ~uint64_t(63);
  for (uint64_t i = 0; i < body; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
  }
  _mm_sfence();
  std::memcpy(dst + body, src + body, n - body);
}

// A persistent pool of host copy threads (spawning threads per 32 MB chunk
// cost a sizeable fraction of the chunk's copy time).  A job is split into
// page-aligned parts; the caller copies part 0 and waits for the rest.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool p(copy_threads());
    return p;
  }
  void run(char* dst, const char* src, uint64_t n) {
    const int nt = (int)workers_.size() + 1;
    const uint64_t part = (n / nt + 4095) & ~4095ull;
    std::unique_lock<std::mutex> lk(mu_);
    dst_ = dst;
    src_ = src;
    n_ = n;
    part_ = part;
    pending_ = nt - 1;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    copy_nt(dst, src, std::min(n, part));
    lk.lock();
    done_cv_.wait(lk, [&] { return pending_ == 0; });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  explicit CopyPool(int nt) {
    for (int t = 1; t < nt; ++t) workers_.emplace_back([this, t] { loop(t); });
  }
  void loop(int t) {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      char* dst = dst_;
      const char* src = src_;
      const uint64_t a = std::min(n_, t * part_), b = std::min(n_, (t + 1) * part_);
      lk.unlock();
      if (b > a) copy_nt(dst + a, src + a, b - a);
      lk.lock();
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  uint64_t gen_ = 0;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  uint64_t n_ = 0, part_ = 0;
  int pending_ = 0;
};

std::mutex g_copy_mu;  // one job at a time in the shared pool

void parallel_memcpy(char* dst, const char* src, uint64_t n) {
  if (n < (4ull << 20) || copy_threads() == 1) {
    std::memcpy(dst, src, n);
    return;
  }
  std::lock_guard<std::mutex> lk(g_copy_mu);
  CopyPool::get().run(dst, src, n);
}

StageRing& stage_ring() {
  static thread_local StageRing r;
  r.init();
  return r;
}

}  // namespace

// Device buffers of the text paths come from a PRIVATE stream-ordered pool
// per device (a 348 MB text buffer costs ~ms through cudaMalloc).  The pool
// keeps up to kTnsPoolKeep bytes cached across calls and returns the rest to
// the device at the next synchronisation, so a large read/write does not pin
// memory the engine's Workspace (cudaMalloc) or other cudaMallocAsync users
// need later; the device's default pool is left untouched.
constexpr uint64_t kTnsPoolKeep = 2ull << 30;
void* tns_dev_alloc(uint64_t bytes, void* stream) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  int dev = 0;
  TNS_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = pools.find(dev);
    if (it == pools.end()) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      TNS_CUDA(cudaMemPoolCreate(&pool, &props));
      uint64_t keep = kTnsPoolKeep;
      TNS_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
      it = pools.emplace(dev, pool).first;
    }
    pool = it->second;
  }
  void* p = nullptr;
  TNS_CUDA(cudaMallocFromPoolAsync(&p, bytes, pool, static_cast<cudaStream_t>(stream)));
  return p;
}
void tns_dev_free(void* p, void* stream) {
  if (p) cudaFreeAsync(p, static_cast<cudaStream_t>(stream));
}

void staged_h2d(void* d_dst, const void* h_src, uint64_t n, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  StageRing& r = stage_ring();
  const uint64_t kStageChunk = stage_chunk();
  for (uint64_t off = 0, i = 0; off < n; off += kStageChunk, ++i) {
    const int k = (int)(i % stage_slots());
    const uint64_t len = std::min(kStageChunk, n - off);
    TNS_CUDA(cudaEventSynchronize(r.ev[k]));  // the slot's previous copy is done
    parallel_memcpy(r.buf[k], static_cast<const char*>(h_src) + off, len);
    TNS_CUDA(cudaMemcpyAsync(static_cast<char*>(d_dst) + off, r.buf[k], len,
                             cudaMemcpyHostToDevice, st));
    TNS_CUDA(cudaEventRecord(r.ev[k], st));
  }
}

// Device -> host through the pinned ring for several (host, device, bytes)
// segments as ONE chunk pipeline (no drain between segments): each chunk's
// DMA runs while earlier chunks are copied out by the host threads.
void staged_d2h_multi(const StageSeg* segs, int nseg, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  StageRing& r = stage_ring();
  const uint64_t kStageChunk = stage_chunk();
  struct Piece {
    char* h;
    const char* d;
    uint64_t len;
  };
  std::vector<Piece> ps;
  for (int s = 0; s < nseg; ++s)
    for (uint64_t off = 0; off < segs[s].n; off += kStageChunk)
      ps.push_back({static_cast<char*>(segs[s].h) + off, static_cast<const char*>(segs[s].d) + off,
                    std::min(kStageChunk, segs[s].n - off)});
  const int kStageSlots = stage_slots();
  auto issue = [&](size_t i) {
    const int k = (int)(i % kStageSlots);
    TNS_CUDA(cudaMemcpyAsync(r.buf[k], ps[i].d, ps[i].len, cudaMemcpyDeviceToHost, st));
    TNS_CUDA(cudaEventRecord(r.ev[k], st));
  };
  for (size_t i = 0; i < std::min<size_t>(ps.size(), kStageSlots); ++i) issue(i);
  for (size_t i = 0; i < ps.size(); ++i) {
    const int k = (int)(i % kStageSlots);
    TNS_CUDA(cudaEventSynchronize(r.ev[k]));
    parallel_memcpy(ps[i].h, r.buf[k], ps[i].len);
    if (i + kStageSlots < ps.size()) issue(i + kStageSlots);
  }
}

void staged_d2h(void* h_dst, const void* d_src, uint64_t n, void* stream) {
  const StageSeg seg{h_dst, d_src, n};
  staged_d2h_multi(&seg, 1, stream);
}

namespace {

struct DevBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  ~DevBuf() {
    if (p) tns_dev_free(p, st);
  }
  template <class T>
  T* alloc(uint64_t bytes, cudaStream_t stream) {
    st = stream;
    p = tns_dev_alloc(std::max<uint64_t>(bytes, 16), stream);
    return static_cast<T*>(p);
  }
};

[[noreturn]] void parse_error(qd_tns_error* err, uint64_t line, uint32_t kind, uint32_t field,
                              uint32_t got, uint32_t expected, uint64_t tb, uint64_t tl,
                              const std::string& what) {
  if (err) {
    err->line = line;
    err->kind = kind;
    err->field = field;
    err->got = got;
    err->expected = expected;
    err->token_offset = tb;
    err->token_len = tl;
  }
  Error e(QD_PARSE_ERROR, "line " + std::to_string(line) + ": " + what);
  e.row = line;
  e.mode = field;
  throw e;
}

}  // namespace

void parse_tns_device(const char* h_text, uint64_t n, const uint32_t* declared,
                      uint32_t declared_rank, bool has_declared, TnsParsed* out,
                      qd_tns_error* err, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const auto t0 = std::chrono::steady_clock::now();
  out->rank = 0;
  out->nnz = 0;
  out->dims.clear();
  out->d_coords = nullptr;
  out->d_values = nullptr;
  if (err) *err = qd_tns_error{};
  if (n && !h_text) invalid("text is null");
  if (has_declared && declared_rank && !declared) invalid("declared dims are null");

  // text in HBM, zero-padded to whole 16-byte words (and one more word)
  const uint64_t n16 = (n + 15) / 16 + 1;
  DevBuf b_text;
  char* d_text = b_text.alloc<char>(n16 * 16, st);
  const uint64_t pad_from = n & ~15ull;  // zero the partial last word and the extra one
  TNS_CUDA(cudaMemsetAsync(d_text + pad_from, 0, n16 * 16 - pad_from, st));
  if (n) staged_h2d(d_text, h_text, n, st);
  static const bool timing = getenv("QD_TNS_TIMING") != nullptr;
  if (timing) {
    TNS_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "qd_read_tns   (text H2D + alloc %8.2f ms)\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                .count());
  }

  // newlines -> line starts
  const uint64_t n_tiles = (n16 + kTileThreads - 1) / kTileThreads;
  DevBuf b_tc, b_to;
  uint32_t* d_tc = b_tc.alloc<uint32_t>(n_tiles * 4, st);
  uint64_t* d_to = b_to.alloc<uint64_t>((n_tiles + 1) * 8, st);
  k_nl_count<<<(unsigned)n_tiles, kTileThreads, 0, st>>>((const uint4*)d_text, n16, d_tc);
  k_scan_excl<<<1, 1024, 0, st>>>(d_tc, n_tiles, d_to);
  uint64_t n_nl = 0;
  TNS_CUDA(cudaMemcpyAsync(&n_nl, d_to + n_tiles, 8, cudaMemcpyDeviceToHost, st));
  TNS_CUDA(cudaStreamSynchronize(st));
  // getline semantics: a final line without '\n' still counts
  const bool tail = n > 0 && h_text[n - 1] != '\n';
  const uint64_t n_lines = n_nl + (tail ? 1 : 0);
  DevBuf b_ls;
  uint64_t* d_ls = b_ls.alloc<uint64_t>((n_nl + 2) * 8, st);
  k_nl_positions<<<(unsigned)n_tiles, kTileThreads, 0, st>>>((const uint4*)d_text, n16, d_to,
                                                            d_ls);

  // classify lines
  const uint64_t n_ctas = std::max<uint64_t>(1, (n_lines + kLineThreads - 1) / kLineThreads);
  DevBuf b_nf, b_cr, b_co, b_small;
  uint32_t* d_nf = b_nf.alloc<uint32_t>(n_lines * 4, st);
  uint32_t* d_cr = b_cr.alloc<uint32_t>(n_ctas * 4, st);
  uint64_t* d_co = b_co.alloc<uint64_t>((n_ctas + 1) * 8, st);
  // small: [0] first data line, [1] error line, [2..] LineError, max_index
  unsigned long long* d_small = b_small.alloc<unsigned long long>(64 + QD_MAX_RANK * 4 + 64, st);
  TNS_CUDA(cudaMemsetAsync(d_small, 0xFF, 16, st));
  uint32_t* d_max = reinterpret_cast<uint32_t*>(d_small + 8);
  TNS_CUDA(cudaMemsetAsync(d_max, 0, QD_MAX_RANK * 4, st));
  LineError* d_lerr = reinterpret_cast<LineError*>(d_small + 2);
  if (n_lines) {
    k_line_classify<<<(unsigned)n_ctas, kLineThreads, 0, st>>>(d_text, n, d_ls, n_nl, n_lines,
                                                               d_nf, d_cr, d_small);
    k_scan_excl<<<1, 1024, 0, st>>>(d_cr, n_ctas, d_co);
  } else {
    TNS_CUDA(cudaMemsetAsync(d_co, 0, (n_ctas + 1) * 8, st));
  }
  uint64_t h2[2] = {0, 0};  // first data line, data rows
  TNS_CUDA(cudaMemcpyAsync(&h2[0], d_small, 8, cudaMemcpyDeviceToHost, st));
  TNS_CUDA(cudaMemcpyAsync(&h2[1], d_co + n_ctas, 8, cudaMemcpyDeviceToHost, st));
  TNS_CUDA(cudaStreamSynchronize(st));
  const uint64_t rows = h2[1];

  if (rows == 0) {  // io.cpp:115-119, then check_valid (coo.cpp:8-16)
    if (!has_declared)
      parse_error(err, n_lines, 8, 0, 0, 0, 0, 0,
                  "empty file: rank is unknowable without declared dimensions");
    if (declared_rank == 0) invalid("tensor rank must be positive");
    for (uint32_t m = 0; m < declared_rank; ++m)
      if (declared[m] == 0) invalid("dimension of mode " + std::to_string(m) + " must be positive");
    out->rank = declared_rank;
    out->dims.assign(declared, declared + declared_rank);
    return;
  }
  const uint64_t first = h2[0];
  uint32_t nf_first = 0;
  TNS_CUDA(cudaMemcpy(&nf_first, d_nf + first, 4, cudaMemcpyDeviceToHost));
  if (nf_first < 2)  // io.cpp:60-64
    parse_error(err, first + 1, 1, 0, nf_first, 0, 0, 0,
                "expected at least one index and a value, got " + std::to_string(nf_first) +
                    " fields");
  if (has_declared && declared_rank != nf_first - 1)  // io.cpp:65-72
    parse_error(err, first + 1, 2, 0, nf_first, declared_rank, 0, 0,
                "file has rank " + std::to_string(nf_first - 1) + " but " +
                    std::to_string(declared_rank) + " dimensions were declared");
  const uint32_t rank = nf_first - 1;
  if (rank > QD_MAX_RANK) invalid("tensor rank must be in 1..64");

  DevBuf b_decl;
  uint32_t* d_decl = nullptr;
  if (has_declared) {
    d_decl = b_decl.alloc<uint32_t>(rank * 4, st);
    TNS_CUDA(cudaMemcpyAsync(d_decl, declared, rank * 4, cudaMemcpyHostToDevice, st));
  }
  uint32_t* d_coords = nullptr;
  double* d_values = nullptr;
  d_coords = static_cast<uint32_t*>(tns_dev_alloc(rows * rank * 4, st));
  try {
    d_values = static_cast<double*>(tns_dev_alloc(rows * 8, st));
  } catch (...) {
    tns_dev_free(d_coords, st);
    throw;
  }
  out->d_coords = d_coords;
  out->d_values = d_values;
  // slow-path list: {line, row} pairs; QD_TNS_SLOW_CAP overrides the capacity
  uint64_t slow_cap = std::min<uint64_t>(rows, 1ull << 20);
  if (const char* ev = getenv("QD_TNS_SLOW_CAP")) slow_cap = strtoull(ev, nullptr, 10);
  DevBuf b_slow;
  uint64_t* d_slow = b_slow.alloc<uint64_t>(std::max<uint64_t>(slow_cap, 1) * 16, st);
  unsigned long long* d_slow_count = d_small + 7;
  TNS_CUDA(cudaMemsetAsync(d_slow_count, 0, 8, st));
  ParseArgs a{d_text, n, d_ls, n_nl, n_lines, d_nf, d_co, nf_first, d_decl,
              d_coords, d_values, d_max, d_small + 1, d_slow_count, d_slow, slow_cap};
  k_line_parse<false><<<(unsigned)n_ctas, kLineThreads, 0, st>>>(a);
  uint64_t slow = 0;
  TNS_CUDA(cudaMemcpyAsync(&slow, d_slow_count, 8, cudaMemcpyDeviceToHost, st));
  TNS_CUDA(cudaStreamSynchronize(st));
  TNS_CUDA(cudaGetLastError());
  if (slow > slow_cap) {  // list overflow: every line again with the slow path inline
    a.slow_cap = 0;
    k_line_parse<true><<<(unsigned)n_ctas, kLineThreads, 0, st>>>(a);
  } else if (slow) {
    k_line_slow<<<(unsigned)((slow + 127) / 128), 128, 0, st>>>(a, slow);
  }
  uint64_t eline = ~0ull;
  TNS_CUDA(cudaMemcpyAsync(&eline, d_small + 1, 8, cudaMemcpyDeviceToHost, st));
  TNS_CUDA(cudaStreamSynchronize(st));
  TNS_CUDA(cudaGetLastError());
  if (eline != ~0ull) {
    k_line_error<<<1, 1, 0, st>>>(a, eline, d_lerr);
    LineError le{};
    TNS_CUDA(cudaMemcpyAsync(&le, d_lerr, sizeof le, cudaMemcpyDeviceToHost, st));
    TNS_CUDA(cudaStreamSynchronize(st));
    const std::string tok(h_text + le.tok_begin, le.tok_len);
    const std::string mode = std::to_string(le.field + 1);
    std::string what;
    switch (le.kind) {  // io.cpp:73-113
      case kErrFieldCount:
        what = "expected " + std::to_string(nf_first) + " fields, got " + std::to_string(le.got);
        break;
      case kErrIndex: what = "invalid index '" + tok + "'"; break;
      case kErrZeroIndex: what = "indices are 1-based; got " + tok + " in mode " + mode; break;
      case kErrExceeds:
        what = "index " + tok + " exceeds declared dimension " +
               std::to_string(declared[le.field]) + " of mode " + mode;
        break;
      default: what = "invalid value '" + tok + "'"; break;
    }
    tns_dev_free(d_coords, st);
    tns_dev_free(d_values, st);
    out->d_coords = nullptr;
    out->d_values = nullptr;
    parse_error(err, eline + 1, le.kind, le.field, le.got, nf_first, le.tok_begin, le.tok_len,
                what);
  }
  out->rank = rank;
  out->nnz = rows;
  if (has_declared) {
    out->dims.assign(declared, declared + rank);
  } else {
    out->dims.resize(rank);
    TNS_CUDA(cudaMemcpy(out->dims.data(), d_max, rank * 4, cudaMemcpyDeviceToHost));
  }
}

// ---- writer: write_tns (io.cpp:128-152) --------------------------------------
namespace {

constexpr int kFmtThreads = 256;
constexpr uint32_t kFmtStage = 40 * 1024;  // CTA text staged in shared memory

__device__ __forceinline__ uint32_t row_text(const uint32_t* coords, const double* values,
                                             uint32_t rank, uint64_t row, char* out) {
  uint32_t p = 0;
  for (uint32_t m = 0; m < rank; ++m) {
    const uint32_t c = coords[row * rank + m] + 1u;  // u32 arithmetic, as io.cpp:141
    p += tns::format_u64(c, out ? out + p : nullptr);
    if (out) out[p] = ' ';
    ++p;
  }
  p += tns::format_f64(values[row], out ? out + p : nullptr);
  if (out) out[p] = '\n';
  return p + 1;
}

__global__ void __launch_bounds__(kFmtThreads)
k_fmt_len(const uint32_t* __restrict__ coords, const double* __restrict__ values, uint32_t rank,
          uint64_t nnz, uint32_t* __restrict__ row_len, uint32_t* __restrict__ cta_len) {
  const uint64_t row = (uint64_t)blockIdx.x * kFmtThreads + threadIdx.x;
  uint32_t len = 0;
  if (row < nnz) {
    len = row_text(coords, values, rank, row, nullptr);
    row_len[row] = len;
  }
  len = __reduce_add_sync(0xffffffffu, len);
  __shared__ uint32_t ws[kFmtThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = len;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int k = 0; k < kFmtThreads / 32; ++k) t += ws[k];
    cta_len[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kFmtThreads)
k_fmt_write(const uint32_t* __restrict__ coords, const double* __restrict__ values,
            uint32_t rank, uint64_t nnz, const uint32_t* __restrict__ row_len,
            const uint64_t* __restrict__ cta_off, char* __restrict__ text) {
  __shared__ uint32_t wsum[kFmtThreads / 32];
  __shared__ __align__(16) char stage[kFmtStage];
  const uint64_t row = (uint64_t)blockIdx.x * kFmtThreads + threadIdx.x;
  const uint32_t len = row < nnz ? row_len[row] : 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t s = len;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, s, d);
    if (lane >= d) s += t;
  }
  if (lane == 31) wsum[warp] = s;
  __syncthreads();
  uint32_t before = s - len, total = 0;
  for (int w = 0; w < kFmtThreads / 32; ++w) {
    if (w < warp) before += wsum[w];
    total += wsum[w];
  }
  const uint64_t base = cta_off[blockIdx.x];
  if (total <= kFmtStage) {
    if (row < nnz) row_text(coords, values, rank, row, stage + before);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < total; i += kFmtThreads) text[base + i] = stage[i];
  } else if (row < nnz) {
    row_text(coords, values, rank, row, text + base + before);
  }
}

}  // namespace

void format_tns_device(uint32_t rank, uint64_t nnz, const uint32_t* h_coords,
                       const double* h_values, char** h_text, uint64_t* n_text, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static const bool timing = getenv("QD_TNS_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!timing) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "qd_write_tns %-12s %8.2f ms\n", what,
            std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  *h_text = nullptr;
  *n_text = 0;
  if (nnz == 0) return;
  DevBuf b_c, b_v, b_len, b_cl, b_co, b_t;
  uint32_t* d_c = b_c.alloc<uint32_t>(nnz * rank * 4, st);
  double* d_v = b_v.alloc<double>(nnz * 8, st);
  staged_h2d(d_c, h_coords, nnz * rank * 4, st);
  staged_h2d(d_v, h_values, nnz * 8, st);
  mark("rows H2D");
  const uint64_t n_ctas = (nnz + kFmtThreads - 1) / kFmtThreads;
  uint32_t* d_len = b_len.alloc<uint32_t>(nnz * 4, st);
  uint32_t* d_cl = b_cl.alloc<uint32_t>(n_ctas * 4, st);
  uint64_t* d_co = b_co.alloc<uint64_t>((n_ctas + 1) * 8, st);
  k_fmt_len<<<(unsigned)n_ctas, kFmtThreads, 0, st>>>(d_c, d_v, rank, nnz, d_len, d_cl);
  k_scan_excl<<<1, 1024, 0, st>>>(d_cl, n_ctas, d_co);
  uint64_t total = 0;
  TNS_CUDA(cudaMemcpyAsync(&total, d_co + n_ctas, 8, cudaMemcpyDeviceToHost, st));
  TNS_CUDA(cudaStreamSynchronize(st));
  mark("lengths");
  char* d_t = b_t.alloc<char>(total, st);
  k_fmt_write<<<(unsigned)n_ctas, kFmtThreads, 0, st>>>(d_c, d_v, rank, nnz, d_len, d_co, d_t);
  TNS_CUDA(cudaGetLastError());
  const uint64_t a = 2ull << 20, cap = (total + a - 1) / a * a;
  char* h = static_cast<char*>(std::aligned_alloc(a, cap));
  if (!h) throw std::bad_alloc();
  madvise(h, cap, MADV_HUGEPAGE);
  mark("format");
  try {
    staged_d2h(h, d_t, total, st);
    TNS_CUDA(cudaStreamSynchronize(st));
    mark("text D2H");
  } catch (...) {
    std::free(h);
    throw;
  }
  *h_text = h;
  *n_text = total;
}

}  // namespace qb200
