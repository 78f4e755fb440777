// Multi-GPU transpose, host C++ over NCCL: one communicator per
// device (one process per GPU, or several devices driven from one process's
// threads), sharded by the range of the output's leading mode sigma1.
//
// Every rank holds a contiguous slice of the global input rows (slices in
// rank order; the global input is simply sorted).  Rank g's output is the
// slice of the global output whose sigma1 values fall in rank g's range, so
// the rank outputs concatenated in rank order equal the reference transpose
// of the global tensor:
//
// * sigma1 == 0 and no mode-0 run straddles two ranks (checked with one
//   allgather of every rank's first/last mode-0 value): the slices are
//   independent — bucket containment (parallel.cpp:125-139
//   lifted to GPUs) — and every rank transposes its own rows, no exchange.
// * otherwise one exchange: sigma1 histogram (device) -> ncclAllReduce ->
//   splitters on the device (balanced output rows at sigma1-value
//   boundaries; a value is never split) -> per-destination row counts,
//   ncclAllGather'd into the world x world count matrix -> stable device
//   partition of the local rows (one k_scatter pass with a lookup digit) ->
//   ONE ncclGroupStart/End of ncclSend + ncclRecv per peer (coordinates and
//   values of each part), received in SOURCE-RANK order, which keeps the
//   received rows a subsequence of the simply sorted global input -> the full
//   local Quesadilla plan.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy torch already
// loaded, else the system one); without it only the emulated transport and
// world size 1 work.  The emulated transport ("hub") runs the ranks as host
// threads of one process on one device — transfers are device copies and the
// ranks meet at host barriers, so no kernel ever waits on another rank's
// kernel — and exists to test this file's logic at world sizes > 1 on a
// single GPU.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "internal.hpp"

namespace qb200 {
namespace {

#define SH_CUDA(x)                                                              \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess)                                                      \
      throw Error(QD_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---- NCCL, resolved at run time ---------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return a;
    auto sym = [&](auto& fn, const char* s) { fn = reinterpret_cast<std::decay_t<decltype(fn)>>(dlsym(a.h, s)); };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.AllGather, "ncclAllGather");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    if (!a.GetUniqueId || !a.CommInitRank || !a.Send || !a.Recv || !a.GroupStart)
      a.h = nullptr;
    return a;
  }();
  if (!api.h) throw Error(QD_NCCL_ERROR, "NCCL (libnccl.so.2) could not be loaded");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(QD_NCCL_ERROR, std::string(what) + ": " +
                                   (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
}

// ---- transports ---------------------------------------------------------------
// One part of an exchange: rows [start, start+count) of the local partitioned
// buffers go to peer p; rows from peer p land at row `at` of the receive buffer.
struct XPart {
  uint64_t send_start = 0, send_count = 0, recv_at = 0, recv_count = 0;
};

struct Transport {
  int nranks = 1, rank = 0;
  virtual ~Transport() = default;
  virtual void allreduce_sum_u64(unsigned long long* d, size_t n, cudaStream_t st) = 0;
  // d_recv[nranks * n]: rank q's n values at q * n
  virtual void allgather_u64(const unsigned long long* d_send, unsigned long long* d_recv,
                             size_t n, cudaStream_t st) = 0;
  // the grouped all-to-allv of rows (coordinates and values)
  virtual void exchange(uint32_t R, const uint32_t* send_c, const double* send_v, uint32_t* recv_c,
                        double* recv_v, const std::vector<XPart>& parts, cudaStream_t st) = 0;
  virtual const char* kind() const = 0;
};

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  ~NcclTransport() override {
    if (comm) nccl().CommDestroy(comm);
  }
  void allreduce_sum_u64(unsigned long long* d, size_t n, cudaStream_t st) override {
    nccl_check(nccl().AllReduce(d, d, n, ncclUint64, ncclSum, comm, st), "ncclAllReduce");
  }
  void allgather_u64(const unsigned long long* s, unsigned long long* r, size_t n,
                     cudaStream_t st) override {
    nccl_check(nccl().AllGather(s, r, n, ncclUint64, comm, st), "ncclAllGather");
  }
  void exchange(uint32_t R, const uint32_t* sc, const double* sv, uint32_t* rc, double* rv,
                const std::vector<XPart>& parts, cudaStream_t st) override {
    const NcclApi& N = nccl();
    // this rank's own part is a local device copy
    const XPart& me = parts[rank];
    if (me.send_count) {
      SH_CUDA(cudaMemcpyAsync(rc + me.recv_at * R, sc + me.send_start * R, me.send_count * R * 4,
                              cudaMemcpyDeviceToDevice, st));
      SH_CUDA(cudaMemcpyAsync(rv + me.recv_at, sv + me.send_start, me.send_count * 8,
                              cudaMemcpyDeviceToDevice, st));
    }
    nccl_check(N.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      const XPart& x = parts[p];
      if (x.send_count) {
        nccl_check(N.Send(sc + x.send_start * R, x.send_count * R, ncclUint32, p, comm, st), "ncclSend");
        nccl_check(N.Send(sv + x.send_start, x.send_count, ncclFloat64, p, comm, st), "ncclSend");
      }
      if (x.recv_count) {
        nccl_check(N.Recv(rc + x.recv_at * R, x.recv_count * R, ncclUint32, p, comm, st), "ncclRecv");
        nccl_check(N.Recv(rv + x.recv_at, x.recv_count, ncclFloat64, p, comm, st), "ncclRecv");
      }
    }
    nccl_check(N.GroupEnd(), "ncclGroupEnd");
  }
  const char* kind() const override { return "nccl"; }
};

}  // namespace

// Emulated ranks: threads of one process on one device, meeting at host
// barriers; every transfer is a device copy between the ranks' buffers.
struct Hub {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  // per-rank posted addresses for the current collective
  std::vector<const void*> a, b;
  std::vector<const std::vector<XPart>*> parts;
  explicit Hub(int n_) : n(n_), a(n_), b(n_), parts(n_) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

namespace {

__global__ void k_add_u64(unsigned long long* dst, const unsigned long long* src, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

struct HubTransport : Transport {
  std::shared_ptr<Hub> hub;
  Workspace* ws = nullptr;  // scratch for the all-reduce
  void allreduce_sum_u64(unsigned long long* d, size_t n, cudaStream_t st) override {
    auto* tmp = static_cast<unsigned long long*>(workspace_buffer(*ws, "hub_tmp", n * 8));
    SH_CUDA(cudaStreamSynchronize(st));
    hub->a[rank] = d;
    hub->barrier();  // every rank's input is final
    SH_CUDA(cudaMemcpyAsync(tmp, hub->a[0], n * 8, cudaMemcpyDeviceToDevice, st));
    for (int q = 1; q < nranks; ++q)
      k_add_u64<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256, 0, st>>>(
          tmp, static_cast<const unsigned long long*>(hub->a[q]), n);
    SH_CUDA(cudaGetLastError());
    SH_CUDA(cudaStreamSynchronize(st));
    hub->barrier();  // every rank has read every input
    SH_CUDA(cudaMemcpyAsync(d, tmp, n * 8, cudaMemcpyDeviceToDevice, st));
    SH_CUDA(cudaStreamSynchronize(st));
  }
  void allgather_u64(const unsigned long long* s, unsigned long long* r, size_t n,
                     cudaStream_t st) override {
    SH_CUDA(cudaStreamSynchronize(st));
    hub->a[rank] = s;
    hub->barrier();
    for (int q = 0; q < nranks; ++q)
      SH_CUDA(cudaMemcpyAsync(r + q * n, hub->a[q], n * 8, cudaMemcpyDeviceToDevice, st));
    SH_CUDA(cudaStreamSynchronize(st));
    hub->barrier();
  }
  void exchange(uint32_t R, const uint32_t* sc, const double* sv, uint32_t* rc, double* rv,
                const std::vector<XPart>& parts, cudaStream_t st) override {
    SH_CUDA(cudaStreamSynchronize(st));
    hub->a[rank] = sc;
    hub->b[rank] = sv;
    hub->parts[rank] = &parts;
    hub->barrier();  // every sender's partitioned rows are final
    // pull part `rank` of every source, in source-rank order
    for (int q = 0; q < nranks; ++q) {
      const XPart& src = (*hub->parts[q])[rank];  // what q sends to me
      const XPart& dst = parts[q];                // where q's rows land here
      if (src.send_count != dst.recv_count)
        throw Error(QD_NCCL_ERROR, "emulated exchange: count mismatch");
      if (!src.send_count) continue;
      SH_CUDA(cudaMemcpyAsync(rc + dst.recv_at * R,
                              static_cast<const uint32_t*>(hub->a[q]) + src.send_start * R,
                              src.send_count * R * 4, cudaMemcpyDeviceToDevice, st));
      SH_CUDA(cudaMemcpyAsync(rv + dst.recv_at, static_cast<const double*>(hub->b[q]) + src.send_start,
                              src.send_count * 8, cudaMemcpyDeviceToDevice, st));
    }
    SH_CUDA(cudaStreamSynchronize(st));
    hub->barrier();  // every receiver is done reading the senders' buffers
  }
  const char* kind() const override { return "emulated"; }
};

// ---- splitters on the device ------------------------------------------------
constexpr int kSplitThreads = 1024;
constexpr uint32_t kSplitTile = 8192;  // values per block in the scan

// per-tile sums of the global histogram
__global__ void __launch_bounds__(kSplitThreads) k_tile_sums(const unsigned long long* h, uint64_t dim,
                                                             unsigned long long* sums) {
  __shared__ unsigned long long s[kSplitThreads / 32];
  const uint64_t b = (uint64_t)blockIdx.x * kSplitTile;
  unsigned long long x = 0;
  for (uint64_t i = b + threadIdx.x; i < min(dim, b + kSplitTile); i += kSplitThreads) x += h[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    x = s[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    if (threadIdx.x == 0) sums[blockIdx.x] = x;
  }
}

// exclusive scan of the tile sums in place (one block; tiles <= 2^32 / 8192)
__global__ void __launch_bounds__(kSplitThreads) k_scan_tiles(unsigned long long* sums, uint32_t nt,
                                                              unsigned long long* total) {
  __shared__ unsigned long long s[kSplitThreads / 32];
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t b = 0; b < nt; b += kSplitThreads) {
    const uint32_t i = b + threadIdx.x;
    const unsigned long long v = i < nt ? sums[i] : 0ull;
    unsigned long long x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s[w] = x;
    __syncthreads();
    if (w == 0) {
      unsigned long long t = s[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, t, o);
        if (lane >= o) t += y;
      }
      s[lane] = t;
    }
    __syncthreads();
    const unsigned long long incl = x + (w ? s[w - 1] : 0ull) + carry;
    if (i < nt) sums[i] = incl - v;
    __syncthreads();
    if (threadIdx.x == kSplitThreads - 1) carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// lookup[v] = the part of sigma1 value v: parts cut the global output rows
// into `parts` balanced ranges, a value going wholly to the part holding the
// midpoint of its rows (monotone in v; an indivisible Zipf head value lands
// once).  Each block rescans its tile serially per warp-chunk.
__global__ void __launch_bounds__(kSplitThreads) k_splitters(const unsigned long long* h, uint64_t dim,
                                                             const unsigned long long* tile_base,
                                                             const unsigned long long* total,
                                                             uint32_t parts, uint32_t* lookup) {
  __shared__ unsigned long long s[kSplitThreads / 32];
  const uint64_t b = (uint64_t)blockIdx.x * kSplitTile;
  const uint64_t e = min(dim, b + kSplitTile);
  const unsigned long long T = *total;
  unsigned long long carry = tile_base[blockIdx.x];
  for (uint64_t c = b; c < e; c += kSplitThreads) {
    const uint64_t i = c + threadIdx.x;
    const unsigned long long v = i < e ? h[i] : 0ull;
    unsigned long long x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s[w] = x;
    __syncthreads();
    if (w == 0) {
      unsigned long long t = s[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, t, o);
        if (lane >= o) t += y;
      }
      s[lane] = t;
    }
    __syncthreads();
    const unsigned long long before = carry + x - v + (w ? s[w - 1] : 0ull);  // rows of values < i
    if (i < e) {
      uint32_t p = 0;
      if (T) {
        // part = floor((before + v/2) * parts / T), in exact integer arithmetic:
        // floor((2*before + v) * parts / (2*T))
        const unsigned __int128 num = (unsigned __int128)(2ull * before + v) * parts;
        const unsigned __int128 q = num / ((unsigned __int128)2 * T);
        p = q < (unsigned __int128)(parts - 1) ? (uint32_t)q : parts - 1;
      }
      lookup[i] = p;
    }
    const unsigned long long block_total = s[kSplitThreads / 32 - 1];
    __syncthreads();
    carry += block_total;
  }
}

// counts[p] += local rows of the values with lookup == p (lookup is monotone:
// runs of one part; a thread adds its run per part change)
__global__ void k_part_counts(const unsigned long long* local, const uint32_t* lookup, uint64_t dim,
                              unsigned long long* counts) {
  const uint64_t per = (dim + (uint64_t)gridDim.x * blockDim.x - 1) / ((uint64_t)gridDim.x * blockDim.x);
  const uint64_t b = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * per;
  const uint64_t e = min(dim, b + per);
  if (b >= e) return;
  uint32_t cur = lookup[b];
  unsigned long long acc = 0;
  for (uint64_t i = b; i < e; ++i) {
    const uint32_t p = lookup[i];
    if (p != cur) {
      if (acc) atomicAdd(counts + cur, acc);
      cur = p;
      acc = 0;
    }
    acc += local[i];
  }
  if (acc) atomicAdd(counts + cur, acc);
}

// [nnz, first mode-0, last mode-0] of this rank's rows
__global__ void k_slice_info(const uint32_t* c, uint32_t R, uint64_t nnz, unsigned long long* out) {
  out[0] = nnz;
  out[1] = nnz ? c[0] : 0u;
  out[2] = nnz ? c[(nnz - 1) * R] : 0u;
}

}  // namespace

struct Comm {
  std::unique_ptr<Transport> t;
  int device = 0;
};

Comm* comm_create_nccl(const unsigned char* id, int nranks, int rank, int device) {
  if (nranks < 1 || rank < 0 || rank >= nranks) invalid("rank must be in 0..nranks-1");
  SH_CUDA(cudaSetDevice(device));
  auto t = std::make_unique<NcclTransport>();
  t->nranks = nranks;
  t->rank = rank;
  ncclUniqueId uid;
  static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(&uid, id, sizeof(uid));
  nccl_check(nccl().CommInitRank(&t->comm, nranks, uid, rank), "ncclCommInitRank");
  auto* c = new Comm;
  c->t = std::move(t);
  c->device = device;
  return c;
}

void comm_unique_id(unsigned char* out) {
  ncclUniqueId uid;
  nccl_check(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(out, &uid, sizeof(uid));
}

Hub* hub_create(int nranks) {
  if (nranks < 1) invalid("hub needs at least one rank");
  return new Hub(nranks);
}
void hub_destroy(Hub* h) { delete h; }

Comm* comm_create_emulated(Hub* hub, int rank, int device, Workspace* ws) {
  if (!hub) invalid("hub is null");
  if (rank < 0 || rank >= hub->n) invalid("rank must be in 0..nranks-1");
  auto t = std::make_unique<HubTransport>();
  t->nranks = hub->n;
  t->rank = rank;
  // non-owning: the hub must outlive its comms (documented in the header)
  t->hub = std::shared_ptr<Hub>(hub, [](Hub*) {});
  t->ws = ws;
  auto* c = new Comm;
  c->t = std::move(t);
  c->device = device;
  return c;
}

void comm_destroy(Comm* c) { delete c; }
int comm_size(const Comm& c) { return c.t->nranks; }
int comm_rank(const Comm& c) { return c.t->rank; }
const char* comm_kind(const Comm& c) { return c.t->kind(); }

void sharded_transpose_device(Comm& comm, Workspace& ws, const TensorView& t, const uint32_t* d_c_in,
                              const double* d_v_in, uint32_t* d_c_out, double* d_v_out,
                              uint64_t out_capacity, uint64_t* n_out,
                              const std::vector<Group>& groups, const uint32_t* target, void* stream,
                              qd_shard_stats* stats) {
  Transport& T = *comm.t;
  const int G = T.nranks, me = T.rank;
  const uint32_t R = t.rank;
  const uint64_t N = t.nnz;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SH_CUDA(cudaSetDevice(workspace_device(ws)));
  qd_shard_stats s{};
  auto finish_local = [&](const uint32_t* c, const double* v, uint64_t n) {
    *n_out = n;
    if (n > out_capacity)
      invalid("output capacity " + std::to_string(out_capacity) + " < " + std::to_string(n) + " rows");
    TensorView lt{R, t.dims, n};
    run_groups(ws, lt, c, v, d_c_out, d_v_out, groups, false, nullptr, nullptr, 0, stream);
  };
  if (G == 1 || groups.empty()) {
    finish_local(d_c_in, d_v_in, N);
    s.rows_out = N;
    if (stats) *stats = s;
    return;
  }
  auto* small = static_cast<unsigned long long*>(workspace_buffer(ws, "shard_small", 64 * 8));
  auto* gath = static_cast<unsigned long long*>(
      workspace_buffer(ws, "shard_gather", (size_t)G * (G + 4) * 8));
  std::vector<unsigned long long> h((size_t)G * (G + 4));
  const uint32_t s1 = target[0];
  bool exchange = true;
  if (s1 == 0) {
    // communication-free when no mode-0 run straddles two ranks
    k_slice_info<<<1, 1, 0, st>>>(d_c_in, R, N, small);
    SH_CUDA(cudaGetLastError());
    workspace_count_launch(ws);
    T.allgather_u64(small, gath, 3, st);
    SH_CUDA(cudaMemcpyAsync(h.data(), gath, (size_t)G * 3 * 8, cudaMemcpyDeviceToHost, st));
    SH_CUDA(cudaStreamSynchronize(st));
    bool aligned = true;
    long prev = -1;  // last non-empty rank
    for (int q = 0; q < G; ++q) {
      if (!h[q * 3]) continue;
      if (prev >= 0 && h[prev * 3 + 2] == h[q * 3 + 1]) aligned = false;
      prev = q;
    }
    exchange = !aligned;
  }
  if (!exchange) {
    finish_local(d_c_in, d_v_in, N);
    s.rows_out = N;
    if (stats) *stats = s;
    return;
  }
  // ---- one exchange keyed on sigma1 ----
  const uint32_t dim = t.dims[s1];
  auto* hist = static_cast<unsigned long long*>(workspace_buffer(ws, "shard_hist", (size_t)dim * 8));
  auto* local = static_cast<unsigned long long*>(workspace_buffer(ws, "shard_local", (size_t)dim * 8));
  auto* lookup = static_cast<uint32_t*>(workspace_buffer(ws, "shard_lookup", (size_t)dim * 4));
  const uint32_t ntile = (uint32_t)((dim + kSplitTile - 1) / kSplitTile);
  auto* tiles = static_cast<unsigned long long*>(workspace_buffer(ws, "shard_tiles", (size_t)ntile * 8 + 8));
  SH_CUDA(cudaMemsetAsync(local, 0, (size_t)dim * 8, st));
  mode_histogram_device(ws, R, N, d_c_in, s1, dim, reinterpret_cast<uint64_t*>(local), stream);
  SH_CUDA(cudaMemcpyAsync(hist, local, (size_t)dim * 8, cudaMemcpyDeviceToDevice, st));
  T.allreduce_sum_u64(hist, dim, st);
  k_tile_sums<<<ntile, kSplitThreads, 0, st>>>(hist, dim, tiles);
  k_scan_tiles<<<1, kSplitThreads, 0, st>>>(tiles, ntile, small);
  k_splitters<<<ntile, kSplitThreads, 0, st>>>(hist, dim, tiles, small, (uint32_t)G, lookup);
  SH_CUDA(cudaMemsetAsync(small + 8, 0, (size_t)G * 8, st));
  {
    const uint32_t th = 256, blocks = (uint32_t)std::min<uint64_t>((dim + th * 64 - 1) / (th * 64), 1024);
    k_part_counts<<<std::max(1u, blocks), th, 0, st>>>(local, lookup, dim, small + 8);
  }
  SH_CUDA(cudaGetLastError());
  for (int k = 0; k < 4; ++k) workspace_count_launch(ws);
  // the world x world count matrix: C[q][p] = rows rank q sends to rank p
  T.allgather_u64(small + 8, gath, (size_t)G, st);
  SH_CUDA(cudaMemcpyAsync(h.data(), gath, (size_t)G * G * 8, cudaMemcpyDeviceToHost, st));
  SH_CUDA(cudaStreamSynchronize(st));
  auto C = [&](int q, int p) { return (uint64_t)h[(size_t)q * G + p]; };
  uint64_t n_recv = 0;
  std::vector<XPart> parts(G);
  uint64_t send_at = 0;
  for (int p = 0; p < G; ++p) {
    parts[p].send_start = send_at;
    parts[p].send_count = C(me, p);
    send_at += C(me, p);
  }
  for (int q = 0; q < G; ++q) {  // source-rank order
    parts[q].recv_at = n_recv;
    parts[q].recv_count = C(q, me);
    n_recv += C(q, me);
  }
  if (send_at != N) throw Error(QD_NCCL_ERROR, "sharded transpose: partition counts do not add up");
  // a rank whose output does not fit fails, and so does everyone else
  // (collectively: nobody is left waiting in the exchange)
  {
    unsigned long long bad = n_recv > out_capacity ? 1ull : 0ull;
    SH_CUDA(cudaMemcpyAsync(small + 1, &bad, 8, cudaMemcpyHostToDevice, st));
    T.allreduce_sum_u64(small + 1, 1, st);
    SH_CUDA(cudaMemcpyAsync(&bad, small + 1, 8, cudaMemcpyDeviceToHost, st));
    SH_CUDA(cudaStreamSynchronize(st));
    *n_out = n_recv;
    if (bad) {
      if (n_recv > out_capacity)
        invalid("output capacity " + std::to_string(out_capacity) + " < " + std::to_string(n_recv) +
                " rows");
      invalid("another rank's output capacity is too small (collective failure)");
    }
  }
  // stable partition of the local rows into destination parts
  auto* sc = static_cast<uint32_t*>(workspace_buffer(ws, "shard_send_c", std::max<uint64_t>(N, 1) * R * 4));
  auto* sv = static_cast<double*>(workspace_buffer(ws, "shard_send_v", std::max<uint64_t>(N, 1) * 8));
  auto* rc = static_cast<uint32_t*>(workspace_buffer(ws, "shard_recv_c", std::max<uint64_t>(n_recv, 1) * R * 4));
  auto* rv = static_cast<double*>(workspace_buffer(ws, "shard_recv_v", std::max<uint64_t>(n_recv, 1) * 8));
  std::vector<uint64_t> pc(G, 0);
  if (N) {
    if ((uint32_t)G > 256) invalid("at most 256 ranks");
    partition_rows_device(ws, R, N, d_c_in, d_v_in, s1, dim, lookup, (uint32_t)G, sc, sv, pc.data(),
                          stream);
  }
  for (int p = 0; p < G; ++p)
    if (pc[p] != C(me, p)) throw Error(QD_NCCL_ERROR, "sharded transpose: partition/count mismatch");
  cudaEvent_t e0, e1;
  SH_CUDA(cudaEventCreate(&e0));
  SH_CUDA(cudaEventCreate(&e1));
  SH_CUDA(cudaEventRecord(e0, st));
  T.exchange(R, sc, sv, rc, rv, parts, st);
  SH_CUDA(cudaEventRecord(e1, st));
  // the received rows, concatenated in source-rank order, are a subsequence
  // of the simply sorted global input: the full local plan finishes them
  finish_local(rc, rv, n_recv);
  float ms = 0;
  SH_CUDA(cudaEventSynchronize(e1));
  SH_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  s.exchanged = 1;
  s.rows_out = n_recv;
  for (int p = 0; p < G; ++p)
    if (p != me) s.bytes_sent += C(me, p) * (4ull * R + 8ull), s.bytes_received += C(p, me) * (4ull * R + 8ull);
  s.exchange_ms = ms;
  if (stats) *stats = s;
}

}  // namespace qb200
