// Microbenchmark: one stable LSD counting pass over 16-byte rows with a WIDE
// digit (up to 11 bits = 2048 bins), the tile sorted in shared memory by two
// ballot-ranked sub-digits (low A bits, then high B bits: LSD inside the
// tile), against the same kernel with one 8-bit sub-digit.  Question: does a
// 2-pass 21-bit sort (11+10) beat the 3-pass one (7+7+7)?
//
// Per tile (T rows, TMA double-buffered like k_scatter):
//   sub-pass A: warp stripes, ballot peers on A bits, per-warp u16 counts,
//               slot -> s_idx[slot] = (row << 11) | digit
//   sub-pass B: same over s_idx on the B high bits -> s_srt
//   heads:      gbase[d] = cursor[d] - j at the first slot of each digit;
//               cursor[d] = gbase[d] + j + 1 at its last slot
//   store:      out[gbase[d] + j] = row, coalesced where bins are populated
// Offsets per (chunk, bin) come from a histogram kernel + host scan (setup).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 wide_digit.cu -o /tmp/wd
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));        \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// ballot peers over BITS bits of d (lanes in `valid` only)
template <int BITS>
__device__ __forceinline__ unsigned peers_of(uint32_t d, unsigned valid) {
  unsigned m = valid;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const unsigned bit = (d >> b) & 1u;
    const unsigned v = __ballot_sync(0xFFFFFFFFu, bit);
    m &= bit ? v : ~v;
  }
  return m;
}

constexpr int NT = 512, NW = NT / 32;

// one ranking sub-pass over n positions: digit(q) -> sub-digit s (SB bits);
// writes dst[slot] = word(q) in stable sub-digit order
template <int SB, class GetW, class GetD>
__device__ __forceinline__ void sub_pass(uint32_t n, uint16_t* hist, uint32_t* wsum, uint32_t* dst,
                                         GetW getw, GetD getd) {
  constexpr int B = 1 << SB;
  const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ipw = (((n + NW - 1) / NW) + 31u) & ~31u;
  const uint32_t lo = w * ipw, hi = min(n, lo + ipw);
  uint16_t* wh = hist + w * B;
  for (int k = lane; k < B; k += 32) wh[k] = 0;
  __syncwarp();
  const unsigned below = (1u << lane) - 1u;
  constexpr int R = 8;  // rounds per warp (T <= NW*32*R)
  uint32_t pk[R], wd[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t p = lo + r * 32 + lane;
    if (lo + r * 32 >= hi) break;
    const bool valid = p < hi;
    const uint32_t x = valid ? getw(p) : 0u;
    const uint32_t s = getd(x);
    const unsigned valid_m = __ballot_sync(0xFFFFFFFFu, valid);
    unsigned peers = peers_of<SB>(s, valid_m);
    const uint32_t c = valid ? wh[s] : 0u;
    __syncwarp();
    if (valid && (peers & below) == 0u) wh[s] = (uint16_t)(c + __popc(peers));
    __syncwarp();
    pk[r] = ((c + __popc(peers & below)) << 16) | s;
    wd[r] = x;
  }
  __syncthreads();
  // warp-exclusive offsets per bin + bin starts (B <= 256: one thread per bin walks the warps)
  if (threadIdx.x < B) {
    uint32_t run = 0;
#pragma unroll
    for (int x = 0; x < NW; ++x) {
      const uint32_t c = hist[x * B + threadIdx.x];
      hist[x * B + threadIdx.x] = (uint16_t)run;
      run += c;
    }
    uint32_t incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(B >= 32 ? 0xFFFFFFFFu : ((1u << B) - 1u), incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    if (lane == 31 || (B < 32 && lane == B - 1)) wsum[w] = incl;
    wsum[8 + threadIdx.x] = incl - run;  // exclusive within its 32-bin group
  }
  __syncthreads();
  if (threadIdx.x < B) {
    uint32_t base = 0;
    for (uint32_t x = 0; x < (threadIdx.x >> 5); ++x) base += wsum[x];
    wsum[8 + threadIdx.x] += base;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t p = lo + r * 32 + lane;
    if (lo + r * 32 >= hi) break;
    if (p < hi) {
      const uint32_t s = pk[r] & 0xFFFFu;
      dst[wsum[8 + s] + wh[s] + (pk[r] >> 16)] = wd[r];
    }
  }
  __syncthreads();
}

template <int A, int Bb>
__global__ void __launch_bounds__(NT, 2) k_wide(const ulonglong2* __restrict__ in,
                                                ulonglong2* __restrict__ out, uint32_t T,
                                                uint32_t CH, uint32_t nchunks, uint64_t N,
                                                const uint32_t* __restrict__ offs,  // [chunk][bin]
                                                uint32_t shift, uint32_t* counter) {
  constexpr int DB = A + Bb;
  constexpr uint32_t BINS = 1u << DB;
  extern __shared__ __align__(128) unsigned char smem[];
  ulonglong2* s_rows = reinterpret_cast<ulonglong2*>(smem);  // [2][T]
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(smem + 2 * T * 16);
  uint32_t* s_srt = s_idx + T;
  uint32_t* s_cur = s_srt + T;   // [BINS] cursor
  int32_t* s_gb = reinterpret_cast<int32_t*>(s_cur + BINS);  // [BINS]
  uint16_t* s_hist = reinterpret_cast<uint16_t*>(s_gb + BINS);  // [NW][<=256]
  uint32_t* s_wsum = reinterpret_cast<uint32_t*>(s_hist + NW * 256);  // 8 + <=256
  unsigned long long* s_bar = reinterpret_cast<unsigned long long*>(s_wsum + 272);
  __shared__ uint32_t s_chunk[2], s_tile[2], s_next;

  const uint32_t adv = NT - 32;
  if (threadIdx.x == adv) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto load = [&](uint32_t b, uint32_t c, uint32_t t) {
    const uint64_t rb = ((uint64_t)c * CH + t) * T;
    const uint32_t n = (uint32_t)min((uint64_t)T, N - rb);
    mbar_expect_tx(&s_bar[b], n * 16);
    bulk_g2s(s_rows + b * T, in + rb, n * 16, &s_bar[b]);
  };
  if (threadIdx.x == adv) {
    s_chunk[0] = blockIdx.x;
    s_tile[0] = 0;
    s_next = gridDim.x + atomicAdd(counter, 1u);
    if (blockIdx.x < nchunks) load(0, blockIdx.x, 0);
  }
  __syncthreads();
  uint32_t phases = 0;
  for (uint32_t it = 0;; ++it) {
    const uint32_t b = it & 1u;
    const uint32_t c = s_chunk[b], t = s_tile[b];
    if (c >= nchunks) break;
    const uint64_t rb = ((uint64_t)c * CH + t) * T;
    const uint32_t n = (uint32_t)min((uint64_t)T, N - rb);
    if (t == 0)
      for (uint32_t k = threadIdx.x; k < BINS; k += NT) s_cur[k] = offs[(size_t)c * BINS + k];
    if (threadIdx.x == adv) {  // next tile
      uint32_t nc = c, nt = t + 1;
      const uint64_t chunk_end = min(N, ((uint64_t)c + 1) * CH * T);
      if (rb + T >= chunk_end) {
        nc = s_next;
        nt = 0;
        if (nc < nchunks) s_next = gridDim.x + atomicAdd(counter, 1u);
      }
      s_chunk[b ^ 1u] = nc;
      s_tile[b ^ 1u] = nt;
      if (nc < nchunks) load(b ^ 1u, nc, nt);
    }
    mbar_wait(&s_bar[b], (phases >> b) & 1u);
    phases ^= 1u << b;
    const ulonglong2* rows = s_rows + b * T;
    const uint32_t dmask = BINS - 1u;
    if (Bb == 0) {
      sub_pass<A>(
          n, s_hist, s_wsum, s_srt,
          [&](uint32_t p) { return (p << 11) | ((uint32_t)(rows[p].x >> shift) & dmask); },
          [&](uint32_t x) { return x & ((1u << A) - 1u); });
    } else {
      sub_pass<A>(
          n, s_hist, s_wsum, s_idx,
          [&](uint32_t p) { return (p << 11) | ((uint32_t)(rows[p].x >> shift) & dmask); },
          [&](uint32_t x) { return x & ((1u << A) - 1u); });
      sub_pass<Bb>(
          n, s_hist, s_wsum, s_srt, [&](uint32_t q) { return s_idx[q]; },
          [&](uint32_t x) { return (x & dmask) >> A; });
    }
    // heads: gbase of every present digit
    for (uint32_t j = threadIdx.x; j < n; j += NT) {
      const uint32_t d = s_srt[j] & dmask;
      if (j == 0 || (s_srt[j - 1] & dmask) != d) s_gb[d] = (int32_t)s_cur[d] - (int32_t)j;
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < n; j += NT) {
      const uint32_t x = s_srt[j];
      const uint32_t d = x & dmask;
      const int32_t g = s_gb[d];
      __stcs(out + (uint32_t)(g + (int32_t)j), rows[x >> 11]);
      if (j + 1 == n || (s_srt[j + 1] & dmask) != d) s_cur[d] = (uint32_t)(g + (int32_t)j + 1);
    }
    __syncthreads();
  }
}

__global__ void k_hist(const ulonglong2* in, uint64_t N, uint32_t T, uint32_t CH, uint32_t bins,
                       uint32_t shift, uint32_t* flat /* [bin][chunk] */, uint32_t nchunks) {
  extern __shared__ uint32_t h[];
  for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    for (uint32_t k = threadIdx.x; k < bins; k += blockDim.x) h[k] = 0;
    __syncthreads();
    const uint64_t b = (uint64_t)c * CH * T, e = min(N, b + (uint64_t)CH * T);
    for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x)
      atomicAdd(h + ((uint32_t)(in[i].x >> shift) & (bins - 1)), 1u);
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < bins; k += blockDim.x) flat[(size_t)k * nchunks + c] = h[k];
    __syncthreads();
  }
}

__global__ void k_fill(ulonglong2* p, uint64_t N, int dist, uint32_t bits) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = i * 0x9E3779B97F4A7C15ull;
    x ^= x >> 29;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 32;
    uint64_t key;
    if (dist == 0) {
      key = x & ((1ull << bits) - 1);
    } else {  // zipf-like: key = floor(2^(bits * u^2)) - 1 (heavy head)
      const double u = (double)(x >> 11) * (1.0 / 9007199254740992.0);
      key = (uint64_t)(exp2((double)bits * u * u)) - 1;
      if (key >= (1ull << bits)) key = (1ull << bits) - 1;
    }
    p[i] = make_ulonglong2(key, i);
  }
}

template <int A, int Bb>
float run(const ulonglong2* in, ulonglong2* out, uint64_t N, uint32_t T, int sms, uint32_t shift,
          bool check, int ctas_per_sm) {
  constexpr uint32_t BINS = 1u << (A + Bb);
  const uint32_t CH = 16;
  const uint32_t nchunks = (uint32_t)((N + (uint64_t)CH * T - 1) / ((uint64_t)CH * T));
  uint32_t *flat, *offs, *counter;
  CK(cudaMalloc(&flat, (size_t)BINS * nchunks * 4));
  CK(cudaMalloc(&offs, (size_t)BINS * nchunks * 4));
  CK(cudaMalloc(&counter, 4));
  k_hist<<<sms * 4, 512, BINS * 4>>>(in, N, T, CH, BINS, shift, flat, nchunks);
  std::vector<uint32_t> h((size_t)BINS * nchunks), o((size_t)BINS * nchunks);
  CK(cudaMemcpy(h.data(), flat, h.size() * 4, cudaMemcpyDeviceToHost));
  uint64_t run = 0;
  for (size_t k = 0; k < h.size(); ++k) {  // [bin][chunk] order = stable
    const uint32_t bin = (uint32_t)(k / nchunks), c = (uint32_t)(k % nchunks);
    o[(size_t)c * BINS + bin] = (uint32_t)run;
    run += h[k];
  }
  CK(cudaMemcpy(offs, o.data(), o.size() * 4, cudaMemcpyHostToDevice));
  const size_t smem = 2 * (size_t)T * 16 + 2 * (size_t)T * 4 + 2 * BINS * 4 + NW * 256 * 2 + 272 * 4 + 16;
  auto fn = k_wide<A, Bb>;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem));
  per_sm = std::min(per_sm, ctas_per_sm);
  const uint32_t grid = std::min<uint32_t>(nchunks, per_sm * sms);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < 4; ++rep) {
    CK(cudaMemset(counter, 0, 4));
    cudaEventRecord(a);
    fn<<<grid, NT, smem>>>(in, out, T, CH, nchunks, N, offs, shift, counter);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = std::min(best, ms);
  }
  CK(cudaGetLastError());
  if (check) {  // sorted by digit, stable (payload = input index increasing within a digit)
    const uint64_t M = std::min<uint64_t>(N, 1ull << 26);
    std::vector<ulonglong2> r(M);
    CK(cudaMemcpy(r.data(), out, M * 16, cudaMemcpyDeviceToHost));
    uint64_t bad = 0;
    for (uint64_t i = 1; i < M; ++i) {
      const uint32_t d0 = (uint32_t)(r[i - 1].x >> shift) & (BINS - 1), d1 = (uint32_t)(r[i].x >> shift) & (BINS - 1);
      if (d1 < d0 || (d1 == d0 && r[i].y <= r[i - 1].y)) ++bad;
    }
    printf("   check: %llu bad of %llu\n", (unsigned long long)bad, (unsigned long long)M);
  }
  printf("A=%d B=%d bins=%4u T=%u grid=%u (%d/SM): %.3f ms  %.1f ps/row  %.0f GB/s\n", A, Bb, BINS,
         T, grid, per_sm, best, best * 1e9 / N, 2.0 * N * 16 / best / 1e6);
  cudaFree(flat);
  cudaFree(offs);
  cudaFree(counter);
  return best;
}

int main(int argc, char** argv) {
  const uint64_t N = argc > 1 ? strtoull(argv[1], 0, 10) : (1ull << 29);
  ulonglong2 *in, *out;
  CK(cudaMalloc(&in, N * 16));
  CK(cudaMalloc(&out, N * 16));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int dist = 0; dist < 2; ++dist) {
    k_fill<<<sms * 8, 256>>>(in, N, dist, 22);
    CK(cudaDeviceSynchronize());
    printf("--- %s digits, N=%llu\n", dist ? "zipf-like" : "uniform", (unsigned long long)N);
    for (int cps : {1, 2}) {
      for (uint32_t T : {2048u, 4096u}) {
        if (cps == 2 && T > 2048) continue;
        run<8, 0>(in, out, N, T, sms, 0, dist == 0 && T == 2048, cps);
        run<4, 4>(in, out, N, T, sms, 0, false, cps);
        run<6, 5>(in, out, N, T, sms, 0, dist == 0 && T == 2048, cps);
        run<6, 5>(in, out, N, T, sms, 11, false, cps);
      }
    }
  }
  return 0;
}
