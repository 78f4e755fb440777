// microbenchmark: MATCH.ANY vs 8-ballot peers vs ATOMS throughput on one SM set
#include <cstdio>
#include <cstdint>
__global__ void k_match(uint32_t* out, int iters, uint32_t mask, int mode) {
  uint32_t x = (threadIdx.x * 2654435761u) ^ blockIdx.x;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    const uint32_t d = (x >> 8) & mask;
    unsigned p;
    if (mode == 0) {
      p = __match_any_sync(0xFFFFFFFFu, d);
    } else {
      p = 0xFFFFFFFFu;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const unsigned bit = (d >> b) & 1u;
        const unsigned v = __ballot_sync(0xFFFFFFFFu, bit);
        p &= bit ? v : ~v;
      }
    }
    acc += p;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  uint32_t* out;
  cudaMalloc(&out, 148 * 32 * 1024 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode)
    for (uint32_t mask : {0u, 3u, 15u, 255u})
      for (int threads : {512, 1024}) {
        const int blocks = 148 * 2;
        k_match<<<blocks, threads>>>(out, iters, mask, mode);
        cudaEventRecord(a);
        k_match<<<blocks, threads>>>(out, iters, mask, mode);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double warp_ops = (double)blocks * threads / 32 * iters;
        const double cyc = ms * 1e-3 * 1.965e9;
        printf("%s mask=%3u threads=%4d: %.2f SM-cycles per warp-op (%.3f ms)\n",
               mode ? "ballot8" : "match  ", mask, threads, cyc * 148 / warp_ops, ms);
      }
  return 0;
}
