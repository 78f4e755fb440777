// Microbenchmark: DRAM efficiency of the chunk-ordered scatter STORE pattern
// as a function of the digit width (bins per pass).  Rows are 16 bytes; each
// CTA takes chunks of CH tiles of T rows; inside a tile the rows are already
// in digit order (as k_scatter's store loop writes them) with T/B rows per
// bin; bin b of chunk c owns the contiguous destination range
// [(b*C + c)*CH*T/B, +CH*T/B) — exactly the destinations of a stable LSD pass
// over uniformly distributed digits.  Reads are coalesced 16-byte loads.
// Built and run by hand: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   scatter_bins.cu -o /tmp/sb && /tmp/sb
#include <cstdio>
#include <cuda_runtime.h>

template <bool CS>
__global__ void k_store(const ulonglong2* __restrict__ in, ulonglong2* __restrict__ out,
                        unsigned long long nchunks, unsigned T, unsigned CH, unsigned B) {
  const unsigned per = T / B;  // rows per bin per tile
  for (unsigned long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
    for (unsigned t = 0; t < CH; ++t) {
      const unsigned long long rb = (c * CH + t) * T;
      for (unsigned j = threadIdx.x; j < T; j += blockDim.x) {
        const ulonglong2 v = __ldcs(in + rb + j);
        const unsigned b = j / per, k = t * per + j % per;
        const unsigned long long dst = ((unsigned long long)b * nchunks + c) * (CH * per) + k;
        if (CS) __stcs(out + dst, v); else out[dst] = v;
      }
    }
  }
}

int main() {
  const unsigned long long N = 1ull << 29;  // 512M rows, 8 GB each way
  ulonglong2 *in, *out;
  cudaMalloc(&in, N * 16);
  cudaMalloc(&out, N * 16);
  cudaMemset(in, 1, N * 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cs = 1; cs >= 0; --cs)
  for (unsigned T : {2048u, 4096u, 8192u}) {
    for (unsigned B : {1u, 256u, 1024u, 2048u, 4096u}) {
      if (B > T) continue;  // needs >= 1 row per bin per tile
      const unsigned CH = 16;
      const unsigned long long nchunks = N / ((unsigned long long)T * CH);
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        if (cs) k_store<true><<<sms * 4, 512>>>(in, out, nchunks, T, CH, B);
        else k_store<false><<<sms * 4, 512>>>(in, out, nchunks, T, CH, B);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("%s T=%u bins=%4u rows/bin/tile=%5.1f  %.3f ms  %.0f GB/s (read+write)\n", cs ? "stcs" : "st  ", T, B,
             (double)T / B, best, 2.0 * N * 16 / best / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
