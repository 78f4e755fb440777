// Microbenchmark: does an L2 evict_last store policy let partially written
// sectors of a wide-digit scatter merge in L2 (consecutive tiles of a chunk
// complete them) instead of costing DRAM read-modify-writes?  Same store
// pattern as scatter_bins.cu (16-byte rows, chunks of 16 tiles, uniform
// digits; loads evict_first) with three store policies: st.global.cs,
// default, and st.global.L2::cache_hint with a createpolicy evict_last.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scatter_policy.cu -o /tmp/sp
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_hint(ulonglong2* p, ulonglong2 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.u64 [%0], {%1, %2}, %3;" ::"l"(p), "l"(v.x), "l"(v.y),
               "l"(pol)
               : "memory");
}

template <int POL>
__global__ void k_store(const ulonglong2* __restrict__ in, ulonglong2* __restrict__ out,
                        unsigned long long nchunks, unsigned T, unsigned CH, unsigned B) {
  unsigned long long pol = 0;
  if (POL == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  const unsigned per = T / B;
  for (unsigned long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
    for (unsigned t = 0; t < CH; ++t) {
      const unsigned long long rb = (c * CH + t) * T;
      for (unsigned j = threadIdx.x; j < T; j += blockDim.x) {
        const ulonglong2 v = __ldcs(in + rb + j);
        const unsigned b = j / per, k = t * per + j % per;
        const unsigned long long dst = ((unsigned long long)b * nchunks + c) * (CH * per) + k;
        if (POL == 0) __stcs(out + dst, v);
        else if (POL == 1) out[dst] = v;
        else st_hint(out + dst, v, pol);
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
  const char* names[3] = {"stcs      ", "default   ", "evict_last"};
  for (int pol = 0; pol < 3; ++pol)
    for (unsigned T : {2048u, 4096u}) {
      for (unsigned B : {256u, 512u, 1024u, 2048u}) {
        const unsigned CH = 16;
        const unsigned long long nchunks = N / ((unsigned long long)T * CH);
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
          cudaEventRecord(a);
          if (pol == 0) k_store<0><<<sms * 4, 512>>>(in, out, nchunks, T, CH, B);
          if (pol == 1) k_store<1><<<sms * 4, 512>>>(in, out, nchunks, T, CH, B);
          if (pol == 2) k_store<2><<<sms * 4, 512>>>(in, out, nchunks, T, CH, B);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        printf("%s T=%u bins=%4u rows/bin/tile=%5.1f  %.3f ms  %.0f GB/s (read+write)\n", names[pol],
               T, B, (double)T / B, best, 2.0 * N * 16 / best / 1e6);
      }
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
