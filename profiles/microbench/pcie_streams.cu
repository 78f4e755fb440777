// Microbenchmark: pinned host<->device copy bandwidth with the transfer split
// over 1, 2 and 4 streams (copy engines), each direction alone and both
// together.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 pcie_streams.cu -o /tmp/ps
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const size_t n = 4ull << 30;  // 4 GB each way
  char *h1, *h2, *d1, *d2;
  cudaMallocHost(&h1, n);
  cudaMallocHost(&h2, n);
  cudaMalloc(&d1, n);
  cudaMalloc(&d2, n);
  cudaStream_t st[8];
  for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int k : {1, 2, 4}) {
    for (int dir = 0; dir < 3; ++dir) {  // 0 H2D, 1 D2H, 2 both
      double best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaDeviceSynchronize();
        const double t0 = now();
        const size_t part = n / k;
        for (int i = 0; i < k; ++i) {
          if (dir != 1) cudaMemcpyAsync(d1 + i * part, h1 + i * part, part, cudaMemcpyHostToDevice, st[i]);
          if (dir != 0) cudaMemcpyAsync(h2 + i * part, d2 + i * part, part, cudaMemcpyDeviceToHost, st[4 + i]);
        }
        cudaDeviceSynchronize();
        best = std::min(best, now() - t0);
      }
      const double bytes = dir == 2 ? 2.0 * n : 1.0 * n;
      printf("%d stream(s) %s: %.1f GB/s\n", k, dir == 0 ? "H2D " : dir == 1 ? "D2H " : "both", bytes / best / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
