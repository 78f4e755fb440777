// Microbenchmark: moving a pageable host buffer (a std::vector) to and from
// the device, the building blocks of the drop-in's synchronous host-buffer
// transpose.  (a) parallel host memcpy throughput (pageable -> pinned, T
// threads); (b) cudaHostRegister + cudaHostUnregister of the buffer in place;
// (c) pinned H2D / D2H; (d) direct pageable cudaMemcpy.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 host_staging.cu -o /tmp/hs -lpthread
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void pmemcpy(char* d, const char* s, size_t n, int T) {
  std::vector<std::thread> th;
  const size_t part = (n / T + 4095) & ~size_t(4095);
  for (int t = 0; t < T; ++t) {
    const size_t a = std::min(n, t * part), b = std::min(n, (t + 1) * part);
    th.emplace_back([=] { if (b > a) std::memcpy(d + a, s + a, b - a); });
  }
  for (auto& x : th) x.join();
}

int main() {
  const size_t n = 600ull << 20;  // 30M rows x 20 B
  std::vector<char> h(n, 1), h2(n, 2);
  char* pin = nullptr;
  cudaMallocHost(&pin, n);
  void* d = nullptr;
  cudaMalloc(&d, n);
  std::memset(pin, 3, n);
  for (int T : {1, 4, 8, 16, 32}) {
    double best = 1e9;
    for (int r = 0; r < 3; ++r) {
      const double t0 = now();
      pmemcpy(pin, h.data(), n, T);
      best = std::min(best, now() - t0);
    }
    printf("memcpy pageable->pinned 600 MB, %2d threads: %.1f ms (%.1f GB/s)\n", T, best * 1e3,
           n / best / 1e9);
  }
  for (int r = 0; r < 3; ++r) {
    double t0 = now();
    cudaHostRegister(h2.data(), n, cudaHostRegisterDefault);
    const double t1 = now();
    cudaMemcpy(d, h2.data(), n, cudaMemcpyHostToDevice);
    const double t2 = now();
    cudaMemcpy(h2.data(), d, n, cudaMemcpyDeviceToHost);
    const double t3 = now();
    cudaHostUnregister(h2.data());
    const double t4 = now();
    printf("register %.1f ms, H2D %.1f ms, D2H %.1f ms, unregister %.1f ms (%s)\n", (t1 - t0) * 1e3,
           (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  for (int r = 0; r < 2; ++r) {
    double t0 = now();
    cudaMemcpy(d, pin, n, cudaMemcpyHostToDevice);
    double t1 = now();
    cudaMemcpy(pin, d, n, cudaMemcpyDeviceToHost);
    double t2 = now();
    cudaMemcpy(d, h.data(), n, cudaMemcpyHostToDevice);
    double t3 = now();
    cudaMemcpy(h.data(), d, n, cudaMemcpyDeviceToHost);
    double t4 = now();
    printf("pinned H2D %.1f D2H %.1f ms; pageable H2D %.1f D2H %.1f ms\n", (t1 - t0) * 1e3,
           (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3);
  }
  return 0;
}
