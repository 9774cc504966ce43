// Host latency of a small device->host read-back after a kernel: pageable vs
// pinned destination (the setup's ~850 read-backs per step).
// nvcc -O2 -gencode arch=compute_100a,code=sm_100a d2h.cu -o d2h
#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
__global__ void bump(int* p) { if (threadIdx.x == 0) p[0] += 1; }
int main() {
  int* d;
  cudaMalloc(&d, 4096);
  cudaMemset(d, 0, 4096);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int* pin;
  cudaHostAlloc(&pin, 4096, cudaHostAllocDefault);
  int page[1024];
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      const int N = 2000;
      auto t0 = std::chrono::steady_clock::now();
      for (int i = 0; i < N; ++i) {
        bump<<<1, 32, 0, s>>>(d);
        int* dst = (mode & 1) ? pin : page;
        size_t bytes = (mode & 2) ? 4096 : 4;
        cudaMemcpyAsync(dst, d, bytes, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
      }
      auto t1 = std::chrono::steady_clock::now();
      if (rep) printf("%s %4zu B: %.2f us per kernel+readback+sync\n", (mode & 1) ? "pinned  " : "pageable",
                      (mode & 2) ? (size_t)4096 : (size_t)4,
                      std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    }
  }
  // kernel + sync only
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 2000; ++i) { bump<<<1, 32, 0, s>>>(d); cudaStreamSynchronize(s); }
  auto t1 = std::chrono::steady_clock::now();
  printf("kernel+sync only: %.2f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / 2000);
  return 0;
}
