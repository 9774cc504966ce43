// Grid-barrier cost on the device: 148 CTAs x 1024 threads, K barriers per
// launch, three barrier flavours.  nvcc -arch=sm_100a -O3 gridbar.cu
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ void bar_acq(unsigned long long* bar, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1ULL);
    unsigned long long v;
    do { asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory"); } while (v < target);
  }
  __syncthreads();
}
__device__ void bar_relaxed(unsigned long long* bar, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" :: "l"(bar) : "memory");
    unsigned long long v;
    do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory"); } while (v < target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
template <int M>
__global__ void __launch_bounds__(1024, 1) k(unsigned long long* bar, int K, double* sink) {
  __shared__ unsigned long long base;
  if (threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
    const unsigned long long span = (unsigned long long)gridDim.x * K;
    base = v - v % span;
  }
  __syncthreads();
  double acc = threadIdx.x;
  for (int s = 0; s < K; ++s) {
    acc = acc * 1.0000001 + 1.0;
    if (M == 0) bar_acq(bar, base + (unsigned long long)gridDim.x * (s + 1));
    else if (M == 1) bar_relaxed(bar, base + (unsigned long long)gridDim.x * (s + 1));
    else cg::this_grid().sync();
  }
  if (acc == 12345.0) sink[0] = acc;
}
template <int M>
float run(int G, int K, unsigned long long* bar, double* sink) {
  cudaMemset(bar, 0, 8);
  void* args[] = {&bar, &K, &sink};
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) cudaLaunchCooperativeKernel((void*)k<M>, G, 1024, args, 0, 0);
  cudaEventRecord(a);
  const int R = 50;
  for (int w = 0; w < R; ++w) cudaLaunchCooperativeKernel((void*)k<M>, G, 1024, args, 0, 0);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  return ms * 1000 / R;
}
int main() {
  unsigned long long* bar; double* sink;
  cudaMalloc(&bar, 8); cudaMemset(bar, 0, 8); cudaMalloc(&sink, 8);
  for (int G : {1, 8, 32, 148}) {
    float t0 = run<0>(G, 1, bar, sink), t6 = run<0>(G, 7, bar, sink);
    float r0 = run<1>(G, 1, bar, sink), r6 = run<1>(G, 7, bar, sink);
    float c0 = run<2>(G, 1, bar, sink), c6 = run<2>(G, 7, bar, sink);
    printf("G=%3d  acq: launch+1 %.2f us, per extra barrier %.2f us | relaxed: %.2f / %.2f | cg: %.2f / %.2f\n",
           G, t0, (t6 - t0) / 6, r0, (r6 - r0) / 6, c0, (c6 - c0) / 6);
  }
  return 0;
}
