// Shared helpers for libairg (B200 / sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <cmath>
#include <cstring>
#include <initializer_list>
#include "../../include/airg.h"

namespace airg {

// Thread-local last-error text, surfaced by airg_last_error().
void set_error(const char* fmt, ...);

#define AIRG_CUDA(call)                                                          \
  do {                                                                           \
    cudaError_t _e = (call);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::airg::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,              \
                        cudaGetErrorString(_e));                                 \
      return AIRG_ERR_CUDA;                                                      \
    }                                                                            \
  } while (0)

#define AIRG_LAUNCH_CHECK()                                                      \
  do {                                                                           \
    cudaError_t _e = cudaGetLastError();                                         \
    if (_e != cudaSuccess) {                                                     \
      ::airg::set_error("%s:%d launch: %s", __FILE__, __LINE__,                  \
                        cudaGetErrorString(_e));                                 \
      return AIRG_ERR_CUDA;                                                      \
    }                                                                            \
  } while (0)

#define AIRG_TRY(call)                                                           \
  do {                                                                           \
    int _s = (call);                                                             \
    if (_s != AIRG_OK) return _s;                                                \
  } while (0)

// SMs of the current device (148 on B200), queried once per device
inline int num_sms() {
  static int cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& v = cache[dev & 63];
  if (v == 0) {
    int n = 0;
    v = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0 ? n : 148;
  }
  return v;
}

inline int blocks_for(long long n, int threads, long long cap = -1) {
  if (cap < 0) cap = (long long)num_sms() * 64;
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}

// Exact (non-contracted) fp64 arithmetic: scipy's sparsetools and numpy
// accumulate with separate multiply and add roundings.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

template <typename T>
__device__ __forceinline__ T warp_sum(T v, unsigned mask = 0xffffffffu) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// The library's own stream-ordered memory pool (one per device), with the
// release threshold raised so freed scratch stays mapped across
// synchronisations (with the default threshold 0 every synchronisation
// unmaps it and the next large allocation pays for re-mapping GBs of HBM).
// A private pool, so the process's default pool -- torch's and every other
// user's -- keeps its own settings.
cudaMemPool_t lib_pool();

// Scratch memory from the library pool (freed by the caller of alloc).
template <typename T>
inline int scratch(T** p, size_t count, cudaStream_t s) {
  if (count == 0) count = 1;
  AIRG_CUDA(cudaMallocFromPoolAsync((void**)p, count * sizeof(T), lib_pool(), s));
  return AIRG_OK;
}
inline void release(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

// Small device -> host read-backs followed by a stream synchronisation,
// staged through a per-thread pinned buffer: a pageable destination costs
// ~1.8 us more per read-back (tools/micro/d2h.cu), and a setup does ~850.
struct ReadBack {
  void* host;
  const void* dev;
  size_t bytes;
};
inline cudaError_t read_back(std::initializer_list<ReadBack> parts, cudaStream_t s) {
  thread_local unsigned char* stage = nullptr;
  thread_local size_t cap = 0;
  size_t need = 0;
  for (const ReadBack& r : parts) need += (r.bytes + 15) & ~(size_t)15;
  if (need > cap) {
    if (stage) cudaFreeHost(stage);
    stage = nullptr;
    cap = 0;
    const size_t c = need > 4096 ? need : 4096;
    if (cudaHostAlloc((void**)&stage, c, cudaHostAllocDefault) == cudaSuccess) cap = c;
    else stage = nullptr;
  }
  if (!stage) {  // no pinned memory: plain copies into the destinations
    for (const ReadBack& r : parts) {
      cudaError_t e = cudaMemcpyAsync(r.host, r.dev, r.bytes, cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) return e;
    }
    return cudaStreamSynchronize(s);
  }
  size_t off = 0;
  for (const ReadBack& r : parts) {
    cudaError_t e = cudaMemcpyAsync(stage + off, r.dev, r.bytes, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return e;
    off += (r.bytes + 15) & ~(size_t)15;
  }
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  off = 0;
  for (const ReadBack& r : parts) {
    memcpy(r.host, stage + off, r.bytes);
    off += (r.bytes + 15) & ~(size_t)15;
  }
  return cudaSuccess;
}
inline cudaError_t read_back(void* host, const void* dev, size_t bytes, cudaStream_t s) {
  return read_back({ReadBack{host, dev, bytes}}, s);
}

// Long-lived plan buffers: pool-backed (no device-wide sync on free).
template <typename T>
inline cudaError_t dmalloc(T** p, size_t bytes) {
  cudaError_t e = cudaMallocFromPoolAsync((void**)p, bytes ? bytes : 1, lib_pool(), 0);
  if (e == cudaSuccess) e = cudaStreamSynchronize(0);
  return e;
}
inline void dfree(void* p) {
  if (p) cudaFreeAsync(p, 0);
}

}  // namespace airg
