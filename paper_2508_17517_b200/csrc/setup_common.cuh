// Shared setup-path infrastructure: device CSR results handed to the caller
// in two phases (info -> caller allocates -> take), CUB scans, PCG64.
#pragma once
#include "airg_common.cuh"
#include <cub/cub.cuh>

// Opaque result: a CSR matrix living in library scratch until taken.
struct airg_csr_result {
  int nrows = 0, ncols = 0;
  long long nnz = 0;
  int* ptr = nullptr;
  int* col = nullptr;
  double* val = nullptr;
  cudaStream_t stream = 0;
};

namespace airg {

// Fork / join of a few side streams so independent launches (per row-size
// class) overlap instead of running back to back with small grids.
struct Fork {
  static constexpr int K = 4;
  cudaStream_t st[K];
  cudaEvent_t ev0, evs[K];
  int begin(cudaStream_t s) {
    static thread_local int dev_init = -1;
    static thread_local cudaStream_t ss[K];
    static thread_local cudaEvent_t e0, es[K];
    int dev = 0;
    AIRG_CUDA(cudaGetDevice(&dev));
    if (dev_init != dev) {
      for (int i = 0; i < K; ++i) {
        AIRG_CUDA(cudaStreamCreateWithFlags(&ss[i], cudaStreamNonBlocking));
        AIRG_CUDA(cudaEventCreateWithFlags(&es[i], cudaEventDisableTiming));
      }
      AIRG_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
      dev_init = dev;
    }
    ev0 = e0;
    for (int i = 0; i < K; ++i) {
      st[i] = ss[i];
      evs[i] = es[i];
    }
    AIRG_CUDA(cudaEventRecord(ev0, s));
    for (int i = 0; i < K; ++i) AIRG_CUDA(cudaStreamWaitEvent(st[i], ev0, 0));
    return AIRG_OK;
  }
  cudaStream_t stream(int c) const { return st[c % K]; }
  int end(cudaStream_t s) {
    for (int i = 0; i < K; ++i) {
      AIRG_CUDA(cudaEventRecord(evs[i], st[i]));
      AIRG_CUDA(cudaStreamWaitEvent(s, evs[i], 0));
    }
    return AIRG_OK;
  }
};

// exclusive scan of `in` (n entries) into out[0..n] (out[n] = total); returns total on host.
int scan_counts(const int* in, int* out, int n, long long* total_h, cudaStream_t s);
// same for 64-bit counts
int scan_counts64(const long long* in, long long* out, int n, long long* total_h, cudaStream_t s);

airg_csr_result* new_result(int nrows, int ncols, cudaStream_t s);
// allocate col/val of a result after its ptr is known (nnz from ptr[nrows])
int result_alloc_entries(airg_csr_result* r, long long nnz, bool values = true);

// ---- PCG64 (numpy's default bit generator), SURVEY App. A.5 ---------------
struct u128 {
  unsigned long long lo, hi;
};

__host__ __device__ __forceinline__ u128 mul128(u128 a, u128 b) {
  u128 r;
#ifdef __CUDA_ARCH__
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
#else
  unsigned __int128 p = (unsigned __int128)a.lo * b.lo;
  r.lo = (unsigned long long)p;
  r.hi = (unsigned long long)(p >> 64) + a.lo * b.hi + a.hi * b.lo;
#endif
  return r;
}
__host__ __device__ __forceinline__ u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}

constexpr unsigned long long kPcgMulHi = 0x2360ED051FC65DA4ull;
constexpr unsigned long long kPcgMulLo = 0x4385DF649FCCF645ull;

// state after `steps` LCG steps from s0 (O(log steps) jump-ahead)
__host__ __device__ __forceinline__ u128 pcg_jump(u128 s0, u128 inc, unsigned long long steps) {
  u128 am = {1ull, 0ull}, aa = {0ull, 0ull};
  u128 cm = {kPcgMulLo, kPcgMulHi}, ca = inc;
  while (steps) {
    if (steps & 1ull) {
      am = mul128(am, cm);
      aa = add128(mul128(aa, cm), ca);
    }
    u128 one = {1ull, 0ull};
    ca = mul128(add128(cm, one), ca);
    cm = mul128(cm, cm);
    steps >>= 1;
  }
  return add128(mul128(am, s0), aa);
}

__host__ __device__ __forceinline__ u128 pcg_step(u128 s, u128 inc) {
  u128 m = {kPcgMulLo, kPcgMulHi};
  return add128(mul128(s, m), inc);
}

__host__ __device__ __forceinline__ double pcg_out_double(u128 s) {
  unsigned long long x = s.hi ^ s.lo;
  unsigned rot = (unsigned)(s.hi >> 58);
  unsigned long long o = (x >> rot) | (x << ((64u - rot) & 63u));
  return (double)(o >> 11) * (1.0 / 9007199254740992.0);
}

// Fill out[i] = a + b * random()_i for i in [0, n): numpy Generator.random()
// (a=0, b=1) or uniform(-1, 1) (a=-1, b=2) bit for bit.  Each thread jumps
// to its chunk then steps sequentially.
int pcg64_fill(u128 s0, u128 inc, long long n, double a, double b, double* out, cudaStream_t s,
               long long start = 0);

}  // namespace airg
