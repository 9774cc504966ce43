// Fused F-smoother chain: e_f = q(A_ff) rhs as ONE persistent kernel.
//
// The reference applies the coefficient polynomial by Horner, one SpMV+axpy
// per degree (polynomial.py:295-300): d passes over A_ff per V-cycle level.
// Here every CTA owns a contiguous block of rows (balanced by nnz + rows, one
// CTA per SM), stages as much of its block's CSR (row offsets, columns,
// values) as fits into shared memory with TMA bulk copies
// (cp.async.bulk + mbarrier) once, and runs all d Horner steps against the
// staged copy, with a grid barrier between steps.  A_ff crosses HBM once per
// V-cycle instead of d times; only the n_f-vectors move per step (through
// L2).  Rows that do not fit are read from global memory every step (they
// are the tail of each CTA's block, so staging covers the block's prefix).
// Fast-mode arithmetic (FMA, lane-split rows), like spmv_vec_kernel.
#pragma once
#include "airg_common.cuh"

namespace airg {

constexpr int kChainMaxDeg = 16;
constexpr int kChainThreads = 1024;
#ifndef CHAIN_U
#define CHAIN_U 4
#endif
constexpr int kChainU = CHAIN_U;  // entries per lane in flight per round

struct ChainArgs {
  int n;                         // rows of A_ff
  const int* ptr;
  const int* col;
  const double* val;
  const double* b;               // rhs (read-only for the whole chain)
  double* t0;                    // ping-pong work vectors (n)
  double* t1;
  double* y;                     // final output, y[ymap ? ymap[i] : i]
  const int* ymap;
  const int* part;               // [3 G + 1]: r0, rs (end of staged prefix), r1 per CTA; max bytes
  unsigned long long* bar;       // grid barrier counter (monotone, per chain)
  int d;                         // Horner degree (steps)
  int smem;                      // dynamic shared memory bytes per CTA
  double coef[kChainMaxDeg + 1];
#ifdef CHAIN_TRACE
  long long* trace;              // [G][4 + 2 d] %globaltimer stamps (tools/micro)
#endif
};

__device__ __forceinline__ void chain_stamp(const ChainArgs& a, int p) {
#ifdef CHAIN_TRACE
  if (threadIdx.x == 0) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[(size_t)blockIdx.x * (4 + 2 * a.d) + p] = t;
  }
#endif
}

// Row partition.  A row costs its rounds of kChainU entries per lane
// (ceil(len / (kChainU VS)): a short row takes a full round trip like a long
// one) plus a fixed overhead; w is the exclusive prefix of that cost, CTA g
// gets rows [r0, r1) with w split evenly, and the staged prefix [r0, rs) is
// the longest that fits `cap` bytes (plan build: cost kernel, device scan,
// one thread per CTA of the chain).
__device__ __forceinline__ long long chain_stage_bytes(const int* ptr, int r0, int rs) {
  const long long k = (long long)__ldg(ptr + rs) - __ldg(ptr + r0);
  return 4LL * (rs - r0 + 1) + 12LL * k + 48;
}
__global__ void chain_cost_kernel(int n, const int* __restrict__ ptr, int vs,
                                  long long* __restrict__ cost) {
  const int step = kChainU * vs;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int len = __ldg(ptr + i + 1) - __ldg(ptr + i);
    cost[i] = (long long)((len + step - 1) / step) * step + 4;
  }
}
// w: exclusive prefix of the row costs (n + 1 entries, w[n] the total)
__global__ void chain_partition_kernel(int n, const int* __restrict__ ptr, int G, long long cap,
                                       const long long* __restrict__ w, int* __restrict__ part) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  const long long W = w[n];
  auto bound = [&](int q) {  // first row i with w[i] >= q W / G
    if (q <= 0) return 0;
    if (q >= G) return n;
    const long long tg = W * q / G;
    int a = 0, b = n;
    while (a < b) {
      const int m = (a + b) >> 1;
      if (w[m] < tg) a = m + 1; else b = m;
    }
    return a;
  };
  const int r0 = bound(g), r1 = bound(g + 1);
  int a = r0, b = r1;  // largest rs in [r0, r1] with bytes(rs) <= cap
  while (a < b) {
    const int m = (a + b + 1) >> 1;
    if (chain_stage_bytes(ptr, r0, m) <= cap) a = m; else b = m - 1;
  }
  part[3 * g] = r0;
  part[3 * g + 1] = a;
  part[3 * g + 2] = r1;
  // shared bytes this CTA stages (+ alignment slack): the launch asks for
  // the maximum, leaving the rest of the SM's 256 KB to L1 (x gathers)
  atomicMax(part + 3 * G, (int)(a > r0 ? chain_stage_bytes(ptr, r0, a) + 64 : 0));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

// copy global bytes [src, src + nbytes) to shared `dst` where
// (dst - src) % 16 == 0: the 16-byte aligned interior by one bulk copy
// (thread 0 arms `mbar`), head and tail elements by the calling threads.
template <typename T>
__device__ __forceinline__ unsigned chain_stage(T* dst, const T* src, long long count,
                                                unsigned long long* mbar, bool issue) {
  const uintptr_t gb = (uintptr_t)src, ge = (uintptr_t)(src + count);
  const uintptr_t ab = (gb + 15) & ~(uintptr_t)15, ae = ge & ~(uintptr_t)15;
  unsigned bytes = 0;
  if (ab < ae) {
    bytes = (unsigned)(ae - ab);
    if (issue) {
      T* d = dst + (ab - gb) / sizeof(T);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              smem_u32(d)),
          "l"(ab), "r"(bytes), "r"(smem_u32(mbar))
          : "memory");
    }
    const long long nh = (long long)(ab - gb) / sizeof(T), nt0 = (long long)(ae - gb) / sizeof(T);
    for (long long j = threadIdx.x; j < nh; j += blockDim.x) dst[j] = src[j];
    for (long long j = nt0 + threadIdx.x; j < count; j += blockDim.x) dst[j] = src[j];
  } else {
    for (long long j = threadIdx.x; j < count; j += blockDim.x) dst[j] = src[j];
  }
  return bytes;
}

// A vector written earlier in the same launch: a coherent (weak, L1-cached)
// load.  The grid barrier's ld.acquire.gpu invalidates the SM's L1
// (CCTL.IVALL), so lines cached before the barrier are never reused after
// it, while the reuse of x among the rows of one step still hits L1.
__device__ __forceinline__ double ld_ca(const double* p) {
  double v;
  asm volatile("ld.global.ca.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// one row group (VS lanes): s = sum_k val * x[col]; xs scales x
// (CG: x was written by this launch -- ld_ca instead of the read-only path)
template <int VS, bool CG>
__device__ __forceinline__ double chain_row(const int* __restrict__ cl, const double* __restrict__ vl,
                                            int b, int e, int lane, const double* __restrict__ x,
                                            double xs) {
  double s = 0.0;
  for (int k0 = b + lane; k0 < e; k0 += kChainU * VS) {
    int c[kChainU];
    double a[kChainU], xv[kChainU];
#pragma unroll
    for (int q = 0; q < kChainU; ++q) {
      const int k = k0 + q * VS;
      c[q] = k < e ? cl[k] : -1;
      a[q] = k < e ? vl[k] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kChainU; ++q) xv[q] = c[q] >= 0 ? (CG ? ld_ca(x + c[q]) : __ldg(x + c[q])) : 0.0;
#pragma unroll
    for (int q = 0; q < kChainU; ++q) s = fma(a[q], xs * xv[q], s);
  }
  if (VS > 1) {
#pragma unroll
    for (int o = VS / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, VS);
  }
  return s;
}

__device__ __forceinline__ void chain_grid_barrier(const ChainArgs& a, int p,
                                                   unsigned long long* bar, unsigned long long target) {
  __syncthreads();
  chain_stamp(a, p);
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1ULL);
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  chain_stamp(a, p + 1);
  __syncthreads();
}

template <int VS>
__global__ void __launch_bounds__(kChainThreads, 1) chain_kernel(const ChainArgs a) {
  extern __shared__ __align__(16) unsigned char chain_sm[];
  unsigned char* sm = chain_sm;
  __shared__ __align__(8) unsigned long long mbar;
  __shared__ unsigned long long base_s;
  const int g = blockIdx.x, G = gridDim.x;
  const int r0 = __ldg(a.part + 3 * g), rs = __ldg(a.part + 3 * g + 1), r1 = __ldg(a.part + 3 * g + 2);
  const int k0 = __ldg(a.ptr + r0), ks = __ldg(a.ptr + rs);
  // shared layout (each array keeps its global 16-byte phase)
  const int nps = rs - r0 + 1;
  int* sp = (int*)sm + ((uintptr_t)(a.ptr + r0) & 15) / 4;
  unsigned char* p1 = sm + (((size_t)nps * 4 + 16 + 15) & ~(size_t)15);
  int* sc = (int*)p1 + ((uintptr_t)(a.col + k0) & 15) / 4;
  unsigned char* p2 = p1 + (((size_t)(ks - k0) * 4 + 16 + 15) & ~(size_t)15);
  double* sv = (double*)p2 + ((uintptr_t)(a.val + k0) & 15) / 8;
  const bool staged = rs > r0;
  chain_stamp(a, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a.bar) : "memory");
    const unsigned long long span = (unsigned long long)G * (a.d - 1);
    base_s = span ? v - v % span : 0;
  }
  __syncthreads();
  if (staged) {
    // byte counts first (no copy), arm the barrier, then issue the copies
    unsigned tx = 0;
    if (threadIdx.x == 0) {
      auto interior = [](const void* p, long long bytes) -> unsigned {
        const uintptr_t gb = (uintptr_t)p, ge = gb + bytes;
        const uintptr_t ab = (gb + 15) & ~(uintptr_t)15, ae = ge & ~(uintptr_t)15;
        return ab < ae ? (unsigned)(ae - ab) : 0u;
      };
      tx = interior(a.ptr + r0, 4LL * nps) + interior(a.col + k0, 4LL * (ks - k0)) +
           interior(a.val + k0, 8LL * (ks - k0));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)),
                   "r"(tx)
                   : "memory");
    }
    const bool t0 = threadIdx.x == 0;
    chain_stage(sp, a.ptr + r0, nps, &mbar, t0);
    chain_stage(sc, a.col + k0, ks - k0, &mbar, t0);
    chain_stage(sv, a.val + k0, ks - k0, &mbar, t0);
  }
  chain_stamp(a, 1);
  const int lane = threadIdx.x & (VS - 1);
  const int grp = threadIdx.x / VS, ngrp = kChainThreads / VS;
  const double* x = a.b;
  double xs = a.coef[a.d];
  for (int step = 0; step < a.d; ++step) {
    const int j = a.d - 1 - step;  // coefficient index of this Horner step
    const bool last = j == 0;
    double* dst = last ? a.y : ((j & 1) ? a.t1 : a.t0);
    const double cj = a.coef[j];
    // unstaged tail rows first (global memory): overlaps the first staging
    // (trip counts are CTA-uniform: the row groups of a warp shuffle together)
    for (int i0 = rs; i0 < r1; i0 += ngrp) {
      const int i = i0 + grp;
      const bool act = i < r1;
      const int b = act ? __ldg(a.ptr + i) : 0, e = act ? __ldg(a.ptr + i + 1) : 0;
      const double s = step == 0 ? chain_row<VS, false>(a.col, a.val, b, e, lane, x, xs)
                                 : chain_row<VS, true>(a.col, a.val, b, e, lane, x, xs);
      if (act && lane == 0) dst[last && a.ymap ? __ldg(a.ymap + i) : i] = fma(cj, __ldg(a.b + i), s);
    }
    if (staged) {
      if (step == 0) {
        unsigned ok = 0;
        while (!ok)
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
              : "=r"(ok)
              : "r"(smem_u32(&mbar))
              : "memory");
        __syncthreads();  // head/tail elements written by plain stores
        chain_stamp(a, 2);
      }
      for (int i0 = r0; i0 < rs; i0 += ngrp) {
        const int i = i0 + grp;
        const bool act = i < rs;
        const int b = act ? sp[i - r0] - k0 : 0, e = act ? sp[i - r0 + 1] - k0 : 0;
        const double s = step == 0 ? chain_row<VS, false>(sc, sv, b, e, lane, x, xs)
                                   : chain_row<VS, true>(sc, sv, b, e, lane, x, xs);
        if (act && lane == 0) dst[last && a.ymap ? __ldg(a.ymap + i) : i] = fma(cj, __ldg(a.b + i), s);
      }
    }
    if (!last) {
      chain_grid_barrier(a, 3 + 2 * step, a.bar, base_s + (unsigned long long)G * (step + 1));
      x = dst;
      xs = 1.0;
    }
#ifdef CHAIN_TRACE
    else {
      __syncthreads();
      chain_stamp(a, 3 + 2 * step);
      chain_stamp(a, 4 + 2 * step);
    }
#endif
  }
}

}  // namespace airg
