// Solve-path kernels: SpMV family with fused epilogues, polynomial apply
// (Horner / Neumann / factored Newton), the V-cycle plan and the Richardson
// driver.  ref: /root/reference/pkg/src/airmg/solve.py:89-167,
// polynomial.py:295-369, sparse.py:206-212.
#include "airg_common.cuh"
#include "chain.cuh"
#include <nccl.h>
#include <vector>
#include <algorithm>
#include <cstring>
#include <string>
#include <mutex>

namespace airg {

static thread_local std::string g_err;
void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

cudaMemPool_t lib_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  cudaMemPool_t& p = pools[dev & 63];
  if (!p) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
      p = nullptr;
      cudaDeviceGetDefaultMemPool(&p, dev);  // fallback: the device pool, untouched
      return p;
    }
    unsigned long long thr = ~0ull;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  return p;
}

// ---------------------------------------------------------------------------
// SpMV with a fused epilogue:
//   out[omap ? omap[i] : i] = alpha * (A (xs*x))_i + beta * v[vmap ? vmap[i] : i]
//   (+ optional out2[omap..] += same value, + optional sum of squares)
// VS lanes cooperate on one row (VS = 1 .. 32).
// ---------------------------------------------------------------------------
struct Epi {
  double* out;
  const int* omap;
  double alpha;
  double beta;
  const double* v;  // may be null
  const int* vmap;
  double* acc;      // optional: acc[o] += value
  double* partial;  // optional: per-block sum of squares of value
  // optional independent scatter done by the same launch (saves a kernel):
  // sc_dst[sc_idx[i]] = sc_src[i], i < sc_n
  const double* sc_src = nullptr;
  const int* sc_idx = nullptr;
  double* sc_dst = nullptr;
  long long sc_n = 0;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ double ld_relaxed_sys_d(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// spin on one peer's message count (relaxed polls, one acquire fence once it
// is reached: an acquire per poll would keep invalidating the SM's L1 under
// the CTAs sharing it); traps (fails the context) after ~20 s instead of
// hanging the device
__device__ __forceinline__ void wait_count(const unsigned long long* flag, unsigned long long want) {
  const long long t0 = clock64();
  while (ld_relaxed_sys(flag) < want) {
    __nanosleep(64);
    if (clock64() - t0 > 40000000000ll) __trap();
  }
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

// Programmatic dependent launch: a kernel launched with the programmatic
// serialization attribute starts while its predecessor drains; it waits here
// (until the predecessor grid completed and its writes are visible) before
// touching any input, then lets its own successor be scheduled.  Both are
// no-ops for a normal launch.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
}

static bool pdl_enabled() {
  static int v = -1;
  if (v < 0) v = getenv("AIRG_PDL") && atoi(getenv("AIRG_PDL")) == 0 ? 0 : 1;
  return v == 1;
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*k)(KArgs...), int grid, int block, cudaStream_t s,
                              Args&&... args) {
  if (!pdl_enabled()) {
    k<<<grid, block, 0, s>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

template <bool E>
__device__ __forceinline__ double madd(double a, double b, double c) {
  return E ? add_rn(c, mul_rn(a, b)) : fma(a, b, c);
}
template <bool E>
__device__ __forceinline__ double mul(double a, double b) {
  return E ? mul_rn(a, b) : a * b;
}

template <int VS, bool E>
__global__ void __launch_bounds__(256) spmv_vec_kernel(int nrows, const int* __restrict__ ptr,
                                                       const int* __restrict__ col,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ x, double xs,
                                                       Epi ep) {
  pdl_enter();
  if (ep.sc_n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < ep.sc_n;
         i += (long long)gridDim.x * blockDim.x)
      ep.sc_dst[ep.sc_idx[i]] = ep.sc_src[i];
  }
  const int lane = threadIdx.x & (VS - 1);
  const long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / VS;
  double s = 0.0;
  if (E && row < nrows) {
    // reference order: s = 0; s = s + a*x, column order, separate roundings
    const int b = __ldg(ptr + row), e = __ldg(ptr + row + 1);
    for (int k = b; k < e; ++k) s = add_rn(s, mul_rn(__ldg(val + k), mul_rn(xs, __ldg(x + __ldg(col + k)))));
  } else if (row < nrows) {
    const int b = __ldg(ptr + row), e = __ldg(ptr + row + 1);
    // rounds of 4 entries per lane: all column/value loads of a round are
    // issued before the gathers, and all gathers before the FMAs, so every
    // lane keeps ~8 independent requests in flight (the kernel is latency-,
    // not issue-bound at these row lengths).
    for (int k0 = b + lane; k0 < e; k0 += 4 * VS) {
      int c[4];
      double a[4], xv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = k0 + q * VS;
        c[q] = k < e ? __ldg(col + k) : -1;
        a[q] = k < e ? __ldg(val + k) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) xv[q] = c[q] >= 0 ? __ldg(x + c[q]) : 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) s = fma(a[q], xs * xv[q], s);
    }
  }
  if (VS > 1) {
#pragma unroll
    for (int o = VS / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  double sq = 0.0;
  if (lane == 0 && row < nrows) {
    double r = mul<E>(ep.alpha, s);
    if (ep.v) r = madd<E>(ep.beta, ep.v[ep.vmap ? ep.vmap[row] : row], r);
    const long long o = ep.omap ? ep.omap[row] : row;
    if (ep.out) ep.out[o] = r;
    if (ep.acc) ep.acc[o] += r;
    sq = r * r;
  }
  if (ep.partial) {
    __shared__ double red[32];
    sq = warp_sum(sq);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x < 32) {
      double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
      t = warp_sum(t);
      if (threadIdx.x == 0) ep.partial[blockIdx.x] = t;
    }
  }
}

// Bitwise scipy csr_matvec: s = 0; s = s + a*x (separate roundings) in column order.
__global__ void spmv_exact_kernel(int nrows, const int* __restrict__ ptr,
                                  const int* __restrict__ col, const double* __restrict__ val,
                                  const double* __restrict__ x, double* __restrict__ y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nrows;
       i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) s = add_rn(s, mul_rn(val[k], x[col[k]]));
    y[i] = s;
  }
}

// lanes per row: about 4-8 entries per lane (one or two unrolled rounds)
static int pick_vs(long long nnz, int nrows) {
  double mean = nrows > 0 ? (double)nnz / nrows : 0.0;
  if (mean <= 6) return 1;
  if (mean <= 12) return 2;
  if (mean <= 24) return 4;
  if (mean <= 48) return 8;
  if (mean <= 96) return 16;
  return 32;
}

// Host-side launcher shared by every solve-path SpMV.
struct Csr {
  int nrows = 0, ncols = 0;
  long long nnz = 0;
  const int* ptr = nullptr;
  const int* col = nullptr;
  const double* val = nullptr;
  int vs = 1;
  // optional ELL copy (fast mode, fixed-width stencil rows): slot k of row i
  // at k * nrows + i; padding slots repeat a valid column with value 0
  int ew = 0;
  const int* ecol = nullptr;
  const double* eval = nullptr;
};

// kernels launched by this thread (per-call deltas are taken on the calling thread)
static thread_local long long g_launches = 0;

// ELL SpMV with the CSR kernel's epilogue (fast mode): one thread per row,
// column-major slots, so the loads of a warp are coalesced and no row
// offsets are read (the stencil operators of the finest level, 2-3 entries
// per row).
__global__ void __launch_bounds__(256) spmv_ell_epi_kernel(int nrows, int w, const int* __restrict__ ecol,
                                                           const double* __restrict__ eval,
                                                           const double* __restrict__ x, double xs,
                                                           Epi ep) {
  pdl_enter();
  if (ep.sc_n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < ep.sc_n;
         i += (long long)gridDim.x * blockDim.x)
      ep.sc_dst[ep.sc_idx[i]] = ep.sc_src[i];
  }
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double sq = 0.0;
  if (row < nrows) {
    int c[4];
    double a[4];
    double s = 0.0;
    for (int k0 = 0; k0 < w; k0 += 4) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool in = k0 + q < w;
        c[q] = in ? __ldg(ecol + (size_t)(k0 + q) * nrows + row) : -1;
        a[q] = in ? __ldg(eval + (size_t)(k0 + q) * nrows + row) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c[q] >= 0) s = fma(a[q], xs * __ldg(x + c[q]), s);
    }
    double r = ep.alpha * s;
    if (ep.v) r = fma(ep.beta, ep.v[ep.vmap ? ep.vmap[row] : row], r);
    const long long o = ep.omap ? ep.omap[row] : row;
    if (ep.out) ep.out[o] = r;
    if (ep.acc) ep.acc[o] += r;
    sq = r * r;
  }
  if (ep.partial) {
    __shared__ double red[32];
    sq = warp_sum(sq);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x < 32) {
      double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
      t = warp_sum(t);
      if (threadIdx.x == 0) ep.partial[blockIdx.x] = t;
    }
  }
}

static int launch_spmv(const Csr& A, const double* x, double xs, const Epi& ep, cudaStream_t s,
                       bool exact = false) {
  if (A.nrows == 0) return AIRG_OK;
  const int threads = 256;
  if (exact) {
    spmv_vec_kernel<1, true><<<(A.nrows + threads - 1) / threads, threads, 0, s>>>(
        A.nrows, A.ptr, A.col, A.val, x, xs, ep);
    ++g_launches;
    AIRG_LAUNCH_CHECK();
    return AIRG_OK;
  }
  if (A.ew > 0) {
    AIRG_CUDA(launch_pdl(spmv_ell_epi_kernel, (A.nrows + threads - 1) / threads, threads, s, A.nrows,
                         A.ew, A.ecol, A.eval, x, xs, ep));
    ++g_launches;
    AIRG_LAUNCH_CHECK();
    return AIRG_OK;
  }
  const long long groups = (long long)A.nrows * A.vs;
  const int blocks = (int)((groups + threads - 1) / threads);
#define AIRG_SPMV_CASE(V)                                                                  \
  case V:                                                                                \
    AIRG_CUDA(launch_pdl(spmv_vec_kernel<V, false>, blocks, threads, s, A.nrows, A.ptr, A.col, \
                         A.val, x, xs, ep));                                             \
    break;
  switch (A.vs) {
    AIRG_SPMV_CASE(1)
    AIRG_SPMV_CASE(2)
    AIRG_SPMV_CASE(4)
    AIRG_SPMV_CASE(8)
    AIRG_SPMV_CASE(16)
    AIRG_SPMV_CASE(32)
    default: set_error("bad vector width"); return AIRG_ERR_ARG;
  }
#undef AIRG_SPMV_CASE
  ++g_launches;
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

static int spmv_blocks(const Csr& A) {
  if (A.ew > 0) return (int)(((long long)A.nrows + 255) / 256);
  return (int)(((long long)A.nrows * A.vs + 255) / 256);
}

// out[omap(i)] = a * x[xmap(i)] + b * y[i]   (elementwise helpers)
template <bool E>
__global__ void axpby_kernel(long long n, double* __restrict__ out, const int* __restrict__ omap,
                             double a, const double* __restrict__ x, const int* __restrict__ xmap,
                             double b, const double* __restrict__ y) {
  pdl_enter();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double r = mul<E>(a, x[xmap ? xmap[i] : i]);
    if (y) r = madd<E>(b, y[i], r);
    out[omap ? omap[i] : i] = r;
  }
}

static int launch_axpby(long long n, double* out, const int* omap, double a, const double* x,
                        const int* xmap, double b, const double* y, cudaStream_t s,
                        bool exact = false) {
  if (n == 0) return AIRG_OK;
  if (exact) axpby_kernel<true><<<blocks_for(n, 256), 256, 0, s>>>(n, out, omap, a, x, xmap, b, y);
  else AIRG_CUDA(launch_pdl(axpby_kernel<false>, blocks_for(n, 256), 256, s, n, out, omap, a, x, xmap, b, y));
  ++g_launches;
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

// Neumann step: t_new = t - ds .* (A t); acc += t_new.
template <bool E>
__global__ void neumann_step_kernel(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                    const double* __restrict__ val, const double* __restrict__ ds,
                                    const double* __restrict__ t, double* __restrict__ tn,
                                    double* __restrict__ acc) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) s = madd<E>(val[k], t[col[k]], s);
    double v = E ? sub_rn(t[i], mul_rn(ds[i], s)) : t[i] - ds[i] * s;
    tn[i] = v;
    acc[i] = E ? add_rn(acc[i], v) : acc[i] + v;
  }
}

// Deterministic sum of per-block partials -> sqrt into out[0].
__global__ void finish_norm_kernel(int nparts, const double* __restrict__ parts,
                                   double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += parts[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) out[0] = sqrt(t);
  }
}

__global__ void sumsq_kernel(long long n, const double* __restrict__ x, double* __restrict__ parts) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    s = fma(x[i], x[i], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) parts[blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------
// Factored Newton application (polynomial.py:312-355) in ONE CTA: the
// per-root max|u| rescale is a block-wide reduction, so the whole root
// sequence runs without leaving the SM.  Vectors live in global memory
// (L1/L2 resident for coarse grids); u, w, z, x are caller scratch.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double block_max(double v, double* red) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_max(t);
    if (threadIdx.x == 0) red[32] = t;
  }
  __syncthreads();
  double r = red[32];
  __syncthreads();
  return r;
}

template <bool E>
__device__ __forceinline__ double row_dot(const int* __restrict__ ptr, const int* __restrict__ col,
                                          const double* __restrict__ val, const double* x, int i) {
  double s = 0.0;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) s = madd<E>(val[k], x[col[k]], s);
  return s;
}

template <bool E>
__global__ void __launch_bounds__(1024) newton_cta_kernel(
    int n, const int* __restrict__ ptr, const int* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ b, double* x, double* u, double* w, double* z, int nunits,
    const int* __restrict__ utype, const double* __restrict__ up1, const double* __restrict__ up2) {
  __shared__ double red[33];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    u[i] = b[i];
    x[i] = 0.0;
  }
  __syncthreads();
  double scale = 1.0;
  for (int k = 0; k < nunits; ++k) {
    double lmax = 0.0;
    if (utype[k] == 0) {
      const double t = up1[k];
      const double sc = scale / t;
      int bad = 0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) bad |= !isfinite(sc * u[i]);
      if (__syncthreads_or(bad)) break;
      for (int i = threadIdx.x; i < n; i += blockDim.x) w[i] = row_dot<E>(ptr, col, val, u, i);
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double ui = u[i];
        x[i] = E ? add_rn(x[i], mul_rn(sc, ui)) : x[i] + sc * ui;
        const double un = E ? sub_rn(ui, __ddiv_rn(w[i], t)) : ui - w[i] / t;
        u[i] = un;
        lmax = fmax(lmax, fabs(un));
      }
    } else {
      const double two_a = up1[k], m2 = up2[k];
      const double sc = scale / m2;
      for (int i = threadIdx.x; i < n; i += blockDim.x) w[i] = row_dot<E>(ptr, col, val, u, i);
      __syncthreads();
      int bad = 0;
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        bad |= !isfinite(mul<E>(sc, E ? sub_rn(mul_rn(two_a, u[i]), w[i]) : two_a * u[i] - w[i]));
      if (__syncthreads_or(bad)) break;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        if (E) x[i] = add_rn(x[i], mul_rn(sc, sub_rn(mul_rn(two_a, u[i]), w[i])));
        else x[i] += sc * (two_a * u[i] - w[i]);
        z[i] = row_dot<E>(ptr, col, val, w, i);
      }
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double un = E ? add_rn(u[i], __ddiv_rn(sub_rn(z[i], mul_rn(two_a, w[i])), m2))
                            : u[i] + (z[i] - two_a * w[i]) / m2;
        u[i] = un;
        lmax = fmax(lmax, fabs(un));
      }
    }
    const double nrm = block_max(lmax, red);  // also orders the u writes above
    if (nrm == 0.0) break;
    if (nrm > 1e150 || nrm < 1e-150) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) u[i] /= nrm;
      scale *= nrm;
      __syncthreads();
      if (!isfinite(scale) || scale == 0.0) break;
    }
  }
}

// NaN-propagating max (np.max semantics)
__device__ __forceinline__ double nanmax(double a, double b) {
  return a != a ? a : (b != b ? b : fmax(a, b));
}

// Single-CTA Newton with u / w / x (and the matrix when it fits) in shared
// memory.  Two barriers per root:
//  * real root:  w = A u | barrier | x += (s/t) u, u -= w/t, local max | max barrier
//    The "delta finite" test is taken from the previous max: with c = s/t,
//    all_i finite(c*u_i) <=> finite(c*max|u|) (rounding is monotone), and the
//    max propagates NaN like np.max.
//  * pair:       w = A u (+ finite test) | barrier_or | z_i = (A w)_i, x, u
//    updated by the owner of row i, local max | max barrier
// The max reduction double-buffers its partials, so no third barrier.
template <bool E>
__global__ void __launch_bounds__(1024) newton_smem_kernel(
    int n, const int* __restrict__ gptr, const int* __restrict__ gcol, const double* __restrict__ gval,
    int mat_smem, const double* __restrict__ b, double* __restrict__ xout, int nunits,
    const int* __restrict__ utype, const double* __restrict__ up1, const double* __restrict__ up2,
    int identity_cols = 0, int* stopped = nullptr) {
  extern __shared__ double sm[];
  __shared__ double red[2][32];
  const int tid = threadIdx.x, nthr = blockDim.x, nw = nthr >> 5;
  // identity_cols: CTA j applies q(A) to e_j and writes column j of Q (column-major)
  const int jcol = identity_cols ? (int)blockIdx.x : -1;
  if (identity_cols) xout += (size_t)jcol * n;
  double* u = sm;
  double* w = u + n;
  double* x = w + n;
  const int* ptr = gptr;
  const int* col = gcol;
  const double* val = gval;
  if (mat_smem) {
    const int nnz = gptr[n];
    double* sval = x + n;
    int* sptr = (int*)(sval + nnz);
    int* scol = sptr + n + 1;
    for (int i = tid; i < nnz; i += nthr) {
      sval[i] = gval[i];
      scol[i] = gcol[i];
    }
    for (int i = tid; i <= n; i += nthr) sptr[i] = gptr[i];
    ptr = sptr;
    col = scol;
    val = sval;
  }
  double lmax = 0.0;
  for (int i = tid; i < n; i += nthr) {
    const double bi = identity_cols ? (i == jcol ? 1.0 : 0.0) : b[i];
    u[i] = bi;
    x[i] = 0.0;
    lmax = nanmax(lmax, fabs(bi));
  }
  constexpr int VS = E ? 1 : 2;  // 512 row groups: coarse grids of <= 512 rows in one pass
  const int g = tid / VS, gl = tid % VS, ng = nthr / VS;
  // every lane of a group must call this (the shuffles name the whole warp);
  // rows past n contribute an empty range
  auto rowdot = [&](const double* v, int r) {
    double s = 0.0;
    const int kb = r < n ? ptr[r] : 0, ke = r < n ? ptr[r + 1] : 0;
    if (E) {
      for (int k = kb; k < ke; ++k) s = add_rn(s, mul_rn(val[k], v[col[k]]));
    } else {
      for (int k = kb + gl; k < ke; k += VS) s = fma(val[k], v[col[k]], s);
#pragma unroll
      for (int o = VS / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, VS);
    }
    return s;
  };
  auto block_max = [&](double v, int parity) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = nanmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((tid & 31) == 0) red[parity][tid >> 5] = v;
    __syncthreads();
    // every warp reduces the partials itself (no serial 32-step loop, no 2nd barrier)
    double m = (tid & 31) < nw ? red[parity][tid & 31] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = nanmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    return m;
  };
  double nrm = block_max(lmax, 1);
  double scale = 1.0;
  const int rows_pad = ((n + ng - 1) / ng) * ng;  // whole groups iterate together (shuffles)
  for (int k = 0; k < nunits; ++k) {
    lmax = 0.0;
    if (utype[k] == 0) {
      const double t = up1[k];
      const double sc = scale / t;
      if (!isfinite(mul<E>(sc, nrm))) {
        if (stopped && tid == 0) atomicOr(stopped, 1);
        break;
      }
      for (int r = g; r < rows_pad; r += ng) {
        const double s = rowdot(u, r);
        if (gl == 0 && r < n) w[r] = s;
      }
      __syncthreads();
      for (int i = tid; i < n; i += nthr) {
        const double ui = u[i];
        x[i] = E ? add_rn(x[i], mul_rn(sc, ui)) : x[i] + sc * ui;
        const double un = E ? sub_rn(ui, __ddiv_rn(w[i], t)) : ui - w[i] / t;
        u[i] = un;
        lmax = nanmax(lmax, fabs(un));
      }
    } else {
      const double two_a = up1[k], m2 = up2[k];
      const double sc = scale / m2;
      int bad = 0;
      for (int r = g; r < rows_pad; r += ng) {
        const double s = rowdot(u, r);
        if (gl == 0 && r < n) {
          w[r] = s;
          const double d = E ? mul_rn(sc, sub_rn(mul_rn(two_a, u[r]), s)) : sc * (two_a * u[r] - s);
          bad |= !isfinite(d);
        }
      }
      if (__syncthreads_or(bad)) {
        if (stopped && tid == 0) atomicOr(stopped, 1);
        break;
      }
      for (int r = g; r < rows_pad; r += ng) {
        const double z = rowdot(w, r);
        if (gl == 0 && r < n) {
          const double ui = u[r], wi = w[r];
          if (E) {
            x[r] = add_rn(x[r], mul_rn(sc, sub_rn(mul_rn(two_a, ui), wi)));
            u[r] = add_rn(ui, __ddiv_rn(sub_rn(z, mul_rn(two_a, wi)), m2));
          } else {
            x[r] += sc * (two_a * ui - wi);
            u[r] = ui + (z - two_a * wi) / m2;
          }
          lmax = nanmax(lmax, fabs(u[r]));
        }
      }
    }
    nrm = block_max(lmax, k & 1);
    if (nrm == 0.0) break;
    if (nrm > 1e150 || nrm < 1e-150) {
      for (int i = tid; i < n; i += nthr) u[i] = E ? __ddiv_rn(u[i], nrm) : u[i] / nrm;
      scale = E ? mul_rn(scale, nrm) : scale * nrm;
      nrm = 1.0;  // max|u/nrm| == 1 exactly
      __syncthreads();
      if (!isfinite(scale) || scale == 0.0) {
        // scale underflowing to 0 only drops terms that would add 0 * u;
        // an infinite scale drops real terms
        if (stopped && tid == 0) atomicOr(stopped, isfinite(scale) ? 2 : 1);
        break;
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < n; i += nthr) xout[i] = x[i];
}

// Multi-CTA Newton for large coarse grids: host loop over roots with the
// scale / stop state kept on the device.
struct NewtonState {
  double scale;
  int stop;
  double nrm;
};

__global__ void newton_init_kernel(int n, const double* __restrict__ b, double* u, double* x,
                                   NewtonState* st) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    u[i] = b[i];
    x[i] = 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->scale = 1.0;
    st->stop = 0;
    st->nrm = 0.0;
  }
}

// flags[0] = any nonfinite delta; partial max in parts
__global__ void newton_check_kernel(int n, int type, double p1, double p2, const double* u,
                                    const double* w, const NewtonState* st, int* flag) {
  if (st->stop) return;
  const double sc = st->scale / (type == 0 ? p1 : p2);
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    bad |= type == 0 ? !isfinite(sc * u[i]) : !isfinite(sc * (p1 * u[i] - w[i]));
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

template <bool E>
__global__ void newton_rowspmv_kernel(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                      const double* __restrict__ val, const double* in, double* out,
                                      const NewtonState* st, const int* flag) {
  if (st->stop || *flag) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = row_dot<E>(ptr, col, val, in, (int)i);
}

template <bool E>
__global__ void newton_update_kernel(int n, int type, double p1, double p2, double* x, double* u,
                                     const double* w, const double* z, const NewtonState* st,
                                     const int* flag, double* parts) {
  __shared__ double red[33];
  if (st->stop || *flag) return;
  const double sc = st->scale / (type == 0 ? p1 : p2);
  double lmax = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double un;
    if (E) {
      if (type == 0) {
        x[i] = add_rn(x[i], mul_rn(sc, u[i]));
        un = sub_rn(u[i], __ddiv_rn(w[i], p1));
      } else {
        x[i] = add_rn(x[i], mul_rn(sc, sub_rn(mul_rn(p1, u[i]), w[i])));
        un = add_rn(u[i], __ddiv_rn(sub_rn(z[i], mul_rn(p1, w[i])), p2));
      }
    } else if (type == 0) {
      x[i] += sc * u[i];
      un = u[i] - w[i] / p1;
    } else {
      x[i] += sc * (p1 * u[i] - w[i]);
      un = u[i] + (z[i] - p1 * w[i]) / p2;
    }
    u[i] = un;
    lmax = fmax(lmax, fabs(un));
  }
  lmax = block_max(lmax, red);
  if (threadIdx.x == 0) parts[blockIdx.x] = lmax;
}

__global__ void newton_rescale_kernel(int n, int nparts, const double* parts, double* u,
                                      NewtonState* st, int* flag) {
  // single block: reduce partial maxima, decide, rescale
  __shared__ double red[33];
  __shared__ int act;
  if (st->stop) return;
  if (*flag) {
    if (threadIdx.x == 0) st->stop = 1;
    return;
  }
  double m = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) m = fmax(m, parts[i]);
  m = block_max(m, red);
  if (threadIdx.x == 0) {
    act = 0;
    if (m == 0.0) st->stop = 1;
    else if (m > 1e150 || m < 1e-150) act = 1;
    st->nrm = m;
  }
  __syncthreads();
  if (act) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) u[i] /= m;
    if (threadIdx.x == 0) {
      double sc = st->scale * m;
      st->scale = sc;
      if (!isfinite(sc) || sc == 0.0) st->stop = 1;
    }
  }
}

__global__ void neumann_scale_kernel(int n, const double* __restrict__ ds, const double* __restrict__ b,
                                     double* __restrict__ t, double* __restrict__ acc) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double v = ds[i] * b[i];
    t[i] = v;
    acc[i] = v;
  }
}

int neumann_scale(int n, const double* ds, const double* b, double* t, double* acc,
                  cudaStream_t s) {
  neumann_scale_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, ds, b, t, acc);
  ++g_launches;
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

// ---------------------------------------------------------------------------
// Polynomial operator (device-side description used by the plan)
// ---------------------------------------------------------------------------
struct Poly {
  int kind = 0;  // 0 coeff (Horner), 1 newton, 2 neumann
  std::vector<double> coef;
  std::vector<int> utype;
  std::vector<double> p1, p2;
  const double* diag_scale = nullptr;
  int* d_utype = nullptr;
  double* d_p1 = nullptr;
  double* d_p2 = nullptr;
};

constexpr int kNewtonCtaMax = 16384;  // single-CTA Newton up to this many rows
constexpr int kDenseCoarseMax = 2048;  // fast mode: dense Q = q(A) up to this many rows

struct Work {
  double* buf = nullptr;
  size_t cap = 0;
};

template <bool E>
static int newton_multi(const Poly& p, const Csr& A, const double* b, double* y, double* t0,
                        double* t1, double* t2, int* iflag, double* parts, NewtonState* nst,
                        cudaStream_t s) {
  const int n = A.nrows;
  const int nunits = (int)p.utype.size();
  const int thr = 256;
  const int nb = blocks_for(n, thr, num_sms() * 8);
  newton_init_kernel<<<nb, thr, 0, s>>>(n, b, t0, y, nst);
  ++g_launches;
  // SpMVs: the reference-order row kernel in exact mode; otherwise the
  // vector SpMV (lanes per row sized to the operator: the coarsest grids of a
  // truncated hierarchy have hundreds of entries per row).  After a stop the
  // vector SpMV still runs but its output is never used (the update and
  // rescale kernels are gated on the state).
  auto spmv = [&](const double* in, double* out) -> int {
    if (E) {
      newton_rowspmv_kernel<E><<<nb, thr, 0, s>>>(n, A.ptr, A.col, A.val, in, out, nst, iflag);
      ++g_launches;
      AIRG_LAUNCH_CHECK();
      return AIRG_OK;
    }
    Epi ep{out, nullptr, 1.0, 0.0, nullptr, nullptr, nullptr, nullptr};
    return launch_spmv(A, in, 1.0, ep, s, false);
  };
  for (int k = 0; k < nunits; ++k) {
    const int ty = p.utype[k];
    AIRG_CUDA(cudaMemsetAsync(iflag, 0, sizeof(int), s));
    if (ty == 1) AIRG_TRY(spmv(t0, t1));
    newton_check_kernel<<<nb, thr, 0, s>>>(n, ty, p.p1[k], p.p2[k], t0, t1, nst, iflag);
    ++g_launches;
    if (ty == 0) AIRG_TRY(spmv(t0, t1));
    else AIRG_TRY(spmv(t1, t2));
    newton_update_kernel<E><<<nb, thr, 0, s>>>(n, ty, p.p1[k], p.p2[k], y, t0, t1, t2, nst, iflag,
                                            parts);
    newton_rescale_kernel<<<1, 1024, 0, s>>>(n, nb, parts, t0, nst, iflag);
    g_launches += 2;
  }
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

// y = q(A) b using scratch t0..t3 (each n doubles).  ymap: optional scatter
// of the result (y[ymap[i]] = ...).  Only the Horner path supports ymap; the
// caller handles others.
// ymap (coefficient polynomials only): the result lands at y[ymap[i]] (the
// V-cycle scatters e[f] = e_f through it instead of a separate kernel)
static int poly_apply_dev(const Poly& p, const Csr& A, const double* b, double* y, double* t0,
                          double* t1, double* t2, double* t3, int* iflag, double* parts,
                          NewtonState* nst, cudaStream_t s, bool exact,
                          const int* ymap = nullptr) {
  const int n = A.nrows;
  if (n == 0) return AIRG_OK;
  if (ymap && p.kind != 0) {
    set_error("an output map needs a coefficient polynomial");
    return AIRG_ERR_ARG;
  }
  if (p.kind == 0) {
    const int d = (int)p.coef.size() - 1;
    if (d < 0) {
      set_error("empty coefficient polynomial");
      return AIRG_ERR_ARG;
    }
    if (d == 0) return launch_axpby(n, y, ymap, p.coef[0], b, nullptr, 0.0, nullptr, s, exact);
    // y_1 = A (c_d b) + c_{d-1} b ; y_{j} = A y_{j-1} + c_j b
    const double* cur = b;
    double xs = p.coef[d];
    double* bufs[2] = {t0, t1};
    for (int j = d - 1; j >= 0; --j) {
      double* dst = (j == 0) ? y : bufs[j & 1];
      Epi ep{dst, j == 0 ? ymap : nullptr, 1.0, p.coef[j], b, nullptr, nullptr, nullptr};
      AIRG_TRY(launch_spmv(A, cur, xs, ep, s, exact));
      cur = dst;
      xs = 1.0;
    }
    return AIRG_OK;
  }
  if (p.kind == 2) {
    // t = ds*b; acc = t; repeat: t = t - ds*(A t); acc += t
    const int order = (int)p.coef.size() - 1;
    const int thr = 256;
    AIRG_TRY(neumann_scale(n, p.diag_scale, b, t0, y, s));
    double* cur = t0;
    double* nxt = t1;
    for (int it = 0; it < order; ++it) {
      if (exact)
        neumann_step_kernel<true><<<blocks_for(n, thr), thr, 0, s>>>(n, A.ptr, A.col, A.val,
                                                                   p.diag_scale, cur, nxt, y);
      else
        neumann_step_kernel<false><<<blocks_for(n, thr), thr, 0, s>>>(n, A.ptr, A.col, A.val,
                                                                    p.diag_scale, cur, nxt, y);
      ++g_launches;
      AIRG_LAUNCH_CHECK();
      std::swap(cur, nxt);
    }
    return AIRG_OK;
  }
  // Newton
  const int nunits = (int)p.utype.size();
  const size_t vec_bytes = (size_t)3 * n * sizeof(double);
  const size_t mat_bytes = (size_t)A.nnz * 12 + (size_t)(n + 1) * 4;
  const size_t smem_cap = 200 * 1024;
  if (vec_bytes <= smem_cap) {
    const int mat_smem = vec_bytes + mat_bytes <= smem_cap ? 1 : 0;
    const size_t shm = vec_bytes + (mat_smem ? mat_bytes : 0);
    const int thr = 1024;
    if (exact) {
      AIRG_CUDA(cudaFuncSetAttribute(newton_smem_kernel<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap));
      newton_smem_kernel<true><<<1, thr, shm, s>>>(n, A.ptr, A.col, A.val, mat_smem, b, y, nunits,
                                                   p.d_utype, p.d_p1, p.d_p2);
    } else {
      AIRG_CUDA(cudaFuncSetAttribute(newton_smem_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap));
      newton_smem_kernel<false><<<1, thr, shm, s>>>(n, A.ptr, A.col, A.val, mat_smem, b, y, nunits,
                                                    p.d_utype, p.d_p1, p.d_p2);
    }
    ++g_launches;
    AIRG_LAUNCH_CHECK();
    return AIRG_OK;
  }
  if (n <= kNewtonCtaMax) {
    if (exact)
      newton_cta_kernel<true><<<1, 1024, 0, s>>>(n, A.ptr, A.col, A.val, b, y, t0, t1, t2, nunits,
                                                 p.d_utype, p.d_p1, p.d_p2);
    else
      newton_cta_kernel<false><<<1, 1024, 0, s>>>(n, A.ptr, A.col, A.val, b, y, t0, t1, t2, nunits,
                                                  p.d_utype, p.d_p1, p.d_p2);
    ++g_launches;
    AIRG_LAUNCH_CHECK();
    return AIRG_OK;
  }
  return exact ? newton_multi<true>(p, A, b, y, t0, t1, t2, iflag, parts, nst, s)
               : newton_multi<false>(p, A, b, y, t0, t1, t2, iflag, parts, nst, s);
}

static int build_poly(Poly& p, int kind, int ncoef, const double* coef_h, int nunits,
                      const int* type_h, const double* p1_h, const double* p2_h,
                      const double* diag_scale) {
  p.kind = kind;
  p.diag_scale = diag_scale;
  if (kind == 0 || kind == 2) {
    if (ncoef < 1 || !coef_h) {
      set_error("coefficient polynomial needs >= 1 coefficient");
      return AIRG_ERR_ARG;
    }
    p.coef.assign(coef_h, coef_h + ncoef);
    if (kind == 2 && !diag_scale) {
      set_error("neumann polynomial needs diag_scale");
      return AIRG_ERR_ARG;
    }
    return AIRG_OK;
  }
  if (kind != 1) {
    set_error("unknown polynomial kind %d", kind);
    return AIRG_ERR_ARG;
  }
  p.utype.assign(type_h, type_h + nunits);
  p.p1.assign(p1_h, p1_h + nunits);
  p.p2.assign(p2_h, p2_h + nunits);
  if (nunits > 0) {
    AIRG_CUDA(dmalloc(&p.d_utype, nunits * sizeof(int)));
    AIRG_CUDA(dmalloc(&p.d_p1, nunits * sizeof(double)));
    AIRG_CUDA(dmalloc(&p.d_p2, nunits * sizeof(double)));
    AIRG_CUDA(cudaMemcpy(p.d_utype, type_h, nunits * sizeof(int), cudaMemcpyHostToDevice));
    AIRG_CUDA(cudaMemcpy(p.d_p1, p1_h, nunits * sizeof(double), cudaMemcpyHostToDevice));
    AIRG_CUDA(cudaMemcpy(p.d_p2, p2_h, nunits * sizeof(double), cudaMemcpyHostToDevice));
  }
  return AIRG_OK;
}

static void free_poly(Poly& p) {
  if (p.d_utype) dfree(p.d_utype);
  if (p.d_p1) dfree(p.d_p1);
  if (p.d_p2) dfree(p.d_p2);
  p.d_utype = nullptr;
  p.d_p1 = p.d_p2 = nullptr;
}

static Csr make_csr(int nrows, int ncols, const int* ptr, const int* col, const double* val,
                    long long nnz) {
  Csr c;
  c.nrows = nrows;
  c.ncols = ncols;
  c.ptr = ptr;
  c.col = col;
  c.val = val;
  c.nnz = nnz;
  c.vs = pick_vs(nnz, nrows);
  return c;
}

static long long read_nnz(const int* ptr, int nrows) {
  int v = 0;
  if (nrows > 0) cudaMemcpy(&v, ptr + nrows, sizeof(int), cudaMemcpyDeviceToHost);
  return v;
}

}  // namespace airg

using namespace airg;

// ---------------------------------------------------------------------------
// Plan
// ---------------------------------------------------------------------------
struct LevelOps {
  int n = 0, n_f = 0, n_c = 0;
  Csr R, Afc, Aff, Asm;
  bool has_asm = false;
  const int* f_idx = nullptr;
  const int* c_idx = nullptr;
  Poly sm;
  // work vectors (owned)
  double* rc = nullptr;   // n_c : restricted residual (input of the next level)
  double* ec = nullptr;   // n_c : coarse error (output of the next level)
  double* rhs = nullptr;  // n_f
  double* ef = nullptr;   // n_f
  double* t0 = nullptr;   // n_f
  double* t1 = nullptr;   // n_f
  double* t2 = nullptr;   // n_f (extra smooths)
  // fused smoother chain (fast mode): CTA row partition + grid-barrier counter
  int chain_G = 0;        // 0: not prepared / not eligible
  int chain_smem = 0;     // dynamic shared bytes of its launches
  int* chain_part = nullptr;
  unsigned long long* chain_bar = nullptr;
};

struct GraphEntry {
  int kind, level;
  const void* a;
  const void* b;
  int fits;
  bool exact;
  cudaGraphExec_t exec;
  long long nk;  // kernels per replay
  unsigned long long used;  // LRU tick
};

// graphs kept per plan (least recently used evicted); the keys use the
// plan's own staging vectors, so a plan needs one per (operation, level,
// smoothing sweeps, arithmetic mode)
constexpr size_t kMaxGraphs = 32;

struct airg_plan {
  cudaStream_t cs = nullptr;  // plan stream: captures and replays
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::vector<GraphEntry> graphs;
  int nlevels = 0;
  std::vector<LevelOps> lv;
  Csr top;
  Csr coarse;
  Poly coarse_poly;
  double *cw0 = nullptr, *cw1 = nullptr, *cw2 = nullptr, *cw3 = nullptr;  // coarse scratch
  double* r = nullptr;  // top residual
  double* e = nullptr;  // top error
  double* parts = nullptr;
  double* norm_d = nullptr;
  double* norm_h = nullptr;
  double norm_hv = 0.0;
  int* iflag = nullptr;
  NewtonState* nst = nullptr;
  int nparts_cap = 0;
  long long launches = 0;
  bool ready_top = false, ready_coarse = false;
  bool exact = false;  // reference arithmetic order (parity mode)
  double* coarseQ = nullptr;  // dense q(A_coarse) for the fast coarse solve
  int dense_state = 0;  // 0 not built, 1 dense q(A) in use, -1 Newton apply (an
                        // identity column stopped early: q(A) is not linear there)
  // staging vectors: Richardson b / x, V-cycle API input / output; the
  // captured graphs name these, never the caller's buffers
  double *sb = nullptr, *sx = nullptr, *vin = nullptr, *vout = nullptr;
  unsigned long long tick = 0;
  bool ell_done = false;
  std::vector<void*> ell_owned;  // ELL copies of the stencil operators (fast mode)
  // plan build: operator nnz read back in ONE synchronisation (pinned slots
  // filled by async copies, resolved by airg_plan_set_coarse)
  int* nnz_h = nullptr;
  int nnz_slots = 0, nnz_used = 0;
  std::vector<std::pair<Csr*, int>> nnz_pend;
};

// An operator of the plan under construction: its nnz (ptr[nrows]) comes back
// by an async copy into the plan's pinned slots; plan_finish_build fills
// nnz and the lanes per row.
static int plan_csr(airg_plan* p, Csr& c, int nrows, int ncols, const int* ptr, const int* col,
                    const double* val) {
  c = Csr();
  c.nrows = nrows;
  c.ncols = ncols;
  c.ptr = ptr;
  c.col = col;
  c.val = val;
  if (nrows <= 0) return AIRG_OK;
  if (p->nnz_used >= p->nnz_slots) {
    set_error("plan nnz slots exhausted");
    return AIRG_ERR_ARG;
  }
  const int slot = p->nnz_used++;
  AIRG_CUDA(cudaMemcpyAsync(p->nnz_h + slot, ptr + nrows, sizeof(int), cudaMemcpyDeviceToHost, 0));
  p->nnz_pend.push_back({&c, slot});
  return AIRG_OK;
}

// plan vectors: stream-ordered on the legacy stream, made visible to every
// stream by the one synchronisation at the end of the build
static int alloc_vec_async(double** q, long long n) {
  AIRG_CUDA(cudaMallocFromPoolAsync((void**)q, (size_t)(n > 0 ? n : 1) * sizeof(double), lib_pool(), 0));
  return AIRG_OK;
}

static int alloc_vec(double** p, long long n) {
  AIRG_CUDA(dmalloc(p, (n > 0 ? n : 1) * sizeof(double)));
  return AIRG_OK;
}

// ---- ELL (fixed width, column-major slots k*n + i) for the fixed-nnz/row
// structured stencils.  Padding slots (value 0, column = row) follow a row's
// real entries, so the exact mode adds only +-0 after the reference's sums:
// bitwise the CSR exact result.
__global__ void csr_to_ell_kernel(int n, int width, const int* __restrict__ ptr, const int* __restrict__ col,
                                  const double* __restrict__ val, int* __restrict__ ecol,
                                  double* __restrict__ eval, int* __restrict__ overflow) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int b = ptr[i], len = ptr[i + 1] - b;
    if (len > width) atomicExch(overflow, 1);
    for (int k = 0; k < width; ++k) {
      const bool real = k < len;
      ecol[(size_t)k * n + i] = real ? col[b + k] : i;
      eval[(size_t)k * n + i] = real ? val[b + k] : 0.0;
    }
  }
}

template <bool E>
__global__ void __launch_bounds__(256) spmv_ell_kernel(int n, int width, const int* __restrict__ ecol,
                                                       const double* __restrict__ eval,
                                                       const double* __restrict__ x, double* __restrict__ y) {
  pdl_enter();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < width; ++k) {
      const double a = __ldg(eval + (size_t)k * n + i);
      const double xv = __ldg(x + __ldg(ecol + (size_t)k * n + i));
      s = E ? add_rn(s, mul_rn(a, xv)) : fma(a, xv, s);
    }
    y[i] = s;
  }
}

extern "C" {

int airg_version(void) { return 1; }

int airg_last_error(char* buf, int len) {
  if (!buf || len <= 0) return (int)airg::g_err.size();
  snprintf(buf, len, "%s", airg::g_err.c_str());
  return (int)airg::g_err.size();
}

int airg_sm_count(void) {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return v;
}

int airg_spmv(int nrows, const int32_t* ptr, const int32_t* col, const double* val,
              const double* x, double* y, int exact, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nrows < 0) {
    set_error("negative row count");
    return AIRG_ERR_ARG;
  }
  if (nrows == 0) return AIRG_OK;
  if (exact) {
    spmv_exact_kernel<<<blocks_for(nrows, 128), 128, 0, s>>>(nrows, ptr, col, val, x, y);
    AIRG_LAUNCH_CHECK();
    return AIRG_OK;
  }
  Csr A = make_csr(nrows, 0, ptr, col, val, read_nnz(ptr, nrows));
  Epi ep{y, nullptr, 1.0, 0.0, nullptr, nullptr, nullptr, nullptr};
  return launch_spmv(A, x, 1.0, ep, s);
}

int airg_csr_to_ell(int nrows, const int32_t* ptr, const int32_t* col, const double* val, int width,
                    int32_t* ell_col, double* ell_val, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nrows < 0 || width < 0) {
    set_error("negative size");
    return AIRG_ERR_ARG;
  }
  if (nrows == 0 || width == 0) return AIRG_OK;
  int* ovf = nullptr;
  AIRG_TRY(scratch(&ovf, 1, s));
  AIRG_CUDA(cudaMemsetAsync(ovf, 0, sizeof(int), s));
  csr_to_ell_kernel<<<blocks_for(nrows, 256), 256, 0, s>>>(nrows, width, ptr, col, val, ell_col, ell_val, ovf);
  AIRG_LAUNCH_CHECK();
  int h = 0;
  AIRG_CUDA(read_back(&h, ovf, sizeof(int), s));
  release(ovf, s);
  if (h) {
    set_error("a row is longer than the ELL width %d", width);
    return AIRG_ERR_VALUE;
  }
  return AIRG_OK;
}

int airg_spmv_ell(int nrows, int width, const int32_t* ell_col, const double* ell_val, const double* x,
                  double* y, int exact, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nrows < 0 || width < 0) {
    set_error("negative size");
    return AIRG_ERR_ARG;
  }
  if (nrows == 0) return AIRG_OK;
  if (exact) AIRG_CUDA(launch_pdl(spmv_ell_kernel<true>, blocks_for(nrows, 256), 256, s, nrows, width, ell_col, ell_val, x, y));
  else AIRG_CUDA(launch_pdl(spmv_ell_kernel<false>, blocks_for(nrows, 256), 256, s, nrows, width, ell_col, ell_val, x, y));
  return AIRG_OK;
}

int airg_norm2(int n, const double* x, double* out_h, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = blocks_for(n, 256, 1024);
  double* parts = nullptr;
  double* d = nullptr;
  AIRG_TRY(scratch(&parts, nb + 1, s));
  d = parts + nb;
  sumsq_kernel<<<nb, 256, 0, s>>>(n, x, parts);
  finish_norm_kernel<<<1, 1024, 0, s>>>(nb, parts, d);
  AIRG_LAUNCH_CHECK();
  AIRG_CUDA(read_back(out_h, d, sizeof(double), s));
  release(parts, s);
  return AIRG_OK;
}

int airg_poly_apply(int kind, int n, const int32_t* ptr, const int32_t* col, const double* val,
                    int ncoef, const double* coef_h, int nunits, const int32_t* type_h,
                    const double* p1_h, const double* p2_h, const double* diag_scale,
                    const double* b, double* y, int exact, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  Poly p;
  AIRG_TRY(build_poly(p, kind, ncoef, coef_h, nunits, type_h, p1_h, p2_h, diag_scale));
  Csr A = make_csr(n, n, ptr, col, val, read_nnz(ptr, n));
  double* w = nullptr;
  const int nb = blocks_for(n, 256, num_sms() * 8);
  AIRG_TRY(scratch(&w, 4LL * (n > 0 ? n : 1) + nb + 8, s));
  double* parts = w + 4LL * (n > 0 ? n : 1);
  int* iflag = (int*)(parts + nb);
  NewtonState* nst = (NewtonState*)(parts + nb + 2);
  const size_t nn = n > 0 ? n : 1;
  int st = poly_apply_dev(p, A, b, y, w, w + nn, w + 2 * nn, w + 3 * nn, iflag, parts, nst, s,
                          exact != 0);
  release(w, s);
  cudaStreamSynchronize(s);
  free_poly(p);
  return st;
}

int airg_plan_create(int nlevels, airg_plan** out) {
  if (nlevels < 0 || !out) {
    set_error("bad plan arguments");
    return AIRG_ERR_ARG;
  }
  airg_plan* p = new airg_plan();
  p->nlevels = nlevels;
  p->lv.resize(nlevels);
  p->nnz_slots = 3 * nlevels + 4;
  AIRG_CUDA(cudaHostAlloc((void**)&p->nnz_h, sizeof(int) * p->nnz_slots, cudaHostAllocDefault));
  p->norm_h = &p->norm_hv;
  AIRG_CUDA(dmalloc(&p->norm_d, sizeof(double)));
  AIRG_CUDA(dmalloc(&p->iflag, sizeof(int)));
  AIRG_CUDA(dmalloc(&p->nst, sizeof(NewtonState)));
  *out = p;
  return AIRG_OK;
}

int airg_plan_destroy(airg_plan* p) {
  if (!p) return AIRG_OK;
  for (auto& g : p->graphs) cudaGraphExecDestroy(g.exec);
  if (p->cs) {
    cudaStreamSynchronize(p->cs);
    cudaStreamDestroy(p->cs);
    cudaEventDestroy(p->ev_in);
    cudaEventDestroy(p->ev_out);
  }
  for (auto& L : p->lv) {
    for (double* q : {L.rc, L.ec, L.rhs, L.ef, L.t0, L.t1, L.t2})
      if (q) dfree(q);
    if (L.chain_part) dfree(L.chain_part);
    if (L.chain_bar) dfree(L.chain_bar);
    free_poly(L.sm);
  }
  free_poly(p->coarse_poly);
  for (double* q : {p->cw0, p->cw1, p->cw2, p->cw3, p->r, p->e, p->parts, p->norm_d, p->coarseQ,
                    p->sb, p->sx, p->vin, p->vout})
    if (q) dfree(q);
  if (p->iflag) dfree(p->iflag);
  if (p->nst) dfree(p->nst);
  for (void* q : p->ell_owned) dfree(q);
  if (p->nnz_h) cudaFreeHost(p->nnz_h);

  delete p;
  return AIRG_OK;
}

int airg_plan_set_top(airg_plan* p, int n, const int32_t* ptr, const int32_t* col,
                      const double* val) {
  AIRG_TRY(plan_csr(p, p->top, n, n, ptr, col, val));
  AIRG_TRY(alloc_vec_async(&p->r, n));
  AIRG_TRY(alloc_vec_async(&p->e, n));
  p->ready_top = true;  // partials buffer sized at the end of the build
  return AIRG_OK;
}

int airg_plan_set_level(airg_plan* p, int level, int n, int n_f, int n_c, const int32_t* R_ptr,
                        const int32_t* R_col, const double* R_val, const int32_t* Afc_ptr,
                        const int32_t* Afc_col, const double* Afc_val, const int32_t* Aff_ptr,
                        const int32_t* Aff_col, const double* Aff_val, const int32_t* f_idx,
                        const int32_t* c_idx, int kind, int ncoef, const double* coef_h,
                        const double* diag_scale, int64_t asm_nnz, const int32_t* asm_ptr,
                        const int32_t* asm_col, const double* asm_val) {
  if (level < 0 || level >= p->nlevels || n_f + n_c != n) {
    set_error("bad level %d (n=%d n_f=%d n_c=%d)", level, n, n_f, n_c);
    return AIRG_ERR_ARG;
  }
  LevelOps& L = p->lv[level];
  L.n = n;
  L.n_f = n_f;
  L.n_c = n_c;
  AIRG_TRY(plan_csr(p, L.R, n_c, n, R_ptr, R_col, R_val));
  AIRG_TRY(plan_csr(p, L.Afc, n_f, n_c, Afc_ptr, Afc_col, Afc_val));
  AIRG_TRY(plan_csr(p, L.Aff, n_f, n_f, Aff_ptr, Aff_col, Aff_val));
  L.has_asm = asm_nnz >= 0;
  if (L.has_asm) L.Asm = make_csr(n_f, n_f, asm_ptr, asm_col, asm_val, asm_nnz);
  L.f_idx = f_idx;
  L.c_idx = c_idx;
  AIRG_TRY(build_poly(L.sm, kind, ncoef, coef_h, 0, nullptr, nullptr, nullptr, diag_scale));
  AIRG_TRY(alloc_vec_async(&L.rc, n_c));
  AIRG_TRY(alloc_vec_async(&L.ec, n_c));
  AIRG_TRY(alloc_vec_async(&L.rhs, n_f));
  AIRG_TRY(alloc_vec_async(&L.ef, n_f));
  AIRG_TRY(alloc_vec_async(&L.t0, n_f));
  AIRG_TRY(alloc_vec_async(&L.t1, n_f));
  AIRG_TRY(alloc_vec_async(&L.t2, n_f));
  return AIRG_OK;
}

int airg_plan_set_coarse(airg_plan* p, int n, const int32_t* ptr, const int32_t* col,
                         const double* val, int kind, int ncoef, const double* coef_h, int nunits,
                         const int32_t* type_h, const double* p1_h, const double* p2_h,
                         const double* diag_scale) {
  AIRG_TRY(plan_csr(p, p->coarse, n, n, ptr, col, val));
  AIRG_TRY(build_poly(p->coarse_poly, kind, ncoef, coef_h, nunits, type_h, p1_h, p2_h,
                      diag_scale));
  AIRG_TRY(alloc_vec_async(&p->cw0, n));
  AIRG_TRY(alloc_vec_async(&p->cw1, n));
  AIRG_TRY(alloc_vec_async(&p->cw2, n));
  AIRG_TRY(alloc_vec_async(&p->cw3, n));
  // end of the build: one synchronisation resolves every operator's nnz and
  // makes the stream-ordered allocations visible to all streams
  AIRG_CUDA(cudaStreamSynchronize(0));
  for (auto& pr : p->nnz_pend) {
    pr.first->nnz = p->nnz_h[pr.second];
    pr.first->vs = pick_vs(pr.first->nnz, pr.first->nrows);
  }
  p->nnz_pend.clear();
  if (!p->parts) {
    const int nb = p->ready_top ? (int)((p->top.nrows * (long long)p->top.vs + 255) / 256) : 0;
    p->nparts_cap = std::max(nb, num_sms() * 8);
    AIRG_TRY(alloc_vec(&p->parts, p->nparts_cap));
  }
  p->ready_coarse = true;
  return AIRG_OK;
}

}  // extern "C"

// ---- fused smoother chain (chain.cuh) ---------------------------------------
namespace airg {
int scan_counts64(const long long* in, long long* out, int n, long long* total_h, cudaStream_t s);
}
static int chain_smem() {
  static int v = 0;
  if (!v) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    v = std::max(48 * 1024, optin - 1024);
  }
  return v;
}
// AIRG_CHAIN: 0 off, 1 (default) where it measured faster, 2 every eligible level
static int chain_mode() {
  const char* e = getenv("AIRG_CHAIN");
  return e ? atoi(e) : 1;
}
// CTAs for a chain: about kb KB of A_ff per CTA, at most one per SM
static int chain_ctas(const Csr& A) {
  const int kb = getenv("AIRG_CHAIN_KB") ? std::max(1, atoi(getenv("AIRG_CHAIN_KB"))) : 64;
  const long long bytes = 12LL * A.nnz + 12LL * A.nrows;
  const long long g = (bytes + kb * 1024LL - 1) / (kb * 1024LL);
  return (int)std::max(1LL, std::min<long long>(g, num_sms()));
}
// Measured per level at 2048^2 (profiles/r02_vcycle.md): the chain wins on
// the short-row levels (<= 8 entries per row: the per-degree kernels there
// are launch- and L2-miss-bound), and loses or ties where rows are long
// (one row's gathers are the latency chain of every step, and a grid barrier
// costs about what a graph-replayed kernel boundary does).
static bool chain_eligible(const LevelOps& L) {
  const int d = (int)L.sm.coef.size() - 1;
  const int mode = chain_mode();
  return mode > 0 && (mode == 2 || L.Aff.vs <= 2) && !L.has_asm && L.sm.kind == 0 && d >= 2 &&
         d <= kChainMaxDeg && L.n_f > 0;
}
static int prepare_chain(LevelOps& L, cudaStream_t s) {
  if (L.chain_G || !chain_eligible(L)) return AIRG_OK;
  const int G = chain_ctas(L.Aff);
  // only where the whole A_ff stages into shared memory: a partly staged
  // chain re-reads the rest every step and measured no faster than the
  // one-launch-per-degree path (tools/micro/chain_bench.cu)
  const bool partial = getenv("AIRG_CHAIN_CAP") || getenv("AIRG_CHAIN_PARTIAL");
  if (!partial && 12LL * L.Aff.nnz + 4LL * L.n_f + 256LL * G > (long long)G * (chain_smem() - 128))
    return AIRG_OK;
  AIRG_CUDA(dmalloc(&L.chain_part, sizeof(int) * (3 * G + 1)));
  AIRG_CUDA(cudaMemsetAsync(L.chain_part + 3 * G, 0, sizeof(int), s));
  AIRG_CUDA(dmalloc(&L.chain_bar, sizeof(unsigned long long)));
  AIRG_CUDA(cudaMemsetAsync(L.chain_bar, 0, sizeof(unsigned long long), s));
  // staging capacity per CTA (AIRG_CHAIN_CAP lowers it: tests of the unstaged rows)
  long long cap = chain_smem() - 128;
  if (getenv("AIRG_CHAIN_CAP")) cap = std::min(cap, atoll(getenv("AIRG_CHAIN_CAP")));
  long long *cost = nullptr, *w = nullptr;
  AIRG_TRY(scratch(&cost, (size_t)L.n_f, s));
  AIRG_TRY(scratch(&w, (size_t)L.n_f + 1, s));
  chain_cost_kernel<<<blocks_for(L.n_f, 256), 256, 0, s>>>(L.n_f, L.Aff.ptr, L.Aff.vs, cost);
  AIRG_LAUNCH_CHECK();
  AIRG_TRY(airg::scan_counts64(cost, w, L.n_f, nullptr, s));
  chain_partition_kernel<<<(G + 127) / 128, 128, 0, s>>>(L.n_f, L.Aff.ptr, G, cap, w, L.chain_part);
  AIRG_LAUNCH_CHECK();
  release(cost, s);
  release(w, s);
  int need = 0;  // one read per level at plan build: the launch's shared bytes
  AIRG_CUDA(read_back(&need, L.chain_part + 3 * G, sizeof(int), s));
  L.chain_smem = std::min(chain_smem(), ((need + 1023) / 1024) * 1024 + 1024);
  L.chain_G = G;
  return AIRG_OK;
}
template <int VS>
static cudaError_t chain_launch_vs(const ChainArgs& a, int G, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(chain_kernel<VS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         chain_smem());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kChainThreads);
  cfg.dynamicSmemBytes = a.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, chain_kernel<VS>, a);
}
// e[ymap] = q(A_ff) rhs in one launch
static int launch_chain(LevelOps& L, const double* rhs, double* y, const int* ymap, cudaStream_t s) {
  ChainArgs a{};
  a.n = L.n_f;
  a.ptr = L.Aff.ptr;
  a.col = L.Aff.col;
  a.val = L.Aff.val;
  a.b = rhs;
  a.t0 = L.t0;
  a.t1 = L.t1;
  a.y = y;
  a.ymap = ymap;
  a.part = L.chain_part;
  a.bar = L.chain_bar;
  a.d = (int)L.sm.coef.size() - 1;
  a.smem = L.chain_smem;
  for (int j = 0; j <= a.d; ++j) a.coef[j] = L.sm.coef[j];
  switch (L.Aff.vs) {
    case 1: AIRG_CUDA(chain_launch_vs<1>(a, L.chain_G, s)); break;
    case 2: AIRG_CUDA(chain_launch_vs<2>(a, L.chain_G, s)); break;
    case 4: AIRG_CUDA(chain_launch_vs<4>(a, L.chain_G, s)); break;
    case 8: AIRG_CUDA(chain_launch_vs<8>(a, L.chain_G, s)); break;
    case 16: AIRG_CUDA(chain_launch_vs<16>(a, L.chain_G, s)); break;
    default: AIRG_CUDA(chain_launch_vs<32>(a, L.chain_G, s)); break;
  }
  ++g_launches;
  return AIRG_OK;
}

// smoother application on one level: ef = q(A_ff) rhs  (or assembled SpMV)
static int smooth_level(airg_plan* p, LevelOps& L, const double* rhs, double* out, cudaStream_t s) {
  if (L.has_asm) {
    Epi ep{out, nullptr, 1.0, 0.0, nullptr, nullptr, nullptr, nullptr};
    return launch_spmv(L.Asm, rhs, 1.0, ep, s, p->exact);
  }
  return poly_apply_dev(L.sm, L.Aff, rhs, out, L.t0, L.t1, L.t2, L.t2, p->iflag, p->parts, p->nst,
                        s, p->exact);
}

// y = Q r, Q column-major n x n (coalesced over rows)
// block = 32 rows x 8 column slices; lanes read 32 consecutive rows (256 B)
__global__ void __launch_bounds__(256) dense_gemv_kernel(int n, const double* __restrict__ Q,
                                                         const double* __restrict__ r,
                                                         double* __restrict__ y) {
  __shared__ double part[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  if (i < n) {
    int j = w;
    for (; j + 24 < n; j += 32) {
#pragma unroll
      for (int q = 0; q < 4; ++q) s[q] = fma(__ldg(Q + (size_t)(j + 8 * q) * n + i), __ldg(r + j + 8 * q), s[q]);
    }
    for (; j < n; j += 8) s[0] = fma(__ldg(Q + (size_t)j * n + i), __ldg(r + j), s[0]);
  }
  part[w][lane] = (s[0] + s[1]) + (s[2] + s[3]);
  __syncthreads();
  if (w == 0 && i < n) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += part[q][lane];
    y[i] = t;
  }
}

// Q = q(A_coarse) applied to every identity column, one CTA per column.
static int build_dense_coarse(airg_plan* p, cudaStream_t s) {
  const int n = p->coarse.nrows;
  AIRG_CUDA(dmalloc(&p->coarseQ, (size_t)n * n * sizeof(double)));
  AIRG_CUDA(cudaMemsetAsync(p->iflag, 0, sizeof(int), s));
  const Poly& cp = p->coarse_poly;
  const Csr& A = p->coarse;
  const size_t vec_bytes = (size_t)3 * n * sizeof(double);
  const size_t mat_bytes = (size_t)A.nnz * 12 + (size_t)(n + 1) * 4;
  const size_t cap = 200 * 1024;
  const int mat_smem = vec_bytes + mat_bytes <= cap ? 1 : 0;
  const size_t shm = vec_bytes + (mat_smem ? mat_bytes : 0);
  AIRG_CUDA(cudaFuncSetAttribute(newton_smem_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)cap));
  newton_smem_kernel<false><<<n, 256, shm, s>>>(n, A.ptr, A.col, A.val, mat_smem, nullptr,
                                                p->coarseQ, (int)cp.utype.size(), cp.d_utype,
                                                cp.d_p1, cp.d_p2, 1, p->iflag);
  ++g_launches;
  AIRG_LAUNCH_CHECK();
  int stopped = 0;
  AIRG_CUDA(read_back(&stopped, p->iflag, sizeof(int), s));
  if (stopped & 1) {  // the reference stops per right-hand side (polynomial.py:312-355)
    dfree(p->coarseQ);
    p->coarseQ = nullptr;
    p->dense_state = -1;
  } else {
    p->dense_state = 1;
  }
  return AIRG_OK;
}

// V-cycle from `level` with residual r (size n_level) -> e (size n_level).
static int vcycle_rec(airg_plan* p, int level, const double* r, double* e, int fits,
                      cudaStream_t s) {
  if (level == p->nlevels) {
    if (!p->ready_coarse) {
      set_error("plan has no coarse solver");
      return AIRG_ERR_ARG;
    }
    if (!p->exact && p->coarse_poly.kind == 1 && p->coarse.nrows <= kDenseCoarseMax &&
        p->dense_state >= 0) {
      // fast mode: y = Q r with Q = q(A_coarse) precomputed column by column
      if (p->dense_state == 0) AIRG_TRY(build_dense_coarse(p, s));
    }
    if (!p->exact && p->coarse_poly.kind == 1 && p->dense_state == 1) {
      const int n = p->coarse.nrows;
      dense_gemv_kernel<<<(n + 31) / 32, 256, 0, s>>>(n, p->coarseQ, r, e);
      ++g_launches;
      AIRG_LAUNCH_CHECK();
      return AIRG_OK;
    }
    return poly_apply_dev(p->coarse_poly, p->coarse, r, e, p->cw0, p->cw1, p->cw2, p->cw3,
                          p->iflag, p->parts, p->nst, s, p->exact);
  }
  LevelOps& L = p->lv[level];
  // r_c = R r
  {
    Epi ep{L.rc, nullptr, 1.0, 0.0, nullptr, nullptr, nullptr, nullptr};
    AIRG_TRY(launch_spmv(L.R, r, 1.0, ep, s, p->exact));
  }
  AIRG_TRY(vcycle_rec(p, level + 1, L.rc, L.ec, fits, s));
  // degree-0 smoother (e.g. the finest level, whose A_ff is diagonal):
  // e[f] = c0 (r[f] - A_fc e_c) straight from the A_fc launch's epilogue,
  // no rhs vector, no second launch (fast mode; exact mode keeps the
  // reference's two roundings)
  if (fits == 1 && !p->exact && !L.has_asm && L.sm.kind == 0 && L.sm.coef.size() == 1 &&
      L.Afc.nrows > 0) {
    const double c0 = L.sm.coef[0];
    Epi ep{e, L.f_idx, -c0, c0, r, L.f_idx, nullptr, nullptr};
    ep.sc_src = L.ec;
    ep.sc_idx = L.c_idx;
    ep.sc_dst = e;
    ep.sc_n = L.n_c;
    return launch_spmv(L.Afc, L.ec, 1.0, ep, s, false);
  }
  // rhs = r[f] - A_fc e_c, and (same launch) the scatter e[c] = e_c
  {
    Epi ep{L.rhs, nullptr, -1.0, 1.0, r, L.f_idx, nullptr, nullptr};
    ep.sc_src = L.ec;
    ep.sc_idx = L.c_idx;
    ep.sc_dst = e;
    ep.sc_n = L.Afc.nrows > 0 ? L.n_c : 0;
    AIRG_TRY(launch_spmv(L.Afc, L.ec, 1.0, ep, s, p->exact));
    if (L.Afc.nrows == 0)
      AIRG_TRY(launch_axpby(L.n_c, e, L.c_idx, 1.0, L.ec, nullptr, 0.0, nullptr, s, p->exact));
  }
  if (fits == 1 && !p->exact && L.chain_G > 0)  // fused chain: A_ff staged once
    return launch_chain(L, L.rhs, e, L.f_idx, s);
  if (fits == 1 && !L.has_asm && L.sm.kind == 0) {
    // e[f] = q(A_ff) rhs written straight through f_idx by the last Horner step
    AIRG_TRY(poly_apply_dev(L.sm, L.Aff, L.rhs, e, L.t0, L.t1, L.t2, L.t2, p->iflag, p->parts,
                            p->nst, s, p->exact, L.f_idx));
    return AIRG_OK;
  }
  AIRG_TRY(smooth_level(p, L, L.rhs, L.ef, s));
  for (int it = 1; it < fits; ++it) {
    // t1 = rhs - A_ff ef ; ef += q(A_ff) t1
    Epi ep{L.t1, nullptr, -1.0, 1.0, L.rhs, nullptr, nullptr, nullptr};
    AIRG_TRY(launch_spmv(L.Aff, L.ef, 1.0, ep, s, p->exact));
    double* tmp = nullptr;
    AIRG_TRY(scratch(&tmp, 2 * (size_t)(L.n_f > 0 ? L.n_f : 1), s));
    AIRG_CUDA(cudaMemcpyAsync(tmp, L.t1, L.n_f * sizeof(double), cudaMemcpyDeviceToDevice, s));
    double* corr = tmp + (L.n_f > 0 ? L.n_f : 1);
    AIRG_TRY(smooth_level(p, L, tmp, corr, s));
    AIRG_TRY(launch_axpby(L.n_f, L.ef, nullptr, 1.0, L.ef, nullptr, 1.0, corr, s, p->exact));
    release(tmp, s);
  }
  // scatter e[f] = ef (e[c] = ec went with the A_fc launch)
  AIRG_TRY(launch_axpby(L.n_f, e, L.f_idx, 1.0, L.ef, nullptr, 0.0, nullptr, s, p->exact));
  return AIRG_OK;
}

// ---------------------------------------------------------------------------
// CUDA-graph replay: a V-cycle is ~170 dependent launches; capturing it once
// per (operation, vectors) removes the host launch gaps between them.
// ---------------------------------------------------------------------------
static bool graphs_enabled() {
  static int v = -1;
  if (v < 0) v = getenv("AIRG_NO_GRAPH") ? 0 : 1;
  return v == 1;
}

static int plan_streams(airg_plan* p) {
  if (!p->cs) {
    AIRG_CUDA(cudaStreamCreateWithFlags(&p->cs, cudaStreamNonBlocking));
    AIRG_CUDA(cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming));
    AIRG_CUDA(cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming));
  }
  return AIRG_OK;
}

// ---- ELL copies of fixed-width operators ------------------------------------
__global__ void row_maxlen_kernel(int n, const int* __restrict__ ptr, int* __restrict__ out) {
  int m = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    m = max(m, ptr[i + 1] - ptr[i]);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}
__global__ void csr_to_ell_pad_kernel(int n, int w, const int* __restrict__ ptr, const int* __restrict__ col,
                                      const double* __restrict__ val, int* __restrict__ ecol,
                                      double* __restrict__ eval) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int b = ptr[i], len = ptr[i + 1] - b;
    const int pad = len > 0 ? col[b + len - 1] : 0;  // a valid column, value 0
    for (int k = 0; k < w; ++k) {
      ecol[(size_t)k * n + i] = k < len ? col[b + k] : pad;
      eval[(size_t)k * n + i] = k < len ? val[b + k] : 0.0;
    }
  }
}
// Give A an ELL copy when its rows are short and nearly uniform (<= 4
// entries, >= AIRG_ELL_FILL of the slots real): the top operator (3 per
// row) and the finest A_fc (2 per row) of the advection hierarchies.  Off
// by default: measured at 2048^2 (tools/vlevels.py) the finest A_fc took
// 40.4 us in ELL vs 38.1 us in CSR and the finest R (fill 0.71) 34.7 vs
// 31.0 us -- the CSR kernel's thread-per-row loads are already coalesced
// for 2-3-entry rows, and the row-offset load it saves is not the
// bottleneck.  AIRG_ELL_FILL=0.9 enables it.
static int make_ell(airg_plan* p, Csr& A, cudaStream_t s) {
  const double fill = getenv("AIRG_ELL_FILL") ? atof(getenv("AIRG_ELL_FILL")) : 2.0;
  if (A.nrows == 0 || A.ew > 0 || fill > 1.0) return AIRG_OK;
  int* d = nullptr;
  AIRG_TRY(scratch(&d, 1, s));
  AIRG_CUDA(cudaMemsetAsync(d, 0, sizeof(int), s));
  row_maxlen_kernel<<<blocks_for(A.nrows, 256), 256, 0, s>>>(A.nrows, A.ptr, d);
  AIRG_LAUNCH_CHECK();
  int w = 0;
  AIRG_CUDA(read_back(&w, d, sizeof(int), s));
  release(d, s);
  if (w < 1 || w > 4 || (double)A.nnz < fill * (double)A.nrows * w) return AIRG_OK;
  int* ecol = nullptr;
  double* eval = nullptr;
  AIRG_CUDA(dmalloc(&ecol, (size_t)w * A.nrows * sizeof(int)));
  AIRG_CUDA(dmalloc(&eval, (size_t)w * A.nrows * sizeof(double)));
  p->ell_owned.push_back(ecol);
  p->ell_owned.push_back(eval);
  csr_to_ell_pad_kernel<<<blocks_for(A.nrows, 256), 256, 0, s>>>(A.nrows, w, A.ptr, A.col, A.val, ecol,
                                                                 eval);
  AIRG_LAUNCH_CHECK();
  A.ew = w;
  A.ecol = ecol;
  A.eval = eval;
  return AIRG_OK;
}

// things a capture must not do (synchronous allocation) are done up front
static int prepare_capture(airg_plan* p, cudaStream_t s) {
  if (!p->exact && p->ready_coarse && p->coarse_poly.kind == 1 &&
      p->coarse.nrows <= kDenseCoarseMax && p->dense_state == 0)
    AIRG_TRY(build_dense_coarse(p, s));
  if (!p->exact) {
    for (auto& L : p->lv) AIRG_TRY(prepare_chain(L, s));
    if (!p->ell_done) {  // the finest level's stencil operators
      p->ell_done = true;
      if (p->ready_top) AIRG_TRY(make_ell(p, p->top, s));
      if (!p->lv.empty()) {
        AIRG_TRY(make_ell(p, p->lv[0].R, s));
        AIRG_TRY(make_ell(p, p->lv[0].Afc, s));
      }
    }
  }
  return AIRG_OK;
}

template <class F>
static int run_graph(airg_plan* p, int kind, int level, const void* a, const void* b, int fits,
                     cudaStream_t cs, F&& issue) {
  if (!graphs_enabled()) return issue(cs);
  GraphEntry* ent = nullptr;
  for (auto& g : p->graphs)
    if (g.kind == kind && g.level == level && g.a == a && g.b == b && g.fits == fits &&
        g.exact == p->exact)
      ent = &g;
  if (!ent && p->graphs.size() >= kMaxGraphs) {  // evict the least recently used
    auto lru = std::min_element(p->graphs.begin(), p->graphs.end(),
                                [](const GraphEntry& x, const GraphEntry& y) { return x.used < y.used; });
    AIRG_CUDA(cudaStreamSynchronize(cs));
    cudaGraphExecDestroy(lru->exec);
    p->graphs.erase(lru);
  }
  if (!ent) {
    const long long l0 = g_launches;
    AIRG_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
    const int st = issue(cs);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
    if (st != AIRG_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    AIRG_CUDA(ce);
    cudaGraphExec_t ex = nullptr;
    AIRG_CUDA(cudaGraphInstantiate(&ex, graph, 0));
    cudaGraphDestroy(graph);
    p->graphs.push_back(GraphEntry{kind, level, a, b, fits, p->exact, ex, g_launches - l0, 0});
    ent = &p->graphs.back();
    g_launches = l0;
  }
  ent->used = ++p->tick;
  AIRG_CUDA(cudaGraphLaunch(ent->exec, cs));
  g_launches += ent->nk;
  return AIRG_OK;
}

extern "C" {

int airg_plan_vcycle(airg_plan* p, int level, const double* r, double* e, int f_smooth_its,
                     void* stream) {
  if (level < 0 || level > p->nlevels) {
    set_error("level %d out of range", level);
    return AIRG_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int fits = f_smooth_its < 1 ? 1 : f_smooth_its;
  AIRG_TRY(plan_streams(p));
  AIRG_TRY(prepare_capture(p, s));
  const int n = level == p->nlevels ? p->coarse.nrows : p->lv[level].n;
  const int nmax = p->nlevels ? p->lv[0].n : p->coarse.nrows;
  if (!p->vin) {
    AIRG_TRY(alloc_vec(&p->vin, nmax));
    AIRG_TRY(alloc_vec(&p->vout, nmax));
  }
  if (r != p->vin)
    AIRG_CUDA(cudaMemcpyAsync(p->vin, r, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  AIRG_CUDA(cudaEventRecord(p->ev_in, s));
  AIRG_CUDA(cudaStreamWaitEvent(p->cs, p->ev_in, 0));
  AIRG_TRY(run_graph(p, 0, level, p->vin, p->vout, fits, p->cs,
                     [&](cudaStream_t t) { return vcycle_rec(p, level, p->vin, p->vout, fits, t); }));
  AIRG_CUDA(cudaEventRecord(p->ev_out, p->cs));
  AIRG_CUDA(cudaStreamWaitEvent(s, p->ev_out, 0));
  if (e != p->vout)
    AIRG_CUDA(cudaMemcpyAsync(e, p->vout, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  return AIRG_OK;
}

// the plan's staging vectors (size of the finest level); a V-cycle called on
// them runs without copying in / out
int airg_plan_staging(airg_plan* p, double** vin, double** vout) {
  const int nmax = p->nlevels ? p->lv[0].n : p->coarse.nrows;
  if (!p->vin) {
    AIRG_TRY(alloc_vec(&p->vin, nmax));
    AIRG_TRY(alloc_vec(&p->vout, nmax));
  }
  *vin = p->vin;
  *vout = p->vout;
  return AIRG_OK;
}

int airg_copy_d2d(void* dst, const void* src, int64_t bytes, void* stream) {
  AIRG_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return AIRG_OK;
}

int airg_plan_graph_count(airg_plan* p) { return p ? (int)p->graphs.size() : 0; }

int airg_plan_coarse_mode(airg_plan* p) {
  // 1: fast-mode coarse solve is the dense q(A) GEMV; 0: Newton apply
  return p && p->dense_state == 1 ? 1 : 0;
}

int64_t airg_plan_launches(airg_plan* p) { return p ? p->launches : 0; }

int airg_plan_set_exact(airg_plan* p, int exact) {
  p->exact = exact != 0;
  return AIRG_OK;
}

}  // extern "C"

// r = b - A x with the fixed-order norm reduction into p->norm_d (stream-ordered)
static int residual_launch(airg_plan* p, const double* b, const double* x, cudaStream_t s) {
  const Csr& A = p->top;
  const int nb = p->exact ? (A.nrows + 255) / 256 : spmv_blocks(A);  // blocks of the launch below
  double* parts = p->parts;
  if (nb > p->nparts_cap) {
    set_error("partials buffer too small");
    return AIRG_ERR_ARG;
  }
  Epi ep{p->r, nullptr, -1.0, 1.0, b, nullptr, nullptr, parts};
  AIRG_TRY(launch_spmv(A, x, 1.0, ep, s, p->exact));
  finish_norm_kernel<<<1, 1024, 0, s>>>(nb, parts, p->norm_d);
  ++g_launches;
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

// r = b - A x, with deterministic norm into p->norm_h (synchronous)
static int residual_norm(airg_plan* p, const double* b, const double* x, double* rnorm,
                         cudaStream_t s) {
  AIRG_TRY(residual_launch(p, b, x, s));
  AIRG_CUDA(read_back(p->norm_h, p->norm_d, sizeof(double), s));
  *rnorm = *p->norm_h;
  return AIRG_OK;
}

static int richardson_body(airg_plan* p, const double* b, double* x, double rtol, double atol,
                           int max_iters, int f_smooth_its, double* history, int* iterations,
                           int* converged, cudaStream_t s);

extern "C" int airg_plan_richardson(airg_plan* p, const double* b, double* x, double rtol,
                                    double atol, int max_iters, int f_smooth_its,
                                    double* history, int* iterations, int* converged,
                                    void* stream) {
  cudaStream_t caller = (cudaStream_t)stream;
  if (!p->ready_top) {
    set_error("plan has no top matrix");
    return AIRG_ERR_ARG;
  }
  AIRG_TRY(plan_streams(p));
  AIRG_TRY(prepare_capture(p, caller));
  AIRG_CUDA(cudaEventRecord(p->ev_in, caller));
  AIRG_CUDA(cudaStreamWaitEvent(p->cs, p->ev_in, 0));
  cudaStream_t s = p->cs;
  const int n = p->top.nrows;
  if (!p->sb) {
    AIRG_TRY(alloc_vec(&p->sb, n));
    AIRG_TRY(alloc_vec(&p->sx, n));
  }
  AIRG_CUDA(cudaMemcpyAsync(p->sb, b, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  AIRG_CUDA(cudaMemcpyAsync(p->sx, x, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  const int st = richardson_body(p, p->sb, p->sx, rtol, atol, max_iters, f_smooth_its, history,
                                 iterations, converged, s);
  cudaMemcpyAsync(x, p->sx, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s);
  cudaEventRecord(p->ev_out, s);
  cudaStreamWaitEvent(caller, p->ev_out, 0);
  return st;
}

static int richardson_body(airg_plan* p, const double* b, double* x, double rtol, double atol,
                           int max_iters, int f_smooth_its, double* history, int* iterations,
                           int* converged, cudaStream_t s) {
  const long long l0 = g_launches;
  const int n = p->top.nrows;
  const int fits = f_smooth_its < 1 ? 1 : f_smooth_its;
  double bnorm = 0.0, rnorm = 0.0;
  {
    // ||b|| with the same fixed-order reduction
    const int nb = blocks_for(n, 256, 1024);
    sumsq_kernel<<<nb, 256, 0, s>>>(n, b, p->parts);
    finish_norm_kernel<<<1, 1024, 0, s>>>(nb, p->parts, p->norm_d);
    g_launches += 2;
    AIRG_LAUNCH_CHECK();
    AIRG_CUDA(read_back(p->norm_h, p->norm_d, sizeof(double), s));
    bnorm = *p->norm_h;
  }
  AIRG_TRY(residual_norm(p, b, x, &rnorm, s));
  history[0] = rnorm;
  const double ref = bnorm > 0 ? bnorm : rnorm;
  const double thr = std::max(rtol * ref, atol);
  *iterations = 0;
  *converged = 0;
  if (!std::isfinite(rnorm)) {
    set_error("non-finite residual at iteration 0");
    return AIRG_ERR_DIVERGED;
  }
  bool conv = rnorm <= thr;
  int its = 0;
  while (!conv && its < max_iters) {
    // x += V-cycle(r); r = b - A x; ||r|| partials -> one captured graph
    AIRG_TRY(run_graph(p, 1, 0, b, x, fits, s, [&](cudaStream_t t) {
      AIRG_TRY(vcycle_rec(p, 0, p->r, p->e, fits, t));
      AIRG_TRY(launch_axpby(n, x, nullptr, 1.0, x, nullptr, 1.0, p->e, t, p->exact));
      return residual_launch(p, b, x, t);
    }));
    AIRG_CUDA(read_back(p->norm_h, p->norm_d, sizeof(double), s));
    rnorm = *p->norm_h;
    ++its;
    history[its] = rnorm;
    *iterations = its;
    if (!std::isfinite(rnorm)) {
      set_error("non-finite residual at iteration %d", its);
      p->launches = g_launches - l0;
      return AIRG_ERR_DIVERGED;
    }
    if (rnorm > 1e8 * history[0]) {
      set_error("residual grew by more than 1e+08 at iteration %d", its);
      p->launches = g_launches - l0;
      return AIRG_ERR_DIVERGED;
    }
    conv = rnorm <= thr;
  }
  *converged = conv ? 1 : 0;
  p->launches = g_launches - l0;
  return AIRG_OK;
}

// ===========================================================================
// Row-strip distributed V-cycle / Richardson.
// Each distributed level keeps R, A_fc, A_ff on local rows with columns in
// the ext space [local | ghost].  Ghost values travel over NVLink by direct
// peer stores: every vector that receives ghosts lives in one cudaMalloc
// arena per rank, shared with the other ranks through CUDA IPC; a put kernel
// gathers the send entries and stores them straight into the peers' ghost
// tails, then publishes a per-(sender, receiver) message count with a
// system-scope release; the consumer's wait kernel acquires it.  Flags flow
// both ways between every pair that shares a halo (also when one direction
// carries no data), which is what makes reusing the ghost tails safe: a
// sender can only overwrite a tail after the receiver's flag for a later
// exchange, which the receiver issues after consuming the tail.  The norm
// allreduce and the replicated-tail gather use the same put/flag scheme, so
// an iteration contains no NCCL call and is one captured CUDA graph.
// NCCL (pack + grouped send/recv) remains as the transport when IPC is not
// available (AIRG_DPLAN_NCCL=1 forces it); it also carries the one-time
// exchange of IPC handles at plan build.
// ===========================================================================
#define AIRG_NCCL(call)                                                          \
  do {                                                                           \
    ncclResult_t _r = (call);                                                    \
    if (_r != ncclSuccess) {                                                     \
      ::airg::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,              \
                        ncclGetErrorString(_r));                                 \
      return AIRG_ERR_CUDA;                                                      \
    }                                                                            \
  } while (0)

namespace airg {

constexpr int kMaxPeers = 8;

struct HaloX {
  int n_loc = 0, nsend = 0, nrecv = 0;
  int* send_idx = nullptr;
  double* sendbuf = nullptr;  // NCCL transport
  std::vector<int> scnt, sofs, rcnt, rofs;
};

// one put: entries [sofs[j], sofs[j+1]) of the gathered send list go to dst[j]
// (idx == nullptr: entry i is x[i - sofs[j]]); rflag[j] (null = local copy)
// receives the new message count for peer[j]
struct PutDesc {
  int nsend = 0;
  const int* idx = nullptr;
  int npeer = 0;
  int sofs[kMaxPeers + 2] = {};
  double* dst[kMaxPeers + 1] = {};
  unsigned long long* rflag[kMaxPeers + 1] = {};
  int peer[kMaxPeers + 1] = {};
};

struct WaitDesc {
  int npeer = 0;
  int peer[kMaxPeers] = {};
};

struct NormDesc {
  int npeer = 0, me = 0, world = 1;
  int peer[kMaxPeers] = {};
  double* slots[kMaxPeers] = {};             // peer's slot array (2 x world)
  unsigned long long* rflag[kMaxPeers] = {};
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// gathers and stores the send entries into the peers' ghost tails, then (last
// CTA) publishes the new message counts, raises the expected counts of the
// messages this exchange receives and waits for them: the kernel completes
// only once the peers' ghost values have landed, so the consuming kernel needs
// no separate wait launch (its griddepcontrol.wait / stream order is the
// acquire edge)
__global__ void put_kernel(PutDesc d, WaitDesc w, const double* __restrict__ x,
                           unsigned long long* sent, unsigned long long* expect,
                           unsigned int* ticket, const unsigned long long* flags) {
  pdl_enter();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d.nsend; i += gridDim.x * blockDim.x) {
    int q = 0;
    while (i >= d.sofs[q + 1]) ++q;
    d.dst[q][i - d.sofs[q]] = d.idx ? x[d.idx[i]] : x[i - d.sofs[q]];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // cumulative over the CTA's stores ordered by the barrier
    const unsigned t = atomicAdd(ticket, 1u);
    if (t == gridDim.x - 1) {  // last CTA: every CTA's stores are fenced
      *ticket = 0u;
      __threadfence_system();
      for (int j = 0; j < d.npeer; ++j)
        if (d.rflag[j]) {
          st_release_sys(d.rflag[j], ++sent[d.peer[j]]);
          ++expect[d.peer[j]];
        }
      for (int j = 0; j < w.npeer; ++j) wait_count(flags + w.peer[j], expect[w.peer[j]]);
    }
  }
}

// ---- LL halo exchange (no system-scope fences) -------------------------------
// Every ghost value travels as one 16-byte slot {lo32, flag, hi32, flag}
// written with a single vector store (NCCL's LL format: each 8-byte
// (data, flag) half lands atomically), so the receiver needs no fence: it polls
// the slots of its own LL region until both flags equal the exchange's
// sequence number and copies the values into the vector's ghost tail.  Each
// message also carries a header slot, so every exchange is a two-way handshake
// between halo partners even when one direction has no data.  Per partner
// pair the sequence number counts the exchanges; its parity selects one of two
// slot banks: the sender can only reuse a bank after the receiver has sent the
// next message, i.e. finished the kernel that drained it.
struct LLDesc {
  int nsend = 0, nrecv = 0;
  const int* idx = nullptr;
  int npeer = 0;
  int peer[kMaxPeers] = {};
  int sofs[kMaxPeers + 1] = {};          // send segments per partner
  int rofs[kMaxPeers + 1] = {};          // ghost-tail segments per partner
  uint4* rdst[kMaxPeers] = {};           // partner's LL region for me
  int rcap[kMaxPeers] = {};              // slots per bank there
  const uint4* lsrc[kMaxPeers] = {};     // my LL region for the partner
  int lcap[kMaxPeers] = {};
  double* ghost = nullptr;               // target vector + n_loc
};

__device__ __forceinline__ void st_ll(uint4* p, double v, unsigned f) {
  const unsigned long long u = __double_as_longlong(v);
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"((unsigned)u), "r"(f),
               "r"((unsigned)(u >> 32)), "r"(f)
               : "memory");
}

__device__ __forceinline__ double ld_ll(const uint4* p, unsigned f) {
  unsigned a, b, c, d;
  const long long t0 = clock64();
  for (;;) {
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "l"(p)
                 : "memory");
    if (b == f && d == f) break;
    if (clock64() - t0 > 40000000000ll) __trap();
  }
  return __longlong_as_double((long long)(((unsigned long long)c << 32) | a));
}

__global__ void ll_halo_kernel(LLDesc d, const double* __restrict__ x, unsigned long long* seq,
                               unsigned int* ticket) {
  pdl_enter();
  unsigned f[kMaxPeers];
#pragma unroll
  for (int j = 0; j < kMaxPeers; ++j) f[j] = j < d.npeer ? (unsigned)seq[d.peer[j]] + 1u : 0u;
  const int stride = gridDim.x * blockDim.x;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = tid; i < d.nsend + d.npeer; i += stride) {
    int j, slot;
    double v = 0.0;
    if (i < d.nsend) {
      j = 0;
      while (i >= d.sofs[j + 1]) ++j;
      slot = 1 + i - d.sofs[j];
      v = x[d.idx[i]];
    } else {
      j = i - d.nsend;
      slot = 0;
    }
    unsigned fj = 0;
#pragma unroll
    for (int q = 0; q < kMaxPeers; ++q)
      if (q == j) fj = f[q];
    st_ll(d.rdst[j] + (size_t)(fj & 1u) * d.rcap[j] + slot, v, fj);
  }
  for (int i = tid; i < d.nrecv + d.npeer; i += stride) {
    int j, slot;
    if (i < d.nrecv) {
      j = 0;
      while (i >= d.rofs[j + 1]) ++j;
      slot = 1 + i - d.rofs[j];
    } else {
      j = i - d.nrecv;
      slot = 0;
    }
    unsigned fj = 0;
#pragma unroll
    for (int q = 0; q < kMaxPeers; ++q)
      if (q == j) fj = f[q];
    const double v = ld_ll(d.lsrc[j] + (size_t)(fj & 1u) * d.lcap[j] + slot, fj);
    if (slot) d.ghost[i] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(ticket, 1u);
    if (t == gridDim.x - 1) {  // every CTA has read the sequence numbers
      *ticket = 0u;
      for (int j = 0; j < d.npeer; ++j) seq[d.peer[j]] += 1ull;
    }
  }
}

// norm allreduce in one single-thread kernel: my partial sum into every
// peer's slot (the parity of the local call count keeps consecutive
// reductions apart), publish, wait for the peers' partials, rank-ordered sum
__global__ void norm_kernel(NormDesc d, WaitDesc w, const double* loc, double* slots_mine,
                            unsigned long long* ncount, unsigned long long* sent,
                            unsigned long long* expect, const unsigned long long* flags, double* out) {
  pdl_enter();
  const int par = (int)(*ncount & 1ull);
  const double v = *loc;
  for (int j = 0; j < d.npeer; ++j) d.slots[j][par * d.world + d.me] = v;
  __threadfence_system();
  for (int j = 0; j < d.npeer; ++j) {
    st_release_sys(d.rflag[j], ++sent[d.peer[j]]);
    ++expect[d.peer[j]];
  }
  for (int j = 0; j < w.npeer; ++j) wait_count(flags + w.peer[j], expect[w.peer[j]]);
  double s = 0.0;
  for (int q = 0; q < d.world; ++q) s += q == d.me ? v : ld_relaxed_sys_d(slots_mine + par * d.world + q);
  *out = s;
  *ncount += 1ull;
}

__global__ void pack_kernel(int n, const int* __restrict__ idx, const double* __restrict__ x,
                            double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = x[idx[i]];
}

__global__ void finish_sum_kernel(int nparts, const double* __restrict__ parts, double* __restrict__ out) {
  pdl_enter();
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += parts[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) out[0] = t;
  }
}

// trecv holds world blocks of tmax entries; out = concatenation of the first
// cnt[q] entries of each block
__global__ void unpad_kernel(int world, int tmax, const int* __restrict__ cnt, const int* __restrict__ ofs,
                             const double* __restrict__ in, double* __restrict__ out) {
  const int q = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt[q]; i += gridDim.x * blockDim.x)
    out[ofs[q] + i] = in[(size_t)q * tmax + i];
}

}  // namespace airg

// P2P halo of one target vector
struct P2PHalo {
  PutDesc put;
  WaitDesc wait;
  LLDesc ll;
};

struct DLev {
  int n_loc = 0, nf = 0, nc = 0;
  Csr R, Afc, Aff;
  HaloX hR, hC, hF;
  const int* f_idx = nullptr;
  const int* c_idx = nullptr;
  std::vector<double> coef;
  double *r_ext = nullptr, *ec_ext = nullptr, *rhs_ext = nullptr, *y0 = nullptr, *y1 = nullptr,
         *e = nullptr;
  bool own_e = false;
  P2PHalo pR, pC, pF[3];  // pF: targets rhs_ext, y0, y1
};

// one NCCL communicator per process, shared by every distributed plan, plus
// the process's IPC arena for the P2P transport: grow-only, laid out by the
// most recent plan (owner); peers' mappings are re-opened only when their
// arena generation changes
struct airg_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  double* arena = nullptr;
  size_t cap = 0;  // doubles
  int gen = 0;
  std::vector<double*> peer_base;
  std::vector<int> peer_gen;
  long long owner = -1, next_id = 0;
};

// Distributed Newton coarse solve (configs[3]: a truncated hierarchy whose
// coarsest grid is too large to replicate): the coarsest operator stays on
// its row strips, u's ghosts travel per SpMV (NCCL send/recv), and the
// per-root decisions of polynomial.py:312-355 (non-finite delta -> stop, max
// |u| -> rescale / stop) need global facts.  They are taken speculatively:
// every rank applies the root, then ONE allreduce(max) of (max|u_new|, bad)
// decides; a root whose delta was non-finite anywhere is undone from the
// saved x / u, which is what stopping before it gives.
struct DCoarse {
  bool on = false;
  int n_loc = 0;
  Csr C;  // local rows, columns [local | ghost]
  HaloX h;
  std::vector<int> utype;
  std::vector<double> p1, p2;
  double *u = nullptr, *w = nullptr, *z = nullptr, *x0 = nullptr, *u0 = nullptr;
  unsigned long long* red = nullptr;  // [0..1] local (max bits, bad), [2..3] global
  double* state = nullptr;            // [0] scale, [1] stop
};

struct airg_dplan {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  bool p2p = false;
  std::vector<DLev> lv;
  Csr top;
  HaloX hT;
  P2PHalo pT, pTail;
  NormDesc nd;
  WaitDesc nwait;
  double *x_ext = nullptr, *r = nullptr, *parts = nullptr, *nrm_loc = nullptr, *nrm_glob = nullptr;
  double norm_h = 0.0;
  int nparts = 0, n_top = 0;
  airg_plan* tail = nullptr;
  std::vector<int> tcnt, tofs;
  int tail_n = 0, tmax = 0;
  int *d_tcnt = nullptr, *d_tofs = nullptr;
  double *tsend = nullptr, *trecv = nullptr, *tr_full = nullptr, *te_full = nullptr;
  // P2P transport state (arena owned by the communicator)
  airg_comm* cm = nullptr;
  long long id = 0;
  int arena_gen = -1;
  double* arena = nullptr;
  std::vector<double*> peer_base;
  double* nslots = nullptr;
  unsigned long long *flags = nullptr, *sent = nullptr, *recvd = nullptr, *ncount = nullptr;
  unsigned int* ticket = nullptr;
  unsigned long long* lseq = nullptr;  // LL exchanges per partner
  unsigned int* llticket = nullptr;
  bool ll = true;
  std::vector<size_t> ll_off;  // my LL region per sender (doubles into the arena)
  std::vector<int> ll_cap;     // its bank size (slots)
  std::vector<void*> owned;  // dmalloc'd buffers freed at destroy
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaGraphExec_t graph = nullptr;
  const void* gkey[2] = {nullptr, nullptr};
  long long launches = 0;
  DCoarse dc;
};

template <typename T>
static int dalloc_owned(airg_dplan* p, T** ptr, size_t count) {
  AIRG_CUDA(dmalloc(ptr, (count ? count : 1) * sizeof(T)));
  p->owned.push_back((void*)*ptr);
  return AIRG_OK;
}

// one P2P exchange: the put kernel stores, publishes and waits (put_kernel)
static int halo_put(airg_dplan* p, const P2PHalo& h, const double* x, cudaStream_t s) {
  const PutDesc& d = h.put;
  if (d.npeer == 0) return AIRG_OK;
  // measured: spreading the gather over CTAs beats one CTA (dependent
  // idx -> x -> remote-store chains); at most 16 CTAs
  AIRG_CUDA(launch_pdl(put_kernel, std::max(1, blocks_for(d.nsend, 256, 16)), 256, s, d, h.wait, x,
                       p->sent, p->recvd, p->ticket, (const unsigned long long*)p->flags));
  ++p->launches;
  return AIRG_OK;
}


// P2P: one put kernel whose last CTA also waits for the incoming ghosts (a
// separate one-CTA wait kernel per exchange measured slower).  Waiting inside the consuming SpMV
// was measured slower both with every CTA polling (2x SpMV time) and with only
// the CTAs that read ghost columns polling (solve 30 vs 21 ms at N = 2: the
// peer wait lands inside the large kernels).  NCCL: pack + send/recv
static int halo_exchange(airg_dplan* p, HaloX& h, const P2PHalo* ph, double* x_ext, cudaStream_t s) {
  if (p->world == 1) return AIRG_OK;
  if (p->p2p && p->ll) {
    const LLDesc& d = ph->ll;
    if (d.npeer == 0) return AIRG_OK;
    AIRG_CUDA(launch_pdl(ll_halo_kernel, std::max(1, blocks_for(d.nsend + d.nrecv, 256, 16)), 256, s, d,
                         (const double*)x_ext, p->lseq, p->llticket));
    ++p->launches;
    return AIRG_OK;
  }
  if (p->p2p) return halo_put(p, *ph, x_ext, s);  // the put kernel also waits
  if (h.nsend) {
    pack_kernel<<<blocks_for(h.nsend, 256, 1024), 256, 0, s>>>(h.nsend, h.send_idx, x_ext, h.sendbuf);
    AIRG_LAUNCH_CHECK();
  }
  AIRG_NCCL(ncclGroupStart());
  for (int q = 0; q < p->world; ++q) {
    if (h.scnt[q]) AIRG_NCCL(ncclSend(h.sendbuf + h.sofs[q], h.scnt[q], ncclDouble, q, p->comm, s));
    if (h.rcnt[q])
      AIRG_NCCL(ncclRecv(x_ext + h.n_loc + h.rofs[q], h.rcnt[q], ncclDouble, q, p->comm, s));
  }
  AIRG_NCCL(ncclGroupEnd());
  return AIRG_OK;
}

// the NCCL form of a halo exchange (pack + grouped send/recv), whatever the
// plan's transport: the distributed coarse solve is not in the P2P layout
static int halo_nccl(airg_dplan* p, HaloX& h, double* x_ext, cudaStream_t s) {
  if (p->world == 1) return AIRG_OK;
  if (h.nsend) {
    pack_kernel<<<blocks_for(h.nsend, 256, 1024), 256, 0, s>>>(h.nsend, h.send_idx, x_ext, h.sendbuf);
    AIRG_LAUNCH_CHECK();
  }
  AIRG_NCCL(ncclGroupStart());
  for (int q = 0; q < p->world; ++q) {
    if (h.scnt[q]) AIRG_NCCL(ncclSend(h.sendbuf + h.sofs[q], h.scnt[q], ncclDouble, q, p->comm, s));
    if (h.rcnt[q])
      AIRG_NCCL(ncclRecv(x_ext + h.n_loc + h.rofs[q], h.rcnt[q], ncclDouble, q, p->comm, s));
  }
  AIRG_NCCL(ncclGroupEnd());
  return AIRG_OK;
}

// nrm_loc -> nrm_glob (sum over ranks)
static int norm_allreduce(airg_dplan* p, cudaStream_t s) {
  if (p->world == 1) {
    AIRG_CUDA(cudaMemcpyAsync(p->nrm_glob, p->nrm_loc, sizeof(double), cudaMemcpyDeviceToDevice, s));
    return AIRG_OK;
  }
  if (!p->p2p) {
    AIRG_NCCL(ncclAllReduce(p->nrm_loc, p->nrm_glob, 1, ncclDouble, ncclSum, p->comm, s));
    return AIRG_OK;
  }
  AIRG_CUDA(launch_pdl(norm_kernel, 1, 1, s, p->nd, p->nwait, (const double*)p->nrm_loc, p->nslots,
                       p->ncount, p->sent, p->recvd, (const unsigned long long*)p->flags, p->nrm_glob));
  ++p->launches;
  return AIRG_OK;
}

__global__ void dn_init_kernel(int n, const double* __restrict__ in, double* __restrict__ u,
                               double* __restrict__ x, double* state, unsigned long long* red) {
  pdl_enter();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    u[i] = in[i];
    x[i] = 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    state[0] = 1.0;
    state[1] = 0.0;
    red[0] = red[1] = 0ull;
  }
}

// x += delta, u = u_new for one unit (real root: p1 = theta; pair: p1 = 2a,
// p2 = |theta|^2), saving the previous x / u; local max|u_new| (as the bits
// of a non-negative double: uint64 order == double order, NaN above inf) and
// the non-finite-delta flag into red[0..1]
__global__ void dn_update_kernel(int n, int type, double p1, double p2, double* __restrict__ x,
                                 double* __restrict__ u, const double* __restrict__ w,
                                 const double* __restrict__ z, double* __restrict__ x0,
                                 double* __restrict__ u0, const double* state,
                                 unsigned long long* red) {
  pdl_enter();
  if (state[1] != 0.0) return;
  const double sc = state[0] / (type == 0 ? p1 : p2);
  double lmax = 0.0;
  int bad = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double ui = u[i], xi = x[i];
    x0[i] = xi;
    u0[i] = ui;
    double d, un;
    if (type == 0) {
      d = sc * ui;
      un = ui - w[i] / p1;
    } else {
      d = sc * (p1 * ui - w[i]);
      un = ui + (z[i] - p1 * w[i]) / p2;
    }
    bad |= !isfinite(d);
    x[i] = xi + d;
    u[i] = un;
    const double a = fabs(un);
    lmax = (a != a || a > lmax) ? a : lmax;
  }
  const unsigned long long bits = (unsigned long long)__double_as_longlong(lmax);
  unsigned long long m = bits;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
    m = y > m ? y : m;
  }
  bad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    if (m) atomicMax(red, m);
    if (bad) atomicOr(red + 1, 1ull);
  }
}

// one CTA: the global decision of the unit (undo + stop / stop / rescale)
__global__ void dn_decide_kernel(int n, double* __restrict__ x, double* __restrict__ u,
                                 const double* __restrict__ x0, const double* __restrict__ u0,
                                 double* state, unsigned long long* red) {
  pdl_enter();
  __shared__ int act;
  __shared__ double nrm;
  if (state[1] != 0.0) return;
  if (threadIdx.x == 0) {
    act = 0;
    if (red[3]) {
      act = 2;  // a non-finite delta somewhere: stop before this unit
    } else {
      const double m = __longlong_as_double((long long)red[2]);
      nrm = m;
      if (m == 0.0) state[1] = 1.0;
      else if (m > 1e150 || m < 1e-150) act = 1;
    }
  }
  __syncthreads();
  if (act == 2) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      x[i] = x0[i];
      u[i] = u0[i];
    }
  } else if (act == 1) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) u[i] /= nrm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (act == 2) state[1] = 1.0;
    if (act == 1) {
      const double sc = state[0] * nrm;
      state[0] = sc;
      if (!isfinite(sc) || sc == 0.0) state[1] = 1.0;
    }
    red[0] = red[1] = 0ull;
  }
}

static int dplan_vcycle(airg_dplan* p, int l, cudaStream_t s);
static int halo_nccl(airg_dplan* p, HaloX& h, double* x_ext, cudaStream_t s);

// e = q(C) r on the row strips of the coarsest operator (see DCoarse)
static int dist_newton(airg_dplan* p, const double* in, double* out, cudaStream_t s) {
  DCoarse& D = p->dc;
  const int n = D.n_loc;
  const int nb = blocks_for(n, 256, num_sms() * 4);
  AIRG_CUDA(launch_pdl(dn_init_kernel, nb, 256, s, n, in, D.u, out, D.state, D.red));
  for (size_t k = 0; k < D.utype.size(); ++k) {
    const int ty = D.utype[k];
    AIRG_TRY(halo_nccl(p, D.h, D.u, s));
    {
      Epi ep{D.w, nullptr, 1.0, 0.0, nullptr, nullptr, nullptr, nullptr};
      AIRG_TRY(launch_spmv(D.C, D.u, 1.0, ep, s));
    }
    if (ty == 1) {
      AIRG_TRY(halo_nccl(p, D.h, D.w, s));
      Epi ep{D.z, nullptr, 1.0, 0.0, nullptr, nullptr, nullptr, nullptr};
      AIRG_TRY(launch_spmv(D.C, D.w, 1.0, ep, s));
    }
    AIRG_CUDA(launch_pdl(dn_update_kernel, nb, 256, s, n, ty, D.p1[k], D.p2[k], out, D.u,
                         (const double*)D.w, (const double*)D.z, D.x0, D.u0,
                         (const double*)D.state, D.red));
    AIRG_NCCL(ncclAllReduce(D.red, D.red + 2, 2, ncclUint64, ncclMax, p->comm, s));
    AIRG_CUDA(launch_pdl(dn_decide_kernel, 1, 1024, s, n, out, D.u, (const double*)D.x0,
                         (const double*)D.u0, D.state, D.red));
    p->launches += 4 + (ty == 1 ? 1 : 0);
  }
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

// V-cycle of the replicated tail: in = local part (tcnt[rank] entries), out = local part
static int dplan_tail(airg_dplan* p, const double* in, double* out, cudaStream_t s) {
  if (p->dc.on) return dist_newton(p, in, out, s);
  const int mine = p->tcnt[p->rank];
  if (p->p2p) {
    AIRG_TRY(halo_put(p, p->pTail, in, s));  // waits for the peers' parts too
  } else {
    AIRG_CUDA(cudaMemcpyAsync(p->tsend, in, (size_t)mine * sizeof(double), cudaMemcpyDeviceToDevice, s));
    AIRG_NCCL(ncclAllGather(p->tsend, p->trecv, p->tmax, ncclDouble, p->comm, s));
    dim3 g(blocks_for(p->tmax, 256, 64), p->world);
    unpad_kernel<<<g, 256, 0, s>>>(p->world, p->tmax, p->d_tcnt, p->d_tofs, p->trecv, p->tr_full);
    AIRG_LAUNCH_CHECK();
  }
  AIRG_TRY(vcycle_rec(p->tail, 0, p->tr_full, p->te_full, 1, s));
  AIRG_CUDA(cudaMemcpyAsync(out, p->te_full + p->tofs[p->rank], (size_t)mine * sizeof(double),
                            cudaMemcpyDeviceToDevice, s));
  return AIRG_OK;
}

// input lv[l].r_ext[0, n_loc), output lv[l].e
static int dplan_vcycle(airg_dplan* p, int l, cudaStream_t s) {
  DLev& L = p->lv[l];
  const bool last = l + 1 == (int)p->lv.size();
  AIRG_TRY(halo_exchange(p, L.hR, &L.pR, L.r_ext, s));
  // restricted residual: the next level's input, or scratch before the tail gather
  double* rc = last ? L.rhs_ext : p->lv[l + 1].r_ext;
  {
    Epi ep{rc, nullptr, 1.0, 0.0, nullptr, nullptr, nullptr, nullptr};
    AIRG_TRY(launch_spmv(L.R, L.r_ext, 1.0, ep, s));
  }
  if (last) AIRG_TRY(dplan_tail(p, rc, L.ec_ext, s));
  else AIRG_TRY(dplan_vcycle(p, l + 1, s));  // writes lv[l+1].e == L.ec_ext
  AIRG_TRY(halo_exchange(p, L.hC, &L.pC, L.ec_ext, s));
  // rhs = r[f] - A_fc e_c
  {
    Epi ep{L.rhs_ext, nullptr, -1.0, 1.0, L.r_ext, L.f_idx, nullptr, nullptr};
    AIRG_TRY(launch_spmv(L.Afc, L.ec_ext, 1.0, ep, s));
  }
  const int d = (int)L.coef.size() - 1;
  if (d == 0) {
    AIRG_TRY(launch_axpby(L.nf, L.e, L.f_idx, L.coef[0], L.rhs_ext, nullptr, 0.0, nullptr, s));
  } else {
    double* cur = L.rhs_ext;
    double xs = L.coef[d];
    double* bufs[2] = {L.y0, L.y1};
    for (int j = d - 1; j >= 0; --j) {
      const P2PHalo* ph = cur == L.rhs_ext ? &L.pF[0] : cur == L.y0 ? &L.pF[1] : &L.pF[2];
      AIRG_TRY(halo_exchange(p, L.hF, ph, cur, s));
      double* dst = j == 0 ? L.e : bufs[j & 1];
      Epi ep{dst, j == 0 ? L.f_idx : nullptr, 1.0, L.coef[j], L.rhs_ext, nullptr, nullptr, nullptr};
      AIRG_TRY(launch_spmv(L.Aff, cur, xs, ep, s));
      cur = dst;
      xs = 1.0;
    }
  }
  AIRG_TRY(launch_axpby(L.nc, L.e, L.c_idx, 1.0, L.ec_ext, nullptr, 0.0, nullptr, s));
  return AIRG_OK;
}

// r = b - A x (halo on x), local sum of squares -> allreduce -> nrm_glob
static int dplan_residual(airg_dplan* p, const double* b, cudaStream_t s) {
  AIRG_TRY(halo_exchange(p, p->hT, &p->pT, p->x_ext, s));
  const int nb = spmv_blocks(p->top);
  // written straight into level 0's input vector (no copy per iteration)
  Epi ep{p->lv[0].r_ext, nullptr, -1.0, 1.0, b, nullptr, nullptr, p->parts};
  AIRG_TRY(launch_spmv(p->top, p->x_ext, 1.0, ep, s));
  AIRG_CUDA(launch_pdl(finish_sum_kernel, 1, 1024, s, nb, (const double*)p->parts, p->nrm_loc));
  return norm_allreduce(p, s);
}

static int dalloc(airg_dplan* p, HaloX& h, int n_loc, int nsend, const int* send_idx,
                  const int* scnt, const int* rcnt, int world) {
  h.n_loc = n_loc;
  h.nsend = nsend;
  h.scnt.assign(scnt, scnt + world);
  h.rcnt.assign(rcnt, rcnt + world);
  h.sofs.assign(world + 1, 0);
  h.rofs.assign(world + 1, 0);
  int a = 0, b = 0;
  for (int q = 0; q < world; ++q) {
    h.sofs[q] = a;
    h.rofs[q] = b;
    a += h.scnt[q];
    b += h.rcnt[q];
  }
  h.sofs[world] = a;
  h.rofs[world] = b;
  h.nrecv = b;
  if (nsend) {
    AIRG_TRY(dalloc_owned(p, &h.send_idx, (size_t)nsend));
    AIRG_CUDA(cudaMemcpy(h.send_idx, send_idx, (size_t)nsend * sizeof(int), cudaMemcpyDeviceToDevice));
    AIRG_TRY(dalloc_owned(p, &h.sendbuf, (size_t)nsend));
  }
  return AIRG_OK;
}

// ---- P2P set-up --------------------------------------------------------------
// Every rank lays its ghost-receiving vectors out in one arena and publishes a
// directory of int64 entries (same layout on every rank):
//   per level: offsets of r_ext, ec_ext, rhs_ext, y0, y1; then for hR, hC, hF:
//              n_loc, rofs[0..W-1]
//   top: offset of x_ext, hT.n_loc, hT.rofs[0..W-1]
//   offsets of tr_full, norm slots, flags
enum { kDirLev = 5 };

// ... then per sender q: offset and bank size (slots) of my LL region for q
static size_t dir_len(int nd, int W) { return (size_t)nd * (kDirLev + 3 * (1 + W)) + (2 + W) + 2 * W + 3; }

static int p2p_peers(const HaloX& h, int me, int W, std::vector<int>& out) {
  out.clear();
  for (int q = 0; q < W; ++q)
    if (q != me && (h.scnt[q] > 0 || h.rcnt[q] > 0)) out.push_back(q);
  if ((int)out.size() > kMaxPeers) {
    set_error("halo spans %d peers (max %d)", (int)out.size(), kMaxPeers);
    return AIRG_ERR_VALUE;
  }
  return AIRG_OK;
}

// put/wait descriptors of halo h into the peers' vector at directory slot
// vec_slot; n_loc/rofs of that halo at dir slot hslot
static int build_p2p_halo(airg_dplan* p, const HaloX& h, const std::vector<long long>& dir, size_t dl,
                          size_t vec_slot, size_t hslot, P2PHalo& out) {
  const int me = p->rank, W = p->world;
  std::vector<int> peers;
  AIRG_TRY(p2p_peers(h, me, W, peers));
  PutDesc d{};
  d.nsend = h.nsend;
  d.idx = h.send_idx;
  d.npeer = (int)peers.size();
  for (int j = 0; j < d.npeer; ++j) {
    const int q = peers[j];
    const long long* D = dir.data() + (size_t)q * dl;
    d.peer[j] = q;
    d.sofs[j] = h.sofs[q];
    d.dst[j] = p->peer_base[q] + D[vec_slot] + D[hslot] + D[hslot + 1 + me];
    d.rflag[j] = (unsigned long long*)(p->peer_base[q] + D[dl - 1]) + me;
  }
  d.sofs[d.npeer] = h.nsend;
  // entries for peers that receive nothing form empty segments in rank order
  for (int j = d.npeer - 1; j >= 0; --j)
    if (h.scnt[d.peer[j]] == 0) d.sofs[j] = d.sofs[j + 1];
  out.put = d;
  out.wait.npeer = d.npeer;
  for (int j = 0; j < d.npeer; ++j) out.wait.peer[j] = peers[j];
  // LL form of the same exchange
  LLDesc l{};
  l.nsend = h.nsend;
  l.nrecv = h.nrecv;
  l.idx = h.send_idx;
  l.npeer = d.npeer;
  const size_t llb = dl - 3 - 2 * (size_t)W;  // directory: LL offsets, then bank sizes
  for (int j = 0; j < l.npeer; ++j) {
    const int q = peers[j];
    const long long* D = dir.data() + (size_t)q * dl;
    l.peer[j] = q;
    l.sofs[j] = h.sofs[q];
    l.rofs[j] = h.rofs[q];
    l.rdst[j] = (uint4*)(p->peer_base[q] + D[llb + me]);
    l.rcap[j] = (int)D[llb + W + me];
    l.lsrc[j] = (const uint4*)(p->arena + p->ll_off[q]);
    l.lcap[j] = p->ll_cap[q];
  }
  l.sofs[l.npeer] = h.nsend;
  l.rofs[l.npeer] = h.nrecv;
  for (int j = l.npeer - 1; j >= 0; --j) {
    if (h.scnt[l.peer[j]] == 0) l.sofs[j] = l.sofs[j + 1];
    if (h.rcnt[l.peer[j]] == 0) l.rofs[j] = l.rofs[j + 1];
  }
  const long long* Dm = dir.data() + (size_t)me * dl;
  l.ghost = p->arena + Dm[vec_slot] + Dm[hslot];
  out.ll = l;
  return AIRG_OK;
}

static int p2p_setup(airg_dplan* p) {
  const int W = p->world, me = p->rank, nd = (int)p->lv.size();
  auto up = [](size_t n) { return (n + 31) & ~(size_t)31; };
  std::vector<long long> mine(dir_len(nd, W), 0);
  size_t off = 0;
  size_t k = 0;
  std::vector<size_t> lev_off(nd * kDirLev);
  for (int l = 0; l < nd; ++l) {
    DLev& L = p->lv[l];
    const size_t sz[kDirLev] = {(size_t)L.n_loc + L.hR.nrecv + 1, (size_t)L.nc + L.hC.nrecv + 1,
                                (size_t)std::max(L.nf, L.nc) + L.hF.nrecv + 1,
                                (size_t)L.nf + L.hF.nrecv + 1, (size_t)L.nf + L.hF.nrecv + 1};
    for (int v = 0; v < kDirLev; ++v) {
      lev_off[l * kDirLev + v] = off;
      mine[k++] = (long long)off;
      off += up(sz[v]);
    }
    for (const HaloX* h : {&L.hR, &L.hC, &L.hF}) {
      mine[k++] = h->n_loc;
      for (int q = 0; q < W; ++q) mine[k++] = h->rofs[q];
    }
  }
  const size_t x_off = off;
  mine[k++] = (long long)off;
  off += up((size_t)p->n_top + p->hT.nrecv + 1);
  mine[k++] = p->hT.n_loc;
  for (int q = 0; q < W; ++q) mine[k++] = p->hT.rofs[q];
  // LL regions: per sender, two banks of (1 header + largest message) 16-byte slots
  p->ll_off.assign(W, 0);
  p->ll_cap.assign(W, 0);
  for (int q = 0; q < W; ++q) {
    if (q == me) continue;
    int mx = p->hT.rcnt[q];
    for (const DLev& L : p->lv) mx = std::max({mx, L.hR.rcnt[q], L.hC.rcnt[q], L.hF.rcnt[q]});
    p->ll_cap[q] = 1 + mx;
    p->ll_off[q] = off;
    off += up((size_t)4 * p->ll_cap[q]);
  }
  for (int q = 0; q < W; ++q) mine[k++] = (long long)p->ll_off[q];
  for (int q = 0; q < W; ++q) mine[k++] = p->ll_cap[q];
  const size_t tr_off = off;
  mine[k++] = (long long)off;
  off += up((size_t)p->tail_n + 1);
  const size_t ns_off = off;
  mine[k++] = (long long)off;
  off += up((size_t)2 * W);
  const size_t fl_off = off;
  mine[k++] = (long long)off;
  off += up((size_t)W);
  airg_comm* cm = p->cm;
  if (off > cm->cap) {  // grow (peers re-open on the generation change)
    AIRG_CUDA(cudaDeviceSynchronize());
    if (cm->arena) AIRG_CUDA(cudaFree(cm->arena));
    cm->arena = nullptr;
    cm->cap = off + off / 4;
    AIRG_CUDA(cudaMalloc((void**)&cm->arena, cm->cap * sizeof(double)));
    ++cm->gen;
  }
  p->arena = cm->arena;
  p->arena_gen = cm->gen;
  cm->owner = p->id;
  // the message counts restart at zero for this layout; the peers cannot
  // write into it before the directory exchange below
  AIRG_CUDA(cudaMemset(p->arena, 0, off * sizeof(double)));
  AIRG_CUDA(cudaDeviceSynchronize());
  for (int l = 0; l < nd; ++l) {
    DLev& L = p->lv[l];
    double** vs[kDirLev] = {&L.r_ext, &L.ec_ext, &L.rhs_ext, &L.y0, &L.y1};
    for (int v = 0; v < kDirLev; ++v) *vs[v] = p->arena + lev_off[l * kDirLev + v];
    if (l > 0) L.e = p->lv[l - 1].ec_ext;  // level l's error is level l-1's e_c
  }
  p->x_ext = p->arena + x_off;
  p->tr_full = p->arena + tr_off;
  p->nslots = p->arena + ns_off;
  p->flags = (unsigned long long*)(p->arena + fl_off);
  // exchange directories + IPC handles (one NCCL all-gather at build time)
  const size_t dl = dir_len(nd, W);
  const size_t rec = dl + 9;  // + 64 bytes of cudaIpcMemHandle_t + arena generation
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  std::vector<long long> hrec(rec);
  std::copy(mine.begin(), mine.end(), hrec.begin());
  cudaIpcMemHandle_t hdl;
  AIRG_CUDA(cudaIpcGetMemHandle(&hdl, p->arena));
  memcpy(hrec.data() + dl, &hdl, 64);
  hrec[dl + 8] = cm->gen;
  long long *dsend = nullptr, *drecv = nullptr;
  AIRG_CUDA(cudaMalloc((void**)&dsend, rec * sizeof(long long)));
  AIRG_CUDA(cudaMalloc((void**)&drecv, rec * W * sizeof(long long)));
  AIRG_CUDA(cudaMemcpy(dsend, hrec.data(), rec * sizeof(long long), cudaMemcpyHostToDevice));
  AIRG_NCCL(ncclAllGather(dsend, drecv, rec * 2, ncclFloat, p->comm, p->cs));  // 8-byte words as 2 floats
  AIRG_CUDA(cudaStreamSynchronize(p->cs));
  std::vector<long long> all(rec * W);
  AIRG_CUDA(cudaMemcpy(all.data(), drecv, rec * W * sizeof(long long), cudaMemcpyDeviceToHost));
  cudaFree(dsend);
  cudaFree(drecv);
  std::vector<long long> dir(dl * W);
  if ((int)cm->peer_base.size() != W) {
    cm->peer_base.assign(W, nullptr);
    cm->peer_gen.assign(W, -1);
  }
  for (int q = 0; q < W; ++q) {
    std::copy(all.begin() + q * rec, all.begin() + q * rec + dl, dir.begin() + q * dl);
    if (q == me) {
      cm->peer_base[q] = p->arena;
      cm->peer_gen[q] = cm->gen;
      continue;
    }
    const int g = (int)all[q * rec + dl + 8];
    if (cm->peer_gen[q] == g && cm->peer_base[q]) continue;
    if (cm->peer_base[q]) cudaIpcCloseMemHandle(cm->peer_base[q]);
    cudaIpcMemHandle_t h;
    memcpy(&h, all.data() + q * rec + dl, 64);
    void* base = nullptr;
    AIRG_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    cm->peer_base[q] = (double*)base;
    cm->peer_gen[q] = g;
  }
  p->peer_base = cm->peer_base;
  // descriptors
  const size_t per_lev = kDirLev + 3 * (1 + W);
  for (int l = 0; l < nd; ++l) {
    DLev& L = p->lv[l];
    const size_t b = (size_t)l * per_lev;
    const size_t hR = b + kDirLev, hC = hR + 1 + W, hF = hC + 1 + W;
    AIRG_TRY(build_p2p_halo(p, L.hR, dir, dl, b + 0, hR, L.pR));
    AIRG_TRY(build_p2p_halo(p, L.hC, dir, dl, b + 1, hC, L.pC));
    for (int v = 0; v < 3; ++v) AIRG_TRY(build_p2p_halo(p, L.hF, dir, dl, b + 2 + v, hF, L.pF[v]));
  }
  const size_t tb = (size_t)nd * per_lev;
  AIRG_TRY(build_p2p_halo(p, p->hT, dir, dl, tb, tb + 1, p->pT));
  // tail gather: my part to every rank's tr_full (self included, no flag)
  {
    PutDesc d{};
    const int n = p->tcnt[me];
    d.idx = nullptr;
    int j = 0;
    for (int q = 0; q < W; ++q) {
      const long long* D = dir.data() + (size_t)q * dl;
      d.peer[j] = q;
      d.sofs[j] = j * n;
      d.dst[j] = p->peer_base[q] + D[dl - 3] + p->tofs[me];
      d.rflag[j] = q == me ? nullptr : (unsigned long long*)(p->peer_base[q] + D[dl - 1]) + me;
      ++j;
    }
    d.npeer = j;
    d.sofs[j] = j * n;
    d.nsend = j * n;
    p->pTail.put = d;
    WaitDesc w{};
    for (int q = 0; q < W; ++q)
      if (q != me) w.peer[w.npeer++] = q;
    p->pTail.wait = w;
    // norm slots
    NormDesc nd_{};
    nd_.me = me;
    nd_.world = W;
    for (int q = 0; q < W; ++q) {
      if (q == me) continue;
      const long long* D = dir.data() + (size_t)q * dl;
      nd_.peer[nd_.npeer] = q;
      nd_.slots[nd_.npeer] = p->peer_base[q] + D[dl - 2];
      nd_.rflag[nd_.npeer] = (unsigned long long*)(p->peer_base[q] + D[dl - 1]) + me;
      ++nd_.npeer;
    }
    p->nd = nd_;
    p->nwait = w;
  }
  if (!p->sent) {
    unsigned long long* ctr = nullptr;
    AIRG_TRY(dalloc_owned(p, &ctr, (size_t)4 * W + 3));
    p->sent = ctr;
    p->recvd = ctr + W;
    p->ncount = ctr + 2 * W;
    p->ticket = (unsigned int*)(ctr + 2 * W + 1);
    p->lseq = ctr + 2 * W + 2;
    p->llticket = (unsigned int*)(ctr + 3 * W + 2);
  }
  AIRG_CUDA(cudaMemset(p->sent, 0, ((size_t)4 * W + 3) * sizeof(unsigned long long)));
  AIRG_CUDA(cudaDeviceSynchronize());
  return AIRG_OK;
}

extern "C" {

int airg_nccl_unique_id(char* out_h) {
  ncclUniqueId id;
  AIRG_NCCL(ncclGetUniqueId(&id));
  memcpy(out_h, id.internal, NCCL_UNIQUE_ID_BYTES);
  return AIRG_OK;
}


int airg_comm_create(const char* id_h, int rank, int world, airg_comm** out) {
  airg_comm* c = new airg_comm();
  c->rank = rank;
  c->world = world;
  ncclUniqueId id;
  memcpy(id.internal, id_h, NCCL_UNIQUE_ID_BYTES);
  AIRG_NCCL(ncclCommInitRank(&c->comm, world, id, rank));
  *out = c;
  return AIRG_OK;
}

int airg_comm_destroy(airg_comm* c) {
  if (!c) return AIRG_OK;
  cudaDeviceSynchronize();
  for (int q = 0; q < (int)c->peer_base.size(); ++q)
    if (q != c->rank && c->peer_base[q]) cudaIpcCloseMemHandle(c->peer_base[q]);
  if (c->arena) cudaFree(c->arena);
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
  return AIRG_OK;
}

int airg_dplan_create(airg_comm* c, int ndist, airg_dplan** out) {
  if (c->world > kMaxPeers + 1) {
    set_error("at most %d ranks", kMaxPeers + 1);
    return AIRG_ERR_VALUE;
  }
  airg_dplan* p = new airg_dplan();
  p->rank = c->rank;
  p->world = c->world;
  p->comm = c->comm;
  p->cm = c;
  p->id = c->next_id++;
  p->lv.resize(ndist);
  AIRG_CUDA(cudaStreamCreateWithFlags(&p->cs, cudaStreamNonBlocking));
  AIRG_CUDA(cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming));
  AIRG_CUDA(cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming));
  AIRG_TRY(dalloc_owned(p, &p->nrm_loc, 2));
  p->nrm_glob = p->nrm_loc + 1;
  *out = p;
  return AIRG_OK;
}

// which: 0 = R (fine space), 1 = A_fc (coarse space), 2 = A_ff (F space), 3 = top A
int airg_dplan_set_halo(airg_dplan* p, int level, int which, int n_loc, int nsend,
                        const int32_t* send_idx, const int32_t* scnt_h, const int32_t* rcnt_h) {
  HaloX* h = which == 3 ? &p->hT : which == 0 ? &p->lv[level].hR : which == 1 ? &p->lv[level].hC
                                                                            : &p->lv[level].hF;
  return dalloc(p, *h, n_loc, nsend, send_idx, scnt_h, rcnt_h, p->world);
}

int airg_dplan_set_level(airg_dplan* p, int level, int n_loc, int nf, int nc, const int32_t* Rp,
                         const int32_t* Rc, const double* Rv, int64_t Rnnz, const int32_t* Fcp,
                         const int32_t* Fcc, const double* Fcv, int64_t Fcnnz, const int32_t* Ffp,
                         const int32_t* Ffc, const double* Ffv, int64_t Ffnnz, const int32_t* f_idx,
                         const int32_t* c_idx, int ncoef, const double* coef_h) {
  DLev& L = p->lv[level];
  L.n_loc = n_loc;
  L.nf = nf;
  L.nc = nc;
  L.R = make_csr(nc, n_loc + L.hR.nrecv, Rp, Rc, Rv, Rnnz);
  L.Afc = make_csr(nf, nc + L.hC.nrecv, Fcp, Fcc, Fcv, Fcnnz);
  L.Aff = make_csr(nf, nf + L.hF.nrecv, Ffp, Ffc, Ffv, Ffnnz);
  L.f_idx = f_idx;
  L.c_idx = c_idx;
  L.coef.assign(coef_h, coef_h + ncoef);
  if (level == 0) {
    AIRG_TRY(dalloc_owned(p, &L.e, (size_t)n_loc + 1));
    L.own_e = true;
  }
  return AIRG_OK;
}

// distributed coarsest grid (Newton coarse solver on row strips): local rows
// with columns [local | ghost] (halo: nsend entries, per-rank counts), the
// units of the Newton form (type, p1, p2 as airg_plan_set_coarse)
int airg_dplan_set_dcoarse(airg_dplan* p, int n_loc, const int32_t* ptr, const int32_t* col,
                           const double* val, int64_t nnz, int nsend, const int32_t* send_idx,
                           const int32_t* scnt_h, const int32_t* rcnt_h, int nunits,
                           const int32_t* type_h, const double* p1_h, const double* p2_h) {
  DCoarse& D = p->dc;
  AIRG_TRY(dalloc(p, D.h, n_loc, nsend, send_idx, scnt_h, rcnt_h, p->world));
  D.n_loc = n_loc;
  D.C = make_csr(n_loc, n_loc + D.h.nrecv, ptr, col, val, nnz);
  D.utype.assign(type_h, type_h + nunits);
  D.p1.assign(p1_h, p1_h + nunits);
  D.p2.assign(p2_h, p2_h + nunits);
  const size_t ext = (size_t)n_loc + D.h.nrecv + 1;
  AIRG_TRY(dalloc_owned(p, &D.u, ext));
  AIRG_TRY(dalloc_owned(p, &D.w, ext));
  AIRG_TRY(dalloc_owned(p, &D.z, (size_t)n_loc + 1));
  AIRG_TRY(dalloc_owned(p, &D.x0, (size_t)n_loc + 1));
  AIRG_TRY(dalloc_owned(p, &D.u0, (size_t)n_loc + 1));
  AIRG_TRY(dalloc_owned(p, &D.red, 4));
  AIRG_TRY(dalloc_owned(p, &D.state, 2));
  D.on = true;
  return AIRG_OK;
}

int airg_dplan_set_top(airg_dplan* p, int n_loc, const int32_t* ptr, const int32_t* col,
                       const double* val, int64_t nnz) {
  p->n_top = n_loc;
  p->top = make_csr(n_loc, n_loc + p->hT.nrecv, ptr, col, val, nnz);
  AIRG_TRY(dalloc_owned(p, &p->r, (size_t)n_loc + 1));
  p->nparts = spmv_blocks(p->top) + 1;
  AIRG_TRY(dalloc_owned(p, &p->parts, (size_t)p->nparts));
  return AIRG_OK;
}

// allocate and link the levels' vectors (level l's coarse error buffer ==
// level l+1's e) and attach the replicated tail plan; counts_h = per-rank
// sizes of the tail level (the coarse size of the last distributed level)
int airg_dplan_finish(airg_dplan* p, airg_plan* tail, const int32_t* counts_h) {
  const int nd = (int)p->lv.size();
  p->tail = tail;
  p->tcnt.assign(counts_h, counts_h + p->world);
  p->tofs.assign(p->world, 0);
  int a = 0, mx = 1;
  for (int q = 0; q < p->world; ++q) {
    p->tofs[q] = a;
    a += p->tcnt[q];
    mx = std::max(mx, p->tcnt[q]);
  }
  p->tail_n = a;
  p->tmax = mx;
  static const bool force_nccl = getenv("AIRG_DPLAN_NCCL") != nullptr;
  p->p2p = p->world > 1 && !force_nccl;
  static const bool no_ll = getenv("AIRG_DPLAN_LL") && atoi(getenv("AIRG_DPLAN_LL")) == 0;
  p->ll = !no_ll;  // AIRG_DPLAN_LL=0: fenced put kernels instead of LL slots
  if (p->p2p) {
    const int rc = p2p_setup(p);
    if (rc != AIRG_OK) return rc;
  } else {
    for (int l = 0; l < nd; ++l) {
      DLev& L = p->lv[l];
      AIRG_TRY(dalloc_owned(p, &L.r_ext, (size_t)L.n_loc + L.hR.nrecv + 1));
      AIRG_TRY(dalloc_owned(p, &L.rhs_ext, (size_t)std::max(L.nf, L.nc) + L.hF.nrecv + 1));
      AIRG_TRY(dalloc_owned(p, &L.y0, (size_t)L.nf + L.hF.nrecv + 1));
      AIRG_TRY(dalloc_owned(p, &L.y1, (size_t)L.nf + L.hF.nrecv + 1));
      AIRG_TRY(dalloc_owned(p, &L.ec_ext, (size_t)L.nc + L.hC.nrecv + 1));
      if (l > 0) L.e = p->lv[l - 1].ec_ext;
    }
    AIRG_TRY(dalloc_owned(p, &p->x_ext, (size_t)p->n_top + p->hT.nrecv + 1));
    AIRG_TRY(dalloc_owned(p, &p->tr_full, (size_t)a + 1));
    AIRG_TRY(dalloc_owned(p, &p->d_tcnt, (size_t)p->world));
    AIRG_TRY(dalloc_owned(p, &p->d_tofs, (size_t)p->world));
    AIRG_CUDA(cudaMemcpy(p->d_tcnt, p->tcnt.data(), p->world * sizeof(int), cudaMemcpyHostToDevice));
    AIRG_CUDA(cudaMemcpy(p->d_tofs, p->tofs.data(), p->world * sizeof(int), cudaMemcpyHostToDevice));
    AIRG_TRY(dalloc_owned(p, &p->tsend, (size_t)mx));
    AIRG_TRY(dalloc_owned(p, &p->trecv, (size_t)mx * p->world));
  }
  AIRG_TRY(dalloc_owned(p, &p->te_full, (size_t)a + 1));
  if (tail) AIRG_TRY(prepare_capture(tail, 0));
  return AIRG_OK;
}

int airg_dplan_destroy(airg_dplan* p) {
  if (!p) return AIRG_OK;
  if (p->cs) cudaStreamSynchronize(p->cs);
  if (p->graph) cudaGraphExecDestroy(p->graph);
  for (void* b : p->owned) dfree(b);  // the arena and the peer mappings belong to the communicator
  if (p->cs) cudaStreamDestroy(p->cs);
  if (p->ev_in) cudaEventDestroy(p->ev_in);
  if (p->ev_out) cudaEventDestroy(p->ev_out);
  delete p;  // the communicator is owned by its airg_comm
  return AIRG_OK;
}

// Richardson with the distributed V-cycle (solve.py:113-167); b, x local (x in/out)
int airg_dplan_richardson(airg_dplan* p, const double* b, double* x, double rtol, double atol,
                          int max_iters, double* history, int* iterations, int* converged,
                          void* stream) {
  cudaStream_t caller = (cudaStream_t)stream;
  cudaStream_t s = p->cs;
  const int n = p->top.nrows;
  if (p->p2p && p->cm->owner != p->id) {
    // a newer plan laid the shared arena out since: lay this plan out again
    // (collective: every rank uses its plans in the same order)
    double* old = p->arena;
    AIRG_TRY(p2p_setup(p));
    if (p->arena != old && p->graph) {
      cudaGraphExecDestroy(p->graph);
      p->graph = nullptr;
    }
  }
  AIRG_CUDA(cudaEventRecord(p->ev_in, caller));
  AIRG_CUDA(cudaStreamWaitEvent(s, p->ev_in, 0));
  AIRG_CUDA(cudaMemcpyAsync(p->x_ext, x, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  // ||b||
  {
    const int nb = blocks_for(n, 256, 1024);
    sumsq_kernel<<<nb, 256, 0, s>>>(n, b, p->parts);
    finish_sum_kernel<<<1, 1024, 0, s>>>(nb, p->parts, p->nrm_loc);
    AIRG_LAUNCH_CHECK();
    AIRG_TRY(norm_allreduce(p, s));
    AIRG_CUDA(read_back(&p->norm_h, p->nrm_glob, sizeof(double), s));
  }
  const double bnorm = std::sqrt(p->norm_h);
  AIRG_TRY(dplan_residual(p, b, s));
  AIRG_CUDA(read_back(&p->norm_h, p->nrm_glob, sizeof(double), s));
  double rn = std::sqrt(p->norm_h);
  history[0] = rn;
  const double thr = std::max(rtol * (bnorm > 0 ? bnorm : rn), atol);
  *iterations = 0;
  *converged = 0;
  int st = AIRG_OK;
  bool conv = rn <= thr;
  int its = 0;
  // With the P2P transport an iteration is kernels only and is captured once
  // per (b, x); capturing the NCCL-bearing iteration costs more than one
  // solve's launch overhead (opt-in: AIRG_DPLAN_GRAPH=1).
  static const bool graph_on = getenv("AIRG_DPLAN_GRAPH") != nullptr;
  const bool use_graph = graphs_enabled() && (p->p2p || graph_on);
  if (use_graph && (p->gkey[0] != b || p->gkey[1] != x) && p->graph) {
    cudaGraphExecDestroy(p->graph);
    p->graph = nullptr;
  }
  auto iteration = [&](cudaStream_t t) -> int {
    DLev& L0 = p->lv[0];
    AIRG_TRY(dplan_vcycle(p, 0, t));
    AIRG_TRY(launch_axpby(n, p->x_ext, nullptr, 1.0, p->x_ext, nullptr, 1.0, L0.e, t));
    return dplan_residual(p, b, t);
  };
  while (!conv && its < max_iters) {
    if (use_graph) {
      if (!p->graph) {
        AIRG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        const int rc = iteration(s);
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(s, &g);
        if (rc != AIRG_OK) {
          if (g) cudaGraphDestroy(g);
          return rc;
        }
        AIRG_CUDA(ce);
        AIRG_CUDA(cudaGraphInstantiate(&p->graph, g, 0));
        cudaGraphDestroy(g);
        p->gkey[0] = b;
        p->gkey[1] = x;
      }
      AIRG_CUDA(cudaGraphLaunch(p->graph, s));
    } else {
      AIRG_TRY(iteration(s));
    }
    AIRG_CUDA(read_back(&p->norm_h, p->nrm_glob, sizeof(double), s));
    rn = std::sqrt(p->norm_h);
    ++its;
    history[its] = rn;
    *iterations = its;
    if (!std::isfinite(rn)) {
      set_error("non-finite residual at iteration %d", its);
      st = AIRG_ERR_DIVERGED;
      break;
    }
    if (rn > 1e8 * history[0]) {
      set_error("residual grew by more than 1e+08 at iteration %d", its);
      st = AIRG_ERR_DIVERGED;
      break;
    }
    conv = rn <= thr;
  }
  *converged = conv ? 1 : 0;
  AIRG_CUDA(cudaMemcpyAsync(x, p->x_ext, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  AIRG_CUDA(cudaEventRecord(p->ev_out, s));
  AIRG_CUDA(cudaStreamWaitEvent(caller, p->ev_out, 0));
  return st;
}

}  // extern "C"
