// Arnoldi (modified Gram-Schmidt with one selective reorthogonalisation
// sweep and the lucky-breakdown rule) for the GMRES-polynomial setup.
// ref: polynomial.py:61-110 (_random_unit_vector, _arnoldi)
//
// Small operators (coarse grids, n <= kArnoldiCta) run the whole Krylov
// recurrence inside ONE CTA: V lives in global memory (L2-resident), every
// dot product is a block reduction, no host round trips.  Large operators
// use a device-resident multi-kernel path: SpMV, fixed-order dot partials,
// axpy, with the reorthogonalisation / breakdown decisions taken on the device.
#include "setup_common.cuh"
#include <cooperative_groups.h>
#include <vector>
#include <cmath>

namespace cg = cooperative_groups;

namespace airg {

constexpr int kArnoldiCta = 1024;  // above: the cooperative grid kernel (measured faster from ~1k rows)

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// block_sum for an 8-warp CTA with ONE barrier: warp totals go to one of two
// alternating slot sets (a fast warp's next write cannot meet a slow warp's
// read of the current set: reusing a set needs the barrier in between), and
// every thread adds the 8 totals in the xor-butterfly order of block_sum's
// final warp_sum (lanes >= 8 contribute exact zeros), so the value is
// bitwise block_sum's.
struct Sum8 {
  double* red;  // 16 slots
  int buf;
  __device__ __forceinline__ double operator()(double v) {
    v = warp_sum(v);
    double* r = red + 8 * buf;
    if ((threadIdx.x & 31) == 0) r[threadIdx.x >> 5] = v;
    buf ^= 1;
    __syncthreads();
    return ((r[0] + r[4]) + (r[2] + r[6])) + ((r[1] + r[5]) + (r[3] + r[7]));
  }
};

__device__ __forceinline__ double rowdot(const int* __restrict__ p, const int* __restrict__ c,
                                         const double* __restrict__ v, const double* x, int i) {
  double s = 0.0;
  for (int k = p[i]; k < p[i + 1]; ++k) s = fma(v[k], x[c[k]], s);
  return s;
}

// H is (m+1) x m row-major.  info[0] = k, info[1] = error code, dinfo[0] = beta
// Thread t owns entries i = t + e*NT (e < E) of the working vector w, kept in
// registers; the Gram-Schmidt step q forms w -= h_q V_q and the next basis
// vector's partial dot in the same pass, with V_{q+1} loaded before the
// reduction of step q, so each step costs one block reduction instead of two
// dependent L2 round trips.  Per-thread summation order is unchanged (entries
// in e order), so H is bitwise what the two-pass loop produced.
// The first vsm basis vectors live in shared memory (after H's column): the
// Gram-Schmidt sweeps re-read every earlier vector, and an order-100
// Arnoldi on a few hundred rows otherwise waits on L2 at every step.
template <int NT, int E>
__global__ void __launch_bounds__(NT) arnoldi_cta_kernel(int n, const int* __restrict__ p,
                                                         const int* __restrict__ c,
                                                         const double* __restrict__ v,
                                                         const double* __restrict__ b, int m,
                                                         double* Vg, double* w, double* H,
                                                         int* info, double* dinfo, int vsm) {
  static_assert(NT == 256, "Sum8 reduces 8 warps");
  __shared__ double red[33];
  __shared__ double red8[16];
  extern __shared__ double hcol[];  // column j of H (m + 1), thread 0 only; then vsm vectors
  double* Vs = hcol + ((m + 2) & ~1);
  auto vrow = [&](int q) -> double* { return q < vsm ? Vs + (size_t)q * n : Vg + (size_t)q * n; };
  double* V = vrow(0);
  Sum8 bsum{red8, 0};
  const int tid = threadIdx.x;
  double sq = 0.0;
  for (int i = tid; i < n; i += NT) sq = fma(b[i], b[i], sq);
  const double beta = sqrt(bsum(sq));
  if (tid == 0) {
    dinfo[0] = beta;
    info[0] = m;
    info[1] = 0;
  }
  if (beta == 0.0) {
    if (tid == 0) info[1] = 1;
    return;
  }
  for (int i = tid; i < n; i += NT) V[i] = b[i] / beta;
  for (int i = tid; i < (m + 1) * m; i += NT) H[i] = 0.0;
  __syncthreads();
  double hmax = 0.0;
  int k = m;
  double wr[E], vq[E], vn[E];
  for (int j = 0; j < m; ++j) {
    const double* Vj = vrow(j);
    sq = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = tid + e * NT;
      wr[e] = 0.0;
      if (i < n) {
        const double t = rowdot(p, c, v, Vj, i);
        wr[e] = t;
        sq = fma(t, t, sq);
      }
    }
    const double before = sqrt(bsum(sq));
    if (tid == 0)
      for (int q = 0; q <= j; ++q) hcol[q] = 0.0;
    double hn = 0.0;
    for (int sweep = 0; sweep < 2; ++sweep) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = tid + e * NT;
        vq[e] = i < n ? V[i] : 0.0;
      }
      for (int q = 0; q <= j; ++q) {
        double d = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (tid + e * NT < n) d = fma(vq[e], wr[e], d);
        if (q < j) {
          const double* Vn = vrow(q + 1);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int i = tid + e * NT;
            vn[e] = i < n ? Vn[i] : 0.0;
          }
        }
        const double h = bsum(d);
        if (tid == 0) hcol[q] += h;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          wr[e] -= h * vq[e];
          vq[e] = vn[e];
        }
      }
      sq = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (tid + e * NT < n) sq = fma(wr[e], wr[e], sq);
      hn = sqrt(bsum(sq));
      if (!(sweep == 0 && hn < 0.7 * before)) break;  // "twice is enough"
    }
    __syncthreads();
    double cn = 0.0;
    if (tid == 0) {
      hcol[j + 1] = hn;
      for (int q = 0; q <= j + 1; ++q) {
        H[q * m + j] = hcol[q];
        cn = fma(hcol[q], hcol[q], cn);
      }
      red[32] = sqrt(cn);
    }
    __syncthreads();
    hmax = fmax(hmax, red[32]);
    __syncthreads();
    if (hn <= 1e-14 * hmax) {
      if (tid == 0) H[(j + 1) * m + j] = 0.0;
      k = j + 1;
      break;
    }
    double* Vn = vrow(j + 1);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = tid + e * NT;
      if (i < n) Vn[i] = wr[e] / hn;
    }
    __syncthreads();
  }
  if (tid == 0) info[0] = k;
}

// ---- one-warp Gram-Schmidt (n <= 512: coarsest grids, order-100 Newton) ----
// The CTA does the SpMV; warp 0 alone runs the Gram-Schmidt sweeps with the
// working vector in registers (E entries per lane), so each of the ~m^2/2
// projections of an order-m Arnoldi costs a 5-step shuffle reduction instead
// of a block barrier (an order-100 Arnoldi on 330 rows: 5 ms -> ~1 ms).
template <int E>
__global__ void __launch_bounds__(256) arnoldi_warp_kernel(int n, const int* __restrict__ p,
                                                           const int* __restrict__ c,
                                                           const double* __restrict__ v,
                                                           const double* __restrict__ b, int m,
                                                           double* Vg, double* H, int* info,
                                                           double* dinfo, int vsm) {
  extern __shared__ double hcol[];  // (m + 2) & ~1 | ws (n, even) | vsm vectors
  __shared__ int done;
  double* ws = hcol + ((m + 2) & ~1);
  double* Vs = ws + ((n + 1) & ~1);
  auto vrow = [&](int q) -> double* { return q < vsm ? Vs + (size_t)q * n : Vg + (size_t)q * n; };
  const int tid = threadIdx.x, lane = tid & 31;
  const bool w0 = tid < 32;
  double wr[E], vq[E], vn[E];
  if (w0) {
    double sq = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = lane + 32 * e;
      wr[e] = i < n ? b[i] : 0.0;
      sq = fma(wr[e], wr[e], sq);
    }
    const double beta = sqrt(warp_sum(sq));
    if (lane == 0) {
      dinfo[0] = beta;
      info[0] = m;
      info[1] = beta == 0.0 ? 1 : 0;
      done = beta == 0.0;
    }
    if (beta != 0.0) {
      double* V0 = vrow(0);
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (lane + 32 * e < n) V0[lane + 32 * e] = wr[e] / beta;
    }
  }
  for (int i = tid; i < (m + 1) * m; i += blockDim.x) H[i] = 0.0;
  __syncthreads();
  if (done) return;
  double hmax = 0.0;
  int k = m;
  for (int j = 0; j < m; ++j) {
    const double* Vj = vrow(j);
    for (int i = tid; i < n; i += blockDim.x) ws[i] = rowdot(p, c, v, Vj, i);
    __syncthreads();
    if (w0) {
      double sq = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = lane + 32 * e;
        wr[e] = i < n ? ws[i] : 0.0;
        sq = fma(wr[e], wr[e], sq);
      }
      const double before = sqrt(warp_sum(sq));
      for (int q = lane; q <= j; q += 32) hcol[q] = 0.0;
      __syncwarp();
      double hn = 0.0;
      for (int sweep = 0; sweep < 2; ++sweep) {
        const double* V0 = vrow(0);
#pragma unroll
        for (int e = 0; e < E; ++e) vq[e] = lane + 32 * e < n ? V0[lane + 32 * e] : 0.0;
        for (int q = 0; q <= j; ++q) {
          double d0 = 0.0, d1 = 0.0;  // two chains: half the dependent FMA latency
#pragma unroll
          for (int e = 0; e < E; e += 2) {
            d0 = fma(vq[e], wr[e], d0);
            if (e + 1 < E) d1 = fma(vq[e + 1], wr[e + 1], d1);
          }
          if (q < j) {
            const double* Vn = vrow(q + 1);
#pragma unroll
            for (int e = 0; e < E; ++e) vn[e] = lane + 32 * e < n ? Vn[lane + 32 * e] : 0.0;
          }
          const double h = warp_sum(d0 + d1);
          if (lane == 0) hcol[q] += h;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            wr[e] -= h * vq[e];
            vq[e] = vn[e];
          }
        }
        sq = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) sq = fma(wr[e], wr[e], sq);
        hn = sqrt(warp_sum(sq));
        if (!(sweep == 0 && hn < 0.7 * before)) break;  // "twice is enough"
      }
      __syncwarp();
      double cn = 0.0;
      if (lane == 0) {
        hcol[j + 1] = hn;
        for (int q = 0; q <= j + 1; ++q) {
          H[q * m + j] = hcol[q];
          cn = fma(hcol[q], hcol[q], cn);
        }
      }
      hmax = fmax(hmax, sqrt(__shfl_sync(0xffffffffu, cn, 0)));
      if (hn <= 1e-14 * hmax) {
        if (lane == 0) {
          H[(j + 1) * m + j] = 0.0;
          done = 1;
        }
        k = j + 1;
      } else {
        double* Vn = vrow(j + 1);
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (lane + 32 * e < n) Vn[lane + 32 * e] = wr[e] / hn;
      }
    }
    __syncthreads();
    if (done) break;
  }
  if (tid == 0) info[0] = k;
}

// ---- multi-kernel path ----------------------------------------------------
// The modified Gram-Schmidt recurrence of the single-CTA kernel, spread over
// the GPU (SpMV, fixed-order dot partials + finish, axpy).  The selective
// second sweep and the lucky-breakdown test are decided on the device by a
// one-thread control kernel; later kernels read the decisions through a
// Gate and exit early, so a whole Arnoldi is enqueued without a host round
// trip (the host reads beta once and H, k at the end).
struct Gate {
  const int* stop;  // skip when *stop != 0 (breakdown reached)
  const int* need;  // skip when need && *need == 0 (no second sweep)
  __device__ __forceinline__ bool off() const { return (stop && *stop) || (need && !*need); }
};

__global__ void dot_partial_kernel(long long n, const double* __restrict__ x, const double* __restrict__ y,
                                   double* __restrict__ parts, Gate g) {
  if (g.off()) return;
  __shared__ double red[33];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    s = fma(x[i], y[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) parts[blockIdx.x] = s;
}

// out = sum(parts) (+ optional accumulate into *acc), fixed order
__global__ void dot_finish_kernel(int np, const double* __restrict__ parts, double* out, double* acc,
                                  Gate g) {
  if (g.off()) return;
  __shared__ double red[33];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += parts[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) {
    *out = s;
    if (acc) *acc += s;
  }
}

__global__ void axpy_dev_kernel(long long n, const double* __restrict__ hptr, const double* __restrict__ x,
                                double* __restrict__ y, Gate g) {
  if (g.off()) return;
  const double h = *hptr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] -= h * x[i];
}

// y = x / d (d by value, or *dptr when given)
__global__ void scale_div_kernel(long long n, const double* __restrict__ x, double d, const double* dptr,
                                 double* __restrict__ y, Gate g) {
  if (g.off()) return;
  const double dd = dptr ? *dptr : d;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = x[i] / dd;
}

// lanes per row from the mean row length (the rule of the solve's SpMV):
// the fine levels' A_ff have 1-8 entries per row, the coarse ones 100+
static int arnoldi_vs(long long nnz, int n) {
  const double mean = n > 0 ? (double)nnz / n : 0.0;
  return mean <= 6 ? 1 : mean <= 12 ? 2 : mean <= 24 ? 4 : mean <= 48 ? 8 : mean <= 96 ? 16 : 32;
}

// y = A x with vs lanes per row (lane-strided FMA, xor-tree over the vs
// lanes).  `gthread` / `gthreads` index the calling threads; trip counts are
// warp-uniform (the row groups of a warp shuffle together).  The grid and
// multi-kernel Arnoldi both use this, so their H stay bitwise equal.
__device__ __forceinline__ void arnoldi_spmv(long long n, const int* __restrict__ p,
                                             const int* __restrict__ c, const double* __restrict__ v,
                                             const double* x, double* y, int vs,
                                             long long gthread, long long gthreads) {
  const int lane = (int)(gthread & 31), sub = lane / vs, sl = lane & (vs - 1);
  const long long per = 32 / vs;  // rows per warp per sweep
  for (long long rb = (gthread >> 5) * per; rb < n; rb += (gthreads >> 5) * per) {
    const long long r = rb + sub;
    double s = 0.0;
    if (r < n)
      for (int k = p[r] + sl; k < p[r + 1]; k += vs) s = fma(v[k], x[c[k]], s);
    for (int o = vs >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, vs);
    if (r < n && sl == 0) y[r] = s;
  }
}

__global__ void spmv_rows_kernel(int n, const int* __restrict__ p, const int* __restrict__ c,
                                 const double* __restrict__ v, const double* __restrict__ x,
                                 double* __restrict__ y, int vs, Gate g) {
  if (g.off()) return;
  arnoldi_spmv(n, p, c, v, x, y, vs, blockIdx.x * (long long)blockDim.x + threadIdx.x,
               (long long)gridDim.x * blockDim.x);
}

// dsc: [0] scratch, [1] projection h, [2] ||w||^2 before, [3] ||w||^2 after, [4] hmax, [5] hn
// ctl: [0] stopped, [1] second sweep, [2] k
__global__ void arnoldi_ctl_kernel(int phase, int j, int m, double* Hd, double* dsc, int* ctl) {
  if (ctl[0]) return;
  const double hn = sqrt(dsc[3]);
  if (phase == 0) {  // after sweep 0: reorthogonalise iff ||w|| dropped below 0.7 of before
    ctl[1] = hn < 0.7 * sqrt(dsc[2]) ? 1 : 0;
    return;
  }
  Hd[(size_t)(j + 1) * m + j] = hn;
  double cn = 0.0;
  for (int q = 0; q <= j + 1; ++q) {
    const double h = Hd[(size_t)q * m + j];
    cn = __dadd_rn(cn, __dmul_rn(h, h));
  }
  dsc[4] = fmax(dsc[4], sqrt(cn));
  if (hn <= 1e-14 * dsc[4]) {  // lucky breakdown
    Hd[(size_t)(j + 1) * m + j] = 0.0;
    ctl[2] = j + 1;
    ctl[0] = 1;
  }
  dsc[5] = hn;
}

struct DotCtx {
  double* parts;
  int np;
};

static int dev_dot(long long n, const double* x, const double* y, double* out, double* acc,
                   const DotCtx& d, Gate g, cudaStream_t s) {
  dot_partial_kernel<<<d.np, 256, 0, s>>>(n, x, y, d.parts, g);
  dot_finish_kernel<<<1, 256, 0, s>>>(d.np, d.parts, out, acc, g);
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

// dot-product partials: one per CTA of the cooperative kernel, which has
// enough threads for one vs-lane group per row (the SpMV), at most 4 per SM
static int arnoldi_parts(int n, int vs) { return blocks_for((long long)n * vs, 256, num_sms() * 4); }

static int arnoldi_multi(int n, const int* p, const int* c, const double* v, const double* b, int m,
                         double* H_h, int* k_h, double* beta_h, int vs, cudaStream_t s) {
  double *V = nullptr, *w = nullptr, *sc = nullptr, *Hd = nullptr;
  int* ctl = nullptr;
  const int np = arnoldi_parts(n, vs);
  AIRG_TRY(scratch(&V, (size_t)(m + 1) * n, s));
  AIRG_TRY(scratch(&w, n, s));
  AIRG_TRY(scratch(&sc, np + 8, s));
  AIRG_TRY(scratch(&Hd, (size_t)(m + 1) * m, s));
  AIRG_TRY(scratch(&ctl, 4, s));
  AIRG_CUDA(cudaMemsetAsync(Hd, 0, (size_t)(m + 1) * m * sizeof(double), s));
  AIRG_CUDA(cudaMemsetAsync(sc, 0, 8 * sizeof(double), s));
  const int ctl0[4] = {0, 0, m, 0};
  AIRG_CUDA(cudaMemcpyAsync(ctl, ctl0, sizeof ctl0, cudaMemcpyHostToDevice, s));
  DotCtx d{sc + 8, np};
  double* dsc = sc;
  const Gate always{nullptr, nullptr};
  const Gate live{ctl, nullptr};        // until the breakdown
  const Gate second{ctl, ctl + 1};      // second sweep only
  double bb = 0;
  AIRG_TRY(dev_dot(n, b, b, dsc, nullptr, d, always, s));
  AIRG_CUDA(read_back(&bb, dsc, sizeof(double), s));
  const double beta = std::sqrt(bb);
  *beta_h = beta;
  if (beta == 0.0) {
    set_error("cannot build a Krylov space from a zero vector");
    return AIRG_ERR_VALUE;
  }
  const int nb = blocks_for(n, 256);
  scale_div_kernel<<<nb, 256, 0, s>>>(n, b, beta, nullptr, V, always);
  for (int j = 0; j < m; ++j) {
    const double* Vj = V + (size_t)j * n;
    spmv_rows_kernel<<<blocks_for((long long)n * vs, 256), 256, 0, s>>>(n, p, c, v, Vj, w, vs, live);
    AIRG_LAUNCH_CHECK();
    AIRG_TRY(dev_dot(n, w, w, dsc + 2, nullptr, d, live, s));
    for (int sweep = 0; sweep < 2; ++sweep) {
      const Gate g = sweep == 0 ? live : second;
      for (int q = 0; q <= j; ++q) {
        const double* Vq = V + (size_t)q * n;
        AIRG_TRY(dev_dot(n, Vq, w, dsc + 1, Hd + q * m + j, d, g, s));
        axpy_dev_kernel<<<nb, 256, 0, s>>>(n, dsc + 1, Vq, w, g);
      }
      AIRG_TRY(dev_dot(n, w, w, dsc + 3, nullptr, d, g, s));
      arnoldi_ctl_kernel<<<1, 1, 0, s>>>(sweep, j, m, Hd, dsc, ctl);
    }
    scale_div_kernel<<<nb, 256, 0, s>>>(n, w, 0.0, dsc + 5, V + (size_t)(j + 1) * n, live);
    AIRG_LAUNCH_CHECK();
  }
  int ctlh[4];
  AIRG_CUDA(read_back({{H_h, Hd, (size_t)(m + 1) * m * sizeof(double)}, {ctlh, ctl, sizeof ctlh}}, s));
  *k_h = ctlh[2];
  release(V, s);
  release(w, s);
  release(sc, s);
  release(Hd, s);
  release(ctl, s);
  return AIRG_OK;
}

// ---- one cooperative kernel for large operators -------------------------
// The multi-kernel recurrence above (same per-element assignment: NP blocks
// of 256 threads, grid-stride; warp per row for the SpMV; dot partials per
// block summed in the dot_finish order), with a grid barrier where a kernel
// boundary was: H and the basis are bitwise the multi-kernel path's, but an
// order-m Arnoldi is one launch instead of ~3 m^2 + 10 m.  The dot reduction
// double-buffers its partials (a block can only rewrite a buffer after the
// barrier of the next dot).  Decisions (second sweep, breakdown) are taken
// redundantly by every block from the same reduced values.
struct ArnoldiGridArgs {
  int n, m;
  const int *p, *c;
  const double* v;
  const double* b;
  double beta;
  double* V;
  double* w;
  double* H;     // (m + 1) x m
  double* parts; // 2 x gridDim.x
  int* info;     // [0] k
  int vs;        // lanes per row of the SpMV
};

__global__ void __launch_bounds__(256) arnoldi_grid_kernel(ArnoldiGridArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[33];
  const int tid = threadIdx.x, np = gridDim.x;
  const long long n = a.n, stride = (long long)np * 256, i0 = (long long)blockIdx.x * 256 + tid;
  int buf = 0;
  auto gdot = [&](const double* x, const double* y) -> double {
    double s = 0.0;
    for (long long i = i0; i < n; i += stride) s = fma(x[i], y[i], s);
    s = block_sum(s, red);
    double* parts = a.parts + (size_t)buf * np;
    buf ^= 1;
    if (tid == 0) parts[blockIdx.x] = s;
    grid.sync();
    double t = 0.0;
    for (int i = tid; i < np; i += 256) t += parts[i];
    return block_sum(t, red);
  };
  const int m = a.m;
  double* V = a.V;
  double* w = a.w;
  for (long long i = i0; i < n; i += stride) V[i] = a.b[i] / a.beta;
  double hmax = 0.0;
  int k = m;
  for (int j = 0; j < m; ++j) {
    grid.sync();  // V_j complete
    const double* Vj = V + (size_t)j * n;
    arnoldi_spmv(n, a.p, a.c, a.v, Vj, w, a.vs, i0, stride);
    grid.sync();  // w complete
    const double before2 = gdot(w, w);
    double hcolj = 0.0;  // unused by blocks > 0
    double after2 = 0.0;
    for (int sweep = 0; sweep < 2; ++sweep) {
      if (sweep == 1 && !(sqrt(after2) < 0.7 * sqrt(before2))) break;
      for (int q = 0; q <= j; ++q) {
        const double* Vq = V + (size_t)q * n;
        const double h = gdot(Vq, w);
        if (blockIdx.x == 0 && tid == 0) a.H[(size_t)q * m + j] += h;
        for (long long i = i0; i < n; i += stride) w[i] -= h * Vq[i];
      }
      after2 = gdot(w, w);
    }
    (void)hcolj;
    const double hn = sqrt(after2);
    // column norm of H(:, j) in the control kernel's order
    grid.sync();  // block 0's H writes visible
    double cn = 0.0;
    for (int q = 0; q <= j; ++q) {
      const double h = a.H[(size_t)q * m + j];
      cn = __dadd_rn(cn, __dmul_rn(h, h));
    }
    cn = __dadd_rn(cn, __dmul_rn(hn, hn));
    hmax = fmax(hmax, sqrt(cn));
    if (hn <= 1e-14 * hmax) {  // lucky breakdown
      k = j + 1;
      break;
    }
    if (blockIdx.x == 0 && tid == 0) a.H[(size_t)(j + 1) * m + j] = hn;
    double* Vn = V + (size_t)(j + 1) * n;
    for (long long i = i0; i < n; i += stride) Vn[i] = w[i] / hn;
  }
  if (blockIdx.x == 0 && tid == 0) a.info[0] = k;
}

static int arnoldi_grid(int n, const int* p, const int* c, const double* v, const double* b, int m,
                        double* H_h, int* k_h, double* beta_h, int vs, cudaStream_t s) {
  double *V = nullptr, *w = nullptr, *sc = nullptr, *Hd = nullptr;
  int* info = nullptr;
  const int np = arnoldi_parts(n, vs);
  AIRG_TRY(scratch(&V, (size_t)(m + 1) * n, s));
  AIRG_TRY(scratch(&w, n, s));
  AIRG_TRY(scratch(&sc, 2 * np + 8, s));
  AIRG_TRY(scratch(&Hd, (size_t)(m + 1) * m, s));
  AIRG_TRY(scratch(&info, 2, s));
  AIRG_CUDA(cudaMemsetAsync(Hd, 0, (size_t)(m + 1) * m * sizeof(double), s));
  // beta with the multi-kernel dot (same partials, same finish)
  DotCtx d{sc + 8, np};
  const Gate always{nullptr, nullptr};
  double bb = 0;
  AIRG_TRY(dev_dot(n, b, b, sc, nullptr, d, always, s));
  AIRG_CUDA(read_back(&bb, sc, sizeof(double), s));
  const double beta = std::sqrt(bb);
  *beta_h = beta;
  if (beta == 0.0) {
    set_error("cannot build a Krylov space from a zero vector");
    return AIRG_ERR_VALUE;
  }
  ArnoldiGridArgs a{n, m, p, c, v, b, beta, V, w, Hd, sc + 8, info, vs};
  void* args[] = {&a};
  AIRG_CUDA(cudaLaunchCooperativeKernel((const void*)arnoldi_grid_kernel, np, 256, args, 0, s));
  int k = 0;
  AIRG_CUDA(read_back({{H_h, Hd, (size_t)(m + 1) * m * sizeof(double)}, {&k, info, sizeof(int)}}, s));
  *k_h = k;
  for (void* q : {(void*)V, (void*)w, (void*)sc, (void*)Hd, (void*)info}) release(q, s);
  return AIRG_OK;
}

// whether the cooperative kernel fits co-resident (it always does on B200:
// at most 592 blocks of 256 threads); otherwise the multi-kernel path
static bool grid_arnoldi_ok(int n, int vs) {
  static int max_blocks = -1;
  if (max_blocks < 0) {
    int per_sm = 0, dev = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    if (!coop ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, arnoldi_grid_kernel, 256, 0) != cudaSuccess)
      per_sm = 0;
    max_blocks = per_sm * num_sms();
  }
  return !getenv("AIRG_ARNOLDI_MULTI") && arnoldi_parts(n, vs) <= max_blocks;
}

}  // namespace airg

using namespace airg;

extern "C" int airg_arnoldi(int n, const int32_t* p, const int32_t* c, const double* v,
                            const double* b, int m, double* H_h, int32_t* k_h, double* beta_h,
                            void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (m < 1 || n < 1) {
    set_error("Arnoldi needs m >= 1 and n >= 1");
    return AIRG_ERR_VALUE;
  }
  if (m > n) m = n;
  int st = AIRG_OK;
  if (n <= kArnoldiCta) {
    double *V = nullptr, *w = nullptr, *H = nullptr, *dinfo = nullptr;
    int* info = nullptr;
    AIRG_TRY(scratch(&V, (size_t)(m + 1) * n, s));
    AIRG_TRY(scratch(&w, n, s));
    AIRG_TRY(scratch(&H, (size_t)(m + 1) * m, s));
    AIRG_TRY(scratch(&dinfo, 1, s));
    AIRG_TRY(scratch(&info, 2, s));
    static_assert(kArnoldiCta <= 256 * 16, "one CTA of 256 threads, 16 entries each");
    // as many basis vectors in shared memory as fit
    const size_t hbytes = (size_t)((m + 2) & ~1) * sizeof(double);
    const size_t cap = 200 * 1024;
    const int vsm = (int)std::min<size_t>((size_t)(m + 1), (cap - hbytes) / ((size_t)n * sizeof(double)));
    const size_t shm = hbytes + (size_t)vsm * n * sizeof(double);
    static bool attr = false;
    if (!attr) {
      AIRG_CUDA(cudaFuncSetAttribute(arnoldi_cta_kernel<256, 16>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap));
      AIRG_CUDA(cudaFuncSetAttribute(arnoldi_cta_kernel<256, 2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap));
      attr = true;
    }
    // up to 512 rows (coarsest grids): one-warp Gram-Schmidt; else 16 entries
    // per thread of the CTA up to 4096
    if (n <= 512 && !getenv("AIRG_ARNOLDI_CTA")) {
      const size_t wbytes = hbytes + (size_t)((n + 1) & ~1) * sizeof(double);
      const int vw = (int)std::min<size_t>((size_t)(m + 1), (cap - wbytes) / ((size_t)n * sizeof(double)));
      const size_t shw = wbytes + (size_t)vw * n * sizeof(double);
      static bool wattr = false;
      if (!wattr) {
        for (auto k : {arnoldi_warp_kernel<4>, arnoldi_warp_kernel<8>, arnoldi_warp_kernel<16>})
          AIRG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap));
        wattr = true;
      }
      auto k = n <= 128 ? arnoldi_warp_kernel<4> : n <= 256 ? arnoldi_warp_kernel<8> : arnoldi_warp_kernel<16>;
      k<<<1, 256, shw, s>>>(n, p, c, v, b, m, V, H, info, dinfo, vw);
    } else if (n <= 512)
      arnoldi_cta_kernel<256, 2><<<1, 256, shm, s>>>(n, p, c, v, b, m, V, w, H, info, dinfo, vsm);
    else
      arnoldi_cta_kernel<256, 16><<<1, 256, shm, s>>>(n, p, c, v, b, m, V, w, H, info, dinfo, vsm);
    AIRG_LAUNCH_CHECK();
    int hi[2];
    AIRG_CUDA(read_back({{H_h, H, (size_t)(m + 1) * m * sizeof(double)}, {hi, info, sizeof hi},
                         {beta_h, dinfo, sizeof(double)}}, s));
    for (void* q : {(void*)V, (void*)w, (void*)H, (void*)dinfo, (void*)info}) release(q, s);
    if (hi[1]) {
      set_error("cannot build a Krylov space from a zero vector");
      return AIRG_ERR_VALUE;
    }
    *k_h = hi[0];
  } else {
    int nnz = 0;
    AIRG_CUDA(read_back(&nnz, p + n, sizeof(int), s));
    const int vs = arnoldi_vs(nnz, n);
    st = grid_arnoldi_ok(n, vs) ? arnoldi_grid(n, p, c, v, b, m, H_h, k_h, beta_h, vs, s)
                                : arnoldi_multi(n, p, c, v, b, m, H_h, k_h, beta_h, vs, s);
    if (st != AIRG_OK) return st;
  }
  // numerically zero on the Krylov space? (polynomial.py:108-109)
  const int k = *k_h;
  double mx = 0.0;
  for (int i = 0; i <= k; ++i)
    for (int j = 0; j < k; ++j) mx = std::max(mx, std::fabs(H_h[(size_t)i * m + j]));
  if (mx == 0.0) {
    set_error("matrix is numerically zero on the Krylov space");
    return AIRG_ERR_VALUE;
  }
  return AIRG_OK;
}
