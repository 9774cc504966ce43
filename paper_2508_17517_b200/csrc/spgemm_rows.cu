// General SpGEMM (Z = -A_cf Ahat, A P, R (A P)) and the fused Galerkin
// product with drop/lump.  Kernel design in spgemm_core.cuh.
// ref: sparse.py:222-240 (spgemm), hierarchy.py:281-286 (coarse_matrix)
#include "spgemm_span.cuh"
#include <vector>
#include <algorithm>

namespace airg {

// ---- row classification ------------------------------------------------------
__global__ void product_ub_kernel(int m, const int* __restrict__ Ap, const int* __restrict__ Ac,
                                  const int* __restrict__ Bp, long long* __restrict__ ub) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    long long s = 0;
    for (int k = Ap[i]; k < Ap[i + 1]; ++k) {
      const int c = Ac[k];
      s += Bp[c + 1] - Bp[c];
    }
    ub[i] = s;
  }
}

// ---- pass 1: structural count -------------------------------------------------
struct CountArgs {
  const int *Ap, *Ac, *Bp, *Bc;
  const int* rows;
  int nrows;
  int bits;  // shared tables (log2 slots); global tables when gtab != nullptr
  int limit;
  int* cnt;
  int* ovf_rows;
  int* ovf_n;
  int* gtab;
  const long long* goff;
  const int* gbits;
};

struct CountCheckOp {
  int* keys;
  int bits;
  int added;
  __device__ __forceinline__ void operator()(double, int c, double) { added += set_insert(keys, bits, c); }
};

// Long rows (product upper bound > 512): one CTA per row sharing one
// shared-memory key set.  Counting has no ordering constraint, so warps take
// chunks of kCountChunk A entries from a shared cursor (dynamic balance: the
// B rows behind the entries vary in length, a static split left warps idle at
// the end-of-row barrier).
constexpr int kCountChunk = 8;
__global__ void __launch_bounds__(256) spgemm_count_block_kernel(CountArgs a) {
  extern __shared__ int keys[];
  __shared__ int total, ovf, cursor;
  const int tid = threadIdx.x, lane = tid & 31;
  const int bits = a.bits, T = 1 << bits;
  for (long long t = blockIdx.x; t < a.nrows; t += gridDim.x) {
    const int row = a.rows[t];
    for (int i = tid; i < T; i += blockDim.x) keys[i] = kEmpty;
    const int ab0 = a.Ap[row], ae = a.Ap[row + 1];
    if (tid == 0) {
      total = 0;
      ovf = 0;
      cursor = ab0;
    }
    __syncthreads();
    // per chunk: the B-row bounds are loaded lane-parallel, the next B row's
    // first 32 columns are prefetched while the current row is inserted
    while (true) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&cursor, kCountChunk);
      base = __shfl_sync(kFull, base, 0);
      if (base >= ae) break;
      int bb = 0, be = 0;
      if (lane < kCountChunk && base + lane < ae) {
        const int k = a.Ac[base + lane];
        bb = a.Bp[k];
        be = a.Bp[k + 1];
      }
      const int cnt = min(kCountChunk, ae - base);
      int cb = __shfl_sync(kFull, bb, 0), ce = __shfl_sync(kFull, be, 0);
      int pc = cb + lane < ce ? a.Bc[cb + lane] : -1;
      int added = 0;
      for (int tt = 0; tt < cnt; ++tt) {
        const int tb = cb, te = ce, c0 = pc;
        if (tt + 1 < cnt) {
          cb = __shfl_sync(kFull, bb, tt + 1);
          ce = __shfl_sync(kFull, be, tt + 1);
          pc = cb + lane < ce ? a.Bc[cb + lane] : -1;
        }
        if (c0 >= 0) added += set_insert(keys, bits, c0);
        for (int jb = tb + 32; jb < te; jb += 96) {
          int cc[3];
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const int jj = jb + 32 * q + lane;
            cc[q] = jj < te ? a.Bc[jj] : -1;
          }
#pragma unroll
          for (int q = 0; q < 3; ++q)
            if (cc[q] >= 0) added += set_insert(keys, bits, cc[q]);
        }
      }
      added = warp_sum(added);
      if (lane == 0 && added) {
        if (atomicAdd(&total, added) + added > a.limit) ovf = 1;
      }
      if (__shfl_sync(kFull, lane == 0 ? *(volatile int*)&ovf : 0, 0)) break;
    }
    __syncthreads();
    if (tid == 0) {
      if (ovf || total > a.limit) a.ovf_rows[atomicAdd(a.ovf_n, 1)] = row;
      else a.cnt[row] = total;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) spgemm_count_kernel(CountArgs a) {
  extern __shared__ int smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (long long t = (long long)blockIdx.x * nw + w; t < a.nrows; t += (long long)gridDim.x * nw) {
    const int row = a.rows[t];
    int* keys;
    int bits;
    if (a.gtab) {
      keys = a.gtab + a.goff[t];
      bits = a.gbits[t];
    } else {
      keys = smem + (size_t)w * (1 << a.bits);
      bits = a.bits;
    }
    const int T = 1 << bits;
    for (int i = lane; i < T; i += 32) keys[i] = kEmpty;
    __syncwarp();
    // walk in chunks of A entries so an overflowing row bails out early
    CountCheckOp op{keys, bits, 0};
    const int ab = a.Ap[row], ae = a.Ap[row + 1];
    bool ovf = false;
    for (int base = ab; base < ae && !ovf; base += 32) {
      // B-row bounds of 32 A entries at once (one per lane)
      int bb = 0, be = 0;
      if (base + lane < ae) {
        const int k = a.Ac[base + lane];
        bb = a.Bp[k];
        be = a.Bp[k + 1];
      }
      const int cnt = min(32, ae - base);
      for (int t = 0; t < cnt; ++t) {
        const int tb = __shfl_sync(kFull, bb, t), te = __shfl_sync(kFull, be, t);
        for (int jb = tb; jb < te; jb += 128) {
          int cc[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int jj = jb + 32 * q + lane;
            cc[q] = jj < te ? a.Bc[jj] : -1;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (cc[q] >= 0) op(0.0, cc[q], 0.0);
        }
      }
      if (!a.gtab) ovf = warp_sum(op.added) > a.limit;
    }
    const int n = warp_sum(op.added);
    if (ovf || (!a.gtab && n > a.limit)) {
      if (lane == 0) a.ovf_rows[atomicAdd(a.ovf_n, 1)] = row;
    } else if (lane == 0) {
      a.cnt[row] = n;
    }
    __syncwarp();
  }
}

// ---- pass 2: numeric + structure --------------------------------------------------
struct NumArgs {
  const int *Ap, *Ac;
  const double* Av;
  const int *Bp, *Bc;
  const double* Bv;
  const int* rows;
  int nrows;
  int bits;
  const int* Cp;
  int* Cc;
  double* Cv;
  int negate;
  int mode;  // 0 plain, 1 fused drop/lump into raw offsets
  double tol;
  int lump;
  int* out_cnt;
  int* any_drop;
  int* gkeys;
  double* gacc;
  const long long* goff;
  const int* gbits;
  int row0;  // global id of local output row 0 (diagonal of the drop/lump epilogue)
};

__global__ void __launch_bounds__(256) spgemm_numeric_kernel(NumArgs a) {
  extern __shared__ double smd[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (long long t = (long long)blockIdx.x * nw + w; t < a.nrows; t += (long long)gridDim.x * nw) {
    const int row = a.rows[t];
    int bits;
    int* keys;
    double* acc;
    int* cnt;
    if (a.gkeys) {
      bits = a.gbits[t];
      keys = a.gkeys + a.goff[t];
      acc = a.gacc + a.goff[t];
      cnt = keys + (1 << bits) - 256;  // global tables are sized >= 2n + 256
    } else {
      bits = a.bits;
      const int T = 1 << bits;
      acc = smd + (size_t)w * ((size_t)T * 3 / 2 + 128);  // T doubles + T ints + 256 ints
      keys = (int*)(acc + T);
      cnt = keys + T;
    }
    const int T = 1 << bits;
    for (int i = lane; i < T; i += 32) {
      keys[i] = kEmpty;
      acc[i] = 0.0;
    }
    __syncwarp();
    AccOp op{keys, acc, bits};
    walk_products<true, true>(a.Ap, a.Ac, a.Av, a.Bp, a.Bc, a.Bv, row, lane, op);
    __syncwarp();
    const int n = compact_slots(keys, acc, T, lane);
    if (n <= 64) {
      int P = 1;
      while (P < n) P <<= 1;
      for (int i = n + lane; i < P; i += 32) keys[i] = 0x7fffffff;
      __syncwarp();
      warp_bitonic(keys, acc, P, lane);
    } else {
      warp_radix_sort(keys, acc, keys + n, acc + n, n, cnt, lane);
    }
    const int o = a.Cp[row];
    if (a.mode == 0) {
      for (int i = lane; i < n; i += 32) {
        a.Cc[o + i] = keys[i];
        const double v = acc[i];
        a.Cv[o + i] = a.negate ? -v : v;
      }
    } else {
      const int wr = drop_lump_row(keys, acc, n, a.row0 + row, a.tol, a.lump, a.Cc, a.Cv,
                                   (long long)o + row, lane, a.any_drop);
      if (lane == 0) a.out_cnt[row] = wr;
    }
    __syncwarp();
  }
}

// Long output rows: one CTA per row, the row's key -> slot table and
// accumulators in shared memory shared by all warps.  Each B row is consumed
// by the whole CTA in one step (threads split its entries); steps are ordered
// by __syncthreads, so every output entry still receives its k in ascending
// order.  The next B row is prefetched into registers during the current
// step.  Warp 0 compacts, sorts and writes the row (a block-wide CUB sort
// was tried: 112 registers/thread cut occupancy to 25% and doubled the time).
template <int NT, int BITS>
__global__ void __launch_bounds__(NT) spgemm_numeric_block_kernel(NumArgs a) {
  constexpr int T = 1 << BITS;
  extern __shared__ double smd[];
  __shared__ int mbb[32], mbe[32];
  __shared__ double mav[32];
  const int tid = threadIdx.x, lane = tid & 31;
  double* acc = smd;
  int* keys = (int*)(acc + T);
  for (long long t = blockIdx.x; t < a.nrows; t += gridDim.x) {
    const int row = a.rows[t];
    for (int i = tid; i < T; i += NT) {
      keys[i] = kEmpty;
      acc[i] = 0.0;
    }
    AccOp op{keys, acc, BITS};
    const int ab = a.Ap[row], ae = a.Ap[row + 1];
    for (int base = ab; base < ae; base += 32) {
      __syncthreads();
      if (tid < 32 && base + tid < ae) {
        const int k = a.Ac[base + tid];
        mav[tid] = a.Av[base + tid];
        mbb[tid] = a.Bp[k];
        mbe[tid] = a.Bp[k + 1];
      }
      __syncthreads();
      const int cnt_k = min(32, ae - base);
      int cb = mbb[0], ce = mbe[0];
      int pc = cb + tid < ce ? a.Bc[cb + tid] : -1;
      double pv = cb + tid < ce ? a.Bv[cb + tid] : 0.0;
      for (int tt = 0; tt < cnt_k; ++tt) {
        const double av = mav[tt];
        const int tb = cb, te = ce, c0 = pc;
        const double v0 = pv;
        if (tt + 1 < cnt_k) {
          cb = mbb[tt + 1];
          ce = mbe[tt + 1];
          pc = cb + tid < ce ? a.Bc[cb + tid] : -1;
          pv = cb + tid < ce ? a.Bv[cb + tid] : 0.0;
        }
        if (c0 >= 0) op(av, c0, v0);
        for (int jj = tb + NT + tid; jj < te; jj += NT) op(av, a.Bc[jj], a.Bv[jj]);
        __syncthreads();
      }
    }
    __syncthreads();
    if (tid < 32) {  // warp 0 compacts, sorts and writes the row
      const int n = compact_slots(keys, acc, T, lane);
      if (n <= 64) {
        int P = 1;
        while (P < n) P <<= 1;
        for (int i = n + lane; i < P; i += 32) keys[i] = 0x7fffffff;
        __syncwarp();
        warp_bitonic(keys, acc, P, lane);
      } else {
        warp_radix_sort(keys, acc, keys + n, acc + n, n, keys + T, lane);
      }
      const int o = a.Cp[row];
      if (a.mode == 0) {
        for (int i = lane; i < n; i += 32) {
          a.Cc[o + i] = keys[i];
          const double v = acc[i];
          a.Cv[o + i] = a.negate ? -v : v;
        }
      } else {
        const int wr = drop_lump_row(keys, acc, n, a.row0 + row, a.tol, a.lump, a.Cc, a.Cv,
                                     (long long)o + row, lane, a.any_drop);
        if (lane == 0) a.out_cnt[row] = wr;
      }
    }
    __syncthreads();
  }
}

__global__ void compact_raw_kernel(int m, const int* __restrict__ rawp, const int* __restrict__ optr,
                                   const int* __restrict__ icol, const double* __restrict__ ival,
                                   int* __restrict__ ocol, double* __restrict__ oval) {
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < m;
       r += ((long long)gridDim.x * blockDim.x) >> 5) {
    const long long src = (long long)rawp[r] + r;
    const int dst = optr[r], n = optr[r + 1] - dst;
    for (int i = lane; i < n; i += 32) {
      ocol[dst + i] = icol[src + i];
      oval[dst + i] = ival[src + i];
    }
  }
}

__global__ void iota_kernel(int n, int* __restrict__ p) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = (int)i;
}

__global__ void ones_kernel(long long n, double* __restrict__ v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v[i] = 1.0;
}

struct Mat {
  int nrows, ncols;
  const int* p;
  const int* c;
  const double* v;
};

static int set_smem(const void* fn, size_t shm) {
  if (shm > 48 * 1024)
    AIRG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  return AIRG_OK;
}

// global-memory tables for rows beyond the shared-memory classes
struct GlobalTables {
  int* rows = nullptr;
  int* bits = nullptr;
  long long* off = nullptr;
  int* keys = nullptr;
  double* acc = nullptr;
  int n = 0;
  void free(cudaStream_t s) {
    for (void* q : {(void*)rows, (void*)bits, (void*)off, (void*)keys, (void*)acc}) release(q, s);
  }
};

// sizes: per-row key counts to hold (table = pow2 >= 2*size)
static int make_tables(const std::vector<int>& rows, const std::vector<long long>& sizes, bool values,
                       GlobalTables& g, cudaStream_t s) {
  const int n = (int)rows.size();
  g.n = n;
  if (!n) return AIRG_OK;
  std::vector<long long> off(n);
  std::vector<int> bits(n);
  long long tot = 0;
  for (int i = 0; i < n; ++i) {
    bits[i] = std::max(5, ceil_log2(2 * std::max(1ll, sizes[i]) + (values ? 256 : 0)));
    off[i] = tot;
    tot += 1ll << bits[i];
  }
  AIRG_TRY(scratch(&g.rows, n, s));
  AIRG_TRY(scratch(&g.bits, n, s));
  AIRG_TRY(scratch(&g.off, n, s));
  AIRG_TRY(scratch(&g.keys, tot, s));
  if (values) AIRG_TRY(scratch(&g.acc, tot, s));
  AIRG_CUDA(cudaMemcpyAsync(g.rows, rows.data(), n * sizeof(int), cudaMemcpyHostToDevice, s));
  AIRG_CUDA(cudaMemcpyAsync(g.bits, bits.data(), n * sizeof(int), cudaMemcpyHostToDevice, s));
  AIRG_CUDA(cudaMemcpyAsync(g.off, off.data(), n * sizeof(long long), cudaMemcpyHostToDevice, s));
  return AIRG_OK;
}

static int gather_ll(const long long* d, const std::vector<int>& rows, std::vector<long long>& out,
                     cudaStream_t s, int m) {
  std::vector<long long> all(m);
  AIRG_CUDA(cudaMemcpyAsync(all.data(), d, m * sizeof(long long), cudaMemcpyDeviceToHost, s));
  AIRG_CUDA(cudaStreamSynchronize(s));
  out.resize(rows.size());
  for (size_t i = 0; i < rows.size(); ++i) out[i] = all[rows[i]];
  return AIRG_OK;
}

// ---- rows with few products: the whole row in registers ---------------------
// G lanes per row (32 / G rows per warp), for rows with at most G products
// and at most G entries in A's row.  Lane t forms product t in scipy's
// generation order (A's row in order, each B row in order); a lane is the
// head of its column if no earlier lane has the column, its output position
// is the number of head columns below it, and the head sums the column's
// products over the lanes in order: 0 + p_1 + p_2 + ... (separate roundings),
// the order of the hash and span kernels -- bitwise the same rows.  Count
// pass: the number of heads.  Numeric pass: the values, written at the
// row's offset (mode 0), or drop/lump (drop_lump_row's rules, dropped values
// summed in column order) at the raw offset Cp[row] + row (mode 1).
struct RegArgs {
  const int *Ap, *Ac;
  const double* Av;
  const int *Bp, *Bc;
  const double* Bv;
  const int* rows;
  int nrows;
  int count_only;
  const int* Cp;
  int* Cc;
  double* Cv;
  int negate, mode;
  double tol;
  int lump;
  int* cnt;       // count pass: unique columns; mode 1: entries written
  int* any_drop;
  int row0;
};

// occupancy cap (CTAs/SM) of the register SpGEMM classes: 5 (48 registers,
// small spills) measured within 1 ms of the setup, 6 spills more; left free
// (an explicit 1 is not the same: it lets ptxas take 80+ registers)
#ifdef AIRG_REG_MINB
#define AIRG_REG_BOUNDS __launch_bounds__(256, AIRG_REG_MINB)
#else
#define AIRG_REG_BOUNDS __launch_bounds__(256)
#endif
template <int G>
__global__ void AIRG_REG_BOUNDS spgemm_reg_kernel(RegArgs a) {
  const int lane = threadIdx.x & 31, j = lane & (G - 1), gbase = lane & ~(G - 1);
  const unsigned gmask = G == 32 ? kFull : ((1u << G) - 1u) << gbase;
  const long long groups = ((long long)gridDim.x * blockDim.x) / G;
  for (long long g0 = ((long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / G; g0 < a.nrows;
       g0 += groups) {  // warp-uniform trip count: the groups of a warp shuffle together
    const long long r = g0 + lane / G;
    const bool live = r < a.nrows;
    const int row = live ? a.rows[r] : 0;
    const int ab = live ? a.Ap[row] : 0, na = live ? a.Ap[row + 1] - ab : 0;
    int bb = 0, bl = 0;
    double av = 0.0;
    if (j < na) {
      const int k = a.Ac[ab + j];
      av = a.Av[ab + j];
      bb = a.Bp[k];
      bl = a.Bp[k + 1] - bb;
    }
    int incl = bl;  // inclusive scan of the B-row lengths over the group
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o, G);
      if (j >= o) incl += y;
    }
    const int excl = incl - bl;
    const int P = __shfl_sync(kFull, incl, G - 1, G);
    // product j: the A entry q with excl_q <= j < incl_q
    int q = 0;
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int ei = __shfl_sync(kFull, excl, i, G), li = __shfl_sync(kFull, bl, i, G);
      if (j >= ei && j < ei + li) q = i;
    }
    const int bq = __shfl_sync(kFull, bb, q, G), eq = __shfl_sync(kFull, excl, q, G);
    const double aq = __shfl_sync(kFull, av, q, G);
    const bool has = j < P;
    const int c = has ? a.Bc[bq + j - eq] : INT_MAX;
    const double pv = has ? mul_rn(aq, a.Bv[bq + j - eq]) : 0.0;
    bool head = has;
    double sum = 0.0;
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int ci = __shfl_sync(kFull, c, i, G);
      const double pi = __shfl_sync(kFull, pv, i, G);
      if (i < j && ci == c) head = false;
      if (i < P && ci == c) sum = add_rn(sum, pi);
    }
    int pos = 0;
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int ci = __shfl_sync(kFull, c, i, G);
      const bool hi = __shfl_sync(kFull, head, i, G);
      if (hi && ci < c) ++pos;
    }
    const int U = __popc(__ballot_sync(kFull, head) & gmask);
    if (a.count_only) {
      if (live && j == 0) a.cnt[row] = U;
      continue;
    }
    if (a.mode == 0) {
      if (head) {
        const long long o = (long long)a.Cp[row] + pos;
        a.Cc[o] = c;
        a.Cv[o] = a.negate ? -sum : sum;
      }
      continue;
    }
    // ---- mode 1: drop / lump (drop_lump_row) ----
    const int diag = a.row0 + row;
    double mx = head ? fabs(sum) : 0.0;
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, o, G));
    const unsigned dball = __ballot_sync(kFull, head && c == diag) & gmask;
    const bool has_diag = dball != 0u;
    const double thr = mul_rn(a.tol, mx);
    const bool drop = head && c != diag && !(fabs(sum) >= thr);
    const unsigned dropb = __ballot_sync(kFull, drop) & gmask;
    const int ndrop = __popc(dropb);
    double lumped = 0.0;  // dropped values in column order (ascending pos)
    const int Umax = __reduce_max_sync(kFull, U);  // warp-uniform trip count
    for (int qq = 0; qq < Umax; ++qq) {
      const unsigned src = __ballot_sync(kFull, head && pos == qq) & gmask;
      const int sl = __ffs(src) - 1 - gbase;
      const double v = __shfl_sync(kFull, sum, sl < 0 ? 0 : sl, G);
      const bool dq = __shfl_sync(kFull, drop, sl < 0 ? 0 : sl, G);
      if (sl >= 0 && dq) lumped = add_rn(lumped, v);
    }
    const bool keep = head && !drop;
    const bool insert = a.lump && ndrop > 0 && !has_diag && lumped != 0.0;
    int krank = 0, before = 0;
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int ci = __shfl_sync(kFull, c, i, G);
      const bool ki = __shfl_sync(kFull, keep, i, G);
      if (ki && ci < c) ++krank;
      if (ki && ci < diag) ++before;
    }
    const long long o = (long long)(live ? a.Cp[row] : 0) + row;
    if (keep) {
      double x = sum;
      if (c == diag && a.lump && ndrop > 0) x = add_rn(x, lumped);
      const int dst = krank + (insert && c > diag ? 1 : 0);
      a.Cc[o + dst] = c;
      a.Cv[o + dst] = x;
    }
    const int kept = __popc(__ballot_sync(kFull, keep) & gmask);
    if (live && j == 0) {
      if (insert) {
        a.Cc[o + before] = diag;
        a.Cv[o + before] = lumped;
      }
      a.cnt[row] = kept + (insert ? 1 : 0);
      if (ndrop && a.any_drop) atomicOr(a.any_drop, 1);
    }
  }
}

template <int G>
static int launch_reg(const RegArgs& a, cudaStream_t s) {
  spgemm_reg_kernel<G><<<blocks_for((long long)a.nrows * G, 256), 256, 0, s>>>(a);
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

// rows of the register classes: not on the span path, <= 8 / <= kRegMax2
// products and A entries (a 32-lane class measured slower than the hash
// warp kernels: three 32-step shuffle loops per row)
#ifndef AIRG_REG2
#define AIRG_REG2 16
#endif
constexpr int kRegMax2 = AIRG_REG2;
__device__ __forceinline__ int reg_class(long long words, long long ub, int na) {
  if (words > 0) return -1;
  if (ub <= 8 && na <= 8) return 0;
  if (ub <= kRegMax2 && na <= kRegMax2) return 1;
  return -1;
}

// count-pass class of a row: span path (window <= 4096 / <= 16384 columns)
// or the hash classes by product upper bound
enum { kCntHash64 = 0, kCntSpan4k = 1, kCntSpan16k = 2, kCntHash512 = 3, kCntHashBlk = 4,
       kCntSpan64k = 5, kCntReg8 = 6, kCntReg32 = 7, kCntClasses = 8 };

__global__ void count_class_kernel(int m, const int* __restrict__ Ap, const long long* __restrict__ ub,
                                   const long long* __restrict__ words, int* __restrict__ ids) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const long long w = words[i], u = ub[i];
    const int rc = reg_class(w, u, Ap[i + 1] - Ap[i]);
    ids[i] = rc >= 0 ? kCntReg8 + rc
           : w > 0 ? (w * 32 <= 4096 ? kCntSpan4k : w * 32 <= 16384 ? kCntSpan16k : kCntSpan64k)
                   : (u <= 64 ? kCntHash64 : u <= 512 ? kCntHash512 : kCntHashBlk);
  }
}

// numeric-pass class: span rows by output length (kSpanCaps), then the hash
// classes (<= 32, <= 128 warp per row; <= 512 ... <= 8192 CTA per row;
// longer: global tables)
constexpr int kNumSpanCls = 10;
__constant__ int kSpanCapsDev[kNumSpanCls] = {128, 256, 384, 512, 768, 1024, 1536, 2048, 3072, 4096};
static const int kSpanCaps[kNumSpanCls] = {128, 256, 384, 512, 768, 1024, 1536, 2048, 3072, 4096};
constexpr int kNumHashCls = 8;
constexpr int kNumRegCls = 2;  // after the span and hash classes
__global__ void numeric_class_kernel(int m, const int* __restrict__ Cp, const int* __restrict__ Ap,
                                     const long long* __restrict__ ub,
                                     const long long* __restrict__ words, int* __restrict__ ids) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const int n = Cp[i + 1] - Cp[i];
    const int rc = reg_class(words[i], ub[i], Ap[i + 1] - Ap[i]);
    int c;
    if (rc >= 0) {
      c = kNumSpanCls + kNumHashCls + rc;
    } else if (words[i] > 0 && n <= kSpanNmax) {
      c = 0;
      while (n > kSpanCapsDev[c]) ++c;
    } else {
      c = kNumSpanCls + (n <= 32 ? 0 : n <= 128 ? 1 : n <= 512 ? 2 : n <= 1024 ? 3 : n <= 2048 ? 4
                         : n <= 4096 ? 5 : n <= 8192 ? 6 : 7);
    }
    ids[i] = c;
  }
}

template <int NW, int KP, int D>
static int launch_span_numeric_nw(const SpanNumArgs& a, cudaStream_t s) {
  const size_t shm = span_num_bytes(a.ncap, a.wcap) * NW;
  static size_t attr = 0;
  if (shm > attr) {
    AIRG_CUDA(cudaFuncSetAttribute(span_numeric_kernel<NW, KP, D>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    attr = shm;
  }
  span_numeric_kernel<NW, KP, D><<<blocks_for(a.nrows, NW, num_sms() * 64), 32 * NW, shm, s>>>(a);
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

// warps per CTA: consecutive output rows share most B rows, so the warps of
// one CTA (same SM, same L1) take consecutive rows; as many as fit in
// shared memory up to AIRG_SPAN_NW (measurement knob)
template <int KP, int D>
static int launch_span_numeric_t(const SpanNumArgs& a, cudaStream_t s) {
  static const int nw_max = getenv("AIRG_SPAN_NW") ? atoi(getenv("AIRG_SPAN_NW")) : 2;
  int nw = nw_max;
  while (nw > 1 && span_num_bytes(a.ncap, a.wcap) * nw > 200 * 1024) nw >>= 1;
  switch (nw) {
    case 8: return launch_span_numeric_nw<8, KP, D>(a, s);
    case 4: return launch_span_numeric_nw<4, KP, D>(a, s);
    case 2: return launch_span_numeric_nw<2, KP, D>(a, s);
    default: return launch_span_numeric_nw<1, KP, D>(a, s);
  }
}

// B-row prefetch shape kd = 10 KP + D (KP x 32 entries, D steps ahead);
// AIRG_SPAN_KD="KP,D" overrides it (measurement only)
static int launch_span_numeric(SpanNumArgs a, int ncap, int kd, cudaStream_t s) {
  a.ncap = ncap;
  if (const char* e = getenv("AIRG_SPAN_KD")) {
    int kp = 4, d = 4;
    sscanf(e, "%d,%d", &kp, &d);
    kd = kp * 10 + d;
  }
  switch (kd) {
    case 82: return launch_span_numeric_t<8, 2>(a, s);
    case 24: return launch_span_numeric_t<2, 4>(a, s);
    default: return launch_span_numeric_t<4, 4>(a, s);
  }
}

template <int NT>
static int launch_span_count(const SpanCountArgs& a, int span, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    AIRG_CUDA(cudaFuncSetAttribute(span_count_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kSpanMax));
    attr = true;
  }
  span_count_kernel<NT><<<std::min(a.nrows, num_sms() * 16), NT, (size_t)span, s>>>(a);
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

// rows with at least this many products may take the span path (below it
// the hash set of 128 slots is cheaper than sweeping a window)
static int span_min_ub() {
  static const int v = getenv("AIRG_SPAN_MIN_UB") ? atoi(getenv("AIRG_SPAN_MIN_UB")) : 65;
  return v;
}

// C = A B (mode 0, optionally negated) or drop_and_lump(A B) (mode 1).
static int spgemm_rows(const Mat& A, const Mat& B, int negate, int mode, double tol, int lump,
                       airg_csr_result** out, cudaStream_t s, int row0 = 0) {
  const int m = A.nrows;
  long long *ub = nullptr, *rl = nullptr, *words = nullptr, *bmoff = nullptr;
  int *cnt = nullptr, *Cp = nullptr, *cmin = nullptr, *ids = nullptr;
  unsigned* gbm = nullptr;
  AIRG_TRY(scratch(&ub, m, s));
  AIRG_TRY(scratch(&cnt, m + 1, s));
  AIRG_TRY(scratch(&Cp, m + 1, s));
  AIRG_TRY(scratch(&cmin, m, s));
  AIRG_TRY(scratch(&words, m, s));
  AIRG_TRY(scratch(&bmoff, m + 1, s));
  AIRG_TRY(scratch(&ids, m, s));
  unsigned long long* tot = nullptr;
  AIRG_TRY(scratch(&tot, 3, s));
  AIRG_CUDA(cudaMemsetAsync(tot, 0, 3 * sizeof(unsigned long long), s));
  if (m > 0)
    span_ub_kernel<8><<<blocks_for((long long)m * 8, 256), 256, 0, s>>>(m, A.p, A.c, B.p, B.c, ub,
                                                                         cmin, words, span_min_ub(), tot);
  AIRG_LAUNCH_CHECK();
  unsigned long long tot_h[3] = {0, 0, 0};
  long long totw = 0;
  AIRG_TRY(scan_counts64(words, bmoff, m, nullptr, s));
  AIRG_CUDA(read_back({{tot_h, tot, sizeof(tot_h)}, {&totw, bmoff + m, sizeof(long long)}}, s));
  release(tot, s);
  // mean B-row length of the span rows sets the numeric prefetch shape: rows
  // longer than 4 x 32 entries would run their tail with exposed latency
  // (KP, D) = (2, 4) up to 48 entries, (4, 4) up to 112, (8, 2) above
  // (measured per level at 2048^2, tools/span_micro.py --kd: levels 3-4 5 %
  // faster with (2, 4), levels 7-8 5-20 % with (8, 2))
  const int span_kd = !tot_h[1] ? 44 : tot_h[0] > 112ull * tot_h[1] ? 82
                    : tot_h[0] > 48ull * tot_h[1] ? 44 : 24;
  AIRG_TRY(scratch(&gbm, totw, s));
  // ---- pass 1 ----
  {
    if (m > 0) count_class_kernel<<<blocks_for(m, 256), 256, 0, s>>>(m, A.p, ub, words, ids);
    AIRG_LAUNCH_CHECK();
    Classes cl;
    AIRG_TRY(classify_ids(m, ids, kCntClasses, cl, s));
    int *ovf_rows = nullptr, *ovf_n = nullptr;
    AIRG_TRY(scratch(&ovf_rows, m > 0 ? m : 1, s));
    AIRG_TRY(scratch(&ovf_n, 1, s));
    AIRG_CUDA(cudaMemsetAsync(ovf_n, 0, sizeof(int), s));
    AIRG_TRY(set_smem((const void*)spgemm_count_kernel, (size_t)8 * 4096 * sizeof(int)));
    Fork fk;
    AIRG_TRY(fk.begin(s));
    for (int c = 0; c < kCntClasses; ++c) {
      const int nr = cl.count[c];
      if (!nr) continue;
      if (c == kCntReg8 || c == kCntReg32) {
        RegArgs a{A.p, A.c, A.v, B.p, B.c, B.v, cl.list(c), nr, 1, nullptr, nullptr, nullptr,
                  0, 0, 0.0, 0, cnt, nullptr, row0};
        AIRG_TRY(c == kCntReg8 ? launch_reg<8>(a, fk.stream(c)) : launch_reg<kRegMax2>(a, fk.stream(c)));
        continue;
      }
      if (c == kCntSpan4k || c == kCntSpan16k || c == kCntSpan64k) {
        SpanCountArgs a{A.p, A.c, B.p, B.c, cl.list(c), nr, cmin, words, bmoff, gbm, cnt};
        if (c == kCntSpan4k) AIRG_TRY((launch_span_count<128>(a, 4096, fk.stream(c))));
        else if (c == kCntSpan16k) AIRG_TRY((launch_span_count<256>(a, 16384, fk.stream(c))));
        else AIRG_TRY((launch_span_count<256>(a, kSpanMax, fk.stream(c))));
        continue;
      }
      const int bits = c == kCntHash64 ? 7 : c == kCntHash512 ? 10 : 12;
      const int warps = c == kCntHashBlk ? 4 : 8;
      const size_t shm = (size_t)warps * (1 << bits) * sizeof(int);
      CountArgs a{A.p, A.c, B.p, B.c, cl.list(c), nr, bits, (1 << bits) * 3 / 4, cnt,
                  ovf_rows, ovf_n, nullptr, nullptr, nullptr};
      if (c == kCntHashBlk) {  // long rows: CTA per row, one shared key set
        // threads per row: swept 64-512 (90 / 53 / 41 / 43 ms); must be a multiple of 32
        static const int cnt_nt = [] {
          const int v = getenv("AIRG_COUNT_NT") ? atoi(getenv("AIRG_COUNT_NT")) : 256;
          return std::max(32, std::min(256, v)) & ~31;
        }();
        spgemm_count_block_kernel<<<std::min(nr, num_sms() * 16), cnt_nt, (size_t)(1 << bits) * 4,
                                    fk.stream(c)>>>(a);
      } else {
        spgemm_count_kernel<<<blocks_for(nr, warps, num_sms() * 32), warps * 32, shm, fk.stream(c)>>>(a);
      }
      AIRG_LAUNCH_CHECK();
    }
    AIRG_TRY(fk.end(s));
    int novf = 0;
    AIRG_CUDA(read_back(&novf, ovf_n, sizeof(int), s));
    if (novf) {
      std::vector<int> rows(novf);
      AIRG_CUDA(cudaMemcpyAsync(rows.data(), ovf_rows, novf * sizeof(int), cudaMemcpyDeviceToHost, s));
      std::vector<long long> sizes;
      AIRG_TRY(gather_ll(ub, rows, sizes, s, m));
      GlobalTables g;
      AIRG_TRY(make_tables(rows, sizes, false, g, s));
      CountArgs a{A.p, A.c, B.p, B.c, g.rows, novf, 0, 0x7fffffff, cnt, ovf_rows, ovf_n, g.keys,
                  g.off, g.bits};
      spgemm_count_kernel<<<blocks_for(novf, 4), 128, 0, s>>>(a);
      AIRG_LAUNCH_CHECK();
      AIRG_CUDA(cudaStreamSynchronize(s));
      g.free(s);
    }
    release(ovf_rows, s);
    release(ovf_n, s);
    release(cl.lists, s);
  }
  // ---- pass 2 ----
  AIRG_TRY(scan_counts(cnt, Cp, m, nullptr, s));
  AIRG_TRY(scratch(&rl, m, s));
  if (m > 0) rowlen_kernel<<<blocks_for(m, 256), 256, 0, s>>>(m, Cp, rl);
  if (m > 0) numeric_class_kernel<<<blocks_for(m, 256), 256, 0, s>>>(m, Cp, A.p, ub, words, ids);
  AIRG_LAUNCH_CHECK();
  Classes cl;
  // the scan total (output nnz) is read back with the class counts: one sync
  int nnz32 = 0;
  AIRG_TRY(classify_ids(m, ids, kNumSpanCls + kNumHashCls + kNumRegCls, cl, s, Cp + m, &nnz32));
  const long long nnz = nnz32;
  airg_csr_result* r = new airg_csr_result();
  r->nrows = m;
  r->ncols = B.ncols;
  r->stream = s;
  int* ocol = nullptr;
  double* oval = nullptr;
  int* anyd = nullptr;
  const long long cap = mode == 1 ? nnz + m : nnz;
  AIRG_TRY(scratch(&ocol, cap, s));
  AIRG_TRY(scratch(&oval, cap, s));
  AIRG_TRY(scratch(&anyd, 1, s));
  AIRG_CUDA(cudaMemsetAsync(anyd, 0, sizeof(int), s));
  {
    Fork fk;
    AIRG_TRY(fk.begin(s));
    for (int c = 0; c < kNumSpanCls; ++c) {
      const int nr = cl.count[c];
      if (!nr) continue;
      SpanNumArgs a{A.p, A.c, A.v, B.p, B.c, B.v, cl.list(c), nr, 0, (int)tot_h[2], cmin, words, bmoff,
                    gbm, Cp, ocol, oval, negate, mode, tol, lump, cnt, anyd, row0};
      AIRG_TRY(launch_span_numeric(a, kSpanCaps[c], span_kd, fk.stream(c)));
    }
    for (int rc = 0; rc < kNumRegCls; ++rc) {
      const int c = kNumSpanCls + kNumHashCls + rc, nr = cl.count[c];
      if (!nr) continue;
      RegArgs a{A.p, A.c, A.v, B.p, B.c, B.v, cl.list(c), nr, 0, Cp, ocol, oval, negate, mode, tol,
                lump, cnt, anyd, row0};
      AIRG_TRY(rc == 0 ? launch_reg<8>(a, fk.stream(c)) : launch_reg<kRegMax2>(a, fk.stream(c)));
    }
    const int cbits[7] = {6, 8, 10, 11, 12, 13, 14}, cwarps[2] = {8, 8};
    constexpr int kGlobalClass = 7;
    AIRG_TRY(set_smem((const void*)spgemm_numeric_kernel, 200 * 1024));
    static bool attr = false;
    if (!attr) {
      const int lim = 200 * 1024;  // >= the 8192-class table (193 KB)
#define AIRG_F3(B) (const void*)spgemm_numeric_block_kernel<64, B>, \
    (const void*)spgemm_numeric_block_kernel<128, B>, (const void*)spgemm_numeric_block_kernel<256, B>
      for (const void* f : {AIRG_F3(10), AIRG_F3(11), AIRG_F3(12), AIRG_F3(13), AIRG_F3(14)})
#undef AIRG_F3
        AIRG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, lim));
      attr = true;
    }
    for (int c = 0; c < kGlobalClass; ++c) {
      const int nr = cl.count[kNumSpanCls + c];
      if (!nr) continue;
      NumArgs a{A.p, A.c, A.v, B.p, B.c, B.v, cl.list(kNumSpanCls + c), nr, cbits[c], Cp, ocol, oval,
                negate, mode, tol, lump, cnt, anyd, nullptr, nullptr, nullptr, nullptr, row0};
      cudaStream_t st = fk.stream(kNumSpanCls + c);
      if (c >= 2) {
        // one CTA per row, table shared by the CTA.  Threads per row measured
        // at 2048^2 (level-5 Galerkin, tools/nt_sweep.sh): the steps carry one
        // B row (~70-200 entries), so 128 threads beat 256 (38 vs 49 ms) for
        // the 512..1024 class; the long classes keep 256.
        const size_t shm = (size_t)(1 << cbits[c]) * 12 + 1024;
        const int grid = std::min(nr, num_sms() * 32);
        static int nts[7] = {0, 0, 128, 128, 256, 256, 256};
        static bool parsed = false;
        if (!parsed) {  // AIRG_NT="t2,t3,t4,t5,t6" overrides (measurement only)
          if (const char* e = getenv("AIRG_NT"))
            sscanf(e, "%d,%d,%d,%d,%d", &nts[2], &nts[3], &nts[4], &nts[5], &nts[6]);
          parsed = true;
        }
        const int nt = nts[c];
#define AIRG_NUMBLK(T, B) spgemm_numeric_block_kernel<T, B><<<grid, T, shm, st>>>(a)
#define AIRG_NUMBLK3(B) \
  if (nt == 64) AIRG_NUMBLK(64, B); else if (nt == 128) AIRG_NUMBLK(128, B); else AIRG_NUMBLK(256, B)
        if (c == 2) { AIRG_NUMBLK3(10); }
        else if (c == 3) { AIRG_NUMBLK3(11); }
        else if (c == 4) { AIRG_NUMBLK3(12); }
        else if (c == 5) { AIRG_NUMBLK3(13); }
        else { AIRG_NUMBLK3(14); }
#undef AIRG_NUMBLK3
#undef AIRG_NUMBLK
      } else {
        const size_t shm = (size_t)cwarps[c] * ((1 << cbits[c]) * 12 + 1024);
        spgemm_numeric_kernel<<<blocks_for(nr, cwarps[c], num_sms() * 32), cwarps[c] * 32, shm, st>>>(a);
      }
      AIRG_LAUNCH_CHECK();
    }
    AIRG_TRY(fk.end(s));
    const int nr = cl.count[kNumSpanCls + kGlobalClass];
    if (nr) {
      std::vector<int> rows(nr);
      AIRG_CUDA(cudaMemcpyAsync(rows.data(), cl.list(kNumSpanCls + kGlobalClass), nr * sizeof(int),
                                cudaMemcpyDeviceToHost, s));
      std::vector<long long> sizes;
      AIRG_TRY(gather_ll(rl, rows, sizes, s, m));
      GlobalTables g;
      AIRG_TRY(make_tables(rows, sizes, true, g, s));
      NumArgs a{A.p, A.c, A.v, B.p, B.c, B.v, g.rows, nr, 0, Cp, ocol, oval, negate, mode, tol, lump,
                cnt, anyd, g.keys, g.acc, g.off, g.bits, row0};
      spgemm_numeric_kernel<<<blocks_for(nr, 4), 128, 0, s>>>(a);
      AIRG_LAUNCH_CHECK();
      AIRG_CUDA(cudaStreamSynchronize(s));
      g.free(s);
    }
    release(cl.lists, s);
  }
  if (mode == 0) {
    r->ptr = Cp;
    r->col = ocol;
    r->val = oval;
    r->nnz = nnz;
  } else {
    AIRG_CUDA(cudaMallocFromPoolAsync((void**)&r->ptr, (size_t)(m + 1) * sizeof(int), lib_pool(), s));
    long long fn = 0;
    AIRG_TRY(scan_counts(cnt, r->ptr, m, &fn, s));
    AIRG_TRY(result_alloc_entries(r, fn, true));
    if (m > 0)
      compact_raw_kernel<<<blocks_for((long long)m * 32, 256), 256, 0, s>>>(m, Cp, r->ptr, ocol, oval,
                                                                           r->col, r->val);
    AIRG_LAUNCH_CHECK();
    release(ocol, s);
    release(oval, s);
    release(Cp, s);
  }
  for (void* q : {(void*)anyd, (void*)ub, (void*)rl, (void*)cnt, (void*)cmin, (void*)words,
                  (void*)bmoff, (void*)ids, (void*)gbm})
    release(q, s);
  *out = r;
  return AIRG_OK;
}

// ---- A P for a one-point P --------------------------------------------------
// P[k, pcol[k]] = 1 (hierarchy.py:250-278), so row i of A P is A's row i with
// its columns mapped through pcol and equal columns merged.  scipy csr_matmat
// semantics with the reference's structural zeros (sparse.py:222-240): the
// unique mapped columns ascending, value = 0 + a_1*1 + a_2*1 + ... in the
// order of A's columns (cancellations stay as +0.0).  Rows are written raw at
// A's offsets and compacted after the scan.
constexpr int kApCap = 1024;

// One warp per row: stage the mapped columns and values of A's row, stable
// LSD radix sort them by column (equal columns keep A's column order), then
// each run of equal columns is summed by the lane holding its head, in A's
// column order -- the sum the first-occurrence merge formed, now in
// O(L log span) instead of O(L x unique).  CAP entries of staging per warp.
template <int CAP, int NW>
__global__ void __launch_bounds__(32 * NW) ap_onepoint_kernel(
    int nr, const int* __restrict__ rows, const int* __restrict__ Ap, const int* __restrict__ Ac,
    const double* __restrict__ Av, const int* __restrict__ pcol, int* __restrict__ rcol,
    double* __restrict__ rval, int* __restrict__ cnt) {
  extern __shared__ unsigned char apsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* base = apsm + (size_t)w * (CAP * 24 + 1024);
  double* as = (double*)base;
  double* v2 = as + CAP;
  int* cs = (int*)(v2 + CAP);
  int* k2 = cs + CAP;
  int* hist = k2 + CAP;
  const unsigned lt = (1u << lane) - 1u;
  for (long long r = (long long)blockIdx.x * NW + w; r < nr; r += (long long)gridDim.x * NW) {
    const int row = rows[r];
    const int b = Ap[row], L = Ap[row + 1] - b;
    for (int j = lane; j < L; j += 32) {
      cs[j] = pcol[Ac[b + j]];
      as[j] = Av[b + j];
    }
    __syncwarp();
    if (L > 1) warp_radix_sort(cs, as, k2, v2, L, hist, lane);
    __syncwarp();
    int U = 0;
    for (int j0 = 0; j0 < L; j0 += 32) {
      const int j = j0 + lane;
      const bool head = j < L && (j == 0 || cs[j] != cs[j - 1]);
      const unsigned bal = __ballot_sync(kFull, head);
      if (head) {
        const int c = cs[j];
        double sum = 0.0;
        for (int jj = j; jj < L && cs[jj] == c; ++jj) sum = add_rn(sum, mul_rn(as[jj], 1.0));
        const int rank = U + __popc(bal & lt);
        rcol[b + rank] = c;
        rval[b + rank] = sum;
      }
      U += __popc(bal);
    }
    if (lane == 0) cnt[row] = U;
    __syncwarp();
  }
}

// Short rows (L <= G entries, G lanes per row, 32 / G rows per warp): the
// merge in registers.  Lane j holds A's j-th entry with its mapped column; a
// lane is the head of its column if no earlier lane has it, its output
// position is the number of head columns below it, and the head sums the
// column's values over the lanes in order -- A's column order, the same sum
// as the sorted-run path above (bitwise).
template <int G>
__global__ void __launch_bounds__(256) ap_small_kernel(
    int nr, const int* __restrict__ rows, const int* __restrict__ Ap, const int* __restrict__ Ac,
    const double* __restrict__ Av, const int* __restrict__ pcol, int* __restrict__ rcol,
    double* __restrict__ rval, int* __restrict__ cnt) {
  const int lane = threadIdx.x & 31, j = lane & (G - 1);
  const long long groups = ((long long)gridDim.x * blockDim.x) / G;
  // warp-uniform trip count: the groups of a warp shuffle together
  for (long long g0 = ((long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / G; g0 < nr;
       g0 += groups) {
    const long long r = g0 + lane / G;
    const bool live = r < nr;
    const int row = live ? rows[r] : 0;
    const int b = live ? Ap[row] : 0, L = live ? Ap[row + 1] - b : 0;
    const bool has = j < L;
    const int c = has ? pcol[Ac[b + j]] : INT_MAX;
    const double a = has ? Av[b + j] : 0.0;
    bool head = has;
    int pos = 0;
    double sum = 0.0;
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int ci = __shfl_sync(kFull, c, i, G);
      const double ai = __shfl_sync(kFull, a, i, G);
      if (i < j && ci == c) head = false;
      if (ci == c) sum = add_rn(sum, mul_rn(ai, 1.0));
    }
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int ci = __shfl_sync(kFull, c, i, G);
      const bool hi = __shfl_sync(kFull, head, i, G);
      if (hi && ci < c) ++pos;
    }
    if (head) {
      rcol[b + pos] = c;
      rval[b + pos] = sum;
    }
    const unsigned bal = __ballot_sync(kFull, head);
    if (live && j == 0) cnt[row] = __popc((bal >> (lane & ~(G - 1))) & (G == 32 ? kFull : ((1u << G) - 1u)));
  }
}

// raw rows (at A's offsets) -> compacted output, vs lanes per row
__global__ void ap_compact_kernel(int n, const int* __restrict__ Ap, const int* __restrict__ Cp,
                                  const int* __restrict__ rcol, const double* __restrict__ rval,
                                  int* __restrict__ oc, double* __restrict__ ov, int vs) {
  const int j = threadIdx.x & (vs - 1);
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / vs; r < n;
       r += ((long long)gridDim.x * blockDim.x) / vs) {
    const int b = Ap[r], o = Cp[r], u = Cp[r + 1] - o;
    for (int q = j; q < u; q += vs) {
      oc[o + q] = rcol[b + q];
      ov[o + q] = rval[b + q];
    }
  }
}

static int ap_onepoint(const Mat& A, int nc, const int* pcol, airg_csr_result** out, cudaStream_t s) {
  const int n = A.nrows;
  // row classes by length (<= 256, <= 1024, longer); nnz(A) read back in the
  // same sync
  long long* len = nullptr;
  AIRG_TRY(scratch(&len, n > 0 ? n : 1, s));
  if (n > 0) rowlen_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, A.p, len);
  AIRG_LAUNCH_CHECK();
  Classes cl;
  int annz32 = 0;
  // classes: <= 8 and <= 32 entries (register merge), <= 256 and <= kApCap
  // (staged radix sort), longer (general product)
  AIRG_TRY(classify(n, len, {8, 32, 256, kApCap}, cl, s, A.p + n, &annz32));
  release(len, s);
  // rows beyond the staging buffer, or (measurement knob AIRG_AP_AVG) a mean
  // row length above the cutoff, go to the general hash product
  static const long long avg_cap = getenv("AIRG_AP_AVG") ? atoll(getenv("AIRG_AP_AVG")) : (1ll << 40);
  const long long annz = annz32;
  if (cl.count[4] > 0 || annz > avg_cap * n) {
    release(cl.lists, s);
    int* Pp = nullptr;
    double* Pv = nullptr;
    AIRG_TRY(scratch(&Pp, A.ncols + 1, s));
    AIRG_TRY(scratch(&Pv, A.ncols > 0 ? A.ncols : 1, s));
    iota_kernel<<<blocks_for(A.ncols + 1, 256), 256, 0, s>>>(A.ncols, Pp);
    ones_kernel<<<blocks_for(A.ncols, 256), 256, 0, s>>>(A.ncols, Pv);
    AIRG_LAUNCH_CHECK();
    Mat P{A.ncols, nc, Pp, pcol, Pv};
    AIRG_TRY(spgemm_rows(A, P, 0, 0, 0.0, 0, out, s));
    release(Pp, s);
    release(Pv, s);
    return AIRG_OK;
  }
  int *rcol = nullptr, *cnt = nullptr;
  double* rval = nullptr;
  AIRG_TRY(scratch(&rcol, annz > 0 ? annz : 1, s));
  AIRG_TRY(scratch(&rval, annz > 0 ? annz : 1, s));
  AIRG_TRY(scratch(&cnt, n + 1, s));
  constexpr int kW0 = 8, kW1 = 2;
  const size_t shm0 = (size_t)kW0 * (256 * 24 + 1024), shm1 = (size_t)kW1 * (kApCap * 24 + 1024);
  static bool attr = false;
  if (!attr) {
    AIRG_CUDA(cudaFuncSetAttribute(ap_onepoint_kernel<256, kW0>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm0));
    AIRG_CUDA(cudaFuncSetAttribute(ap_onepoint_kernel<kApCap, kW1>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm1));
    attr = true;
  }
  Fork fk;
  AIRG_TRY(fk.begin(s));
  if (cl.count[0])
    ap_small_kernel<8><<<blocks_for((long long)cl.count[0] * 8, 256), 256, 0, fk.stream(0)>>>(
        cl.count[0], cl.list(0), A.p, A.c, A.v, pcol, rcol, rval, cnt);
  AIRG_LAUNCH_CHECK();
  if (cl.count[1])
    ap_small_kernel<32><<<blocks_for((long long)cl.count[1] * 32, 256), 256, 0, fk.stream(1)>>>(
        cl.count[1], cl.list(1), A.p, A.c, A.v, pcol, rcol, rval, cnt);
  AIRG_LAUNCH_CHECK();
  if (cl.count[2])
    ap_onepoint_kernel<256, kW0><<<blocks_for(cl.count[2], kW0, num_sms() * 4), 32 * kW0, shm0, fk.stream(2)>>>(
        cl.count[2], cl.list(2), A.p, A.c, A.v, pcol, rcol, rval, cnt);
  AIRG_LAUNCH_CHECK();
  if (cl.count[3])
    ap_onepoint_kernel<kApCap, kW1><<<blocks_for(cl.count[3], kW1, num_sms() * 4), 32 * kW1, shm1,
                                      fk.stream(3)>>>(cl.count[3], cl.list(3), A.p, A.c, A.v, pcol,
                                                      rcol, rval, cnt);
  AIRG_LAUNCH_CHECK();
  AIRG_TRY(fk.end(s));
  release(cl.lists, s);
  airg_csr_result* r = new_result(n, nc, s);
  long long nnz = 0;
  AIRG_TRY(scan_counts(cnt, r->ptr, n, &nnz, s));
  AIRG_TRY(result_alloc_entries(r, nnz, true));
  if (n > 0) {
    const int vs = annz <= 4LL * n ? 4 : annz <= 16LL * n ? 8 : 32;  // lanes per row
    ap_compact_kernel<<<blocks_for((long long)n * vs, 256), 256, 0, s>>>(n, A.p, r->ptr, rcol, rval,
                                                                        r->col, r->val, vs);
  }
  AIRG_LAUNCH_CHECK();
  release(rcol, s);
  release(rval, s);
  release(cnt, s);
  *out = r;
  return AIRG_OK;
}

}  // namespace airg

using namespace airg;

extern "C" {

int airg_spgemm(int m, int k, int n, const int32_t* Ap, const int32_t* Ac, const double* Av,
                const int32_t* Bp, const int32_t* Bc, const double* Bv, int negate,
                airg_csr_result** out, void* stream) {
  Mat A{m, k, Ap, Ac, Av}, B{k, n, Bp, Bc, Bv};
  return spgemm_rows(A, B, negate, 0, 0.0, 0, out, (cudaStream_t)stream);
}

// General product with the optional fused drop/lump epilogue and a global
// row offset (row-strip operators).  mode 0: C = A B (negate); mode 1:
// drop_and_lump(A B, tol, lump) with diagonal column = row0 + local row.
int airg_spgemm_ex(int m, int k, int n, const int32_t* Ap, const int32_t* Ac, const double* Av,
                   const int32_t* Bp, const int32_t* Bc, const double* Bv, int negate, int mode,
                   double tol, int lump, int row0, airg_csr_result** out, void* stream) {
  Mat A{m, k, Ap, Ac, Av}, B{k, n, Bp, Bc, Bv};
  return spgemm_rows(A, B, negate, mode, tol, lump, out, (cudaStream_t)stream, row0);
}

int airg_galerkin(int n, int nc, const int32_t* Rp, const int32_t* Rc, const double* Rv,
                  const int32_t* Ap, const int32_t* Ac, const double* Av, const int32_t* pcol,
                  double a_drop, int lump, airg_csr_result** out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  Mat A{n, n, Ap, Ac, Av};
  airg_csr_result* AP = nullptr;
  AIRG_TRY(ap_onepoint(A, nc, pcol, &AP, s));
  Mat R{nc, n, Rp, Rc, Rv}, APm{n, nc, AP->ptr, AP->col, AP->val};
  AIRG_TRY(spgemm_rows(R, APm, 0, a_drop == 0.0 ? 0 : 1, a_drop, lump, out, s));
  airg_result_free(AP);
  return AIRG_OK;
}

// A P for a one-point prolongator given by pcol (rows of A on a strip with
// ext columns: pcol has one entry per ext column); ref hierarchy.py:281-286
int airg_ap_onepoint(int m, int k, int nc, const int32_t* Ap, const int32_t* Ac, const double* Av,
                     const int32_t* pcol, airg_csr_result** out, void* stream) {
  Mat A{m, k, Ap, Ac, Av};
  return ap_onepoint(A, nc, pcol, out, (cudaStream_t)stream);
}

}  // extern "C"
