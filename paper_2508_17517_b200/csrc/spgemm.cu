// Bit-exact sparse products for the AIRG setup on sm_100a.
//
//   * spgemm C = A B with the structural pattern (cancellation zeros kept),
//     values summed k-ascending with separate mul/add roundings exactly as
//     scipy's csr_matmat: a warp owns a row; lanes split
//     the entries of ONE B row (distinct output columns) and the A row is
//     walked sequentially, so every output entry sees its k in order.
//     Symbolic: shared-memory open-addressing key set -> count -> sort.
//     Numeric: static shared-memory lookup (column -> position in the sorted
//     row) and an fp64 accumulator per output entry.
//   * fused Galerkin epilogue: drop_and_lump on the RAP row in registers /
//     shared memory, so raw R(AP) rows are never materialised in HBM.
//   * masked polynomial assembly sum_k c_k mask(A^k) row by row, all powers
//     of one row kept in shared memory (polynomial.py:372-416).
//   * extract, drop_and_lump, restriction assembly.
// ref: sparse.py:222-352, polynomial.py:372-416, hierarchy.py:211-286
#include "setup_common.cuh"
#include <vector>
#include <algorithm>

namespace airg {

constexpr int kEmpty = -1;

__device__ __forceinline__ unsigned hash_of(int key, int bits) {
  return ((unsigned)key * 0x9E3779B1u) >> (32 - bits);
}

// insert key into an open-addressing set; returns 1 when newly inserted,
// 0 when present, 1<<20 when the table is full (caller flags overflow)
__device__ __forceinline__ int set_insert(int* keys, int bits, int key) {
  const unsigned mask = (1u << bits) - 1u;
  unsigned h = hash_of(key, bits);
  for (unsigned probe = 0; probe <= mask; ++probe) {
    int prev = atomicCAS(keys + h, kEmpty, key);
    if (prev == kEmpty) return 1;
    if (prev == key) return 0;
    h = (h + 1u) & mask;
  }
  return 1 << 20;
}

__device__ __forceinline__ int map_find(const int* keys, const int* vals, int bits, int key) {
  const unsigned mask = (1u << bits) - 1u;
  unsigned h = hash_of(key, bits);
  while (true) {
    int k = keys[h];
    if (k == key) return vals[h];
    if (k == kEmpty) return -1;
    h = (h + 1u) & mask;
  }
}

__device__ __forceinline__ void map_insert(int* keys, int* vals, int bits, int key, int v) {
  const unsigned mask = (1u << bits) - 1u;
  unsigned h = hash_of(key, bits);
  while (true) {
    int prev = atomicCAS(keys + h, kEmpty, key);
    if (prev == kEmpty || prev == key) {
      vals[h] = v;
      return;
    }
    h = (h + 1u) & mask;
  }
}

// warp-wide bitonic sort of buf[0..P) ascending (P power of two)
__device__ void warp_bitonic(int* buf, int P, int lane) {
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < P; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int a = buf[i], b = buf[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            buf[i] = b;
            buf[ixj] = a;
          }
        }
      }
      __syncwarp();
    }
  }
}

__host__ __device__ __forceinline__ int ceil_log2(long long x) {
  int b = 0;
  while ((1ll << b) < x) ++b;
  return b;
}

// ----------------------------------------------------------------------------
// row classification
// ----------------------------------------------------------------------------
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

// append row ids to per-class lists by thresholds on size[i]
__global__ void classify_kernel(int m, const long long* __restrict__ size, const long long* __restrict__ th,
                                int ncls, int* __restrict__ lists, int* __restrict__ counts) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const long long v = size[i];
    int c = 0;
    while (c < ncls - 1 && v > th[c]) ++c;
    const int slot = atomicAdd(counts + c, 1);
    lists[(long long)c * m + slot] = (int)i;
  }
}

__global__ void int_to_ll_kernel(int m, const int* __restrict__ ptr, long long* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = ptr[i + 1] - ptr[i];
}

struct Classes {
  std::vector<int> count;
  int* lists = nullptr;  // ncls * m
  int m = 0;
  const int* list(int c) const { return lists + (long long)c * m; }
};

static int classify(int m, const long long* size, const std::vector<long long>& th, Classes& out,
                    cudaStream_t s) {
  const int ncls = (int)th.size() + 1;
  long long* dth = nullptr;
  int* cnt = nullptr;
  AIRG_TRY(scratch(&out.lists, (size_t)ncls * (m > 0 ? m : 1), s));
  AIRG_TRY(scratch(&dth, th.size() + 1, s));
  AIRG_TRY(scratch(&cnt, ncls, s));
  if (!th.empty())
    AIRG_CUDA(cudaMemcpyAsync(dth, th.data(), th.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
  AIRG_CUDA(cudaMemsetAsync(cnt, 0, ncls * sizeof(int), s));
  if (m > 0) classify_kernel<<<blocks_for(m, 256), 256, 0, s>>>(m, size, dth, ncls, out.lists, cnt);
  AIRG_LAUNCH_CHECK();
  out.count.assign(ncls, 0);
  AIRG_CUDA(cudaMemcpyAsync(out.count.data(), cnt, ncls * sizeof(int), cudaMemcpyDeviceToHost, s));
  AIRG_CUDA(cudaStreamSynchronize(s));
  out.m = m;
  release(dth, s);
  release(cnt, s);
  return AIRG_OK;
}

// ----------------------------------------------------------------------------
// symbolic phase
// ----------------------------------------------------------------------------
// Tables: shared memory (bits <= 14) or a global pool (gtab != nullptr, one
// table of 2^gbits[r] ints per listed row at goff[r]).
struct SymArgs {
  const int *Ap, *Ac, *Bp, *Bc;
  const int* rows;
  int nrows;
  int bits;          // shared-table size (log2), 0 for global tables
  int limit;         // max keys before overflow (shared tables)
  int* cnt;          // per row count (output)
  int* ovf_rows;     // overflow list
  int* ovf_n;
  int* gtab;         // global tables
  const long long* goff;
  const int* gbits;
  const int* optr;   // fill mode: output row offsets
  int* ocol;         // fill mode: output columns
};

template <bool FILL>
__global__ void __launch_bounds__(256) spgemm_symbolic_kernel(SymArgs a) {
  extern __shared__ int smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ int wcount[8];
  __shared__ int wovf[8];
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
    if (lane == 0) {
      wcount[w] = 0;
      wovf[w] = 0;
    }
    __syncwarp();
    const int ab = a.Ap[row], ae = a.Ap[row + 1];
    for (int kk = ab; kk < ae; ++kk) {
      const int k = a.Ac[kk];
      const int bb = a.Bp[k], be = a.Bp[k + 1];
      int added = 0;
      for (int jj = bb + lane; jj < be; jj += 32) added += set_insert(keys, bits, a.Bc[jj]);
      added = warp_sum(added);
      if (lane == 0) wcount[w] += added;
      __syncwarp();
      if (!a.gtab && wcount[w] > a.limit) {
        if (lane == 0) wovf[w] = 1;
        break;
      }
    }
    __syncwarp();
    if (wovf[w]) {
      if (!FILL && lane == 0) a.ovf_rows[atomicAdd(a.ovf_n, 1)] = row;
      __syncwarp();
      continue;
    }
    const int n = wcount[w];
    if (!FILL) {
      if (lane == 0) a.cnt[row] = n;
      __syncwarp();
      continue;
    }
    // in-place compaction of occupied slots to keys[0..n)
    int wpos = 0;
    for (int base = 0; base < T; base += 32) {
      const int v = keys[base + lane];
      const bool occ = v != kEmpty;
      const unsigned bal = __ballot_sync(0xffffffffu, occ);
      __syncwarp();
      if (occ) keys[wpos + __popc(bal & ((1u << lane) - 1u))] = v;
      wpos += __popc(bal);
      __syncwarp();
    }
    int P = 1;
    while (P < n) P <<= 1;
    for (int i = n + lane; i < P; i += 32) keys[i] = 0x7fffffff;
    __syncwarp();
    warp_bitonic(keys, P, lane);
    const int o = a.optr[row];
    for (int i = lane; i < n; i += 32) a.ocol[o + i] = keys[i];
    __syncwarp();
  }
}

// ----------------------------------------------------------------------------
// numeric phase
// ----------------------------------------------------------------------------
// mode 0: C_val[pos] = acc (optionally negated)
// mode 1: fused drop_and_lump(tol, lump) on the sorted row, kept entries written
//         at the raw offsets (out_col/out_val) with out_cnt[row] = kept count.
struct NumArgs {
  const int *Ap, *Ac;
  const double* Av;
  const int *Bp, *Bc;
  const double* Bv;
  const int *Cp, *Cc;  // symbolic result (sorted)
  double* Cv;
  const int* rows;
  int nrows;
  int bits;            // shared lookup table bits, 0 => global
  int acc_cap;         // shared accumulator capacity
  int negate;
  int mode;
  double tol;
  int lump;
  int* out_col;
  double* out_val;
  int* out_cnt;
  // global fallback storage
  int* gkeys;
  int* gvals;
  double* gacc;
  const long long* goff;   // table offset per listed row
  const long long* gaoff;  // accumulator offset per listed row
  const int* gbits;
};

__global__ void __launch_bounds__(256) spgemm_numeric_kernel(NumArgs a) {
  extern __shared__ unsigned char smraw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (long long t = (long long)blockIdx.x * nw + w; t < a.nrows; t += (long long)gridDim.x * nw) {
    const int row = a.rows[t];
    int *keys, *vals;
    double* acc;
    int bits;
    if (a.gkeys) {
      bits = a.gbits[t];
      keys = a.gkeys + a.goff[t];
      vals = a.gvals + a.goff[t];
      acc = a.gacc + a.gaoff[t];
    } else {
      bits = a.bits;
      const size_t T = (size_t)1 << bits;
      unsigned char* base = smraw + (size_t)w * (T * 8 + (size_t)a.acc_cap * 8);
      acc = (double*)base;
      keys = (int*)(base + (size_t)a.acc_cap * 8);
      vals = keys + T;
    }
    const int T = 1 << bits;
    const int cb = a.Cp[row], ce = a.Cp[row + 1], nc = ce - cb;
    for (int i = lane; i < T; i += 32) keys[i] = kEmpty;
    __syncwarp();
    for (int i = lane; i < nc; i += 32) {
      map_insert(keys, vals, bits, a.Cc[cb + i], i);
      acc[i] = 0.0;
    }
    __syncwarp();
    const int ab = a.Ap[row], ae = a.Ap[row + 1];
    for (int kk = ab; kk < ae; ++kk) {
      const int k = a.Ac[kk];
      const double av = a.Av[kk];
      const int bb = a.Bp[k], be = a.Bp[k + 1];
      for (int jj = bb + lane; jj < be; jj += 32) {
        const int p = map_find(keys, vals, bits, a.Bc[jj]);
        acc[p] = add_rn(acc[p], mul_rn(av, a.Bv[jj]));
      }
      __syncwarp();
    }
    if (a.mode == 0) {
      for (int i = lane; i < nc; i += 32) {
        const double v = acc[i];
        a.Cv[cb + i] = a.negate ? -v : v;
      }
      __syncwarp();
      continue;
    }
    // ---- fused drop_and_lump (sparse.py:307-352) on the sorted row ----
    double mx = 0.0;
    int dpos = -1;
    for (int i = lane; i < nc; i += 32) {
      mx = fmax(mx, fabs(acc[i]));
      if (a.Cc[cb + i] == row) dpos = i;
    }
    mx = warp_max(mx);
    dpos = __reduce_max_sync(0xffffffffu, dpos);
    const double thr = mul_rn(a.tol, mx);
    // sequential lump of dropped values in column order (np.bincount)
    double lumped = 0.0;
    int ndrop = 0;
    if (lane == 0) {
      for (int i = 0; i < nc; ++i) {
        const double v = acc[i];
        if (i != dpos && !(fabs(v) >= thr)) {
          lumped = add_rn(lumped, v);
          ++ndrop;
        }
      }
    }
    lumped = __shfl_sync(0xffffffffu, lumped, 0);
    ndrop = __shfl_sync(0xffffffffu, ndrop, 0);
    const bool insert = a.lump && ndrop > 0 && dpos < 0 && lumped != 0.0;
    int o = cb;  // raw offsets are an upper bound (+1 slot reserved per row for insertion)
    o += row;    // one spare slot per row before this one
    int written = 0;
    for (int base = 0; base < nc; base += 32) {
      const int i = base + lane;
      bool keep = false;
      double v = 0.0;
      int c = 0;
      if (i < nc) {
        v = acc[i];
        c = a.Cc[cb + i];
        keep = i == dpos || fabs(v) >= thr;
        if (i == dpos && a.lump && ndrop > 0) v = add_rn(v, lumped);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        int dst = written + __popc(bal & ((1u << lane) - 1u));
        if (insert && c > row) ++dst;
        a.out_col[o + dst] = c;
        a.out_val[o + dst] = v;
      }
      written += __popc(bal);
    }
    if (insert) {
      // position = number of kept columns < row
      int before = 0;
      for (int i = lane; i < nc; i += 32) {
        const double v = acc[i];
        before += (fabs(v) >= thr) && a.Cc[cb + i] < row;
      }
      before = warp_sum(before);
      if (lane == 0) {
        a.out_col[o + before] = row;
        a.out_val[o + before] = lumped;
      }
      ++written;
    }
    if (lane == 0) a.out_cnt[row] = written;
    __syncwarp();
  }
}

__global__ void compact_rows_kernel(int m, const int* __restrict__ rawp, const int* __restrict__ optr,
                                    const int* __restrict__ icol, const double* __restrict__ ival,
                                    int* __restrict__ ocol, double* __restrict__ oval) {
  // warp per row
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

// ----------------------------------------------------------------------------
// host driver
// ----------------------------------------------------------------------------
struct Mat {
  int nrows, ncols;
  const int* p;
  const int* c;
  const double* v;
};

static int smem_limit() { return 200 * 1024; }

static int launch_symbolic(const Mat& A, const Mat& B, const Classes& cl, int* cnt, const int* optr,
                           int* ocol, bool fill, cudaStream_t s, std::vector<int>* ovf_out,
                           const std::vector<int>* ovf_in, const long long* ub) {
  // class -> shared table bits (ub thresholds 64 / 512 / rest)
  const int bits_of[3] = {7, 10, 12};
  int* ovf_rows = nullptr;
  int* ovf_n = nullptr;
  AIRG_TRY(scratch(&ovf_rows, cl.m > 0 ? cl.m : 1, s));
  AIRG_TRY(scratch(&ovf_n, 1, s));
  AIRG_CUDA(cudaMemsetAsync(ovf_n, 0, sizeof(int), s));
  for (int c = 0; c < 3; ++c) {
    const int nr = cl.count[c];
    if (!nr) continue;
    const int bits = bits_of[c];
    const int warps = 8;
    const size_t shm = (size_t)warps * (1 << bits) * sizeof(int);
    SymArgs a{A.p, A.c, B.p, B.c, cl.list(c), nr, bits, (1 << bits) * 3 / 4, cnt, ovf_rows, ovf_n,
              nullptr, nullptr, nullptr, optr, ocol};
    if (fill) {
      if (shm > 48 * 1024)
        AIRG_CUDA(cudaFuncSetAttribute(spgemm_symbolic_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
      spgemm_symbolic_kernel<true><<<blocks_for(nr, warps, 148 * 16), warps * 32, shm, s>>>(a);
    } else {
      if (shm > 48 * 1024)
        AIRG_CUDA(cudaFuncSetAttribute(spgemm_symbolic_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
      spgemm_symbolic_kernel<false><<<blocks_for(nr, warps, 148 * 16), warps * 32, shm, s>>>(a);
    }
    AIRG_LAUNCH_CHECK();
  }
  (void)ovf_in;
  (void)ub;
  int novf = 0;
  AIRG_CUDA(cudaMemcpyAsync(&novf, ovf_n, sizeof(int), cudaMemcpyDeviceToHost, s));
  AIRG_CUDA(cudaStreamSynchronize(s));
  if (ovf_out) {
    ovf_out->resize(novf);
    if (novf)
      AIRG_CUDA(cudaMemcpyAsync(ovf_out->data(), ovf_rows, novf * sizeof(int), cudaMemcpyDeviceToHost, s));
    AIRG_CUDA(cudaStreamSynchronize(s));
  }
  release(ovf_rows, s);
  release(ovf_n, s);
  return AIRG_OK;
}

// global-table symbolic for overflow rows (count or fill)
static int symbolic_global(const Mat& A, const Mat& B, const std::vector<int>& rows,
                           const long long* ub_d, int* cnt, const int* optr, int* ocol, bool fill,
                           cudaStream_t s) {
  const int nr = (int)rows.size();
  if (!nr) return AIRG_OK;
  std::vector<long long> ubh(nr);
  // fetch ub of these rows
  std::vector<long long> all;
  for (int i = 0; i < nr; ++i)
    AIRG_CUDA(cudaMemcpyAsync(&ubh[i], ub_d + rows[i], sizeof(long long), cudaMemcpyDeviceToHost, s));
  AIRG_CUDA(cudaStreamSynchronize(s));
  std::vector<long long> off(nr);
  std::vector<int> gb(nr);
  long long tot = 0;
  for (int i = 0; i < nr; ++i) {
    gb[i] = std::max(5, ceil_log2(2 * std::max(1ll, ubh[i])));
    off[i] = tot;
    tot += 1ll << gb[i];
  }
  int *drows = nullptr, *dgb = nullptr, *tab = nullptr;
  long long* doff = nullptr;
  AIRG_TRY(scratch(&drows, nr, s));
  AIRG_TRY(scratch(&dgb, nr, s));
  AIRG_TRY(scratch(&doff, nr, s));
  AIRG_TRY(scratch(&tab, tot, s));
  AIRG_CUDA(cudaMemcpyAsync(drows, rows.data(), nr * sizeof(int), cudaMemcpyHostToDevice, s));
  AIRG_CUDA(cudaMemcpyAsync(dgb, gb.data(), nr * sizeof(int), cudaMemcpyHostToDevice, s));
  AIRG_CUDA(cudaMemcpyAsync(doff, off.data(), nr * sizeof(long long), cudaMemcpyHostToDevice, s));
  SymArgs a{A.p, A.c, B.p, B.c, drows, nr, 0, 0x7fffffff, cnt, nullptr, nullptr, tab, doff, dgb,
            optr, ocol};
  if (fill) spgemm_symbolic_kernel<true><<<blocks_for(nr, 4), 128, 0, s>>>(a);
  else spgemm_symbolic_kernel<false><<<blocks_for(nr, 4), 128, 0, s>>>(a);
  AIRG_LAUNCH_CHECK();
  AIRG_CUDA(cudaStreamSynchronize(s));
  release(drows, s);
  release(dgb, s);
  release(doff, s);
  release(tab, s);
  return AIRG_OK;
}

// Structural product C = A*B: returns C_ptr (m+1) and sorted C_col.
static int spgemm_structure(const Mat& A, const Mat& B, int** Cp_out, int** Cc_out, long long* nnz_out,
                            long long** ub_out, cudaStream_t s) {
  const int m = A.nrows;
  long long* ub = nullptr;
  int* cnt = nullptr;
  int* Cp = nullptr;
  AIRG_TRY(scratch(&ub, m, s));
  AIRG_TRY(scratch(&cnt, m + 1, s));
  AIRG_TRY(scratch(&Cp, m + 1, s));
  if (m > 0) product_ub_kernel<<<blocks_for(m, 256), 256, 0, s>>>(m, A.p, A.c, B.p, ub);
  AIRG_LAUNCH_CHECK();
  Classes cl;
  AIRG_TRY(classify(m, ub, {64, 512}, cl, s));
  std::vector<int> ovf;
  AIRG_TRY(launch_symbolic(A, B, cl, cnt, nullptr, nullptr, false, s, &ovf, nullptr, ub));
  AIRG_TRY(symbolic_global(A, B, ovf, ub, cnt, nullptr, nullptr, false, s));
  long long nnz = 0;
  AIRG_TRY(scan_counts(cnt, Cp, m, &nnz, s));
  int* Cc = nullptr;
  AIRG_TRY(scratch(&Cc, nnz, s));
  AIRG_TRY(launch_symbolic(A, B, cl, cnt, Cp, Cc, true, s, nullptr, nullptr, ub));
  AIRG_TRY(symbolic_global(A, B, ovf, ub, cnt, Cp, Cc, true, s));
  release(cl.lists, s);
  release(cnt, s);
  *Cp_out = Cp;
  *Cc_out = Cc;
  *nnz_out = nnz;
  if (ub_out) *ub_out = ub;
  else release(ub, s);
  return AIRG_OK;
}

// Numeric pass over the structure (mode 0: values into Cv; mode 1: fused drop/lump)
static int spgemm_numeric(const Mat& A, const Mat& B, const int* Cp, const int* Cc, double* Cv,
                          int negate, int mode, double tol, int lump, int* out_col, double* out_val,
                          int* out_cnt, cudaStream_t s) {
  const int m = A.nrows;
  long long* rl = nullptr;
  AIRG_TRY(scratch(&rl, m, s));
  if (m > 0) int_to_ll_kernel<<<blocks_for(m, 256), 256, 0, s>>>(m, Cp, rl);
  Classes cl;
  AIRG_TRY(classify(m, rl, {64, 512, 2048}, cl, s));
  const int cls_bits[3] = {7, 10, 12};
  const int cls_acc[3] = {64, 512, 2048};
  const int cls_warps[3] = {8, 8, 4};
  for (int c = 0; c < 3; ++c) {
    const int nr = cl.count[c];
    if (!nr) continue;
    const int bits = cls_bits[c];
    const size_t per = ((size_t)1 << bits) * 8 + (size_t)cls_acc[c] * 8;
    const size_t shm = per * cls_warps[c];
    NumArgs a{A.p, A.c, A.v, B.p, B.c, B.v, Cp, Cc, Cv, cl.list(c), nr, bits, cls_acc[c], negate,
              mode, tol, lump, out_col, out_val, out_cnt, nullptr, nullptr, nullptr, nullptr,
              nullptr, nullptr};
    if (shm > 48 * 1024)
      AIRG_CUDA(cudaFuncSetAttribute(spgemm_numeric_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)shm));
    spgemm_numeric_kernel<<<blocks_for(nr, cls_warps[c], 148 * 16), cls_warps[c] * 32, shm, s>>>(a);
    AIRG_LAUNCH_CHECK();
  }
  // global fallback for very long output rows
  const int nr = cl.count[3];
  if (nr) {
    std::vector<int> rows(nr);
    AIRG_CUDA(cudaMemcpyAsync(rows.data(), cl.list(3), nr * sizeof(int), cudaMemcpyDeviceToHost, s));
    std::vector<int> ph(m + 1);
    AIRG_CUDA(cudaMemcpyAsync(ph.data(), Cp, (m + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
    AIRG_CUDA(cudaStreamSynchronize(s));
    std::vector<long long> off(nr), aoff(nr);
    std::vector<int> gb(nr);
    long long tt = 0, ta = 0;
    for (int i = 0; i < nr; ++i) {
      const int len = ph[rows[i] + 1] - ph[rows[i]];
      gb[i] = ceil_log2(2ll * len);
      off[i] = tt;
      tt += 1ll << gb[i];
      aoff[i] = ta;
      ta += len;
    }
    int *drows = nullptr, *dgb = nullptr, *gk = nullptr, *gv = nullptr;
    long long *doff = nullptr, *daoff = nullptr;
    double* gacc = nullptr;
    AIRG_TRY(scratch(&drows, nr, s));
    AIRG_TRY(scratch(&dgb, nr, s));
    AIRG_TRY(scratch(&doff, nr, s));
    AIRG_TRY(scratch(&daoff, nr, s));
    AIRG_TRY(scratch(&gk, tt, s));
    AIRG_TRY(scratch(&gv, tt, s));
    AIRG_TRY(scratch(&gacc, ta, s));
    AIRG_CUDA(cudaMemcpyAsync(drows, rows.data(), nr * sizeof(int), cudaMemcpyHostToDevice, s));
    AIRG_CUDA(cudaMemcpyAsync(dgb, gb.data(), nr * sizeof(int), cudaMemcpyHostToDevice, s));
    AIRG_CUDA(cudaMemcpyAsync(doff, off.data(), nr * sizeof(long long), cudaMemcpyHostToDevice, s));
    AIRG_CUDA(cudaMemcpyAsync(daoff, aoff.data(), nr * sizeof(long long), cudaMemcpyHostToDevice, s));
    NumArgs a{A.p, A.c, A.v, B.p, B.c, B.v, Cp, Cc, Cv, drows, nr, 0, 0, negate, mode, tol, lump,
              out_col, out_val, out_cnt, gk, gv, gacc, doff, daoff, dgb};
    spgemm_numeric_kernel<<<blocks_for(nr, 4), 128, 0, s>>>(a);
    AIRG_LAUNCH_CHECK();
    AIRG_CUDA(cudaStreamSynchronize(s));
    for (void* q : {(void*)drows, (void*)dgb, (void*)doff, (void*)daoff, (void*)gk, (void*)gv,
                    (void*)gacc})
      release(q, s);
  }
  release(cl.lists, s);
  release(rl, s);
  return AIRG_OK;
}

static int spgemm_full(const Mat& A, const Mat& B, int negate, airg_csr_result** out, cudaStream_t s) {
  airg_csr_result* r = new airg_csr_result();
  r->nrows = A.nrows;
  r->ncols = B.ncols;
  r->stream = s;
  long long nnz = 0;
  AIRG_TRY(spgemm_structure(A, B, &r->ptr, &r->col, &nnz, nullptr, s));
  r->nnz = nnz;
  AIRG_TRY(scratch(&r->val, nnz, s));
  AIRG_TRY(spgemm_numeric(A, B, r->ptr, r->col, r->val, negate, 0, 0.0, 0, nullptr, nullptr,
                          nullptr, s));
  *out = r;
  return AIRG_OK;
}

// R (A P) with fused drop_and_lump; P is the one-point prolongator (pcol per row).
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

// ----------------------------------------------------------------------------
// drop_and_lump on an existing CSR (sparse.py:307-352), warp per row
// ----------------------------------------------------------------------------
__global__ void drop_lump_kernel(int m, const int* __restrict__ p, const int* __restrict__ c,
                                 const double* __restrict__ v, double tol, int lump,
                                 int* __restrict__ out_col, double* __restrict__ out_val,
                                 int* __restrict__ out_cnt, int* __restrict__ any_drop) {
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < m;
       r += ((long long)gridDim.x * blockDim.x) >> 5) {
    const int row = (int)r;
    const int b = p[row], e = p[row + 1], nc = e - b;
    double mx = 0.0;
    int dpos = -1;
    for (int i = lane; i < nc; i += 32) {
      mx = fmax(mx, fabs(v[b + i]));
      if (c[b + i] == row) dpos = i;
    }
    mx = warp_max(mx);
    dpos = __reduce_max_sync(0xffffffffu, dpos);
    const double thr = mul_rn(tol, mx);
    double lumped = 0.0;
    int ndrop = 0;
    if (lane == 0) {
      for (int i = 0; i < nc; ++i) {
        const double x = v[b + i];
        if (i != dpos && !(fabs(x) >= thr)) {
          lumped = add_rn(lumped, x);
          ++ndrop;
        }
      }
      if (ndrop) atomicOr(any_drop, 1);
    }
    lumped = __shfl_sync(0xffffffffu, lumped, 0);
    ndrop = __shfl_sync(0xffffffffu, ndrop, 0);
    const bool insert = lump && ndrop > 0 && dpos < 0 && lumped != 0.0;
    const long long o = (long long)b + row;
    int written = 0;
    int before = 0;
    for (int base = 0; base < nc; base += 32) {
      const int i = base + lane;
      bool keep = false;
      double x = 0.0;
      int cc = 0;
      if (i < nc) {
        x = v[b + i];
        cc = c[b + i];
        keep = i == dpos || fabs(x) >= thr;
        if (i == dpos && lump && ndrop > 0) x = add_rn(x, lumped);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      before += __popc(__ballot_sync(0xffffffffu, keep && cc < row));
      if (keep) {
        int dst = written + __popc(bal & ((1u << lane) - 1u));
        if (insert && cc > row) ++dst;
        out_col[o + dst] = cc;
        out_val[o + dst] = x;
      }
      written += __popc(bal);
    }
    if (insert) {
      if (lane == 0) {
        out_col[o + before] = row;
        out_val[o + before] = lumped;
      }
      ++written;
    }
    if (lane == 0) out_cnt[row] = written;
  }
}

static int finish_raw(int m, int ncols, const int* rawp, int* cnt, int* rcol, double* rval,
                      airg_csr_result** out, cudaStream_t s) {
  airg_csr_result* r = new_result(m, ncols, s);
  if (!r) return AIRG_ERR_CUDA;
  long long nnz = 0;
  AIRG_TRY(scan_counts(cnt, r->ptr, m, &nnz, s));
  AIRG_TRY(result_alloc_entries(r, nnz, true));
  if (m > 0)
    compact_rows_kernel<<<blocks_for((long long)m * 32, 256), 256, 0, s>>>(m, rawp, r->ptr, rcol, rval,
                                                                          r->col, r->val);
  AIRG_LAUNCH_CHECK();
  *out = r;
  return AIRG_OK;
}

// ----------------------------------------------------------------------------
// masked products: spgemm_fixed_sparsity and the polynomial assembly
// ----------------------------------------------------------------------------
// pattern = A + diag (sorted), count / fill
__global__ void pattern_diag_kernel(int n, const int* __restrict__ p, const int* __restrict__ c,
                                    const int* __restrict__ optr, int* __restrict__ ocol,
                                    int* __restrict__ cnt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int b = p[i], e = p[i + 1];
    bool has = false;
    for (int k = b; k < e; ++k) has |= c[k] == i;
    if (cnt) cnt[i] = e - b + (has ? 0 : 1);
    if (ocol) {
      int o = optr[i];
      bool done = has;
      for (int k = b; k < e; ++k) {
        if (!done && c[k] > i) {
          ocol[o++] = (int)i;
          done = true;
        }
        ocol[o++] = c[k];
      }
      if (!done) ocol[o++] = (int)i;
    }
  }
}

// Per row (warp): positions of the pattern row in shared memory; for each
// power k = 2..d: next[pos(j)] += P_{k-1}[i,q] * A[q,j] over q ascending
// (present entries only), lanes over A row q.  Accumulate
// s = ((c0 I + c1 A) + c2 P2) + ... with absent terms skipped; keep an entry
// iff it was present in some term and s != 0 (csr + prunes exact zeros).
// mode_masked=1: plain masked product P = A*B restricted to `pattern`
// (A row given by the pattern-relative current power = A row itself).
struct PolyArgs {
  int n;
  const int *Ap, *Ac;
  const double* Av;
  const int *Pp, *Pc;  // pattern (sorted)
  const double* coef;  // device coefficients (ncoef)
  int ncoef;
  int cap;             // max pattern row length handled in shared memory
  int bits;            // lookup table bits
  double* out_val;     // pattern-sized values
  unsigned char* out_keep;
  int* out_cnt;
  // masked-product mode: left operand rows (Lp, Lc, Lv), right (Ap...)
  int masked;
  const int *Lp, *Lc;
  const double* Lv;
};

__global__ void __launch_bounds__(128) poly_assemble_kernel(PolyArgs a) {
  extern __shared__ unsigned char smraw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int T = 1 << a.bits;
  const int cap = a.cap;
  // per warp: keys[T], pos[T], cur[cap], nxt[cap], acc[cap], flags cur/nxt/acc (3*cap bytes)
  const size_t per = (size_t)T * 8 + (size_t)cap * 24 + (size_t)cap * 3;
  unsigned char* base = smraw + (size_t)w * ((per + 15) & ~(size_t)15);
  double* cur = (double*)base;
  double* nxt = cur + cap;
  double* acc = nxt + cap;
  int* keys = (int*)(acc + cap);
  int* pv = keys + T;
  unsigned char* fcur = (unsigned char*)(pv + T);
  unsigned char* fnxt = fcur + cap;
  unsigned char* facc = fnxt + cap;
  for (long long r = (long long)blockIdx.x * nw + w; r < a.n; r += (long long)gridDim.x * nw) {
    const int row = (int)r;
    const int pb = a.Pp[row], pe = a.Pp[row + 1], m = pe - pb;
    if (m > cap) continue;  // handled by the global pass (flag via out_cnt = -1)
    for (int i = lane; i < T; i += 32) keys[i] = kEmpty;
    __syncwarp();
    for (int i = lane; i < m; i += 32) {
      map_insert(keys, pv, a.bits, a.Pc[pb + i], i);
      cur[i] = 0.0;
      nxt[i] = 0.0;
      acc[i] = 0.0;
      fcur[i] = 0;
      fnxt[i] = 0;
      facc[i] = 0;
    }
    __syncwarp();
    if (a.masked) {
      // one masked product: left row L_i, right rows A_q
      const int lb = a.Lp[row], le = a.Lp[row + 1];
      for (int qq = lb; qq < le; ++qq) {
        const int q = a.Lc[qq];
        const double lv = a.Lv[qq];
        for (int jj = a.Ap[q] + lane; jj < a.Ap[q + 1]; jj += 32) {
          const int p = map_find(keys, pv, a.bits, a.Ac[jj]);
          if (p >= 0) {
            nxt[p] = add_rn(nxt[p], mul_rn(lv, a.Av[jj]));
            fnxt[p] = 1;
          }
        }
        __syncwarp();
      }
      int c = 0;
      for (int i = lane; i < m; i += 32) {
        a.out_val[pb + i] = nxt[i];
        a.out_keep[pb + i] = fnxt[i];
        c += fnxt[i];
      }
      c = warp_sum(c);
      if (lane == 0) a.out_cnt[row] = c;
      __syncwarp();
      continue;
    }
    const int d = a.ncoef - 1;
    // term 0: c0 * I (diagonal is always in the pattern)
    const double c0 = a.coef[0];
    if (lane == 0) {
      const int p = map_find(keys, pv, a.bits, row);
      acc[p] = add_rn(acc[p], c0);  // 0 + c0 (=c0; -0 -> +0 is pruned anyway)
      facc[p] = 1;
    }
    __syncwarp();
    if (d >= 1) {
      const double c1 = a.coef[1];
      for (int kk = a.Ap[row] + lane; kk < a.Ap[row + 1]; kk += 32) {
        const int p = map_find(keys, pv, a.bits, a.Ac[kk]);
        const double v = a.Av[kk];
        acc[p] = add_rn(acc[p], mul_rn(c1, v));
        facc[p] = 1;
        cur[p] = v;
        fcur[p] = 1;
      }
      __syncwarp();
    }
    for (int k = 2; k <= d; ++k) {
      // nxt = mask(cur * A): walk present entries of cur in column (= position) order
      for (int q = 0; q < m; ++q) {
        if (!fcur[q]) continue;
        const int col_q = a.Pc[pb + q];
        const double lv = cur[q];
        for (int jj = a.Ap[col_q] + lane; jj < a.Ap[col_q + 1]; jj += 32) {
          const int p = map_find(keys, pv, a.bits, a.Ac[jj]);
          if (p >= 0) {
            nxt[p] = add_rn(nxt[p], mul_rn(lv, a.Av[jj]));
            fnxt[p] = 1;
          }
        }
        __syncwarp();
      }
      const double ck = a.coef[k];
      for (int i = lane; i < m; i += 32) {
        if (fnxt[i]) {
          acc[i] = add_rn(acc[i], mul_rn(ck, nxt[i]));
          facc[i] = 1;
        }
        cur[i] = nxt[i];
        fcur[i] = fnxt[i];
        nxt[i] = 0.0;
        fnxt[i] = 0;
      }
      __syncwarp();
    }
    int c = 0;
    for (int i = lane; i < m; i += 32) {
      const bool keep = d == 0 ? (bool)facc[i] : (facc[i] && acc[i] != 0.0);
      a.out_val[pb + i] = acc[i];
      a.out_keep[pb + i] = keep;
      c += keep;
    }
    c = warp_sum(c);
    if (lane == 0) a.out_cnt[row] = c;
    __syncwarp();
  }
}

__global__ void compact_keep_kernel(int m, const int* __restrict__ pp, const int* __restrict__ pc,
                                    const double* __restrict__ pv, const unsigned char* __restrict__ keep,
                                    const int* __restrict__ optr, int* __restrict__ oc,
                                    double* __restrict__ ov) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    int o = optr[i];
    for (int k = pp[i]; k < pp[i + 1]; ++k)
      if (keep[k]) {
        oc[o] = pc[k];
        ov[o] = pv[k];
        ++o;
      }
  }
}

__global__ void max_rowlen_kernel(int m, const int* __restrict__ p, int* __restrict__ mx) {
  int v = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x)
    v = max(v, p[i + 1] - p[i]);
  v = __reduce_max_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) atomicMax(mx, v);
}

static int max_row_len(int m, const int* p, int* out, cudaStream_t s) {
  int* d = nullptr;
  AIRG_TRY(scratch(&d, 1, s));
  AIRG_CUDA(cudaMemsetAsync(d, 0, sizeof(int), s));
  if (m > 0) max_rowlen_kernel<<<blocks_for(m, 256, 148 * 8), 256, 0, s>>>(m, p, d);
  AIRG_LAUNCH_CHECK();
  AIRG_CUDA(cudaMemcpyAsync(out, d, sizeof(int), cudaMemcpyDeviceToHost, s));
  AIRG_CUDA(cudaStreamSynchronize(s));
  release(d, s);
  return AIRG_OK;
}

static int run_poly_kernel(PolyArgs& a, int maxlen, cudaStream_t s) {
  int cap = 32;
  while (cap < maxlen) cap <<= 1;
  a.cap = cap;
  a.bits = ceil_log2(2ll * cap);
  const size_t T = (size_t)1 << a.bits;
  const size_t per = (T * 8 + (size_t)cap * 27 + 15) & ~(size_t)15;
  int warps = 4;
  while (warps > 1 && per * warps > (size_t)smem_limit()) warps >>= 1;
  if (per > (size_t)smem_limit()) {
    set_error("pattern row of %d entries exceeds the shared-memory assembly kernel", maxlen);
    return AIRG_ERR_VALUE;
  }
  const size_t shm = per * warps;
  if (shm > 48 * 1024)
    AIRG_CUDA(cudaFuncSetAttribute(poly_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)shm));
  poly_assemble_kernel<<<blocks_for(a.n, warps, 148 * 32), warps * 32, shm, s>>>(a);
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

// ----------------------------------------------------------------------------
// extract / restriction assembly
// ----------------------------------------------------------------------------
__global__ void extract_kernel(int nr, const int* __restrict__ rows, const int* __restrict__ p,
                               const int* __restrict__ c, const double* __restrict__ v,
                               const int* __restrict__ colmap, const int* __restrict__ optr,
                               int* __restrict__ oc, double* __restrict__ ov, int* __restrict__ cnt) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nr;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = rows[t];
    int o = optr ? optr[t] : 0, n = 0;
    for (int k = p[i]; k < p[i + 1]; ++k) {
      const int m = colmap[c[k]];
      if (m < 0) continue;
      if (oc) {
        oc[o + n] = m;
        ov[o + n] = v[k];
      }
      ++n;
    }
    if (cnt) cnt[t] = n;
  }
}

__global__ void colmap_kernel(int n, const signed char* __restrict__ labels, signed char want,
                              const int* __restrict__ pos, int* __restrict__ map) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    map[i] = labels[i] == want ? pos[i] : -1;
}

// R row j = [Z row j mapped through f_idx | 1 at c_idx[j]] in fine ordering
__global__ void restriction_kernel(int nc, const int* __restrict__ zp, const int* __restrict__ zc,
                                   const double* __restrict__ zv, const int* __restrict__ f_idx,
                                   const int* __restrict__ c_idx, int* __restrict__ rp,
                                   int* __restrict__ rc, double* __restrict__ rv) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < nc;
       j += (long long)gridDim.x * blockDim.x) {
    const int b = zp[j], e = zp[j + 1];
    const int cj = c_idx[j];
    long long o = (long long)b + j;
    rp[j] = (int)o;
    if (j == nc - 1) rp[nc] = (int)(e + nc);
    bool done = false;
    for (int k = b; k < e; ++k) {
      const int col = f_idx[zc[k]];
      if (!done && col > cj) {
        rc[o] = cj;
        rv[o] = 1.0;
        ++o;
        done = true;
      }
      rc[o] = col;
      rv[o] = zv[k];
      ++o;
    }
    if (!done) {
      rc[o] = cj;
      rv[o] = 1.0;
    }
  }
}

}  // namespace airg

using namespace airg;

extern "C" {

int airg_spgemm(int m, int k, int n, const int32_t* Ap, const int32_t* Ac, const double* Av,
                const int32_t* Bp, const int32_t* Bc, const double* Bv, int negate,
                airg_csr_result** out, void* stream) {
  Mat A{m, k, Ap, Ac, Av}, B{k, n, Bp, Bc, Bv};
  return spgemm_full(A, B, negate, out, (cudaStream_t)stream);
}

int airg_spgemm_masked(int m, int k, int n, const int32_t* Ap, const int32_t* Ac, const double* Av,
                       const int32_t* Bp, const int32_t* Bc, const double* Bv, const int32_t* Pp,
                       const int32_t* Pc, airg_csr_result** out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int maxlen = 0;
  AIRG_TRY(max_row_len(m, Pp, &maxlen, s));
  int pnnz = 0;
  if (m > 0) AIRG_CUDA(cudaMemcpyAsync(&pnnz, Pp + m, sizeof(int), cudaMemcpyDeviceToHost, s));
  AIRG_CUDA(cudaStreamSynchronize(s));
  double* pv = nullptr;
  unsigned char* keep = nullptr;
  int* cnt = nullptr;
  AIRG_TRY(scratch(&pv, pnnz, s));
  AIRG_TRY(scratch(&keep, pnnz, s));
  AIRG_TRY(scratch(&cnt, m + 1, s));
  PolyArgs a{};
  a.n = m;
  a.Ap = Bp;
  a.Ac = Bc;
  a.Av = Bv;
  a.Pp = Pp;
  a.Pc = Pc;
  a.out_val = pv;
  a.out_keep = keep;
  a.out_cnt = cnt;
  a.masked = 1;
  a.Lp = Ap;
  a.Lc = Ac;
  a.Lv = Av;
  AIRG_TRY(run_poly_kernel(a, maxlen, s));
  airg_csr_result* r = new_result(m, n, s);
  long long nnz = 0;
  AIRG_TRY(scan_counts(cnt, r->ptr, m, &nnz, s));
  AIRG_TRY(result_alloc_entries(r, nnz, true));
  if (m > 0) compact_keep_kernel<<<blocks_for(m, 256), 256, 0, s>>>(m, Pp, Pc, pv, keep, r->ptr, r->col, r->val);
  AIRG_LAUNCH_CHECK();
  release(pv, s);
  release(keep, s);
  release(cnt, s);
  *out = r;
  return AIRG_OK;
}

int airg_poly_assemble(int n, const int32_t* Ap, const int32_t* Ac, const double* Av, int ncoef,
                       const double* coef_h, airg_csr_result** out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (ncoef < 1) {
    set_error("need at least one coefficient");
    return AIRG_ERR_VALUE;
  }
  int *cnt = nullptr, *Pp = nullptr, *Pc = nullptr;
  AIRG_TRY(scratch(&cnt, n + 1, s));
  AIRG_TRY(scratch(&Pp, n + 1, s));
  const int nb = blocks_for(n, 256);
  if (n > 0) pattern_diag_kernel<<<nb, 256, 0, s>>>(n, Ap, Ac, nullptr, nullptr, cnt);
  long long pnnz = 0;
  AIRG_TRY(scan_counts(cnt, Pp, n, &pnnz, s));
  AIRG_TRY(scratch(&Pc, pnnz, s));
  if (n > 0) pattern_diag_kernel<<<nb, 256, 0, s>>>(n, Ap, Ac, Pp, Pc, nullptr);
  AIRG_LAUNCH_CHECK();
  int maxlen = 0;
  AIRG_TRY(max_row_len(n, Pp, &maxlen, s));
  double *pv = nullptr, *dcoef = nullptr;
  unsigned char* keep = nullptr;
  AIRG_TRY(scratch(&pv, pnnz, s));
  AIRG_TRY(scratch(&keep, pnnz, s));
  AIRG_TRY(scratch(&dcoef, ncoef, s));
  AIRG_CUDA(cudaMemcpyAsync(dcoef, coef_h, ncoef * sizeof(double), cudaMemcpyHostToDevice, s));
  PolyArgs a{};
  a.n = n;
  a.Ap = Ap;
  a.Ac = Ac;
  a.Av = Av;
  a.Pp = Pp;
  a.Pc = Pc;
  a.coef = dcoef;
  a.ncoef = ncoef;
  a.out_val = pv;
  a.out_keep = keep;
  a.out_cnt = cnt;
  AIRG_TRY(run_poly_kernel(a, maxlen, s));
  airg_csr_result* r = new_result(n, n, s);
  long long nnz = 0;
  AIRG_TRY(scan_counts(cnt, r->ptr, n, &nnz, s));
  AIRG_TRY(result_alloc_entries(r, nnz, true));
  if (n > 0) compact_keep_kernel<<<nb, 256, 0, s>>>(n, Pp, Pc, pv, keep, r->ptr, r->col, r->val);
  AIRG_LAUNCH_CHECK();
  for (void* q : {(void*)cnt, (void*)Pp, (void*)Pc, (void*)pv, (void*)keep, (void*)dcoef}) release(q, s);
  *out = r;
  return AIRG_OK;
}

int airg_drop_lump(int m, int ncols, const int32_t* p, const int32_t* c, const double* v,
                   double tol, int lump, airg_csr_result** out, int32_t* changed_h, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (tol < 0) {
    set_error("rel_tol must be non-negative");
    return AIRG_ERR_VALUE;
  }
  if (lump && m != ncols) {
    set_error("lumping requires a square matrix");
    return AIRG_ERR_VALUE;
  }
  int nnz = 0;
  if (m > 0) AIRG_CUDA(cudaMemcpyAsync(&nnz, p + m, sizeof(int), cudaMemcpyDeviceToHost, s));
  AIRG_CUDA(cudaStreamSynchronize(s));
  int *rcol = nullptr, *cnt = nullptr, *anyd = nullptr;
  double* rval = nullptr;
  const long long raw = (long long)nnz + m;
  AIRG_TRY(scratch(&rcol, raw, s));
  AIRG_TRY(scratch(&rval, raw, s));
  AIRG_TRY(scratch(&cnt, m + 1, s));
  AIRG_TRY(scratch(&anyd, 1, s));
  AIRG_CUDA(cudaMemsetAsync(anyd, 0, sizeof(int), s));
  if (m > 0)
    drop_lump_kernel<<<blocks_for((long long)m * 32, 256), 256, 0, s>>>(m, p, c, v, tol, lump, rcol, rval,
                                                                       cnt, anyd);
  AIRG_LAUNCH_CHECK();
  AIRG_TRY(finish_raw(m, ncols, p, cnt, rcol, rval, out, s));
  int ad = 0;
  AIRG_CUDA(cudaMemcpyAsync(&ad, anyd, sizeof(int), cudaMemcpyDeviceToHost, s));
  AIRG_CUDA(cudaStreamSynchronize(s));
  if (changed_h) *changed_h = ad;
  for (void* q : {(void*)rcol, (void*)rval, (void*)cnt, (void*)anyd}) release(q, s);
  return AIRG_OK;
}

int airg_galerkin(int n, int nc, const int32_t* Rp, const int32_t* Rc, const double* Rv,
                  const int32_t* Ap, const int32_t* Ac, const double* Av, const int32_t* pcol,
                  double a_drop, int lump, airg_csr_result** out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  // P as CSR (one unit entry per row)
  int* Pp = nullptr;
  double* Pv = nullptr;
  AIRG_TRY(scratch(&Pp, n + 1, s));
  AIRG_TRY(scratch(&Pv, n, s));
  iota_kernel<<<blocks_for(n + 1, 256), 256, 0, s>>>(n, Pp);
  ones_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, Pv);
  AIRG_LAUNCH_CHECK();
  Mat A{n, n, Ap, Ac, Av}, P{n, nc, Pp, pcol, Pv};
  airg_csr_result* AP = nullptr;
  AIRG_TRY(spgemm_full(A, P, 0, &AP, s));
  Mat R{nc, n, Rp, Rc, Rv}, APm{n, nc, AP->ptr, AP->col, AP->val};
  int *Cp = nullptr, *Cc = nullptr;
  long long nnz = 0;
  AIRG_TRY(spgemm_structure(R, APm, &Cp, &Cc, &nnz, nullptr, s));
  if (a_drop == 0.0) {
    airg_csr_result* r = new airg_csr_result();
    r->nrows = nc;
    r->ncols = nc;
    r->stream = s;
    r->ptr = Cp;
    r->col = Cc;
    r->nnz = nnz;
    AIRG_TRY(scratch(&r->val, nnz, s));
    AIRG_TRY(spgemm_numeric(R, APm, Cp, Cc, r->val, 0, 0, 0.0, 0, nullptr, nullptr, nullptr, s));
    *out = r;
  } else {
    int *rcol = nullptr, *cnt = nullptr;
    double* rval = nullptr;
    AIRG_TRY(scratch(&rcol, nnz + nc, s));
    AIRG_TRY(scratch(&rval, nnz + nc, s));
    AIRG_TRY(scratch(&cnt, nc + 1, s));
    AIRG_TRY(spgemm_numeric(R, APm, Cp, Cc, nullptr, 0, 1, a_drop, lump, rcol, rval, cnt, s));
    AIRG_TRY(finish_raw(nc, nc, Cp, cnt, rcol, rval, out, s));
    for (void* q : {(void*)rcol, (void*)rval, (void*)cnt, (void*)Cp, (void*)Cc}) release(q, s);
  }
  airg_result_free(AP);
  release(Pp, s);
  release(Pv, s);
  return AIRG_OK;
}

int airg_extract(int nr_sel, const int32_t* rows, const int32_t* p, const int32_t* c,
                 const double* v, const int32_t* colmap, int ncols_sel, airg_csr_result** out,
                 void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  airg_csr_result* r = new_result(nr_sel, ncols_sel, s);
  int* cnt = nullptr;
  AIRG_TRY(scratch(&cnt, nr_sel + 1, s));
  const int nb = blocks_for(nr_sel, 256);
  if (nr_sel > 0)
    extract_kernel<<<nb, 256, 0, s>>>(nr_sel, rows, p, c, v, colmap, nullptr, nullptr, nullptr, cnt);
  long long nnz = 0;
  AIRG_TRY(scan_counts(cnt, r->ptr, nr_sel, &nnz, s));
  AIRG_TRY(result_alloc_entries(r, nnz, true));
  if (nr_sel > 0)
    extract_kernel<<<nb, 256, 0, s>>>(nr_sel, rows, p, c, v, colmap, r->ptr, r->col, r->val, nullptr);
  AIRG_LAUNCH_CHECK();
  release(cnt, s);
  *out = r;
  return AIRG_OK;
}

int airg_label_colmap(int n, const int8_t* labels, int which, const int32_t* pos, int32_t* map,
                      void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n > 0)
    colmap_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, (const signed char*)labels,
                                                      (signed char)which, pos, map);
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

int airg_restriction(int n, int nc, const int32_t* zp, const int32_t* zc, const double* zv,
                     const int32_t* f_idx, const int32_t* c_idx, airg_csr_result** out,
                     void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int znnz = 0;
  if (nc > 0) AIRG_CUDA(cudaMemcpyAsync(&znnz, zp + nc, sizeof(int), cudaMemcpyDeviceToHost, s));
  AIRG_CUDA(cudaStreamSynchronize(s));
  airg_csr_result* r = new_result(nc, n, s);
  AIRG_TRY(result_alloc_entries(r, (long long)znnz + nc, true));
  if (nc > 0)
    restriction_kernel<<<blocks_for(nc, 256), 256, 0, s>>>(nc, zp, zc, zv, f_idx, c_idx, r->ptr, r->col,
                                                          r->val);
  else
    AIRG_CUDA(cudaMemsetAsync(r->ptr, 0, sizeof(int), s));
  AIRG_LAUNCH_CHECK();
  *out = r;
  return AIRG_OK;
}

}  // extern "C"
