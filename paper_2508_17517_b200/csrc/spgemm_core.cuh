// Row-wise Gustavson SpGEMM core, bit-exact with scipy's csr_matmat.
//
// Pass 1 (count): warp per row, shared-memory open-addressing key set.
// Pass 2 (numeric + structure): warp per row, key -> slot table with an fp64
//   accumulator per slot; the A row is walked in order and lanes split ONE B
//   row at a time (distinct output columns), so every output entry receives
//   its k contributions in ascending order with separate mul/add roundings.
//   The occupied slots are compacted and bitonic-sorted by column in shared
//   memory and written once (optionally negated, or through the fused
//   drop_and_lump epilogue).
// Latency: A-row metadata (k, a_ik, B row bounds) is fetched 32 entries at a
// time, one per lane, and the first 32 entries of the next B row are loaded
// before the current one is processed.
#pragma once
#include "setup_common.cuh"
#include <vector>

namespace airg {

constexpr int kEmpty = -1;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned hash_of(int key, int bits) {
  return ((unsigned)key * 0x9E3779B1u) >> (32 - bits);
}

// returns 1 when newly inserted, 0 when present, 1<<20 when the table is full
__device__ __forceinline__ int set_insert(int* keys, int bits, int key) {
  const unsigned mask = (1u << bits) - 1u;
  unsigned h = hash_of(key, bits);
  for (unsigned probe = 0; probe <= mask; ++probe) {
    const int cur = keys[h];  // most products hit a present key: read before CAS
    if (cur == key) return 0;
    if (cur == kEmpty) {
      const int prev = atomicCAS(keys + h, kEmpty, key);
      if (prev == kEmpty) return 1;
      if (prev == key) return 0;
    }
    h = (h + 1u) & mask;
  }
  return 1 << 20;
}

// slot of key (inserting it); the table always has room in pass 2
__device__ __forceinline__ int slot_of(int* keys, int bits, int key) {
  const unsigned mask = (1u << bits) - 1u;
  unsigned h = hash_of(key, bits);
  while (true) {
    const int cur = keys[h];
    if (cur == key) return (int)h;
    if (cur == kEmpty) {
      const int prev = atomicCAS(keys + h, kEmpty, key);
      if (prev == kEmpty || prev == key) return (int)h;
    }
    h = (h + 1u) & mask;
  }
}

__device__ __forceinline__ int map_find(const int* keys, const int* vals, int bits, int key) {
  const unsigned mask = (1u << bits) - 1u;
  unsigned h = hash_of(key, bits);
  while (true) {
    const int k = keys[h];
    if (k == key) return vals[h];
    if (k == kEmpty) return -1;
    h = (h + 1u) & mask;
  }
}

__device__ __forceinline__ void map_insert(int* keys, int* vals, int bits, int key, int v) {
  const unsigned mask = (1u << bits) - 1u;
  unsigned h = hash_of(key, bits);
  while (true) {
    const int prev = atomicCAS(keys + h, kEmpty, key);
    if (prev == kEmpty || prev == key) {
      vals[h] = v;
      return;
    }
    h = (h + 1u) & mask;
  }
}

// warp-wide bitonic sort of buf[0..P) ascending (P power of two); optional payload
template <typename V>
__device__ void warp_bitonic(int* buf, V* pay, int P, int lane) {
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
            if (pay) {
              const V t = pay[i];
              pay[i] = pay[ixj];
              pay[ixj] = t;
            }
          }
        }
      }
      __syncwarp();
    }
  }
}

// Warp-level stable LSD radix sort of (k, v)[0..n) by k (8-bit digits of
// k - min k), ping-ponging through (k2, v2)[0..n); cnt = 256 ints of scratch.
// The sorted result is left in (k, v).
template <typename V>
__device__ void warp_radix_sort(int* k, V* v, int* k2, V* v2, int n, int* cnt, int lane) {
  int mn = 0x7fffffff, mx = -0x7fffffff - 1;
  for (int i = lane; i < n; i += 32) {
    mn = min(mn, k[i]);
    mx = max(mx, k[i]);
  }
  mn = __reduce_min_sync(kFull, mn);
  mx = __reduce_max_sync(kFull, mx);
  const unsigned span = (unsigned)(mx - mn);
  const int bits = span ? 32 - __clz(span) : 0;
  const int passes = (bits + 7) / 8;
  int *src = k, *dst = k2;
  V *vs = v, *vd = v2;
  const unsigned lt = (1u << lane) - 1u;
  for (int p = 0; p < passes; ++p) {
    const int sh = 8 * p;
    for (int i = lane; i < 256; i += 32) cnt[i] = 0;
    __syncwarp();
    for (int i = lane; i < n; i += 32) atomicAdd(cnt + ((((unsigned)(src[i] - mn)) >> sh) & 255u), 1);
    __syncwarp();
    // exclusive scan of the 256 counters: 8 per lane
    int loc[8], s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      loc[j] = s;
      s += cnt[lane * 8 + j];
    }
    int inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    const int excl = inc - s;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j) cnt[lane * 8 + j] = excl + loc[j];
    __syncwarp();
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const bool ok = i < n;
      const int key = ok ? src[i] : 0;
      const int d = ok ? (int)((((unsigned)(key - mn)) >> sh) & 255u) : 256 + lane;
      const unsigned peers = __match_any_sync(kFull, d);
      int off = 0;
      if (ok) {
        off = cnt[d] + __popc(peers & lt);
        dst[off] = key;
        vd[off] = vs[i];
      }
      __syncwarp();
      if (ok && lane == __ffs(peers) - 1) cnt[d] += __popc(peers);
      __syncwarp();
    }
    int* tk = src;
    src = dst;
    dst = tk;
    V* tv = vs;
    vs = vd;
    vd = tv;
  }
  if (src != k) {
    for (int i = lane; i < n; i += 32) {
      k[i] = src[i];
      v[i] = vs[i];
    }
    __syncwarp();
  }
}

// Predicated global loads straight into the destination register (value
// kept when the predicate is off).  Written as PTX so the compiler cannot
// load into a temporary and move it to the destination, which would wait
// for the load and defeat a software-pipelined walk.
__device__ __forceinline__ void ld_pred(int& v, const int* p, bool pr) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.b32 %0, [%1];\n\t}"
               : "+r"(v) : "l"(p), "r"((int)pr));
}
__device__ __forceinline__ void ld_pred(double& v, const double* p, bool pr) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.f64 %0, [%1];\n\t}"
               : "+d"(v) : "l"(p), "r"((int)pr));
}

__host__ __device__ __forceinline__ int ceil_log2(long long x) {
  int b = 0;
  while ((1ll << b) < x) ++b;
  return b;
}

// Walk the products of A row `row` with B: f(a_ik, col, b_kj) per product,
// lanes split one B row, rows in A order; SYNC orders successive B rows.
template <bool SYNC, bool VALUES, class F>
__device__ __forceinline__ void walk_products(const int* __restrict__ Ap, const int* __restrict__ Ac,
                                              const double* __restrict__ Av,
                                              const int* __restrict__ Bp, const int* __restrict__ Bc,
                                              const double* __restrict__ Bv, int row, int lane,
                                              F& f) {
  const int ab = Ap[row], ae = Ap[row + 1];
  for (int base = ab; base < ae; base += 32) {
    const int kk = base + lane;
    int bb = 0, be = 0;
    double av = 0.0;
    if (kk < ae) {
      const int k = Ac[kk];
      if (VALUES) av = Av[kk];
      bb = Bp[k];
      be = Bp[k + 1];
    }
    const int cnt = min(32, ae - base);
    // the first kPre*32 entries of the next B row live in registers one step ahead
    constexpr int kPre = 1;
    int cb = __shfl_sync(kFull, bb, 0), ce = __shfl_sync(kFull, be, 0);
    int pc[kPre];
    double pv[kPre];
#pragma unroll
    for (int q = 0; q < kPre; ++q) {
      const int jj = cb + 32 * q + lane;
      pc[q] = jj < ce ? Bc[jj] : -1;
      pv[q] = (VALUES && jj < ce) ? Bv[jj] : 0.0;
    }
    for (int t = 0; t < cnt; ++t) {
      const double a = VALUES ? __shfl_sync(kFull, av, t) : 0.0;
      const int tb = cb, te = ce;
      int c0[kPre];
      double v0[kPre];
#pragma unroll
      for (int q = 0; q < kPre; ++q) {
        c0[q] = pc[q];
        v0[q] = pv[q];
      }
      if (t + 1 < cnt) {  // prefetch the next B row
        cb = __shfl_sync(kFull, bb, t + 1);
        ce = __shfl_sync(kFull, be, t + 1);
#pragma unroll
        for (int q = 0; q < kPre; ++q) {
          const int jj = cb + 32 * q + lane;
          pc[q] = jj < ce ? Bc[jj] : -1;
          if (VALUES) pv[q] = jj < ce ? Bv[jj] : 0.0;
        }
      }
#pragma unroll
      for (int q = 0; q < kPre; ++q)
        if (c0[q] >= 0) f(a, c0[q], v0[q]);
      for (int jb = tb + 32 * kPre; jb < te; jb += 96) {
        int cc[3];
        double vv[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int jj = jb + 32 * q + lane;
          cc[q] = jj < te ? Bc[jj] : -1;
          vv[q] = (VALUES && jj < te) ? Bv[jj] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 3; ++q)
          if (cc[q] >= 0) f(a, cc[q], vv[q]);
      }
      if (SYNC) __syncwarp();
    }
  }
}

struct CountOp {
  int* keys;
  int bits;
  int added;
  __device__ __forceinline__ void operator()(double, int c, double) { added += set_insert(keys, bits, c); }
};

struct AccOp {
  int* keys;
  double* acc;
  int bits;
  __device__ __forceinline__ void operator()(double a, int c, double v) {
    const int s = slot_of(keys, bits, c);
    acc[s] = add_rn(acc[s], mul_rn(a, v));
  }
};

// In-place compaction of occupied slots (keys + payload) to [0, n).
template <typename V>
__device__ __forceinline__ int compact_slots(int* keys, V* pay, int T, int lane) {
  int wpos = 0;
  for (int base = 0; base < T; base += 32) {
    const int k = keys[base + lane];
    V v{};
    if (pay) v = pay[base + lane];
    const bool occ = k != kEmpty;
    const unsigned bal = __ballot_sync(kFull, occ);
    __syncwarp();
    if (occ) {
      const int d = wpos + __popc(bal & ((1u << lane) - 1u));
      keys[d] = k;
      if (pay) pay[d] = v;
    }
    wpos += __popc(bal);
    __syncwarp();
  }
  return wpos;
}

// drop_and_lump (sparse.py:307-352) of one sorted row held in (col, val)[0..n):
// keep = diagonal | |v| >= tol*max|v|; dropped values summed sequentially in
// column order onto the diagonal (inserted when absent and the sum != 0).
// Writes kept entries to out_col/out_val[o...]; returns the written count.
__device__ static int drop_lump_row(const int* col, double* val, int n, int row, double tol, int lump,
                             int* __restrict__ out_col, double* __restrict__ out_val, long long o,
                             int lane, int* any_drop) {
  double mx = 0.0;
  int dpos = -1;
  for (int i = lane; i < n; i += 32) {
    mx = fmax(mx, fabs(val[i]));
    if (col[i] == row) dpos = i;
  }
  mx = warp_max(mx);
  dpos = __reduce_max_sync(kFull, dpos);
  const double thr = mul_rn(tol, mx);
  // dropped values, in column order, are packed into val[n ..) (callers'
  // tables hold >= 2n slots) and summed one by one by lane 0: the serial
  // chain is one add per dropped entry with its loads pipelined
  double* dropped = val + n;
  int ndrop = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const double x = i < n ? val[i] : 0.0;
    const bool d = i < n && i != dpos && !(fabs(x) >= thr);
    const unsigned bal = __ballot_sync(kFull, d);
    if (d) dropped[ndrop + __popc(bal & ((1u << lane) - 1u))] = x;
    ndrop += __popc(bal);
  }
  __syncwarp();
  double lumped = 0.0;
  if (lane == 0) {
#pragma unroll 8
    for (int i = 0; i < ndrop; ++i) lumped = add_rn(lumped, dropped[i]);
    if (ndrop && any_drop) atomicOr(any_drop, 1);
  }
  lumped = __shfl_sync(kFull, lumped, 0);
  const bool insert = lump && ndrop > 0 && dpos < 0 && lumped != 0.0;
  int written = 0, before = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    bool keep = false;
    double x = 0.0;
    int cc = 0;
    if (i < n) {
      x = val[i];
      cc = col[i];
      keep = i == dpos || fabs(x) >= thr;
      if (i == dpos && lump && ndrop > 0) x = add_rn(x, lumped);
    }
    const unsigned bal = __ballot_sync(kFull, keep);
    before += __popc(__ballot_sync(kFull, keep && cc < row));
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
  return written;
}

// ---- row classification by size (shared by the SpGEMM and assembly kernels) ----
static __global__ void rowlen_kernel(int m, const int* __restrict__ ptr, long long* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = ptr[i + 1] - ptr[i];
}

constexpr int kMaxCls = 24;

// block-aggregated append of row ids to per-class lists (lists[c*m + ...])
static __global__ void classify_kernel(int m, const long long* __restrict__ size, const long long* __restrict__ th,
                                int ncls, int* __restrict__ lists, int* __restrict__ counts) {
  __shared__ int scnt[kMaxCls], sbase[kMaxCls];
  if (threadIdx.x < ncls) scnt[threadIdx.x] = 0;
  __syncthreads();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int c = 0, slot = 0;
  if (i < m) {
    const long long v = size[i];
    while (c < ncls - 1 && v > th[c]) ++c;
    slot = atomicAdd(scnt + c, 1);
  }
  __syncthreads();
  if (threadIdx.x < ncls) sbase[threadIdx.x] = atomicAdd(counts + threadIdx.x, scnt[threadIdx.x]);
  __syncthreads();
  if (i < m) lists[(long long)c * m + sbase[c] + slot] = (int)i;
}

// same with a precomputed class id per row
static __global__ void classify_ids_kernel(int m, const int* __restrict__ ids, int ncls,
                                           int* __restrict__ lists, int* __restrict__ counts) {
  __shared__ int scnt[kMaxCls], sbase[kMaxCls];
  if (threadIdx.x < ncls) scnt[threadIdx.x] = 0;
  __syncthreads();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int c = 0, slot = 0;
  if (i < m) {
    c = ids[i];
    slot = atomicAdd(scnt + c, 1);
  }
  __syncthreads();
  if (threadIdx.x < ncls) sbase[threadIdx.x] = atomicAdd(counts + threadIdx.x, scnt[threadIdx.x]);
  __syncthreads();
  if (i < m) lists[(long long)c * m + sbase[c] + slot] = (int)i;
}

struct Classes {
  std::vector<int> count;
  int* lists = nullptr;
  int m = 0;
  const int* list(int c) const { return lists + (long long)c * m; }
};

// extra_dev/extra_h: one more device int read back with the same synchronisation
static int classify(int m, const long long* size, const std::vector<long long>& th, Classes& out,
                    cudaStream_t s, const int* extra_dev = nullptr, int* extra_h = nullptr) {
  const int ncls = (int)th.size() + 1;
  long long* dth = nullptr;
  int* cnt = nullptr;
  AIRG_TRY(scratch(&out.lists, (size_t)ncls * (m > 0 ? m : 1), s));
  AIRG_TRY(scratch(&dth, th.size() + 1, s));
  AIRG_TRY(scratch(&cnt, ncls, s));
  if (!th.empty())
    AIRG_CUDA(cudaMemcpyAsync(dth, th.data(), th.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
  AIRG_CUDA(cudaMemsetAsync(cnt, 0, ncls * sizeof(int), s));
  if (m > 0) classify_kernel<<<(m + 255) / 256, 256, 0, s>>>(m, size, dth, ncls, out.lists, cnt);
  AIRG_LAUNCH_CHECK();
  out.count.assign(ncls, 0);
  if (extra_dev)
    AIRG_CUDA(read_back({{out.count.data(), cnt, ncls * sizeof(int)}, {extra_h, extra_dev, sizeof(int)}}, s));
  else
    AIRG_CUDA(read_back(out.count.data(), cnt, ncls * sizeof(int), s));
  out.m = m;
  release(dth, s);
  release(cnt, s);
  return AIRG_OK;
}

// class lists from per-row ids in [0, ncls); extra_dev as in classify
static int classify_ids(int m, const int* ids, int ncls, Classes& out, cudaStream_t s,
                        const int* extra_dev = nullptr, int* extra_h = nullptr) {
  int* cnt = nullptr;
  AIRG_TRY(scratch(&out.lists, (size_t)ncls * (m > 0 ? m : 1), s));
  AIRG_TRY(scratch(&cnt, ncls, s));
  AIRG_CUDA(cudaMemsetAsync(cnt, 0, ncls * sizeof(int), s));
  if (m > 0) classify_ids_kernel<<<(m + 255) / 256, 256, 0, s>>>(m, ids, ncls, out.lists, cnt);
  AIRG_LAUNCH_CHECK();
  out.count.assign(ncls, 0);
  if (extra_dev)
    AIRG_CUDA(read_back({{out.count.data(), cnt, ncls * sizeof(int)}, {extra_h, extra_dev, sizeof(int)}}, s));
  else
    AIRG_CUDA(read_back(out.count.data(), cnt, ncls * sizeof(int), s));
  out.m = m;
  release(cnt, s);
  return AIRG_OK;
}

}  // namespace airg
