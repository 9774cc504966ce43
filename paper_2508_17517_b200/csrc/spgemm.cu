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
#include "spgemm_core.cuh"
#include <vector>
#include <type_traits>
#include <algorithm>

namespace airg {


// raw rows live at [ptr[r] + r, ...) (one spare slot per row for a lumped diagonal)
__global__ void compact_rows_kernel(int m, const int* __restrict__ rawp, const int* __restrict__ optr,
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
                                    int* __restrict__ cnt, int row0 = 0) {
  for (long long li = blockIdx.x * (long long)blockDim.x + threadIdx.x; li < n;
       li += (long long)gridDim.x * blockDim.x) {
    const int b = p[li], e = p[li + 1];
    const int i = row0 + (int)li;  // global id of the diagonal
    bool has = false;
    for (int k = b; k < e; ++k) has |= c[k] == i;
    if (cnt) cnt[li] = e - b + (has ? 0 : 1);
    if (ocol) {
      int o = optr[li];
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

// Position of a column in the (sorted) pattern row of the current row, held
// in shared memory: a hash table (any column window) or a bitmap of the
// row's window [pmin, pmax] (windows <= kPolySpan columns -- every row of the
// advection hierarchies).  The bitmap answers with a bit test (misses, most
// products) and a rank (hits); the hash table needs a probe sequence, which
// for a miss runs until an empty slot.
constexpr int kPolySpan = 8192;
constexpr int kPolyWords = kPolySpan / 32;

struct HashPos {
  int* keys;
  int* pv;
  int bits;
  static __host__ __device__ size_t bytes(int cap) { return (size_t)8 << ceil_log2(2ll * cap); }
  __device__ void bind(unsigned char* p, int cap) {
    bits = ceil_log2(2ll * cap);
    keys = (int*)p;
    pv = keys + (1 << bits);
  }
  __device__ void clear(const int*, int, int, int tid, int nt) {
    for (int i = tid; i < (1 << bits); i += nt) keys[i] = kEmpty;
  }
  __device__ void insert(const int* pc, int i) { map_insert(keys, pv, bits, pc[i], i); }
  __device__ int find(int c) const { return map_find(keys, pv, bits, c); }
};

struct BitPos {
  uint2* bm;  // per window word: (position of its first column, bits)
  int pmin;
  unsigned span;
  static __host__ __device__ size_t bytes(int) { return (size_t)kPolyWords * sizeof(uint2); }
  __device__ void bind(unsigned char* p, int) { bm = (uint2*)p; }
  // pc: the pattern row (m sorted columns)
  __device__ void clear(const int* pc, int m, int, int tid, int nt) {
    pmin = m ? pc[0] : 0;
    span = m ? (unsigned)(pc[m - 1] - pmin + 1) : 0u;
    for (int i = tid; i < (int)((span + 31) >> 5); i += nt) bm[i] = make_uint2(0u, 0u);
  }
  __device__ void insert(const int* pc, int i) {
    const unsigned off = (unsigned)(pc[i] - pmin);
    atomicOr(&bm[off >> 5].y, 1u << (off & 31u));
    if (i == 0 || ((unsigned)(pc[i - 1] - pmin) >> 5) != (off >> 5)) bm[off >> 5].x = (unsigned)i;
  }
  __device__ int find(int c) const {
    const unsigned off = (unsigned)(c - pmin);
    if (off >= span) return -1;
    const uint2 e = bm[off >> 5];
    if (!((e.y >> (off & 31u)) & 1u)) return -1;
    return (int)e.x + __popc(e.y & ((1u << (off & 31u)) - 1u));
  }
};

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
  // row-strip operation: global id of local row 0 and global column -> row
  // of Ap (local rows first, then fetched ghost rows); null = identity
  int row0;
  const int* rowmap;
  // rows handled by this launch (one length class); null = all n rows
  const int* rows;
  int nrows;
  // block kernel only: per-CTA working set in global memory (rows whose
  // working set exceeds shared memory), gstride bytes per CTA; null = smem
  unsigned char* gmem;
  size_t gstride;
};

// One power of the warp-per-row assembly: nxt[pos(j)] += cur[q] * A[q, j]
// over the present positions q in ascending order, lanes splitting the A
// row of col_q (distinct columns -> distinct positions; rows in order, so
// the summation order is the reference's).  Software-pipelined: while the
// products of one A row are formed, the first KP x 32 entries of the
// next present row are already loading into the other register set (two
// named sets, no register copies of pending loads), and the next 32-position
// block's row bounds are fetched when a block is entered.  Entries beyond
// KP x 32 of a row load in place (KP from the class's pattern length).
template <int KP>
struct PolyRowRegs {
  int c[KP];
  double v[KP];
  int b, e;
  double l;
};

template <class PM, int KP>
__device__ __forceinline__ void poly_power_walk(const PolyArgs& a, const PM& pm, int pb, int m,
                                                int lane, const double* cur,
                                                const unsigned char* fcur, double* nxt,
                                                unsigned char* fnxt) {
  // block metadata (per lane: position base + lane)
  auto meta = [&](int base, int& rb, int& re, double& lv) -> unsigned {
    const int q = base + lane;
    const bool pres = q < m && fcur[q];
    rb = re = 0;
    lv = 0.0;
    if (pres) {
      const int col_q = a.Pc[pb + q];
      const int rq = a.rowmap ? a.rowmap[col_q] : col_q;
      rb = a.Ap[rq];
      re = a.Ap[rq + 1];
      lv = cur[q];
    }
    return __ballot_sync(0xffffffffu, pres);
  };
  int base = 0, rb, re, nrb = 0, nre = 0;
  double lv, nlv = 0.0;
  unsigned todo = meta(0, rb, re, lv), ntodo = 0;
  if (m > 32) ntodo = meta(32, nrb, nre, nlv);
  // next present position: (row bounds, coefficient) broadcast from its lane
  auto next = [&](int& b, int& e, double& l) -> bool {
    while (!todo) {
      base += 32;
      if (base >= m) return false;
      todo = ntodo;
      rb = nrb;
      re = nre;
      lv = nlv;
      ntodo = 0;
      if (base + 32 < m) ntodo = meta(base + 32, nrb, nre, nlv);
    }
    const int t = __ffs(todo) - 1;
    todo &= todo - 1;
    b = __shfl_sync(0xffffffffu, rb, t);
    e = __shfl_sync(0xffffffffu, re, t);
    l = __shfl_sync(0xffffffffu, lv, t);
    return true;
  };
  auto issue = [&](PolyRowRegs<KP>& R) {
    const int len = R.e - R.b;
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const bool p = 32 * q + lane < len;
      R.c[q] = -1;
      R.v[q] = 0.0;
      ld_pred(R.c[q], a.Ac + R.b + 32 * q + lane, p);
      ld_pred(R.v[q], a.Av + R.b + 32 * q + lane, p);
    }
  };
  auto process = [&](const PolyRowRegs<KP>& R) {
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      if (R.c[q] >= 0) {
        const int p = pm.find(R.c[q]);
        if (p >= 0) {
          nxt[p] = add_rn(nxt[p], mul_rn(R.l, R.v[q]));
          fnxt[p] = 1;
        }
      }
    }
    for (int jj = R.b + 32 * KP + lane; jj < R.e; jj += 32) {
      const int p = pm.find(a.Ac[jj]);
      if (p >= 0) {
        nxt[p] = add_rn(nxt[p], mul_rn(R.l, a.Av[jj]));
        fnxt[p] = 1;
      }
    }
    __syncwarp();
  };
  PolyRowRegs<KP> A, B;
  if (!next(A.b, A.e, A.l)) return;
  issue(A);
  while (true) {
    if (!next(B.b, B.e, B.l)) {
      process(A);
      return;
    }
    issue(B);
    process(A);
    if (!next(A.b, A.e, A.l)) {
      process(B);
      return;
    }
    issue(A);
    process(B);
  }
}

template <class PM, int KP>
// KP = 8 (pattern rows of 129-511 entries): 6 CTAs per SM caps it at 85
// registers (the shared-memory limit of the class is 6 CTAs too); left free
// it took 96 and ran 5.  Polynomial phase 68.8-69.2 -> 67.1 ms on one box;
// 8 CTAs (64 registers) spills and loses (78.9 ms).
#ifndef AIRG_POLY_MINB8
#define AIRG_POLY_MINB8 6
#endif
// KP = 4 (65-128 entries): 8 CTAs per SM caps it at 63 registers (80 free),
// no spills; polynomial phase 61.7-62.4 -> 60.2-61.0 ms (7 compiles the same;
// 10 CTAs = 48 registers spills, 66.8 ms)
#ifndef AIRG_POLY_MINB4
#define AIRG_POLY_MINB4 8
#endif
// KP = 1 / 2 (<= 64 entries): the same 8-CTA cap (48-56 registers, from
// 61-76; no spills): polynomial phase 60.5 -> 59.0-59.6 ms at 2048², the DG
// problem's 0.65 -> 0.63 s
#ifndef AIRG_POLY_MINB21
#define AIRG_POLY_MINB21 8
#endif
__global__ void __launch_bounds__(128, KP == 8 ? AIRG_POLY_MINB8 : KP == 4 ? AIRG_POLY_MINB4 : AIRG_POLY_MINB21)
    poly_assemble_kernel(PolyArgs a) {
  extern __shared__ unsigned char smraw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int cap = a.cap;
  // per warp: position map, cur[cap], nxt[cap], acc[cap], flags cur/nxt/acc (3*cap bytes)
  const size_t per = PM::bytes(cap) + (size_t)cap * 24 + (size_t)cap * 3;
  unsigned char* base = smraw + (size_t)w * ((per + 15) & ~(size_t)15);
  double* cur = (double*)base;
  double* nxt = cur + cap;
  double* acc = nxt + cap;
  PM pm;
  pm.bind((unsigned char*)(acc + cap), cap);
  unsigned char* fcur = (unsigned char*)(acc + cap) + PM::bytes(cap);
  unsigned char* fnxt = fcur + cap;
  unsigned char* facc = fnxt + cap;
  for (long long r = (long long)blockIdx.x * nw + w; r < a.nrows; r += (long long)gridDim.x * nw) {
    const int row = a.rows ? a.rows[r] : (int)r;
    const int pb = a.Pp[row], pe = a.Pp[row + 1], m = pe - pb;
    if (m > cap) continue;  // handled by the global pass (flag via out_cnt = -1)
    pm.clear(a.Pc + pb, m, cap, lane, 32);
    __syncwarp();
    for (int i = lane; i < m; i += 32) {
      pm.insert(a.Pc + pb, i);
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
          const int p = pm.find(a.Ac[jj]);
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
      const int p = pm.find(a.row0 + row);
      acc[p] = add_rn(acc[p], c0);  // 0 + c0 (=c0; -0 -> +0 is pruned anyway)
      facc[p] = 1;
    }
    __syncwarp();
    if (d >= 1) {
      const double c1 = a.coef[1];
      for (int kk = a.Ap[row] + lane; kk < a.Ap[row + 1]; kk += 32) {
        const int p = pm.find(a.Ac[kk]);
        const double v = a.Av[kk];
        acc[p] = add_rn(acc[p], mul_rn(c1, v));
        facc[p] = 1;
        cur[p] = v;
        fcur[p] = 1;
      }
      __syncwarp();
    }
    for (int k = 2; k <= d; ++k) {
      // nxt = mask(cur * A): the present entries of cur in column (= position)
      // order, software-pipelined (poly_power_walk)
      poly_power_walk<PM, KP>(a, pm, pb, m, lane, cur, fcur, nxt, fnxt);
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

// Long pattern rows (cap >= 256): one CTA per row.  Same recurrence and
// summation order as poly_assemble_kernel: within a power the present
// positions q are consumed in ascending order, all threads splitting the A
// row of col_q (distinct columns -> distinct positions), a barrier between
// consecutive q.  The present positions of a power and their A-row bounds are
// staged in shared memory first, so a step issues no dependent global loads.
// Working set per CTA (block_bytes): position map, cur/nxt/acc cap doubles,
// list/rb/re cap ints, flags 3 cap bytes -- in shared memory, or for rows
// beyond it (any length, as the reference, polynomial.py:379-416) in a
// global-memory slab per CTA.  masked=1: the plain masked product, one
// barrier per left-row entry.
template <class PM>
__host__ __device__ __forceinline__ size_t block_bytes(int cap) {
  return (PM::bytes(cap) + (size_t)cap * (24 + 12 + 3) + 15) & ~(size_t)15;
}

template <class PM>
__global__ void __launch_bounds__(256) poly_assemble_block_kernel(PolyArgs a) {
  extern __shared__ unsigned char smraw[];
  __shared__ int s_np, s_cnt;
  const int tid = threadIdx.x, NT = blockDim.x;
  const int cap = a.cap;
  unsigned char* wbase = a.gmem ? a.gmem + (size_t)blockIdx.x * a.gstride : smraw;
  double* cur = (double*)wbase;
  double* nxt = cur + cap;
  double* acc = nxt + cap;
  PM pm;
  pm.bind((unsigned char*)(acc + cap), cap);
  int* list = (int*)((unsigned char*)(acc + cap) + PM::bytes(cap));
  int* rbs = list + cap;
  int* res = rbs + cap;
  unsigned char* fcur = (unsigned char*)(res + cap);
  unsigned char* fnxt = fcur + cap;
  unsigned char* facc = fnxt + cap;
  for (long long r = blockIdx.x; r < a.nrows; r += gridDim.x) {
    const int row = a.rows ? a.rows[r] : (int)r;
    const int pb = a.Pp[row], pe = a.Pp[row + 1], m = pe - pb;
    pm.clear(a.Pc + pb, m, cap, tid, NT);
    __syncthreads();
    for (int i = tid; i < m; i += NT) {
      pm.insert(a.Pc + pb, i);
      cur[i] = 0.0;
      nxt[i] = 0.0;
      acc[i] = 0.0;
      fcur[i] = 0;
      fnxt[i] = 0;
      facc[i] = 0;
    }
    __syncthreads();
    if (a.masked) {  // one masked product: left row L_i (in order), right rows A_q
      for (int qq = a.Lp[row]; qq < a.Lp[row + 1]; ++qq) {
        const int q = a.Lc[qq];
        const double lv = a.Lv[qq];
        for (int jj = a.Ap[q] + tid; jj < a.Ap[q + 1]; jj += NT) {
          const int p = pm.find(a.Ac[jj]);
          if (p >= 0) {
            nxt[p] = add_rn(nxt[p], mul_rn(lv, a.Av[jj]));
            fnxt[p] = 1;
          }
        }
        __syncthreads();
      }
      if (tid == 0) s_cnt = 0;
      __syncthreads();
      int c = 0;
      for (int i = tid; i < m; i += NT) {
        a.out_val[pb + i] = nxt[i];
        a.out_keep[pb + i] = fnxt[i];
        c += fnxt[i];
      }
      c = warp_sum(c);
      if ((tid & 31) == 0 && c) atomicAdd(&s_cnt, c);
      __syncthreads();
      if (tid == 0) a.out_cnt[row] = s_cnt;
      __syncthreads();
      continue;
    }
    const int d = a.ncoef - 1;
    if (tid == 0) {  // term 0: c0 * I (the diagonal is always in the pattern)
      const int p = pm.find(a.row0 + row);
      acc[p] = add_rn(acc[p], a.coef[0]);
      facc[p] = 1;
    }
    __syncthreads();
    if (d >= 1) {
      const double c1 = a.coef[1];
      for (int kk = a.Ap[row] + tid; kk < a.Ap[row + 1]; kk += NT) {
        const int p = pm.find(a.Ac[kk]);
        const double v = a.Av[kk];
        acc[p] = add_rn(acc[p], mul_rn(c1, v));
        facc[p] = 1;
        cur[p] = v;
        fcur[p] = 1;
      }
      __syncthreads();
    }
    for (int k = 2; k <= d; ++k) {
      // present positions in ascending order + their A-row bounds
      if (tid < 32) {
        int np = 0;
        for (int base = 0; base < m; base += 32) {
          const int q = base + tid;
          const bool pres = q < m && fcur[q];
          const unsigned bal = __ballot_sync(0xffffffffu, pres);
          if (pres) list[np + __popc(bal & ((1u << tid) - 1u))] = q;
          np += __popc(bal);
        }
        if (tid == 0) s_np = np;
      }
      __syncthreads();
      const int np = s_np;
      for (int t = tid; t < np; t += NT) {
        const int q = list[t];
        const int col_q = a.Pc[pb + q];
        const int rq = a.rowmap ? a.rowmap[col_q] : col_q;
        rbs[t] = a.Ap[rq];
        res[t] = a.Ap[rq + 1];
      }
      __syncthreads();
      for (int t = 0; t < np; ++t) {
        const double l = cur[list[t]];
        const int rb = rbs[t], re = res[t];
        for (int jj = rb + tid; jj < re; jj += NT) {
          const int p = pm.find(a.Ac[jj]);
          if (p >= 0) {
            nxt[p] = add_rn(nxt[p], mul_rn(l, a.Av[jj]));
            fnxt[p] = 1;
          }
        }
        __syncthreads();
      }
      const double ck = a.coef[k];
      for (int i = tid; i < m; i += NT) {
        if (fnxt[i]) {
          acc[i] = add_rn(acc[i], mul_rn(ck, nxt[i]));
          facc[i] = 1;
        }
        cur[i] = nxt[i];
        fcur[i] = fnxt[i];
        nxt[i] = 0.0;
        fnxt[i] = 0;
      }
      __syncthreads();
    }
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    int c = 0;
    for (int i = tid; i < m; i += NT) {
      const bool keep = d == 0 ? (bool)facc[i] : (facc[i] && acc[i] != 0.0);
      a.out_val[pb + i] = acc[i];
      a.out_keep[pb + i] = keep;
      c += keep;
    }
    c = warp_sum(c);
    if ((tid & 31) == 0 && c) atomicAdd(&s_cnt, c);
    __syncthreads();
    if (tid == 0) a.out_cnt[row] = s_cnt;
    __syncthreads();
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
  if (m > 0) max_rowlen_kernel<<<blocks_for(m, 256, num_sms() * 8), 256, 0, s>>>(m, p, d);
  AIRG_LAUNCH_CHECK();
  AIRG_CUDA(read_back(out, d, sizeof(int), s));
  release(d, s);
  return AIRG_OK;
}

// Rows are classified by pattern length (caps 32, 64, ..., next pow2 >= the
// longest row) and by column window (bitmap position map when the window is
// <= kPolySpan, hash table otherwise), and each class runs with its own
// working-set size, so a few long rows do not cut the occupancy of every row
// of the level.  Warp per row below kPolyBlockCap entries, CTA per row above;
// CTA rows whose working set exceeds the shared-memory opt-in limit run from
// global memory.
static const int kPolyBlockCap = getenv("AIRG_POLY_BLOCK_CAP") ? atoi(getenv("AIRG_POLY_BLOCK_CAP")) : 512;

// Short pattern rows (<= G entries, G lanes per row, 32 / G rows per warp):
// every power in registers.  Lane j owns pattern position j (column c_j) and
// its cur / nxt / acc values and flags; a power walks the present positions
// q in order, loads A's row of col_q G entries at a time and each lane picks
// the entry with its column (distinct columns: at most one) -- the same
// products added in the same order as the warp and CTA kernels, bitwise.
template <int G>
// occupancy cap of the register assembly classes: 5 / 6 CTAs per SM measured
// within noise of the setup; left free
#ifdef AIRG_PSMALL_MINB
#define AIRG_PSMALL_BOUNDS __launch_bounds__(256, AIRG_PSMALL_MINB)
#else
#define AIRG_PSMALL_BOUNDS __launch_bounds__(256)
#endif
__global__ void AIRG_PSMALL_BOUNDS poly_small_kernel(PolyArgs a) {
  const int lane = threadIdx.x & 31, j = lane & (G - 1), gbase = lane & ~(G - 1);
  const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << gbase;
  const long long groups = ((long long)gridDim.x * blockDim.x) / G;
  for (long long g0 = ((long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / G; g0 < a.nrows;
       g0 += groups) {  // warp-uniform trip count
    const long long r = g0 + lane / G;
    const bool live = r < a.nrows;
    const int row = live ? (a.rows ? a.rows[r] : (int)r) : 0;
    const int pb = live ? a.Pp[row] : 0, m = live ? a.Pp[row + 1] - pb : 0;
    const int cj = j < m ? a.Pc[pb + j] : INT_MAX;
    const int d = a.ncoef - 1;
    double acc = 0.0, cur = 0.0, nxt = 0.0;
    bool facc = false, fcur = false, fnxt = false;
    if (cj == a.row0 + row) {  // c0 I (the diagonal is always in the pattern)
      acc = add_rn(acc, a.coef[0]);
      facc = true;
    }
    // lane j's value in a row of A (b..e): the entry with column c_j, if any
    auto pick = [&](int b, int e, double& v) -> bool {
      bool hit = false;
      const int len = e - b;
      const int lmax = __reduce_max_sync(0xffffffffu, len);
      for (int t0 = 0; t0 < lmax; t0 += G) {
        const int t = t0 + j;
        const int ct = t < len ? __ldg(a.Ac + b + t) : -1;
        const double vt = t < len ? __ldg(a.Av + b + t) : 0.0;
#pragma unroll
        for (int i = 0; i < G; ++i) {
          const int ci = __shfl_sync(0xffffffffu, ct, i, G);
          const double vi = __shfl_sync(0xffffffffu, vt, i, G);
          if (ci == cj) {
            v = vi;
            hit = true;
          }
        }
      }
      return hit;
    };
    if (d >= 1) {
      const double c1 = a.coef[1];
      double v = 0.0;
      const int ab = live ? a.Ap[row] : 0, ae = live ? a.Ap[row + 1] : 0;
      if (pick(ab, ae, v) && cj != INT_MAX) {
        acc = add_rn(acc, mul_rn(c1, v));
        facc = true;
        cur = v;
        fcur = true;
      }
    }
    const int mmax = __reduce_max_sync(0xffffffffu, m);
    for (int k = 2; k <= d; ++k) {
      nxt = 0.0;
      fnxt = false;
      for (int q = 0; q < mmax; ++q) {  // present positions in order
        const bool pq = __shfl_sync(0xffffffffu, fcur, q, G) && q < m;
        const double lq = __shfl_sync(0xffffffffu, cur, q, G);
        const int colq = __shfl_sync(0xffffffffu, cj, q, G);
        int b = 0, e = 0;
        if (pq) {
          const int rq = a.rowmap ? a.rowmap[colq] : colq;
          b = a.Ap[rq];
          e = a.Ap[rq + 1];
        }
        double v = 0.0;
        if (pick(b, e, v) && cj != INT_MAX) {
          nxt = add_rn(nxt, mul_rn(lq, v));
          fnxt = true;
        }
      }
      if (fnxt) {
        acc = add_rn(acc, mul_rn(a.coef[k], nxt));
        facc = true;
      }
      cur = nxt;
      fcur = fnxt;
    }
    const bool keep = d == 0 ? facc : (facc && acc != 0.0);
    if (j < m) {
      a.out_val[pb + j] = acc;
      a.out_keep[pb + j] = keep;
    }
    const int c = __popc(__ballot_sync(0xffffffffu, keep && j < m) & gmask);
    if (live && j == 0) a.out_cnt[row] = c;
  }
}

// class of a pattern row: register classes for <= 8 / <= 16 entries (plain
// assembly only), else the pow2 caps x (bitmap | hash) position map; the top
// cap class takes every longer row (its cap is the level's longest row)
__global__ void poly_class_kernel(int n, const int* __restrict__ Pp, const int* __restrict__ Pc,
                                  int ncap, int reg, int* __restrict__ ids) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int b = Pp[i], m = Pp[i + 1] - b;
    if (reg && m <= 16) {
      ids[i] = 2 * ncap + (m <= 8 ? 0 : 1);
      continue;
    }
    int c = 0;
    while (c < ncap - 1 && (32 << c) < m) ++c;
    const bool bit = m == 0 || (long long)Pc[b + m - 1] - Pc[b] < kPolySpan;
    ids[i] = c + (bit ? 0 : ncap);
  }
}

// dynamic shared memory a kernel of this file may request: the device opt-in
// limit less room for the kernels' static shared variables
static int smem_optin() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
      v = 227 * 1024;
    v -= 1024;
  }
  return v;
}

template <class PM>
static int launch_poly_class(PolyArgs b, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    for (auto k : {poly_assemble_kernel<PM, 1>, poly_assemble_kernel<PM, 2>, poly_assemble_kernel<PM, 4>,
                   poly_assemble_kernel<PM, 8>})
      AIRG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin()));
    AIRG_CUDA(cudaFuncSetAttribute(poly_assemble_block_kernel<PM>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin()));
    attr = true;
  }
  const size_t per = (PM::bytes(b.cap) + (size_t)b.cap * 27 + 15) & ~(size_t)15;
  // hash-map rows (windows > kPolySpan) keep the CTA kernel from 256 entries:
  // the warp kernel's probe loops lost there (upwind DG, configs[4])
  const int block_cap = std::is_same<PM, BitPos>::value ? kPolyBlockCap : 256;
  if (b.cap < block_cap && per <= (size_t)smem_optin()) {
    int warps = 4;
    while (warps > 1 && per * warps > (size_t)smem_optin()) warps >>= 1;
    // A-row entries held per lane in the pipeline: the class's row length
    static const int kp8 = getenv("AIRG_POLY_KP8") ? atoi(getenv("AIRG_POLY_KP8")) : 1;
    auto k = b.cap <= 32 ? poly_assemble_kernel<PM, 1>
           : b.cap <= 64 ? poly_assemble_kernel<PM, 2>
           : (b.cap <= 128 || !kp8) ? poly_assemble_kernel<PM, 4> : poly_assemble_kernel<PM, 8>;
    k<<<blocks_for(b.nrows, warps, num_sms() * 32), warps * 32, per * warps, st>>>(b);
    AIRG_LAUNCH_CHECK();
    return AIRG_OK;
  }
  static const int nt128 = getenv("AIRG_POLY_NT128") ? atoi(getenv("AIRG_POLY_NT128")) : 64;
  static const int nt256 = getenv("AIRG_POLY_NT256") ? atoi(getenv("AIRG_POLY_NT256")) : 128;
  const int nt = b.cap >= 512 ? 256 : b.cap >= 256 ? nt256 : nt128;
  const size_t shm = block_bytes<PM>(b.cap);
  if (shm <= (size_t)smem_optin()) {
    poly_assemble_block_kernel<PM><<<std::min(b.nrows, num_sms() * 16), nt, shm, st>>>(b);
    AIRG_LAUNCH_CHECK();
    return AIRG_OK;
  }
  // one working set per CTA, at most ~2 GB of them
  const int grid = (int)std::max<long long>(
      1, std::min<long long>(std::min(b.nrows, num_sms() * 2), (2ll << 30) / (long long)shm));
  AIRG_TRY(scratch(&b.gmem, shm * grid, st));
  b.gstride = shm;
  poly_assemble_block_kernel<PM><<<grid, 256, 0, st>>>(b);
  AIRG_LAUNCH_CHECK();
  release(b.gmem, st);
  return AIRG_OK;
}

static int run_poly_kernel(PolyArgs& a, int maxlen, cudaStream_t s) {
  // pow2 caps 32 .. 32 << (kPolyCaps - 1); rows beyond go to the top class
  // with the longest row as its cap (global-memory working set), so any row
  // length assembles, as the reference's does (polynomial.py:379-416)
  constexpr int kPolyCaps = (kMaxCls - 2) / 2;
  int ncap = 1;
  while (ncap < kPolyCaps && (32 << (ncap - 1)) < maxlen) ++ncap;
  int* ids = nullptr;
  AIRG_TRY(scratch(&ids, a.n > 0 ? a.n : 1, s));
  const int reg = a.masked ? 0 : 1;  // register classes: plain assembly only
  if (a.n > 0)
    poly_class_kernel<<<blocks_for(a.n, 256), 256, 0, s>>>(a.n, a.Pp, a.Pc, ncap, reg, ids);
  AIRG_LAUNCH_CHECK();
  Classes cl;
  AIRG_TRY(classify_ids(a.n, ids, 2 * ncap + 2, cl, s));
  Fork fk;
  AIRG_TRY(fk.begin(s));
  for (int c = 0; c < 2 * ncap + 2; ++c) {
    const int nr = cl.count[c];
    if (!nr) continue;
    PolyArgs b = a;
    b.rows = cl.list(c);
    b.nrows = nr;
    if (c >= 2 * ncap) {
      if (c == 2 * ncap)
        poly_small_kernel<8><<<blocks_for((long long)nr * 8, 256), 256, 0, fk.stream(c)>>>(b);
      else
        poly_small_kernel<16><<<blocks_for((long long)nr * 16, 256), 256, 0, fk.stream(c)>>>(b);
      AIRG_LAUNCH_CHECK();
      continue;
    }
    b.cap = 32 << (c % ncap);
    if (c % ncap == ncap - 1) b.cap = std::max(b.cap, maxlen);
    if (c < ncap) AIRG_TRY(launch_poly_class<BitPos>(b, fk.stream(c)));
    else AIRG_TRY(launch_poly_class<HashPos>(b, fk.stream(c)));
  }
  AIRG_TRY(fk.end(s));
  release(ids, s);
  release(cl.lists, s);
  return AIRG_OK;
}

// ----------------------------------------------------------------------------
// extract / restriction assembly
// ----------------------------------------------------------------------------
// VS lanes per selected row (coalesced walk of the row, ballot compaction of
// the kept entries in column order); one group per row, no grid stride so
// every lane of a warp reaches the ballots
template <int VS>
__global__ void extract_kernel(int nr, const int* __restrict__ rows, const int* __restrict__ p,
                               const int* __restrict__ c, const double* __restrict__ v,
                               const int* __restrict__ colmap, const int* __restrict__ optr,
                               int* __restrict__ oc, double* __restrict__ ov, int* __restrict__ cnt) {
  const long long t = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / VS;
  const int lane = threadIdx.x & 31, g = lane & (VS - 1), sh = lane - g;
  const unsigned gmask = (VS == 32 ? 0xffffffffu : ((1u << VS) - 1u)) << sh;
  int b = 0, e = 0, o = 0;
  if (t < nr) {
    const int i = rows[t];
    b = p[i];
    e = p[i + 1];
    if (optr) o = optr[t];
  }
  int n = 0;
  for (int j0 = b; __any_sync(0xffffffffu, j0 < e); j0 += VS) {
    const int k = j0 + g;
    const int m = k < e ? colmap[c[k]] : -1;
    const unsigned bal = __ballot_sync(0xffffffffu, m >= 0) & gmask;
    if (m >= 0 && oc) {
      const int d = o + n + __popc(bal & ((1u << lane) - 1u));
      oc[d] = m;
      ov[d] = v[k];
    }
    n += __popc(bal);
  }
  if (cnt && g == 0 && t < nr) cnt[t] = n;
}

__global__ void colmap_kernel(int n, const signed char* __restrict__ labels, signed char want,
                              const int* __restrict__ pos, int* __restrict__ map) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    map[i] = labels[i] == want ? pos[i] : -1;
}

// R row j = [Z row j mapped through f_idx | 1 at c_idx[j]] in fine ordering:
// the unit entry goes before the first mapped column > c_idx[j] (or last).
// VS lanes per row (from the mean row length); the loads of 4 chunks are
// issued before any is used (the f_idx gather depends on the column load),
// then the chunks are placed in order, the insertion point found by ballot.
template <int VS>
__global__ void restriction_kernel(int nc, const int* __restrict__ zp, const int* __restrict__ zc,
                                   const double* __restrict__ zv, const int* __restrict__ f_idx,
                                   const int* __restrict__ c_idx, int* __restrict__ rp,
                                   int* __restrict__ rc, double* __restrict__ rv) {
  constexpr int U = 4;
  const long long j = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / VS;
  const int lane = threadIdx.x & 31, g = lane & (VS - 1), sh = lane - g;
  const unsigned gmask = (VS == 32 ? 0xffffffffu : ((1u << VS) - 1u)) << sh;
  int b = 0, e = 0, cj = 0;
  if (j < nc) {
    b = zp[j];
    e = zp[j + 1];
    cj = c_idx[j];
    if (g == 0) {
      rp[j] = (int)(b + j);
      if (j == nc - 1) rp[nc] = (int)(e + nc);
    }
  }
  const long long o = (long long)b + j;
  bool done = false;  // unit entry already placed (uniform within the group)
  for (int k0 = b; __any_sync(0xffffffffu, k0 < e); k0 += U * VS) {
    int col[U];
    double val[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int k = k0 + q * VS + g;
      col[q] = k < e ? zc[k] : -1;
      val[q] = k < e ? zv[k] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) col[q] = col[q] >= 0 ? f_idx[col[q]] : -1;
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int k = k0 + q * VS + g;
      const bool in = k < e;
      const unsigned gt = __ballot_sync(0xffffffffu, in && col[q] > cj) & gmask;
      int shift = done ? 1 : 0;
      if (!done && gt) {
        const int first = __ffs(gt) - 1;  // lane holding the first column > cj
        if (lane >= first) shift = 1;
        if (lane == first) {
          rc[o + (k - b)] = cj;
          rv[o + (k - b)] = 1.0;
        }
      }
      if (in) {
        rc[o + (k - b) + shift] = col[q];
        rv[o + (k - b) + shift] = val[q];
      }
      done = done || gt != 0;
    }
  }
  if (j < nc && !done && g == 0) {
    rc[o + (e - b)] = cj;
    rv[o + (e - b)] = 1.0;
  }
}

}  // namespace airg

using namespace airg;

extern "C" {

int airg_spgemm_masked(int m, int k, int n, const int32_t* Ap, const int32_t* Ac, const double* Av,
                       const int32_t* Bp, const int32_t* Bc, const double* Bv, const int32_t* Pp,
                       const int32_t* Pc, airg_csr_result** out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int maxlen = 0;
  AIRG_TRY(max_row_len(m, Pp, &maxlen, s));
  int pnnz = 0;
  if (m > 0) AIRG_CUDA(read_back(&pnnz, Pp + m, sizeof(int), s));
  else AIRG_CUDA(cudaStreamSynchronize(s));
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

static int poly_assemble_impl(int n, const int32_t* Ap, const int32_t* Ac, const double* Av,
                              int ncoef, const double* coef_h, const int32_t* Qp,
                              const int32_t* Qc, int row0, const int32_t* rowmap,
                              airg_csr_result** out, cudaStream_t s);

int airg_poly_assemble(int n, const int32_t* Ap, const int32_t* Ac, const double* Av, int ncoef,
                       const double* coef_h, const int32_t* Qp, const int32_t* Qc,
                       airg_csr_result** out, void* stream) {
  return poly_assemble_impl(n, Ap, Ac, Av, ncoef, coef_h, Qp, Qc, 0, nullptr, out,
                            (cudaStream_t)stream);
}

// Row-strip assembly: rows [0, n) of Ap are the local rows (global row
// row0 + i), further rows are fetched ghost rows; column ids are global and
// rowmap[global column] gives the row of Ap holding it.
int airg_poly_assemble_ex(int n, int row0, const int32_t* Ap, const int32_t* Ac, const double* Av,
                          const int32_t* rowmap, int ncoef, const double* coef_h,
                          const int32_t* Qp, const int32_t* Qc, airg_csr_result** out,
                          void* stream) {
  return poly_assemble_impl(n, Ap, Ac, Av, ncoef, coef_h, Qp, Qc, row0, rowmap, out,
                            (cudaStream_t)stream);
}

}  // extern "C"

static int poly_assemble_impl(int n, const int32_t* Ap, const int32_t* Ac, const double* Av,
                              int ncoef, const double* coef_h, const int32_t* Qp,
                              const int32_t* Qc, int row0, const int32_t* rowmap,
                              airg_csr_result** out, cudaStream_t s) {
  if (ncoef < 1) {
    set_error("need at least one coefficient");
    return AIRG_ERR_VALUE;
  }
  if (!Qp) {  // the mask comes from the base matrix itself (arnoldi_coeff kind)
    Qp = Ap;
    Qc = Ac;
  }
  int *cnt = nullptr, *Pp = nullptr, *Pc = nullptr;
  AIRG_TRY(scratch(&cnt, n + 1, s));
  AIRG_TRY(scratch(&Pp, n + 1, s));
  const int nb = blocks_for(n, 256);
  if (n > 0) pattern_diag_kernel<<<nb, 256, 0, s>>>(n, Qp, Qc, nullptr, nullptr, cnt, row0);
  long long pnnz = 0;
  AIRG_TRY(scan_counts(cnt, Pp, n, &pnnz, s));
  AIRG_TRY(scratch(&Pc, pnnz, s));
  if (n > 0) pattern_diag_kernel<<<nb, 256, 0, s>>>(n, Qp, Qc, Pp, Pc, nullptr, row0);
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
  a.row0 = row0;
  a.rowmap = rowmap;
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

extern "C" {

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
  if (m > 0) AIRG_CUDA(read_back(&nnz, p + m, sizeof(int), s));
  else AIRG_CUDA(cudaStreamSynchronize(s));
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
  AIRG_CUDA(read_back(&ad, anyd, sizeof(int), s));
  if (changed_h) *changed_h = ad;
  for (void* q : {(void*)rcol, (void*)rval, (void*)cnt, (void*)anyd}) release(q, s);
  return AIRG_OK;
}

int airg_extract_ex(int nr_sel, const int32_t* rows, const int32_t* p, const int32_t* c,
                    const double* v, const int32_t* colmap, int ncols_sel, double mean_len,
                    airg_csr_result** out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  airg_csr_result* r = new_result(nr_sel, ncols_sel, s);
  int* cnt = nullptr;
  AIRG_TRY(scratch(&cnt, nr_sel + 1, s));
  // lanes per row: ~2-4 entries per lane and round (8 without a hint)
  const int vs = mean_len <= 0 ? 8 : mean_len <= 12 ? 4 : mean_len <= 48 ? 8 : mean_len <= 96 ? 16 : 32;
  const int nb = (int)(((long long)nr_sel * vs + 255) / 256);
  auto launch = [&](const int* optr, int* oc, double* ov, int* cn) {
    switch (vs) {
      case 4: extract_kernel<4><<<nb, 256, 0, s>>>(nr_sel, rows, p, c, v, colmap, optr, oc, ov, cn); break;
      case 16: extract_kernel<16><<<nb, 256, 0, s>>>(nr_sel, rows, p, c, v, colmap, optr, oc, ov, cn); break;
      case 32: extract_kernel<32><<<nb, 256, 0, s>>>(nr_sel, rows, p, c, v, colmap, optr, oc, ov, cn); break;
      default: extract_kernel<8><<<nb, 256, 0, s>>>(nr_sel, rows, p, c, v, colmap, optr, oc, ov, cn);
    }
  };
  if (nr_sel > 0) launch(nullptr, nullptr, nullptr, cnt);
  long long nnz = 0;
  AIRG_TRY(scan_counts(cnt, r->ptr, nr_sel, &nnz, s));
  AIRG_TRY(result_alloc_entries(r, nnz, true));
  if (nr_sel > 0) launch(r->ptr, r->col, r->val, nullptr);
  AIRG_LAUNCH_CHECK();
  release(cnt, s);
  *out = r;
  return AIRG_OK;
}

int airg_extract(int nr_sel, const int32_t* rows, const int32_t* p, const int32_t* c,
                 const double* v, const int32_t* colmap, int ncols_sel, airg_csr_result** out,
                 void* stream) {
  return airg_extract_ex(nr_sel, rows, p, c, v, colmap, ncols_sel, 0.0, out, stream);
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
  if (nc > 0) AIRG_CUDA(read_back(&znnz, zp + nc, sizeof(int), s));
  else AIRG_CUDA(cudaStreamSynchronize(s));
  airg_csr_result* r = new_result(nc, n, s);
  AIRG_TRY(result_alloc_entries(r, (long long)znnz + nc, true));
  const double mean = nc > 0 ? (double)znnz / nc : 0.0;  // lanes per row: 4 entries per lane
  if (nc > 0 && mean > 64)
    restriction_kernel<32><<<(int)(((long long)nc * 32 + 255) / 256), 256, 0, s>>>(
        nc, zp, zc, zv, f_idx, c_idx, r->ptr, r->col, r->val);
  else if (nc > 0 && mean > 16)
    restriction_kernel<8><<<(int)(((long long)nc * 8 + 255) / 256), 256, 0, s>>>(
        nc, zp, zc, zv, f_idx, c_idx, r->ptr, r->col, r->val);
  else if (nc > 0)
    restriction_kernel<2><<<(int)(((long long)nc * 2 + 255) / 256), 256, 0, s>>>(
        nc, zp, zc, zv, f_idx, c_idx, r->ptr, r->col, r->val);
  else
    AIRG_CUDA(cudaMemsetAsync(r->ptr, 0, sizeof(int), s));
  AIRG_LAUNCH_CHECK();
  *out = r;
  return AIRG_OK;
}

}  // extern "C"
