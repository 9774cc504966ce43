// Span-indexed SpGEMM rows (the dense levels of R (A P) and Z = -A_cf Ahat).
//
// The output columns of one row of these products lie in a bounded window
// [cmin, cmax] (the coarse points are numbered in fine-grid order, so a row's
// stencil covers a few grid rows: span <= ~15k columns at every level of the
// 2048^2 hierarchy, tools/spgemm_stats.py), but only 2-10 % of the window is
// occupied.  So instead of hashing every product twice (count, then
// numeric), a row is handled through a BITMAP of its window:
//
//   count   (CTA per row): one byte flag per window column in shared memory,
//           set by plain byte stores (no atomics, no probing; warps take
//           chunks of the A row from a shared cursor); a sweep packs the
//           flags into 32-bit bitmap words, written to global scratch, and
//           their popcount is the row length.
//   numeric (warp per row): the bitmap is loaded back with an exclusive
//           popcount prefix per word; the output position of column c is
//           prefix[w] + popc(bits[w] & below(c)) -- a rank, not a search.
//           Accumulators are indexed by that rank, i.e. already in column
//           order: no compaction and no sort at the end of the row.
//
// Summation order is the one of spgemm_core.cuh (A row in order, lanes
// split ONE B row, __syncwarp between B rows): every output entry receives
// its k in ascending order with separate mul/add roundings, so the result is
// bitwise scipy's csr_matmat (sparse.py:222-240), structural zeros included
// (the structure comes from the flags, not from the values).
#pragma once
#include "spgemm_core.cuh"

namespace airg {

constexpr int kSpanMax = 65536;              // window columns handled here (the 4096^2
                                             // hierarchy's windows reach ~30k)
constexpr int kSpanWords = kSpanMax / 32;    // bitmap words per row (max)
constexpr int kSpanNmax = 4096;              // longest output row handled here

// bytes b0..b3 in {0,1} of x -> bits 0..3 (no carries: the partial products
// land on distinct bit positions)
__device__ __forceinline__ unsigned flag_nibble(unsigned x) { return (x * 0x10204080u) >> 28; }

// rank of window offset `off` in the bitmap (prefix, bits) pairs
__device__ __forceinline__ int span_rank(const uint2* bm, unsigned off) {
  const uint2 e = bm[off >> 5];
  return (int)e.x + __popc(e.y & ((1u << (off & 31u)) - 1u));
}

// Per row: product upper bound, window [cmin, cmax] and bitmap words (0 when
// the row is not handled by the span path: few products, a window beyond
// kSpanMax, a window much wider than the products, or B rows averaging
// fewer than 8 entries, where the per-step work of the span walk does not pay).
template <int VS>
__global__ void span_ub_kernel(int m, const int* __restrict__ Ap, const int* __restrict__ Ac,
                               const int* __restrict__ Bp, const int* __restrict__ Bc,
                               long long* __restrict__ ub, int* __restrict__ cmin_out,
                               long long* __restrict__ words, int span_min_ub,
                               unsigned long long* __restrict__ totals) {
  const int sub = threadIdx.x & (VS - 1);
  const unsigned gmask = VS == 32 ? 0xffffffffu : (((1u << VS) - 1u) << (threadIdx.x & 31 & ~(VS - 1)));
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / VS; r < m;
       r += ((long long)gridDim.x * blockDim.x) / VS) {
    long long s = 0;
    int mn = 0x7fffffff, mx = -1;
    const int ab = Ap[r], ae = Ap[r + 1];
    for (int kk = ab + sub; kk < ae; kk += VS) {
      const int k = Ac[kk];
      const int b = Bp[k], e = Bp[k + 1];
      if (e > b) {
        s += e - b;
        mn = min(mn, Bc[b]);
        mx = max(mx, Bc[e - 1]);
      }
    }
#pragma unroll
    for (int o = VS / 2; o > 0; o >>= 1) {
      s += __shfl_xor_sync(gmask, s, o);
      mn = min(mn, __shfl_xor_sync(gmask, mn, o));
      mx = max(mx, __shfl_xor_sync(gmask, mx, o));
    }
    if (sub == 0) {
      ub[r] = s;
      cmin_out[r] = mn;
      const long long span = (long long)mx - mn + 1;
      const bool use = s >= span_min_ub && span > 0 && span <= kSpanMax && span <= 32 * s &&
                       s >= 8ll * (ae - ab);
      words[r] = use ? (span + 31) / 32 : 0;
      if (use) {  // products and steps of the span rows (B-row prefetch shape), widest window
        atomicAdd(totals, (unsigned long long)s);
        atomicAdd(totals + 1, (unsigned long long)(ae - ab));
        atomicMax(totals + 2, (unsigned long long)((span + 31) / 32));
      }
    }
  }
}

struct SpanCountArgs {
  const int *Ap, *Ac, *Bp, *Bc;
  const int* rows;
  int nrows;
  const int* cmin;
  const long long* words;   // bitmap words per row
  const long long* bmoff;   // offset of the row's bitmap in gbm
  unsigned* gbm;
  int* cnt;
};

// Count pass: one CTA (NT threads) per row sharing kSpanMax byte flags.
// Counting has no order constraint, so warps take chunks of kSpanChunk A
// entries from a shared cursor (the B rows behind the entries vary in length).
constexpr int kSpanChunk = 8;
template <int NT>
__global__ void __launch_bounds__(NT) span_count_kernel(SpanCountArgs a) {
  extern __shared__ uint4 span_flags4[];
  __shared__ int cursor, total;
  unsigned char* flags = (unsigned char*)span_flags4;
  const int tid = threadIdx.x, lane = tid & 31;
  for (long long t = blockIdx.x; t < a.nrows; t += gridDim.x) {
    const int row = a.rows[t];
    const int cmin = a.cmin[row];
    const int nw = (int)a.words[row];
    const int ab = a.Ap[row], ae = a.Ap[row + 1];
    for (int i = tid; i < 2 * nw; i += NT) span_flags4[i] = make_uint4(0u, 0u, 0u, 0u);
    if (tid == 0) {
      cursor = ab;
      total = 0;
    }
    __syncthreads();
    while (true) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&cursor, kSpanChunk);
      base = __shfl_sync(kFull, base, 0);
      if (base >= ae) break;
      int bb = 0, be = 0;
      if (lane < kSpanChunk && base + lane < ae) {
        const int k = a.Ac[base + lane];
        bb = a.Bp[k];
        be = a.Bp[k + 1];
      }
      const int cnt = min(kSpanChunk, ae - base);
      int cb = __shfl_sync(kFull, bb, 0), ce = __shfl_sync(kFull, be, 0);
      int p0 = cb + lane < ce ? a.Bc[cb + lane] : -1;
      int p1 = cb + 32 + lane < ce ? a.Bc[cb + 32 + lane] : -1;
      for (int tt = 0; tt < cnt; ++tt) {
        const int tb = cb, te = ce, c0 = p0, c1 = p1;
        if (tt + 1 < cnt) {  // next B row's head (64 entries) one step ahead
          cb = __shfl_sync(kFull, bb, tt + 1);
          ce = __shfl_sync(kFull, be, tt + 1);
          p0 = cb + lane < ce ? a.Bc[cb + lane] : -1;
          p1 = cb + 32 + lane < ce ? a.Bc[cb + 32 + lane] : -1;
        }
        if (c0 >= 0) flags[c0 - cmin] = 1;
        if (c1 >= 0) flags[c1 - cmin] = 1;
        for (int jb = tb + 64; jb < te; jb += 96) {
          int cc[3];
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const int jj = jb + 32 * q + lane;
            cc[q] = jj < te ? a.Bc[jj] : -1;
          }
#pragma unroll
          for (int q = 0; q < 3; ++q)
            if (cc[q] >= 0) flags[cc[q] - cmin] = 1;
        }
      }
    }
    __syncthreads();
    // pack 32 flags per bitmap word
    unsigned* out = a.gbm + a.bmoff[row];
    int n = 0;
    for (int i = tid; i < nw; i += NT) {
      const uint4 x0 = span_flags4[2 * i], x1 = span_flags4[2 * i + 1];
      const unsigned bits = flag_nibble(x0.x) | flag_nibble(x0.y) << 4 | flag_nibble(x0.z) << 8 |
                            flag_nibble(x0.w) << 12 | flag_nibble(x1.x) << 16 |
                            flag_nibble(x1.y) << 20 | flag_nibble(x1.z) << 24 | flag_nibble(x1.w) << 28;
      out[i] = bits;
      n += __popc(bits);
    }
    n = warp_sum(n);
    if (lane == 0 && n) atomicAdd(&total, n);
    __syncthreads();
    if (tid == 0) a.cnt[row] = total;
  }
}

// Numeric walk of one row through the bitmap rank, software-pipelined: the B
// rows of the next D steps are held in registers (KP x 32 entries each;
// longer B rows load their tail in place), so a step does not wait for its
// own loads (L2, ~250+ cycles) -- the kernel is occupancy-limited by shared
// memory, so the registers are free.  Per step the KP x 32 entries are first
// ranked, then all accumulators are loaded, then all updated and stored: the
// entries of one B row are distinct columns, so within a lane the
// read-modify-writes never alias and their latency chains overlap.  Lanes
// without an entry update the dummy slot acc[n] (never output).
template <int KP, int D>
__device__ __forceinline__ void span_walk_numeric(const int* __restrict__ Ap, const int* __restrict__ Ac,
                                                  const double* __restrict__ Av,
                                                  const int* __restrict__ Bp, const int* Bc,
                                                  const double* Bv, int row, int lane,
                                                  const uint2* bm, double* acc, int cmin, int n) {
  const int ab = Ap[row], S = Ap[row + 1] - ab;
  if (S <= 0) return;
  // 32-entry chunk metadata at the issue pointer (i*) and of the next chunk (n*)
  int ic = 0, ibb = 0, ibe = 0, nbb = 0, nbe = 0;
  double iav = 0.0, nav = 0.0;
  if (lane < S) {
    const int k = Ac[ab + lane];
    iav = Av[ab + lane];
    ibb = Bp[k];
    ibe = Bp[k + 1];
  }
  if (32 + lane < S) {
    const int k = Ac[ab + 32 + lane];
    nav = Av[ab + 32 + lane];
    nbb = Bp[k];
    nbe = Bp[k + 1];
  }
  // keep the B base pointers in registers (otherwise they are re-read from
  // the parameter bank every step, and the move of a just-loaded pointer
  // stalls like a global load)
  asm volatile("" : "+l"(Bc), "+l"(Bv));
  int col[D][KP];
  double val[D][KP];
  int rb[D], re[D];
  double ra[D];
  // issue() is branch-free around the buffer registers (predicated loads
  // only): a branch merging a buffer's old value with a pending load makes
  // the compiler insert register moves that wait for the load, which
  // serialises the pipeline.  Steps past the row issue nothing (len 0).
  auto issue = [&](int s, int& b, int& e, double& a, int* cc, double* vv) {
    const bool live = s < S;
    if (live && (s >> 5) != ic) {  // warp-uniform: the issue pointer enters the next chunk
      ++ic;
      ibb = nbb;
      ibe = nbe;
      iav = nav;
      nbb = nbe = 0;
      nav = 0.0;
      const int k2 = (ic + 1) * 32 + lane;
      if (k2 < S) {
        const int k = Ac[ab + k2];
        nav = Av[ab + k2];
        nbb = Bp[k];
        nbe = Bp[k + 1];
      }
    }
    const int ln = s & 31;
    b = __shfl_sync(kFull, ibb, ln);
    e = __shfl_sync(kFull, ibe, ln);
    a = __shfl_sync(kFull, iav, ln);
    e = live ? e : b;
    const int len = e - b;
    const int* pc = Bc + b + lane;
    const double* pv = Bv + b + lane;
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const bool p = 32 * q + lane < len;
      cc[q] = -1;
      vv[q] = 0.0;
      ld_pred(cc[q], pc + 32 * q, p);
      ld_pred(vv[q], pv + 32 * q, p);
    }
    // entries beyond KP x 32: pull their lines into L1 now (one line per
    // lane; columns 32 per line, values 16 per line)
    if (len > 32 * KP) {  // warp-uniform
      for (int j = 32 * KP + 32 * lane; j < len; j += 32 * 32)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(Bc + b + j));
      for (int j = 32 * KP + 16 * lane; j < len; j += 16 * 32)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(Bv + b + j));
    }
  };
#pragma unroll
  for (int d = 0; d < D; ++d) issue(d, rb[d], re[d], ra[d], col[d], val[d]);
  for (int s0 = 0; s0 < S; s0 += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int s = s0 + d;
      if (s < S) {
        const double a = ra[d];
        const int len = re[d] - rb[d];
        int pos[KP];
        double x[KP];
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          if (32 * q < len) {
            const int c = col[d][q];
            pos[q] = c >= 0 ? span_rank(bm, (unsigned)(c - cmin)) : n;
          }
        }
#pragma unroll
        for (int q = 0; q < KP; ++q)
          if (32 * q < len) x[q] = acc[pos[q]];
#pragma unroll
        for (int q = 0; q < KP; ++q)
          if (32 * q < len) acc[pos[q]] = add_rn(x[q], mul_rn(a, val[d][q]));
        for (int jj = rb[d] + 32 * KP + lane; jj < re[d]; jj += 32) {  // long B rows
          const int p = span_rank(bm, (unsigned)(Bc[jj] - cmin));
          acc[p] = add_rn(acc[p], mul_rn(a, Bv[jj]));
        }
        __syncwarp();
        issue(s + D, rb[d], re[d], ra[d], col[d], val[d]);
      }
    }
  }
}

struct SpanNumArgs {
  const int *Ap, *Ac;
  const double* Av;
  const int *Bp, *Bc;
  const double* Bv;
  const int* rows;
  int nrows;
  int ncap;  // longest output row of this launch (sizes the accumulators)
  int wcap;  // widest window of this product in bitmap words (sizes the bitmap)
  const int* cmin;
  const long long* words;
  const long long* bmoff;
  const unsigned* gbm;
  const int* Cp;
  int* Cc;
  double* Cv;
  int negate;
  int mode;  // 0 plain, 1 fused drop/lump into raw offsets (Cp[row] + row)
  double tol;
  int lump;
  int* out_cnt;
  int* any_drop;
  int row0;
};

// shared memory per warp of the numeric kernel: bitmap (prefix, bits) pairs,
// ncap + 1 accumulators (the last one the dummy slot), the drop mask
__host__ __device__ __forceinline__ size_t span_num_bytes(int ncap, int wcap) {
  return ((size_t)wcap * sizeof(uint2) + (size_t)(ncap + 2) * sizeof(double) +
          (size_t)(ncap / 32 + 1) * sizeof(unsigned) + 15) & ~(size_t)15;
}

// drop_and_lump (sparse.py:307-352) of one accumulated row, positions in
// column order, column of a position from the bitmap.  keep = diagonal |
// |v| >= tol * max|v|; the dropped values are summed sequentially in column
// order (lane 0, from the drop mask) and added to the diagonal, which is
// inserted when absent and the sum is nonzero.  Same rule and order as
// drop_lump_row (spgemm_core.cuh).  Returns the number of entries written.
__device__ __forceinline__ int span_drop_lump_row(const uint2* bm, int nw, const double* acc, int n,
                                                  int cmin, int row, double tol, int lump,
                                                  unsigned* dmask, int* __restrict__ out_col,
                                                  double* __restrict__ out_val, long long o, int lane,
                                                  int* any_drop) {
  double mx = 0.0;
  for (int i = lane; i < n; i += 32) mx = fmax(mx, fabs(acc[i]));
  mx = warp_max(mx);
  int dpos = -1;
  {
    const long long off = (long long)row - cmin;
    if (off >= 0 && off < 32ll * nw) {
      const uint2 e = bm[off >> 5];
      if (e.y >> (off & 31) & 1u) dpos = span_rank(bm, (unsigned)off);
    }
  }
  const double thr = mul_rn(tol, mx);
  int ndrop = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const bool d = i < n && i != dpos && !(fabs(acc[i]) >= thr);
    const unsigned bal = __ballot_sync(kFull, d);
    if (lane == 0) dmask[base >> 5] = bal;
    ndrop += __popc(bal);
  }
  __syncwarp();
  double lumped = 0.0;
  if (lane == 0 && ndrop) {
    for (int wd = 0; wd < (n + 31) >> 5; ++wd) {
      unsigned m = dmask[wd];
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1u;
        lumped = add_rn(lumped, acc[wd * 32 + b]);
      }
    }
    if (any_drop) atomicOr(any_drop, 1);
  }
  lumped = __shfl_sync(kFull, lumped, 0);
  const bool insert = lump && ndrop > 0 && dpos < 0 && lumped != 0.0;
  // kept entries, walked by bitmap word (lane = word): count, scan, write
  int written = 0, before = 0;
  for (int b0 = 0; b0 < nw; b0 += 32) {
    const int i = b0 + lane;
    const uint2 e = i < nw ? bm[i] : make_uint2(0u, 0u);
    int kc = 0, kb = 0;
    {
      unsigned bits = e.y;
      int p = (int)e.x;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1u;
        const int pi = p++;
        const bool d = (dmask[pi >> 5] >> (pi & 31)) & 1u;
        if (!d) {
          ++kc;
          if (cmin + i * 32 + b < row) ++kb;
        }
      }
    }
    int inc = kc;
#pragma unroll
    for (int sh = 1; sh < 32; sh <<= 1) {
      const int y = __shfl_up_sync(kFull, inc, sh);
      if (lane >= sh) inc += y;
    }
    int q = written + inc - kc;
    {
      unsigned bits = e.y;
      int p = (int)e.x;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1u;
        const int pi = p++;
        if ((dmask[pi >> 5] >> (pi & 31)) & 1u) continue;
        const int cc = cmin + i * 32 + b;
        double x = acc[pi];
        if (pi == dpos && lump && ndrop > 0) x = add_rn(x, lumped);
        const int dst = q + (insert && cc > row ? 1 : 0);
        out_col[o + dst] = cc;
        out_val[o + dst] = x;
        ++q;
      }
    }
    written += __shfl_sync(kFull, inc, 31);
    before += warp_sum(kb);
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

// Numeric pass: warp per row, output length <= a.ncap (runtime: one kernel,
// any class granularity; NW warps per CTA).
template <int NW, int KP, int D>
// Occupancy: 8 CTAs of two warps per SM caps the kernel at 128 registers
// (16 warps/SM); left free it took more and ran 12 warps/SM.  Measured on
// the 2048^2 products of levels 4-9 (tools/span_micro.py): 104.5 -> 93.0 ms
// despite a small spill of the deep-prefetch variant; capping harder (20 or
// 32 warps/SM) spills more and measured 126-200 ms.
#ifndef AIRG_SPAN_MINB
#define AIRG_SPAN_MINB 8
#endif
__global__ void __launch_bounds__(32 * NW, (AIRG_SPAN_MINB * 2 / NW) > 0 ? (AIRG_SPAN_MINB * 2 / NW) : 1) span_numeric_kernel(SpanNumArgs a) {
  extern __shared__ uint4 span_smem4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* base = (unsigned char*)span_smem4 + (size_t)w * span_num_bytes(a.ncap, a.wcap);
  uint2* bm = (uint2*)base;
  double* acc = (double*)(base + (size_t)a.wcap * sizeof(uint2));
  unsigned* dm = (unsigned*)(acc + a.ncap + 2);
  for (long long t = (long long)blockIdx.x * NW + w; t < a.nrows; t += (long long)gridDim.x * NW) {
    const int row = a.rows[t];
    const int cmin = a.cmin[row];
    const int nw = (int)a.words[row];
    const unsigned* g = a.gbm + a.bmoff[row];
    // bitmap + exclusive popcount prefix
    int run = 0;
    for (int b0 = 0; b0 < nw; b0 += 32) {
      const int i = b0 + lane;
      const unsigned bits = i < nw ? g[i] : 0u;
      const int c = __popc(bits);
      int inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
      }
      if (i < nw) bm[i] = make_uint2((unsigned)(run + inc - c), bits);
      run += __shfl_sync(kFull, inc, 31);
    }
    const int n = run;
    for (int i = lane; i <= n; i += 32) acc[i] = 0.0;
    __syncwarp();
    span_walk_numeric<KP, D>(a.Ap, a.Ac, a.Av, a.Bp, a.Bc, a.Bv, row, lane, bm, acc, cmin,
                                       n);
    if (a.mode == 0) {
      const int o = a.Cp[row];
      for (int i = lane; i < n; i += 32) {
        const double v = acc[i];
        a.Cv[o + i] = a.negate ? -v : v;
      }
      for (int i = lane; i < nw; i += 32) {  // columns, by bitmap word
        const uint2 e = bm[i];
        unsigned bits = e.y;
        int p = o + (int)e.x;
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1u;
          a.Cc[p++] = cmin + i * 32 + b;
        }
      }
    } else {
      const int wr = span_drop_lump_row(bm, nw, acc, n, cmin, a.row0 + row, a.tol, a.lump, dm, a.Cc,
                                        a.Cv, (long long)a.Cp[row] + row, lane, a.any_drop);
      if (lane == 0) a.out_cnt[row] = wr;
    }
    __syncwarp();
  }
}

}  // namespace airg
