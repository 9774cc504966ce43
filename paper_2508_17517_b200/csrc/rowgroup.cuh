// Row kernels with VS lanes per row shared by the serial and the row-strip
// CF splitting (split.cu, dist_kernels.cu): coalesced row walks, ballot
// compaction, order-preserving sums.  ref: splitting.py:86-109, 162-207
#pragma once
#include "setup_common.cuh"

namespace airg {

// VS lanes per row (one group per row, no grid stride: every lane of a warp
// reaches the shuffles and ballots)
#define AIRG_GROUP(VS)                                                              \
  const int lane = threadIdx.x & 31, g = lane & (VS - 1), sh = lane - g;           \
  const unsigned gmask = (VS == 32 ? 0xffffffffu : ((1u << VS) - 1u)) << sh;       \
  (void)gmask

// strong couplings of row i (diagonal = column row0 + i)
template <int VS>
__global__ void strength_count_kernel(int n, int row0, const int* __restrict__ ptr,
                                      const int* __restrict__ col, const double* __restrict__ val,
                                      double theta, unsigned char* __restrict__ keep,
                                      int* __restrict__ cnt) {
  AIRG_GROUP(VS);
  const long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / VS;
  const long long gi = row0 + i;
  int b = 0, e = 0;
  if (i < n) {
    b = ptr[i];
    e = ptr[i + 1];
  }
  double mx = 0.0;  // max is order-free: lanes stride the row, then reduce
  for (int k = b + g; k < e; k += VS)
    if (col[k] != gi) mx = fmax(mx, fabs(val[k]));
#pragma unroll
  for (int o = VS / 2; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const double thr = mul_rn(theta, mx);
  int c = 0;
  for (int k0 = b; __any_sync(0xffffffffu, k0 < e); k0 += VS) {
    const int k = k0 + g;
    bool st = false;
    if (k < e) {
      const double v = val[k];
      st = col[k] != gi && v != 0.0 && fabs(v) >= thr;
      keep[k] = st;
    }
    c += __popc(__ballot_sync(0xffffffffu, st) & gmask);
  }
  if (i < n && g == 0) cnt[i] = c;
}

template <int VS>
__global__ void compact_cols_kernel(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                    const unsigned char* __restrict__ keep,
                                    const int* __restrict__ optr, int* __restrict__ ocol) {
  AIRG_GROUP(VS);
  const long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / VS;
  int b = 0, e = 0, o = 0;
  if (i < n) {
    b = ptr[i];
    e = ptr[i + 1];
    o = optr[i];
  }
  for (int k0 = b; __any_sync(0xffffffffu, k0 < e); k0 += VS) {
    const int k = k0 + g;
    const bool kp = k < e && keep[k];
    const unsigned bal = __ballot_sync(0xffffffffu, kp) & gmask;
    if (kp) ocol[o + __popc(bal & ((1u << lane) - 1u))] = col[k];
    o += __popc(bal);
  }
}

static inline int group_blocks(long long n, int vs) { return (int)((n * vs + 255) / 256); }

// VS lanes load a row chunk coalesced; the group's first lane adds the
// off-diagonal F entries in entry order (bincount's sequential sum)
// (bad records the global row row0 + i of a zero diagonal)
template <int VS>
__global__ void ddc_ratio_kernel(int nf, int row0, const int* __restrict__ f_idx, const int* __restrict__ ptr,
                                 const int* __restrict__ col, const double* __restrict__ val,
                                 const signed char* __restrict__ labels, double* __restrict__ ratio,
                                 int* __restrict__ bad) {
  AIRG_GROUP(VS);
  const long long t = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / VS;
  int i = 0, b = 0, e = 0;
  if (t < nf) {
    i = f_idx[t];
    b = ptr[i];
    e = ptr[i + 1];
  }
  double sum = 0.0, d = 0.0;
  for (int k0 = b; __any_sync(0xffffffffu, k0 < e); k0 += VS) {
    const int k = k0 + g;
    bool off = false, dia = false;
    double a = 0.0;
    if (k < e) {
      const int j = col[k];
      if (labels[j] == 0) {
        a = val[k];
        dia = j == i;
        off = !dia;
      }
    }
    const unsigned bo = __ballot_sync(0xffffffffu, off) & gmask;
    const unsigned bd = __ballot_sync(0xffffffffu, dia) & gmask;
    if (bd) d = __shfl_sync(0xffffffffu, a, __ffs(bd) - 1);
    else __shfl_sync(0xffffffffu, a, lane);  // keep every lane in the shuffle
    const double fa = fabs(a);
#pragma unroll
    for (int q = 0; q < VS; ++q) {
      const double x = __shfl_sync(0xffffffffu, fa, sh + q);
      if ((bo >> (sh + q)) & 1u) sum = add_rn(sum, x);
    }
  }
  if (t < nf && g == 0) {
    if (d == 0.0) atomicMin(bad, row0 + i);
    ratio[t] = __ddiv_rn(sum, fabs(d));
  }
}

}  // namespace airg
