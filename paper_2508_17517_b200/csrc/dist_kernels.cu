// Row-strip (domain-decomposed) variants of the setup kernels.  A rank owns
// global rows [row0, row0 + n_loc); its matrices keep local rows with column
// ids either GLOBAL or renumbered to the extended space [local | ghost]
// (ext id i < n_loc <=> global row0 + i).  Everything else reuses the serial
// kernels on ext-renumbered arrays.  Semantics are the serial ones row by row,
// so a distributed hierarchy equals the serial one bit for bit.
// ref: splitting.py:86-207, problems.py:48-85
#include "setup_common.cuh"
#include "rowgroup.cuh"
#include <vector>

namespace airg {

// rows [r0, r1) of the 2-D upwind stencil, ptr relative to r0
__global__ void advection_rows_kernel(int nx, long long r0, long long r1, double vx, double vy,
                                      long long base, int* __restrict__ ptr, int* __restrict__ col,
                                      double* __restrict__ val) {
  const double dg = add_rn(vx, vy);
  for (long long idx = r0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < r1;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx % nx, j = idx / nx;
    long long before = idx;
    if (vx > 0) before += j * (nx - 1) + (i > 0 ? i - 1 : 0);
    if (vy > 0) before += idx - nx > 0 ? idx - nx : 0;
    long long k = before - base;
    ptr[idx - r0] = (int)k;
    if (vy > 0 && j > 0) {
      col[k] = (int)(idx - nx);
      val[k] = -vy;
      ++k;
    }
    if (vx > 0 && i > 0) {
      col[k] = (int)(idx - 1);
      val[k] = -vx;
      ++k;
    }
    col[k] = (int)idx;
    val[k] = dg;
    ++k;
    if (idx == r1 - 1) ptr[r1 - r0] = (int)k;
  }
}

static long long stencil_before(long long idx, int nx, double vx, double vy) {
  const long long i = idx % nx, j = idx / nx;
  long long before = idx;
  if (vx > 0) before += j * (nx - 1) + (i > 0 ? i - 1 : 0);
  if (vy > 0) before += idx - nx > 0 ? idx - nx : 0;
  return before;
}

__global__ void union_sorted_rows_kernel(int n, const int* __restrict__ ap, const int* __restrict__ ac,
                                         const int* __restrict__ bp, const int* __restrict__ bc,
                                         const int* __restrict__ optr, int* __restrict__ ocol,
                                         int* __restrict__ cnt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int x = ap[i], xe = ap[i + 1], y = bp[i], ye = bp[i + 1];
    int o = optr ? optr[i] : 0, c = 0;
    while (x < xe || y < ye) {
      int v;
      if (y >= ye || (x < xe && ac[x] < bc[y])) v = ac[x++];
      else if (x >= xe || bc[y] < ac[x]) v = bc[y++];
      else {
        v = ac[x++];
        ++y;
      }
      if (ocol) ocol[o + c] = v;
      ++c;
    }
    if (cnt) cnt[i] = c;
  }
}

__global__ void luby_weights_rows_kernel(int n, long long row0, const int* __restrict__ ptr, u128 s0,
                                         u128 inc, double* __restrict__ w) {
  // chunked jump-ahead to the global position of each local row
  const long long chunk = 64;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long i0 = t * chunk;
  if (i0 >= n) return;
  const long long i1 = i0 + chunk < n ? i0 + chunk : n;
  u128 st = pcg_jump(s0, inc, (unsigned long long)(row0 + i0));
  for (long long i = i0; i < i1; ++i) {
    st = pcg_step(st, inc);
    const double d = (double)(ptr[i + 1] - ptr[i]);
    w[i] = add_rn(pcg_out_double(st), __ddiv_rn(d, add_rn(d, 1.0)));
  }
}

__device__ __forceinline__ bool beats_g(double wi, int gi, double wj, int gj) {
  return wi > wj || (wi == wj && gi < gj);
}

// phase 0: select new F (mark) among undecided local rows; ext arrays w/st/gid
__global__ void luby_select_ext_kernel(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                       const double* __restrict__ w, const int* __restrict__ gid,
                                       signed char* st, signed char mark) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (st[i] != 0) continue;
    const double wi = w[i];
    const int gi = gid[i];
    bool win = true;
    for (int k = ptr[i]; k < ptr[i + 1] && win; ++k) {
      const int j = col[k];
      const signed char sj = st[j];
      if ((sj == 0 || sj == mark) && !beats_g(wi, gi, w[j], gid[j])) win = false;
    }
    if (win) st[i] = mark;
  }
}

__global__ void luby_block_ext_kernel(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                      signed char* st, signed char mark, int* __restrict__ remaining) {
  int left = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (st[i] != 0) continue;
    bool blocked = false;
    for (int k = ptr[i]; k < ptr[i + 1]; ++k)
      if (st[col[k]] == mark) {
        blocked = true;
        break;
      }
    if (blocked) st[i] = 2;
    else ++left;
  }
  left = warp_sum(left);
  if ((threadIdx.x & 31) == 0 && left) atomicAdd(remaining, left);
}

__global__ void luby_finish_ext_kernel(int n, const signed char* __restrict__ st,
                                       signed char* __restrict__ labels) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const signed char v = st[i];
    labels[i] = (v == 1 || v >= 3) ? 0 : 1;
  }
}

__global__ void ddc_hist_ext_kernel(int nf, const double* __restrict__ ratio,
                                    const double* __restrict__ edges, int nedges,
                                    unsigned long long* __restrict__ hist) {
  extern __shared__ unsigned long long sh[];
  double* se = (double*)(sh + nedges + 1);
  for (int k = threadIdx.x; k <= nedges; k += blockDim.x) sh[k] = 0ull;
  for (int k = threadIdx.x; k < nedges; k += blockDim.x) se[k] = edges[k];
  __syncthreads();
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nf;
       t += (long long)gridDim.x * blockDim.x) {
    const double r = ratio[t];
    int lo = 0, hi = nedges;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (se[mid] < r) lo = mid + 1;
      else hi = mid;
    }
    atomicAdd(sh + lo, 1ull);
  }
  __syncthreads();
  for (int k = threadIdx.x; k <= nedges; k += blockDim.x)
    if (sh[k]) atomicAdd(hist + k, sh[k]);
}

__global__ void ddc_convert_ext_kernel(int nf, const int* __restrict__ f_loc, const double* __restrict__ ratio,
                                       double cut, int all, signed char* __restrict__ labels,
                                       int* __restrict__ converted) {
  int c = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nf;
       t += (long long)gridDim.x * blockDim.x) {
    if (all || ratio[t] > cut) {
      labels[f_loc[t]] = 1;
      ++c;
    }
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(converted, c);
}

__global__ void minmaxsum_kernel(int n, const double* __restrict__ x, double* __restrict__ parts) {
  __shared__ double rmin[32], rmax[32], rsum[32];
  double mn = INFINITY, mx = -INFINITY, sm = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = x[i];
    mn = fmin(mn, v);
    mx = fmax(mx, v);
    sm += v;
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    rmin[w] = mn;
    rmax[w] = mx;
    rsum[w] = sm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) {
      mn = fmin(mn, rmin[q]);
      mx = fmax(mx, rmax[q]);
      sm += rsum[q];
    }
    parts[3 * blockIdx.x] = mn;
    parts[3 * blockIdx.x + 1] = mx;
    parts[3 * blockIdx.x + 2] = sm;
  }
}

// out[i] = map[in[i]] (int32 gather), used for renumbering column arrays
__global__ void gather_int_kernel(long long n, const int* __restrict__ in, const int* __restrict__ map,
                                  int* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int v = in[i];
    out[i] = v >= 0 ? map[v] : v;
  }
}

}  // namespace airg

using namespace airg;

extern "C" {

int airg_advection_2d_rows(int nx, int ny, double vx, double vy, int64_t row_begin, int64_t row_end,
                           int32_t* ptr, int32_t* col, double* val, int64_t* nnz_h, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const long long n = (long long)nx * ny;
  if (row_begin < 0 || row_end > n || row_begin > row_end) {
    set_error("bad row range");
    return AIRG_ERR_VALUE;
  }
  // entries before row idx (valid up to idx = n, where it is the total nnz)
  const long long base = stencil_before(row_begin, nx, vx, vy);
  if (nnz_h) *nnz_h = stencil_before(row_end, nx, vx, vy) - base;
  if (!ptr) return AIRG_OK;  // size query
  if (row_end == row_begin) {
    AIRG_CUDA(cudaMemsetAsync(ptr, 0, sizeof(int), s));
    return AIRG_OK;
  }
  advection_rows_kernel<<<blocks_for(row_end - row_begin, 256), 256, 0, s>>>(
      nx, row_begin, row_end, vx, vy, base, ptr, col, val);
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

int airg_strength_rows(int n, int row0, const int32_t* ptr, const int32_t* col, const double* val,
                       int64_t nnz, double theta, airg_csr_result** S_out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  unsigned char* keep = nullptr;
  int* cnt = nullptr;
  AIRG_TRY(scratch(&keep, nnz, s));
  AIRG_TRY(scratch(&cnt, n + 1, s));
  const int nb = blocks_for(n, 256);
  if (n > 0) strength_count_kernel<8><<<group_blocks(n, 8), 256, 0, s>>>(n, row0, ptr, col, val, theta, keep, cnt);
  AIRG_LAUNCH_CHECK();
  airg_csr_result* S = new_result(n, 0, s);
  long long snnz = 0;
  AIRG_TRY(scan_counts(cnt, S->ptr, n, &snnz, s));
  AIRG_TRY(result_alloc_entries(S, snnz, false));
  if (n > 0) compact_cols_kernel<8><<<group_blocks(n, 8), 256, 0, s>>>(n, ptr, col, keep, S->ptr, S->col);
  AIRG_LAUNCH_CHECK();
  release(keep, s);
  release(cnt, s);
  *S_out = S;
  return AIRG_OK;
}

int airg_union_rows(int n, const int32_t* ap, const int32_t* ac, const int32_t* bp, const int32_t* bc,
                    airg_csr_result** out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int* cnt = nullptr;
  AIRG_TRY(scratch(&cnt, n + 1, s));
  const int nb = blocks_for(n, 256);
  if (n > 0) union_sorted_rows_kernel<<<nb, 256, 0, s>>>(n, ap, ac, bp, bc, nullptr, nullptr, cnt);
  airg_csr_result* r = new_result(n, 0, s);
  long long nnz = 0;
  AIRG_TRY(scan_counts(cnt, r->ptr, n, &nnz, s));
  AIRG_TRY(result_alloc_entries(r, nnz, false));
  if (n > 0) union_sorted_rows_kernel<<<nb, 256, 0, s>>>(n, ap, ac, bp, bc, r->ptr, r->col, nullptr);
  AIRG_LAUNCH_CHECK();
  release(cnt, s);
  *out = r;
  return AIRG_OK;
}

int airg_luby_weights(int n, int64_t row0, const int32_t* cptr, uint64_t state_hi, uint64_t state_lo,
                      uint64_t inc_hi, uint64_t inc_lo, double* w, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n <= 0) return AIRG_OK;
  u128 s0 = {state_lo, state_hi}, inc = {inc_lo, inc_hi};
  const long long threads = (n + 63) / 64;
  luby_weights_rows_kernel<<<(int)((threads + 255) / 256), 256, 0, s>>>(n, row0, cptr, s0, inc, w);
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

// phase 0 = select, phase 1 = block (remaining_h = local undecided count)
int airg_luby_round(int n, const int32_t* cptr, const int32_t* ccol_ext, const double* w_ext,
                    const int32_t* gid_ext, int8_t* st_ext, int mark, int phase, int32_t* remaining_h,
                    void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = blocks_for(n, 256);
  if (phase == 0) {
    if (n > 0)
      luby_select_ext_kernel<<<nb, 256, 0, s>>>(n, cptr, ccol_ext, w_ext, gid_ext, (signed char*)st_ext,
                                                (signed char)mark);
    AIRG_LAUNCH_CHECK();
    return AIRG_OK;
  }
  int* rem = nullptr;
  AIRG_TRY(scratch(&rem, 1, s));
  AIRG_CUDA(cudaMemsetAsync(rem, 0, sizeof(int), s));
  if (n > 0)
    luby_block_ext_kernel<<<nb, 256, 0, s>>>(n, cptr, ccol_ext, (signed char*)st_ext, (signed char)mark,
                                             rem);
  AIRG_LAUNCH_CHECK();
  if (remaining_h) {  // null: no convergence check this round (no host sync)
    AIRG_CUDA(read_back(remaining_h, rem, sizeof(int), s));
  }
  release(rem, s);
  return AIRG_OK;
}

int airg_luby_finish(int n, const int8_t* st, int8_t* labels, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n > 0)
    luby_finish_ext_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, (const signed char*)st,
                                                              (signed char*)labels);
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

int airg_ddc_ratios(int nf, int row0, const int32_t* f_loc, const int32_t* ptr, const int32_t* col_ext,
                    const double* val, const int8_t* labels_ext, double* ratio, int32_t* bad_h,
                    double* minmaxsum_h, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int* bad = nullptr;
  const int np = blocks_for(nf, 256, 512);
  double* parts = nullptr;
  AIRG_TRY(scratch(&bad, 1, s));
  AIRG_TRY(scratch(&parts, 3 * (size_t)np, s));
  const int init = 0x7fffffff;
  AIRG_CUDA(cudaMemcpyAsync(bad, &init, sizeof(int), cudaMemcpyHostToDevice, s));
  if (nf > 0) {
    ddc_ratio_kernel<8><<<group_blocks(nf, 8), 256, 0, s>>>(nf, row0, f_loc, ptr, col_ext, val,
                                                            (const signed char*)labels_ext, ratio, bad);
    minmaxsum_kernel<<<np, 256, 0, s>>>(nf, ratio, parts);
  }
  AIRG_LAUNCH_CHECK();
  std::vector<double> h(3 * (size_t)np);
  AIRG_CUDA(cudaMemcpyAsync(bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  if (nf > 0)
    AIRG_CUDA(read_back(h.data(), parts, h.size() * sizeof(double), s));
  else
    AIRG_CUDA(cudaStreamSynchronize(s));
  double mn = INFINITY, mx = -INFINITY, sm = 0.0;
  for (int b = 0; nf > 0 && b < np; ++b) {
    mn = std::min(mn, h[3 * b]);
    mx = std::max(mx, h[3 * b + 1]);
    sm += h[3 * b + 2];
  }
  minmaxsum_h[0] = mn;
  minmaxsum_h[1] = mx;
  minmaxsum_h[2] = sm;
  release(bad, s);
  release(parts, s);
  return AIRG_OK;
}

int airg_ddc_hist(int nf, const double* ratio, const double* edges_h, int nedges, uint64_t* hist,
                  void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  double* de = nullptr;
  AIRG_TRY(scratch(&de, nedges, s));
  AIRG_CUDA(cudaMemcpyAsync(de, edges_h, nedges * sizeof(double), cudaMemcpyHostToDevice, s));
  AIRG_CUDA(cudaMemsetAsync(hist, 0, (nedges + 1) * sizeof(uint64_t), s));
  const size_t shm = (size_t)(nedges + 1) * sizeof(unsigned long long) + nedges * sizeof(double);
  if (shm > 200 * 1024) {
    set_error("too many DDC bins for the shared-memory histogram");
    return AIRG_ERR_VALUE;
  }
  AIRG_CUDA(cudaFuncSetAttribute(ddc_hist_ext_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(200 * 1024)));
  if (nf > 0)
    ddc_hist_ext_kernel<<<blocks_for(nf, 256, num_sms() * 2), 256, shm, s>>>(nf, ratio, de, nedges,
                                                                       (unsigned long long*)hist);
  AIRG_LAUNCH_CHECK();
  release(de, s);
  return AIRG_OK;
}

int airg_ddc_convert(int nf, const int32_t* f_loc, const double* ratio, double cut, int all,
                     int8_t* labels, int32_t* converted_h, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int* c = nullptr;
  AIRG_TRY(scratch(&c, 1, s));
  AIRG_CUDA(cudaMemsetAsync(c, 0, sizeof(int), s));
  if (nf > 0)
    ddc_convert_ext_kernel<<<blocks_for(nf, 256), 256, 0, s>>>(nf, f_loc, ratio, cut, all,
                                                               (signed char*)labels, c);
  AIRG_LAUNCH_CHECK();
  if (converted_h) {  // NULL: no host read (the caller counts the labels itself)
    AIRG_CUDA(read_back(converted_h, c, sizeof(int), s));
  }
  release(c, s);
  return AIRG_OK;
}

// elements [start, start + n) of the numpy PCG64 stream: out = a + b*random()
int airg_pcg64_fill_at(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                       int64_t start, int64_t n, double a, double b, double* out, void* stream) {
  u128 s0 = {state_lo, state_hi}, inc = {inc_lo, inc_hi};
  return pcg64_fill(s0, inc, n, a, b, out, (cudaStream_t)stream, start);
}

int airg_gather_int(int64_t n, const int32_t* in, const int32_t* map, int32_t* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n > 0) gather_int_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, in, map, out);
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}

}  // extern "C"
