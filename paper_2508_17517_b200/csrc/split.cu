// CF splitting on the GPU: strength graph + symmetric closure, PMISR Luby
// rounds with numpy-exact PCG64 weights, DDC cleanup, repair, split index
// maps and the one-point prolongator.
// ref: splitting.py:86-238, hierarchy.py:250-305
#include "setup_common.cuh"
#include "rowgroup.cuh"
#include <vector>
#include <cmath>

namespace airg {

// ---- strength graph (splitting.py:86-109) ----------------------------------
__global__ void col_count_kernel(long long nnz, const int* __restrict__ col, int* __restrict__ cnt) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz;
       k += (long long)gridDim.x * blockDim.x)
    atomicAdd(cnt + col[k], 1);
}

__global__ void transpose_fill_kernel(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                      const int* __restrict__ tptr, int* __restrict__ fillpos,
                                      int* __restrict__ tcol) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
      const int j = col[k];
      tcol[tptr[j] + atomicAdd(fillpos + j, 1)] = (int)i;
    }
}

// small per-row insertion sort (transpose rows of strength graphs are short)
__global__ void sort_rows_kernel(int n, const int* __restrict__ ptr, int* __restrict__ col) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int b = ptr[i], e = ptr[i + 1];
    for (int k = b + 1; k < e; ++k) {
      int v = col[k], m = k - 1;
      while (m >= b && col[m] > v) {
        col[m + 1] = col[m];
        --m;
      }
      col[m + 1] = v;
    }
  }
}

// union of two sorted rows: count (out==nullptr) or write
__global__ void union_rows_kernel(int n, const int* __restrict__ ap, const int* __restrict__ ac,
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

__global__ void fill_ones_kernel(long long n, double* __restrict__ v) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x)
    v[k] = 1.0;
}

// Builds S (strong couplings) and pattern(S + S^T).  Values are not stored.
static int strength_closure(int n, const int* ptr, const int* col, const double* val, long long nnz,
                            double theta, airg_csr_result** S_out, airg_csr_result** C_out,
                            cudaStream_t s) {
  unsigned char* keep = nullptr;
  int *cnt = nullptr, *tcnt = nullptr, *tptr = nullptr, *tcol = nullptr;
  AIRG_TRY(scratch(&keep, nnz, s));
  AIRG_TRY(scratch(&cnt, n + 1, s));
  const int nb = blocks_for(n, 256);
  strength_count_kernel<8><<<group_blocks(n, 8), 256, 0, s>>>(n, 0, ptr, col, val, theta, keep, cnt);
  AIRG_LAUNCH_CHECK();
  airg_csr_result* S = new_result(n, n, s);
  if (!S) return AIRG_ERR_CUDA;
  long long snnz = 0;
  AIRG_TRY(scan_counts(cnt, S->ptr, n, &snnz, s));
  AIRG_TRY(result_alloc_entries(S, snnz, false));
  compact_cols_kernel<8><<<group_blocks(n, 8), 256, 0, s>>>(n, ptr, col, keep, S->ptr, S->col);
  AIRG_LAUNCH_CHECK();
  // transpose
  AIRG_TRY(scratch(&tcnt, n + 1, s));
  AIRG_TRY(scratch(&tptr, n + 1, s));
  AIRG_TRY(scratch(&tcol, snnz, s));
  AIRG_CUDA(cudaMemsetAsync(tcnt, 0, (size_t)(n + 1) * sizeof(int), s));
  col_count_kernel<<<blocks_for(snnz, 256), 256, 0, s>>>(snnz, S->col, tcnt);
  AIRG_TRY(scan_counts(tcnt, tptr, n, nullptr, s));
  AIRG_CUDA(cudaMemsetAsync(tcnt, 0, (size_t)(n + 1) * sizeof(int), s));
  transpose_fill_kernel<<<nb, 256, 0, s>>>(n, S->ptr, S->col, tptr, tcnt, tcol);
  sort_rows_kernel<<<nb, 256, 0, s>>>(n, tptr, tcol);
  AIRG_LAUNCH_CHECK();
  // closure = union
  airg_csr_result* Cl = new_result(n, n, s);
  if (!Cl) return AIRG_ERR_CUDA;
  union_rows_kernel<<<nb, 256, 0, s>>>(n, S->ptr, S->col, tptr, tcol, nullptr, nullptr, cnt);
  long long cnnz = 0;
  AIRG_TRY(scan_counts(cnt, Cl->ptr, n, &cnnz, s));
  AIRG_TRY(result_alloc_entries(Cl, cnnz, false));
  union_rows_kernel<<<nb, 256, 0, s>>>(n, S->ptr, S->col, tptr, tcol, Cl->ptr, Cl->col, nullptr);
  AIRG_LAUNCH_CHECK();
  release(keep, s);
  release(cnt, s);
  release(tcnt, s);
  release(tptr, s);
  release(tcol, s);
  if (S_out) *S_out = S;
  else airg_result_free(S);
  *C_out = Cl;
  return AIRG_OK;
}

// ---- PMISR (splitting.py:112-159) ------------------------------------------
// state: 0 undecided, 1 fine, 2 coarse, 3/4 new-fine marker of the current round
__global__ void luby_weight_kernel(int n, const int* __restrict__ ptr, double* __restrict__ w) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double d = (double)(ptr[i + 1] - ptr[i]);
    w[i] = add_rn(w[i], __ddiv_rn(d, add_rn(d, 1.0)));  // random() + deg/(deg+1)
  }
}

__device__ __forceinline__ bool beats(double wi, int i, double wj, int j) {
  return wi > wj || (wi == wj && i < j);
}

__global__ void luby_select_kernel(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                   const double* __restrict__ w, signed char* st, signed char mark) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (st[i] != 0) continue;
    const double wi = w[i];
    bool win = true;
    for (int k = ptr[i]; k < ptr[i + 1] && win; ++k) {
      const int j = col[k];
      const signed char sj = st[j];
      if ((sj == 0 || sj == mark) && !beats(wi, (int)i, w[j], j)) win = false;
    }
    if (win) st[i] = mark;
  }
}

__global__ void luby_block_kernel(int n, const int* __restrict__ ptr, const int* __restrict__ col,
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

__global__ void luby_normalise_kernel(int n, signed char* st) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (st[i] >= 3) st[i] = 1;
}

__global__ void luby_finish_kernel(int n, const signed char* __restrict__ st,
                                   signed char* __restrict__ labels, int cap_to_coarse) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const signed char v = st[i];
    labels[i] = (v == 1 || v >= 3) ? 0 : 1;  // F_POINT = 0, C_POINT = 1
  }
}

static int pmisr_run(int n, const int* cptr, const int* ccol, u128 s0, u128 inc, int max_loops,
                     signed char* labels, int* loops_h, cudaStream_t s) {
  double* w = nullptr;
  signed char* st = nullptr;
  // rounds are enqueued kLubyBatch (2; 1/2/4/8 measured within 1 ms of
  // cf_split over the 2048² setup) at a time, each counting the undecided
  // rows left in its own slot, with one read-back per batch: a round after
  // the last one finds no undecided row and changes nothing
  static const int kLubyBatch = getenv("AIRG_LUBY_BATCH") ? std::max(1, atoi(getenv("AIRG_LUBY_BATCH"))) : 2;
  int* rem = nullptr;
  AIRG_TRY(scratch(&w, n, s));
  AIRG_TRY(scratch(&st, n, s));
  AIRG_TRY(scratch(&rem, kLubyBatch, s));
  AIRG_TRY(pcg64_fill(s0, inc, n, 0.0, 1.0, w, s));
  const int nb = blocks_for(n, 256);
  luby_weight_kernel<<<nb, 256, 0, s>>>(n, cptr, w);
  AIRG_CUDA(cudaMemsetAsync(st, 0, (size_t)n, s));
  int loops = 0;
  bool more = n > 0;
  std::vector<int> left(kLubyBatch);
  while (more) {
    if (max_loops >= 0 && loops >= max_loops) break;  // leftovers -> C in finish
    const int r = max_loops >= 0 ? std::min(kLubyBatch, max_loops - loops) : kLubyBatch;
    AIRG_CUDA(cudaMemsetAsync(rem, 0, r * sizeof(int), s));
    for (int q = 0; q < r; ++q) {
      const int l = loops + q;
      // per-round new-F marker; earlier markers read as decided F
      const signed char mark = (signed char)(3 + l % 120);
      if (l > 0 && l % 120 == 0) luby_normalise_kernel<<<nb, 256, 0, s>>>(n, st);
      luby_select_kernel<<<nb, 256, 0, s>>>(n, cptr, ccol, w, st, mark);
      luby_block_kernel<<<nb, 256, 0, s>>>(n, cptr, ccol, st, mark, rem + q);
    }
    AIRG_LAUNCH_CHECK();
    AIRG_CUDA(read_back(left.data(), rem, r * sizeof(int), s));
    int q = 0;
    while (q < r && left[q] > 0) ++q;
    if (q < r) {
      loops += q + 1;  // the round that left no undecided row
      more = false;
    } else {
      loops += r;
    }
  }
  luby_finish_kernel<<<nb, 256, 0, s>>>(n, st, labels, 1);
  AIRG_LAUNCH_CHECK();
  release(w, s);
  release(st, s);
  release(rem, s);
  if (loops_h) *loops_h = loops;
  return AIRG_OK;
}

// ---- split index maps ----------------------------------------------------
__global__ void label_flags_kernel(int n, const signed char* __restrict__ labels, int* __restrict__ fl) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    fl[i] = labels[i] == 0;
}

// pos[i] = rank of i within its class; f_idx / c_idx optional
__global__ void split_pos_kernel(int n, const signed char* __restrict__ labels,
                                 const int* __restrict__ fscan, int* __restrict__ pos,
                                 int* __restrict__ f_idx, int* __restrict__ c_idx) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int fr = fscan[i];
    if (labels[i] == 0) {
      if (pos) pos[i] = fr;
      if (f_idx) f_idx[fr] = (int)i;
    } else {
      const int cr = (int)i - fr;
      if (pos) pos[i] = cr;
      if (c_idx) c_idx[cr] = (int)i;
    }
  }
}

int split_index(int n, const signed char* labels, int* pos, int* f_idx, int* c_idx, int* nf_h,
                cudaStream_t s) {
  int *fl = nullptr, *fs = nullptr;
  AIRG_TRY(scratch(&fl, n + 1, s));
  AIRG_TRY(scratch(&fs, n + 1, s));
  const int nb = blocks_for(n, 256);
  label_flags_kernel<<<nb, 256, 0, s>>>(n, labels, fl);
  long long nf = 0;
  AIRG_TRY(scan_counts(fl, fs, n, &nf, s));
  split_pos_kernel<<<nb, 256, 0, s>>>(n, labels, fs, pos, f_idx, c_idx);
  AIRG_LAUNCH_CHECK();
  release(fl, s);
  release(fs, s);
  if (nf_h) *nf_h = (int)nf;
  return AIRG_OK;
}

// ---- DDC (splitting.py:162-207) --------------------------------------------
// b = #{edges < r} per ratio (binary search over the edges in shared
// memory); 32-bit shared bins, lanes of a warp with the same bin add once
// (__match_any_sync: the ratios cluster in few bins, and same-address shared
// atomics serialise), one global 64-bit add per non-empty bin and block
__global__ void ddc_hist_kernel(int nf, const double* __restrict__ ratio, const double* __restrict__ edges,
                                int nedges, unsigned long long* __restrict__ hist) {
  extern __shared__ unsigned long long sh64[];
  unsigned* sh = (unsigned*)sh64;
  double* se = (double*)(sh64 + nedges + 1);
  for (int k = threadIdx.x; k <= nedges; k += blockDim.x) sh[k] = 0u;
  for (int k = threadIdx.x; k < nedges; k += blockDim.x) se[k] = edges[k];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (long long t0 = blockIdx.x * (long long)blockDim.x; t0 < nf; t0 += (long long)gridDim.x * blockDim.x) {
    const long long t = t0 + threadIdx.x;
    int b = -1;
    if (t < nf) {
      const double r = ratio[t];
      int lo = 0, hi = nedges;
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (se[mid] < r) lo = mid + 1;
        else hi = mid;
      }
      b = lo;
    }
    const unsigned m = __match_any_sync(0xffffffffu, b);
    if (b >= 0 && lane == __ffs(m) - 1) atomicAdd(sh + b, (unsigned)__popc(m));
  }
  __syncthreads();
  for (int k = threadIdx.x; k <= nedges; k += blockDim.x)
    if (sh[k]) atomicAdd(hist + k, (unsigned long long)sh[k]);
}

__global__ void ddc_convert_kernel(int nf, const int* __restrict__ f_idx, const double* __restrict__ ratio,
                                   double cut, int all, signed char* __restrict__ labels,
                                   int* __restrict__ converted) {
  int c = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nf;
       t += (long long)gridDim.x * blockDim.x) {
    if (all || ratio[t] > cut) {
      labels[f_idx[t]] = 1;
      ++c;
    }
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(converted, c);
}

__global__ void sum_kernel(int n, const double* __restrict__ x, double* __restrict__ parts) {
  __shared__ double red[32];
  double v = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v += x[i];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) parts[blockIdx.x] = t;
  }
}

static int ddc_pass_run(int n, const int* ptr, const int* col, const double* val,
                        signed char* labels, double frac, int nbins, double* stats,
                        cudaStream_t s) {
  if (!(frac > 0.0 && frac < 1.0)) {
    set_error("fraction must lie in (0, 1)");
    return AIRG_ERR_VALUE;
  }
  if (nbins < 1) {
    set_error("nbins must be positive");
    return AIRG_ERR_VALUE;
  }
  int nf = 0;
  int* f_idx = nullptr;
  AIRG_TRY(scratch(&f_idx, n, s));
  AIRG_TRY(split_index(n, labels, nullptr, f_idx, nullptr, &nf, s));
  if (nf == 0) {
    release(f_idx, s);
    set_error("zero-size array to reduction operation minimum which has no identity");
    return AIRG_ERR_VALUE;
  }
  double* ratio = nullptr;
  int* ibuf = nullptr;  // [0] bad, [1] converted
  AIRG_TRY(scratch(&ratio, nf, s));
  AIRG_TRY(scratch(&ibuf, 2, s));
  int init[2] = {0x7fffffff, 0};
  AIRG_CUDA(cudaMemcpyAsync(ibuf, init, sizeof init, cudaMemcpyHostToDevice, s));
  const int nb = blocks_for(nf, 256);
  if (nf > 0)
    ddc_ratio_kernel<8><<<group_blocks(nf, 8), 256, 0, s>>>(nf, 0, f_idx, ptr, col, val, labels, ratio, ibuf);
  AIRG_LAUNCH_CHECK();
  // min / max / mean, read back with the zero-diagonal flag (one sync)
  int bad = 0;
  double lo = 0, hi = 0, mean = 0;
  {
    double* mm = nullptr;
    AIRG_TRY(scratch(&mm, 2 + 1024, s));
    void* tmp = nullptr;
    size_t b1 = 0, b2 = 0;
    AIRG_CUDA(cub::DeviceReduce::Min(tmp, b1, ratio, mm, nf, s));
    AIRG_CUDA(cub::DeviceReduce::Max(tmp, b2, ratio, mm + 1, nf, s));
    AIRG_CUDA(cudaMallocFromPoolAsync(&tmp, b1 > b2 ? b1 : b2, lib_pool(), s));
    AIRG_CUDA(cub::DeviceReduce::Min(tmp, b1, ratio, mm, nf, s));
    AIRG_CUDA(cub::DeviceReduce::Max(tmp, b2, ratio, mm + 1, nf, s));
    const int pb = blocks_for(nf, 256, 1024);
    sum_kernel<<<pb, 256, 0, s>>>(nf, ratio, mm + 2);
    std::vector<double> h(2 + pb);
    AIRG_CUDA(read_back({{h.data(), mm, (2 + pb) * sizeof(double)}, {&bad, ibuf, sizeof(int)}}, s));
    cudaFreeAsync(tmp, s);
    release(mm, s);
    if (bad != 0x7fffffff) {
      release(f_idx, s);
      release(ratio, s);
      release(ibuf, s);
      set_error("zero diagonal in fine-fine block (fine row %d); splitting is not usable for "
                "reduction", bad);
      return AIRG_ERR_VALUE;
    }
    lo = h[0];
    hi = h[1];
    double sm = 0;
    for (int i = 0; i < pb; ++i) sm += h[2 + i];
    mean = nf > 0 ? sm / nf : NAN;
  }
  const double target = frac * (double)nf;
  double cut;
  int all = 0;
  bool convert_any = true;
  if (lo == hi) {
    const bool conv = std::fabs((double)nf - target) < target;
    all = conv ? 1 : 0;
    convert_any = conv;
    cut = conv ? lo : hi;
  } else {
    std::vector<double> edges(nbins + 1);
    for (int k = 0; k <= nbins; ++k) {
      volatile double t = (hi - lo) * (double)k;  // (hi-lo)*k, then /nbins, then lo + .
      volatile double q = t / (double)nbins;
      edges[k] = lo + q;
    }
    double* de = nullptr;
    unsigned long long* hist = nullptr;
    AIRG_TRY(scratch(&de, nbins + 1, s));
    AIRG_TRY(scratch(&hist, nbins + 2, s));
    AIRG_CUDA(cudaMemcpyAsync(de, edges.data(), (nbins + 1) * sizeof(double), cudaMemcpyHostToDevice, s));
    AIRG_CUDA(cudaMemsetAsync(hist, 0, (nbins + 2) * sizeof(unsigned long long), s));
    const size_t shm = (size_t)(nbins + 2) * sizeof(unsigned long long) + (nbins + 1) * sizeof(double);
    if (shm > 200 * 1024) {
      set_error("too many DDC bins for the shared-memory histogram");
      return AIRG_ERR_VALUE;
    }
    if (shm > 48 * 1024)
      AIRG_CUDA(cudaFuncSetAttribute(ddc_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    ddc_hist_kernel<<<blocks_for(nf, 256, num_sms() * 2), 256, shm, s>>>(nf, ratio, de, nbins + 1, hist);
    AIRG_LAUNCH_CHECK();
    std::vector<unsigned long long> hh(nbins + 2);
    AIRG_CUDA(read_back(hh.data(), hist, (nbins + 2) * sizeof(unsigned long long), s));
    release(de, s);
    release(hist, s);
    // above_k = #{ratio > edge_k} = sum_{b > k} hist[b]
    std::vector<long long> above(nbins + 1);
    long long acc = 0;
    for (int k = nbins + 1; k >= 1; --k) {
      acc += (long long)hh[k];
      above[k - 1] = acc;
    }
    // argmin over the reversed array: largest k among equal minima
    int best = nbins;
    double bd = std::fabs((double)above[nbins] - target);
    for (int k = nbins - 1; k >= 0; --k) {
      const double d = std::fabs((double)above[k] - target);
      if (d < bd) {
        bd = d;
        best = k;
      }
    }
    cut = edges[best];
  }
  int converted = 0;
  if (convert_any && nf > 0) {
    ddc_convert_kernel<<<nb, 256, 0, s>>>(nf, f_idx, ratio, cut, all, labels, ibuf + 1);
    AIRG_LAUNCH_CHECK();
    AIRG_CUDA(read_back(&converted, ibuf + 1, sizeof(int), s));
  }
  release(f_idx, s);
  release(ratio, s);
  release(ibuf, s);
  stats[0] = nf;
  stats[1] = converted;
  stats[2] = lo;
  stats[3] = hi;
  stats[4] = mean;
  stats[5] = cut;
  return AIRG_OK;
}

// ---- repair (hierarchy.py:289-305) and one-point P (hierarchy.py:250-278) ----
__global__ void repair_kernel(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                              const signed char* __restrict__ lab_in, signed char* __restrict__ lab_out,
                              int* __restrict__ changed) {
  int c = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    signed char v = lab_in[i];
    if (v == 0) {
      bool has_c = false;
      for (int k = ptr[i]; k < ptr[i + 1] && !has_c; ++k) has_c = lab_in[col[k]] == 1;
      if (!has_c) {
        v = 1;
        ++c;
      }
    }
    lab_out[i] = v;
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(changed, c);
}

// VS lanes per row: each lane keeps its first maximum of |a_ij| over the C
// neighbours it strides over, then the group keeps the larger value, the
// earlier entry on ties -- the sequential "first maximum wins" scan.
template <int VS>
__global__ void onepoint_kernel(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                const double* __restrict__ val, const signed char* __restrict__ labels,
                                const int* __restrict__ pos, int* __restrict__ pcol,
                                int* __restrict__ bad) {
  AIRG_GROUP(VS);
  const long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / VS;
  const bool fine = i < n && labels[i] != 1;
  int b = 0, e = 0;
  if (fine) {
    b = ptr[i];
    e = ptr[i + 1];
  }
  double bm = -1.0;
  int bk = 0x7fffffff;
  for (int k = b + g; k < e; k += VS) {
    const int j = col[k];
    if (labels[j] != 1) continue;
    const double a = fabs(val[k]);
    if (a > bm) {
      bm = a;
      bk = k;
    }
  }
#pragma unroll
  for (int o = VS / 2; o > 0; o >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, bm, o);
    const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
    if (om > bm || (om == bm && ok < bk)) {
      bm = om;
      bk = ok;
    }
  }
  if (i < n && g == 0) {
    if (!fine) {
      pcol[i] = pos[i];
    } else {
      const int best = bk != 0x7fffffff ? pos[col[bk]] : -1;
      pcol[i] = best;
      if (best < 0) atomicMin(bad, (int)i);
    }
  }
}

}  // namespace airg

using namespace airg;

extern "C" {

int airg_strength(int n, const int32_t* ptr, const int32_t* col, const double* val, int64_t nnz,
                  double theta, airg_csr_result** S_out, airg_csr_result** closure_out,
                  void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!(theta >= 0.0 && theta <= 1.0)) {
    set_error("theta must lie in [0, 1]");
    return AIRG_ERR_VALUE;
  }
  airg_csr_result *S = nullptr, *Cl = nullptr;
  AIRG_TRY(strength_closure(n, ptr, col, val, nnz, theta, &S, &Cl, s));
  for (airg_csr_result* r : {S, Cl}) {
    AIRG_CUDA(cudaMallocFromPoolAsync((void**)&r->val, (size_t)(r->nnz > 0 ? r->nnz : 1) * sizeof(double), lib_pool(), s));
    fill_ones_kernel<<<blocks_for(r->nnz, 256), 256, 0, s>>>(r->nnz, r->val);
  }
  AIRG_LAUNCH_CHECK();
  *S_out = S;
  *closure_out = Cl;
  return AIRG_OK;
}

int airg_pmisr(int n, const int32_t* cptr, const int32_t* ccol, uint64_t state_hi,
               uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int max_loops,
               int8_t* labels, int32_t* loops_h, void* stream) {
  u128 s0 = {state_lo, state_hi}, inc = {inc_lo, inc_hi};
  return pmisr_run(n, cptr, ccol, s0, inc, max_loops, (signed char*)labels, loops_h,
                   (cudaStream_t)stream);
}

int airg_cf_pmisr(int n, const int32_t* ptr, const int32_t* col, const double* val, int64_t nnz,
                  double theta, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                  uint64_t inc_lo, int max_loops, int8_t* labels, int32_t* loops_h, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!(theta >= 0.0 && theta <= 1.0)) {
    set_error("theta must lie in [0, 1]");
    return AIRG_ERR_VALUE;
  }
  airg_csr_result* Cl = nullptr;
  AIRG_TRY(strength_closure(n, ptr, col, val, nnz, theta, nullptr, &Cl, s));
  u128 s0 = {state_lo, state_hi}, inc = {inc_lo, inc_hi};
  int st = pmisr_run(n, Cl->ptr, Cl->col, s0, inc, max_loops, (signed char*)labels, loops_h, s);
  airg_result_free(Cl);
  return st;
}

int airg_ddc_pass(int n, const int32_t* ptr, const int32_t* col, const double* val, int8_t* labels,
                  double fraction, int nbins, double* stats_h, void* stream) {
  return ddc_pass_run(n, ptr, col, val, (signed char*)labels, fraction, nbins, stats_h,
                      (cudaStream_t)stream);
}

int airg_split_index(int n, const int8_t* labels, int32_t* pos, int32_t* f_idx, int32_t* c_idx,
                     int32_t* nf_h, void* stream) {
  return split_index(n, (const signed char*)labels, pos, f_idx, c_idx, nf_h, (cudaStream_t)stream);
}

int airg_repair_split(int n, const int32_t* ptr, const int32_t* col, int8_t* labels,
                      int32_t* changed_h, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  signed char* tmp = nullptr;
  int* ch = nullptr;
  AIRG_TRY(scratch(&tmp, n, s));
  AIRG_TRY(scratch(&ch, 1, s));
  AIRG_CUDA(cudaMemsetAsync(ch, 0, sizeof(int), s));
  repair_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, ptr, col, (const signed char*)labels, tmp, ch);
  AIRG_LAUNCH_CHECK();
  AIRG_CUDA(cudaMemcpyAsync(labels, tmp, (size_t)n, cudaMemcpyDeviceToDevice, s));
  AIRG_CUDA(read_back(changed_h, ch, sizeof(int), s));
  release(tmp, s);
  release(ch, s);
  return AIRG_OK;
}

int airg_prolong_onepoint(int n, const int32_t* ptr, const int32_t* col, const double* val,
                          const int8_t* labels, const int32_t* pos, int32_t* pcol, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int* bad = nullptr;
  AIRG_TRY(scratch(&bad, 1, s));
  int init = 0x7fffffff;
  AIRG_CUDA(cudaMemcpyAsync(bad, &init, sizeof(int), cudaMemcpyHostToDevice, s));
  onepoint_kernel<8><<<group_blocks(n, 8), 256, 0, s>>>(n, ptr, col, val, (const signed char*)labels,
                                                        pos, pcol, bad);
  AIRG_LAUNCH_CHECK();
  int b = 0;
  AIRG_CUDA(read_back(&b, bad, sizeof(int), s));
  release(bad, s);
  if (b != 0x7fffffff) {
    set_error("fine point %d has no coupling to any coarse point; the splitting is invalid for "
              "a one-point prolongator", b);
    return AIRG_ERR_VALUE;
  }
  return AIRG_OK;
}

}  // extern "C"
