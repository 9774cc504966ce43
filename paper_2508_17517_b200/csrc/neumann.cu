// Neumann-series pieces of the fixed-sparsity assembly (nAIR variant):
// base = I + (-D^-1 A) with exact zeros pruned (scipy CSR +), and the final
// right scaling by D^-1.  ref: polynomial.py:396-415
#include "setup_common.cuh"

namespace airg {

// per row: entries of -ds_i * a_ij, diagonal 1 + (-ds_i a_ii) (inserted as 1
// when absent), exact zeros dropped; count (ocol == nullptr) or write
__global__ void neumann_base_kernel(int n, const int* __restrict__ p, const int* __restrict__ c,
                                    const double* __restrict__ v, const double* __restrict__ ds,
                                    const int* __restrict__ optr, int* __restrict__ ocol,
                                    double* __restrict__ oval, int* __restrict__ cnt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double s = -ds[i];
    int o = optr ? optr[i] : 0, m = 0;
    bool diag_done = false;
    auto emit = [&](int col, double val) {
      if (val != 0.0) {
        if (ocol) {
          ocol[o + m] = col;
          oval[o + m] = val;
        }
        ++m;
      }
    };
    for (int k = p[i]; k < p[i + 1]; ++k) {
      const int j = c[k];
      const double sv = mul_rn(s, v[k]);
      if (!diag_done && j > i) {
        emit((int)i, 1.0);
        diag_done = true;
      }
      if (j == i) {
        emit(j, add_rn(1.0, sv));
        diag_done = true;
      } else {
        emit(j, sv);  // 0 + s_ij
      }
    }
    if (!diag_done) emit((int)i, 1.0);
    if (cnt) cnt[i] = m;
  }
}

__global__ void scale_columns_kernel(long long nnz, const int* __restrict__ c, const double* __restrict__ ds,
                                     double* __restrict__ v) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz;
       k += (long long)gridDim.x * blockDim.x)
    v[k] = mul_rn(v[k], ds[c[k]]);
}

}  // namespace airg

using namespace airg;

extern "C" int airg_neumann_base(int n, const int32_t* p, const int32_t* c, const double* v,
                                 const double* diag_scale, airg_csr_result** out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  airg_csr_result* r = new_result(n, n, s);
  if (!r) return AIRG_ERR_CUDA;
  int* cnt = nullptr;
  AIRG_TRY(scratch(&cnt, n + 1, s));
  const int nb = blocks_for(n, 256);
  if (n > 0) neumann_base_kernel<<<nb, 256, 0, s>>>(n, p, c, v, diag_scale, nullptr, nullptr, nullptr, cnt);
  long long nnz = 0;
  AIRG_TRY(scan_counts(cnt, r->ptr, n, &nnz, s));
  AIRG_TRY(result_alloc_entries(r, nnz, true));
  if (n > 0) neumann_base_kernel<<<nb, 256, 0, s>>>(n, p, c, v, diag_scale, r->ptr, r->col, r->val, nullptr);
  AIRG_LAUNCH_CHECK();
  release(cnt, s);
  *out = r;
  return AIRG_OK;
}

extern "C" int airg_scale_columns(int64_t nnz, const int32_t* c, const double* diag_scale, double* v,
                                  void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nnz > 0) scale_columns_kernel<<<blocks_for(nnz, 256), 256, 0, s>>>(nnz, c, diag_scale, v);
  AIRG_LAUNCH_CHECK();
  return AIRG_OK;
}
