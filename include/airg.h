/* libairg -- B200 (sm_100a) kernels for the AIRG reduction-multigrid path.
 *
 * C ABI: plain pointers and sizes, no torch types.  Every pointer argument is
 * a DEVICE pointer unless its name ends in `_h` (host).  `stream` is a
 * cudaStream_t passed as void*; every call is stream-ordered and returns an
 * airg status (0 = ok).  airg_last_error() gives the message, which the
 * Python layer maps to the reference's exception types (ValueError /
 * DivergenceError).
 *
 * Index arrays are int32 (rows/cols/offsets), values fp64.  Variable-size
 * outputs are two-phase: a *_count/_symbolic call writes per-row counts or a
 * total, the caller allocates, then the *_fill/_numeric call writes.
 *
 * Reference interfaces replaced (Python, /root/reference/pkg/src/airmg/):
 * see the comment above each entry point ("ref: file:line").
 */
#ifndef AIRG_H
#define AIRG_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AIRG_OK 0
#define AIRG_ERR_ARG 1
#define AIRG_ERR_CUDA 2
#define AIRG_ERR_VALUE 3     /* maps to ValueError */
#define AIRG_ERR_DIVERGED 4  /* maps to DivergenceError */

/* ---- library ---------------------------------------------------------- */
int airg_version(void);
/* Copies the last error message (thread-local) into buf; returns its length. */
int airg_last_error(char* buf_h, int len);
int airg_sm_count(void);

/* ---- sparse kernels ---------------------------------------------------- */
/* y = A x.  exact=1: one thread per row, sequential column-order sum with
 * separate mul/add rounding == scipy csr_matvec bitwise.  exact=0: adaptive
 * vector CSR with FMA (solve path).  ref: sparse.py:206-212 */
int airg_spmv(int nrows, const int32_t* ptr, const int32_t* col, const double* val,
              const double* x, double* y, int exact, void* stream);

/* Euclidean norm of x (deterministic fixed-order reduction) into out_h. */
int airg_norm2(int n, const double* x, double* out_h, void* stream);

/* ---- polynomial application (polynomial.py:295-369) ---------------------
 * kind: 0 = arnoldi_coeff (Horner, ncoef monomial coefficients in coef_h),
 *       1 = newton_roots (nunits units: type_h[k]=0 real root p1=theta,
 *           type_h[k]=1 conjugate pair p1=2*Re, p2=|theta|^2),
 *       2 = neumann (ncoef = order+1, diag_scale device vector).
 * y = q(A) b.  ref: polynomial.py:358 apply_matrix_free */
int airg_poly_apply(int kind, int n, const int32_t* ptr, const int32_t* col, const double* val,
                    int ncoef, const double* coef_h, int nunits, const int32_t* type_h,
                    const double* p1_h, const double* p2_h, const double* diag_scale,
                    const double* b, double* y, void* stream);

/* ---- V-cycle / Richardson plan (solve.py:95-167) ------------------------
 * A plan holds device pointers to the retained operators of a hierarchy
 * (the caller keeps them alive) plus its own work vectors. */
typedef struct airg_plan airg_plan;
int airg_plan_create(int nlevels, airg_plan** out_h);
int airg_plan_destroy(airg_plan* plan);
int airg_plan_set_top(airg_plan* plan, int n, const int32_t* ptr, const int32_t* col,
                      const double* val);
/* One reduction level: R (n_c x n), A_fc (n_f x n_c), A_ff (n_f x n_f), the
 * sorted index sets f_idx/c_idx and the smoother (same encoding as
 * airg_poly_apply).  asm_* is the optional assembled smoother (nnz<0: none).
 */
int airg_plan_set_level(airg_plan* plan, int level, int n, int n_f, int n_c,
                        const int32_t* R_ptr, const int32_t* R_col, const double* R_val,
                        const int32_t* Afc_ptr, const int32_t* Afc_col, const double* Afc_val,
                        const int32_t* Aff_ptr, const int32_t* Aff_col, const double* Aff_val,
                        const int32_t* f_idx, const int32_t* c_idx,
                        int kind, int ncoef, const double* coef_h, const double* diag_scale,
                        int64_t asm_nnz, const int32_t* asm_ptr, const int32_t* asm_col,
                        const double* asm_val);
int airg_plan_set_coarse(airg_plan* plan, int n, const int32_t* ptr, const int32_t* col,
                         const double* val, int kind, int ncoef, const double* coef_h,
                         int nunits, const int32_t* type_h, const double* p1_h,
                         const double* p2_h, const double* diag_scale);
/* e = V-cycle(level, r) for vectors of the level's size. ref: solve.py:95 */
int airg_plan_vcycle(airg_plan* plan, int level, const double* r, double* e,
                     int f_smooth_its, void* stream);
/* Undamped Richardson preconditioned by one V-cycle (solve.py:113-167).
 * x is updated in place.  history_h must hold max_iters+1 doubles.
 * Returns AIRG_ERR_DIVERGED (iteration in *iterations_h) on a non-finite or
 * 1e8-times-grown residual. */
int airg_plan_richardson(airg_plan* plan, const double* b, double* x, double rtol,
                         double atol, int max_iters, int f_smooth_its, double* history_h,
                         int* iterations_h, int* converged_h, void* stream);
/* Number of kernel launches issued by the last airg_plan_richardson call. */
int64_t airg_plan_launches(airg_plan* plan);

#ifdef __cplusplus
}
#endif
#endif /* AIRG_H */
