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
/* ELL storage for the fixed-nnz/row structured stencils: width slots per row,
 * column-major (slot k of row i at k*nrows + i), padding (value 0, column =
 * row) after a row's entries.  airg_csr_to_ell fails (status 3) when a row is
 * longer than width.  airg_spmv_ell: y = A x; exact = 1 gives the CSR exact
 * (scipy csr_matvec) result bitwise.  ref: sparse.py:206-212 */
int airg_csr_to_ell(int nrows, const int32_t* ptr, const int32_t* col, const double* val, int width,
                    int32_t* ell_col, double* ell_val, void* stream);
int airg_spmv_ell(int nrows, int width, const int32_t* ell_col, const double* ell_val, const double* x,
                  double* y, int exact, void* stream);

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
                    const double* b, double* y, int exact, void* stream);

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
/* exact=1: every solve kernel follows the reference's arithmetic order
 * (sequential row sums, separate mul/add roundings) so x is bitwise the
 * reference's for the same hierarchy; exact=0 (default): vector SpMV + FMA. */
int airg_plan_set_exact(airg_plan* plan, int exact);
/* Number of kernel launches issued by the last airg_plan_richardson call. */
int64_t airg_plan_launches(airg_plan* plan);
/* 1 when the fast-mode coarse solve of this plan is the dense q(A) GEMV,
 * 0 when it runs the Newton apply (exact mode, a large coarse grid, or an
 * identity column of q(A) that stopped early, polynomial.py:312-355). */
int airg_plan_coarse_mode(airg_plan* plan);
/* Number of CUDA graphs the plan holds (bounded: least recently used evicted). */
int airg_plan_graph_count(airg_plan* plan);
/* The plan's staging vectors (finest-level size): airg_plan_vcycle called
 * with r = *vin, e = *vout runs the captured V-cycle without copying the
 * caller's vectors in and out (measurement). */
int airg_plan_staging(airg_plan* plan, double** vin, double** vout);
/* Stream-ordered device-to-device copy (bench / test helper). */
int airg_copy_d2d(void* dst, const void* src, int64_t bytes, void* stream);

/* ---- distributed (row-strip) solve over NCCL ----------------
 * One plan per rank: per distributed level R / A_fc / A_ff on local rows with
 * columns in [local | ghost], halo plans (send indices + per-peer counts;
 * ghost values land in the tail of the operand vector), the top operator,
 * and the replicated serial plan of the coarse tail. */
typedef struct airg_dplan airg_dplan;
typedef struct airg_comm airg_comm;
int airg_nccl_unique_id(char* out_h /* 128 bytes */);
/* one NCCL communicator per process (ncclCommInitRank), shared by plans */
int airg_comm_create(const char* id_h, int rank, int world, airg_comm** out_h);
int airg_comm_destroy(airg_comm* comm);
int airg_dplan_create(airg_comm* comm, int ndist, airg_dplan** out_h);
/* which: 0 = R (fine space), 1 = A_fc (coarse space), 2 = A_ff (F space), 3 = top */
int airg_dplan_set_halo(airg_dplan* plan, int level, int which, int n_loc, int nsend,
                        const int32_t* send_idx, const int32_t* scnt_h, const int32_t* rcnt_h);
int airg_dplan_set_level(airg_dplan* plan, int level, int n_loc, int nf, int nc, const int32_t* Rp,
                         const int32_t* Rc, const double* Rv, int64_t Rnnz, const int32_t* Fcp,
                         const int32_t* Fcc, const double* Fcv, int64_t Fcnnz, const int32_t* Ffp,
                         const int32_t* Ffc, const double* Ffv, int64_t Ffnnz, const int32_t* f_idx,
                         const int32_t* c_idx, int ncoef, const double* coef_h);
int airg_dplan_set_top(airg_dplan* plan, int n_loc, const int32_t* ptr, const int32_t* col,
                       const double* val, int64_t nnz);
/* Distributed coarsest grid for a Newton coarse solver (configs[3]): the
 * rank's rows of the coarsest operator with columns [local | ghost], its halo
 * (as airg_dplan_set_halo) and the Newton units (as airg_plan_set_coarse).
 * The tail V-cycle then applies q(C) on the row strips instead of gathering
 * the coarsest grid (ref: polynomial.py:312-355, hierarchy.py:308-362). */
int airg_dplan_set_dcoarse(airg_dplan* plan, int n_loc, const int32_t* ptr, const int32_t* col,
                           const double* val, int64_t nnz, int nsend, const int32_t* send_idx,
                           const int32_t* scnt_h, const int32_t* rcnt_h, int nunits,
                           const int32_t* type_h, const double* p1_h, const double* p2_h);
int airg_dplan_finish(airg_dplan* plan, airg_plan* tail, const int32_t* counts_h);
int airg_dplan_richardson(airg_dplan* plan, const double* b, double* x, double rtol, double atol,
                          int max_iters, double* history_h, int* iterations_h, int* converged_h,
                          void* stream);
int airg_dplan_destroy(airg_dplan* plan);

/* ---- variable-size CSR results (setup path) ------------------------------
 * Producers return an opaque airg_csr_result held in library scratch;
 * airg_result_info gives its shape, the caller allocates ptr[nrows+1],
 * col[nnz], val[nnz] and airg_result_take copies them out and frees the
 * result (val may be NULL to drop values). */
typedef struct airg_csr_result airg_csr_result;
int airg_result_info(airg_csr_result* r, int32_t* nrows_h, int32_t* ncols_h, int64_t* nnz_h);
int airg_result_take(airg_csr_result* r, int32_t* ptr, int32_t* col, double* val, void* stream);
int airg_result_free(airg_csr_result* r);
/* Zero-copy hand-over: the result's three device buffers (library pool)
 * become the caller's; each is returned with airg_buffer_free when the
 * caller is done (val is NULL for a pattern-only result).  The result is
 * ready on `stream` when this returns. */
int airg_result_detach(airg_csr_result* r, int32_t** ptr, int32_t** col, double** val, void* stream);
int airg_buffer_free(void* p, void* stream);

/* numpy Generator(PCG64(SeedSequence(seed))) stream: out[i] = a + b*random()_i
 * (a=0,b=1: .random(n); a=-1,b=2: .uniform(-1,1,n)); the 128-bit state and
 * increment come from the host's SeedSequence.  ref: polynomial.py:61-65,
 * splitting.py:119 */
int airg_pcg64_fill(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                    int64_t n, double a, double b, double* out, void* stream);

/* Random unit vector: uniform(-1, 1, n) / ||.|| (norm_h may be NULL).
 * ref: polynomial.py:61-65 */
int airg_random_unit(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                     int64_t n, double* out, double* norm_h, void* stream);
/* Pre-grow the library's stream-ordered scratch pool by `bytes` (kept mapped). */
int airg_reserve(int64_t bytes, void* stream);
/* Main diagonal (structurally missing entries are 0).  ref: sparse.py:360-367 */
int airg_diagonal(int n, const int32_t* p, const int32_t* c, const double* v, double* d,
                  void* stream);

/* 2-D upwind advection stencil (nnz = n + [vx>0](nx-1)ny + [vy>0]nx(ny-1)).
 * ref: problems.py:48-85 */
int airg_advection_2d(int nx, int ny, double vx, double vy, int32_t* ptr, int32_t* col,
                      double* val, void* stream);

/* ---- CF splitting (splitting.py:86-238) --------------------------------- */
/* S and pattern(S + S^T) with unit values.  ref: splitting.py:86-109 */
int airg_strength(int n, const int32_t* ptr, const int32_t* col, const double* val, int64_t nnz,
                  double theta, airg_csr_result** S_out, airg_csr_result** closure_out,
                  void* stream);
/* Luby rounds on a symmetric closure; labels int8 F=0 / C=1; max_loops<0 =
 * unlimited.  ref: splitting.py:127-159 */
int airg_pmisr(int n, const int32_t* cptr, const int32_t* ccol, uint64_t state_hi,
               uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int max_loops,
               int8_t* labels, int32_t* loops_h, void* stream);
/* strength + closure + PMISR fused (closure never leaves the library). */
int airg_cf_pmisr(int n, const int32_t* ptr, const int32_t* col, const double* val, int64_t nnz,
                  double theta, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                  uint64_t inc_lo, int max_loops, int8_t* labels, int32_t* loops_h, void* stream);
/* One DDC pass, labels updated in place; stats_h[6] = n_f_before, converted,
 * ratio_min, ratio_max, ratio_mean, cut.  ref: splitting.py:162-207 */
int airg_ddc_pass(int n, const int32_t* ptr, const int32_t* col, const double* val, int8_t* labels,
                  double fraction, int nbins, double* stats_h, void* stream);
/* pos[i] = rank of i inside its class; f_idx / c_idx = sorted index sets
 * (any of the three may be NULL).  ref: splitting.py:53-58 (CFSplit.from_labels) */
int airg_split_index(int n, const int8_t* labels, int32_t* pos, int32_t* f_idx, int32_t* c_idx,
                     int32_t* nf_h, void* stream);
/* F rows without a C coupling become C.  ref: hierarchy.py:289-305 */
int airg_repair_split(int n, const int32_t* ptr, const int32_t* col, int8_t* labels,
                      int32_t* changed_h, void* stream);
/* One-point prolongator column per row (coarse numbering).  ref: hierarchy.py:250-278 */
int airg_prolong_onepoint(int n, const int32_t* ptr, const int32_t* col, const double* val,
                          const int8_t* labels, const int32_t* pos, int32_t* pcol, void* stream);

/* ---- sparse products (sparse.py:222-352, polynomial.py:372-416) ---------- */
/* C = A B (m x k times k x n), structural pattern with cancellation zeros
 * kept, entries summed k-ascending with separate roundings (== scipy
 * csr_matmat); negate=1 stores -C (hierarchy.py:200-202,236). */
int airg_spgemm(int m, int k, int n, const int32_t* Ap, const int32_t* Ac, const double* Av,
                const int32_t* Bp, const int32_t* Bc, const double* Bv, int negate,
                airg_csr_result** out, void* stream);
/* A B restricted to the stored positions of pattern P.  ref: sparse.py:243-263 */
int airg_spgemm_masked(int m, int k, int n, const int32_t* Ap, const int32_t* Ac, const double* Av,
                       const int32_t* Bp, const int32_t* Bc, const double* Bv, const int32_t* Pp,
                       const int32_t* Pc, airg_csr_result** out, void* stream);
/* sum_k c_k mask(A^k), mask = pattern(A) + diagonal, exact zeros pruned.
 * ref: polynomial.py:372-416 (arnoldi_coeff kind) */
int airg_poly_assemble(int n, const int32_t* Ap, const int32_t* Ac, const double* Av, int ncoef,
                       const double* coef_h, const int32_t* Qp, const int32_t* Qc,
                       airg_csr_result** out, void* stream);
/* Neumann base I + (-D^-1 A) with exact zeros pruned (the mask for its
 * powers is pattern(A) + diag: pass A as Q to airg_poly_assemble), and the
 * final right scaling v *= ds[col].  ref: polynomial.py:396-415 */
int airg_neumann_base(int n, const int32_t* p, const int32_t* c, const double* v,
                      const double* diag_scale, airg_csr_result** out, void* stream);
int airg_scale_columns(int64_t nnz, const int32_t* c, const double* diag_scale, double* v,
                       void* stream);
/* Row-relative drop (+ sequential lump onto the diagonal); changed_h = any
 * entry dropped.  ref: sparse.py:307-352 */
int airg_drop_lump(int m, int ncols, const int32_t* p, const int32_t* c, const double* v,
                   double tol, int lump, airg_csr_result** out, int32_t* changed_h, void* stream);
/* Galerkin coarse matrix drop_and_lump(R (A P), a_drop, lump) with the
 * one-point P given as pcol[n]; the drop/lump runs in the numeric epilogue.
 * ref: hierarchy.py:281-286 */
int airg_galerkin(int n, int nc, const int32_t* Rp, const int32_t* Rc, const double* Rv,
                  const int32_t* Ap, const int32_t* Ac, const double* Av, const int32_t* pcol,
                  double a_drop, int lump, airg_csr_result** out, void* stream);
/* 2-D upwind DG advection operator (nodal Q1 at the cell corners, 4 unknowns per
 * cell, cell e = j*nx + i, unknown 4e + d) from the host-computed 4x4 cell
 * blocks blocks_h[48] = {D, W, S} row-major (own cell, west and south
 * inflow neighbours).  SURVEY 8(d) cfg 5 (no reference generator). */
int airg_advection_dg(int nx, int ny, const double* blocks_h, int west, int south,
                      airg_csr_result** out, void* stream);
/* A P for the one-point prolongator P[j, pcol[j]] = 1 (A: m x k, pcol[k],
 * result m x nc): columns mapped and merged, values summed in A's column
 * order, cancellation zeros kept.  ref: hierarchy.py:281-286 (A @ P),
 * sparse.py:222-240 */
int airg_ap_onepoint(int m, int k, int nc, const int32_t* Ap, const int32_t* Ac, const double* Av,
                     const int32_t* pcol, airg_csr_result** out, void* stream);
/* A[rows, cols] with colmap[old col] = new col or -1.  ref: sparse.py:278-304 */
int airg_extract(int nr_sel, const int32_t* rows, const int32_t* p, const int32_t* c,
                 const double* v, const int32_t* colmap, int ncols_sel, airg_csr_result** out,
                 void* stream);
/* the same with A's mean row length (nnz / rows) as a hint: lanes per row */
int airg_extract_ex(int nr_sel, const int32_t* rows, const int32_t* p, const int32_t* c,
                    const double* v, const int32_t* colmap, int ncols_sel, double mean_len,
                    airg_csr_result** out, void* stream);
/* map[i] = labels[i] == which ? pos[i] : -1 */
int airg_label_colmap(int n, const int8_t* labels, int which, const int32_t* pos, int32_t* map,
                      void* stream);
/* R = [Z | I] scattered into the fine ordering.  ref: hierarchy.py:239-244 */
int airg_restriction(int n, int nc, const int32_t* zp, const int32_t* zc, const double* zv,
                     const int32_t* f_idx, const int32_t* c_idx, airg_csr_result** out,
                     void* stream);

/* ---- row-strip (multi-GPU) variants --------------------------------------
 * A rank owns global rows [row0, row0 + n); column ids are global or
 * renumbered to the extended space [local | ghost].  Same per-row semantics
 * as the serial entry points (hence bitwise-identical hierarchies). */
/* rows [row_begin, row_end) of the 2-D stencil; ptr == NULL: nnz query */
int airg_advection_2d_rows(int nx, int ny, double vx, double vy, int64_t row_begin, int64_t row_end,
                           int32_t* ptr, int32_t* col, double* val, int64_t* nnz_h, void* stream);
/* strong couplings of local rows (global column ids).  ref: splitting.py:86-104 */
int airg_strength_rows(int n, int row0, const int32_t* ptr, const int32_t* col, const double* val,
                       int64_t nnz, double theta, airg_csr_result** S_out, void* stream);
/* union of two row-sorted patterns (closure S + S^T).  ref: splitting.py:106 */
int airg_union_rows(int n, const int32_t* ap, const int32_t* ac, const int32_t* bp, const int32_t* bc,
                    airg_csr_result** out, void* stream);
/* Luby weights of local rows at their global stream positions.  ref: splitting.py:119-120 */
int airg_luby_weights(int n, int64_t row0, const int32_t* cptr, uint64_t state_hi, uint64_t state_lo,
                      uint64_t inc_hi, uint64_t inc_lo, double* w, void* stream);
/* one half-round of PMISR on ext arrays (phase 0 select, 1 block).  ref: splitting.py:144-157 */
int airg_luby_round(int n, const int32_t* cptr, const int32_t* ccol_ext, const double* w_ext,
                    const int32_t* gid_ext, int8_t* st_ext, int mark, int phase, int32_t* remaining_h,
                    void* stream);
int airg_luby_finish(int n, const int8_t* st, int8_t* labels, void* stream);
/* DDC pieces (ratios + local min/max/sum, histogram over host edges, convert).
 * ref: splitting.py:162-203 */
int airg_ddc_ratios(int nf, int row0, const int32_t* f_loc, const int32_t* ptr, const int32_t* col_ext,
                    const double* val, const int8_t* labels_ext, double* ratio, int32_t* bad_h,
                    double* minmaxsum_h, void* stream);
int airg_ddc_hist(int nf, const double* ratio, const double* edges_h, int nedges, uint64_t* hist,
                  void* stream);
/* converted_h may be NULL (no host read, no stream synchronisation) */
int airg_ddc_convert(int nf, const int32_t* f_loc, const double* ratio, double cut, int all,
                     int8_t* labels, int32_t* converted_h, void* stream);
/* elements [start, start+n) of the PCG64 stream (a + b*random()) */
int airg_pcg64_fill_at(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                       int64_t start, int64_t n, double a, double b, double* out, void* stream);
/* C = A B (mode 0, optional negate) or drop_and_lump(A B) (mode 1) with the
 * diagonal of local output row i at column row0 + i. */
int airg_spgemm_ex(int m, int k, int n, const int32_t* Ap, const int32_t* Ac, const double* Av,
                   const int32_t* Bp, const int32_t* Bc, const double* Bv, int negate, int mode,
                   double tol, int lump, int row0, airg_csr_result** out, void* stream);
/* fixed-sparsity assembly of local rows [0, n) (global row row0 + i); rows
 * of A beyond n are fetched ghost rows, rowmap[global col] -> row of A. */
int airg_poly_assemble_ex(int n, int row0, const int32_t* Ap, const int32_t* Ac, const double* Av,
                          const int32_t* rowmap, int ncoef, const double* coef_h,
                          const int32_t* Qp, const int32_t* Qc, airg_csr_result** out,
                          void* stream);
/* out[i] = map[in[i]] (negative ids pass through) */
int airg_gather_int(int64_t n, const int32_t* in, const int32_t* map, int32_t* out, void* stream);

/* ---- Krylov (polynomial.py:68-110) --------------------------------------
 * MGS Arnoldi from start vector b (device), m = min(order+1, n) steps, one
 * reorthogonalisation sweep when ||w|| < 0.7 ||A v||, lucky breakdown at
 * h_{j+1,j} <= 1e-14 max column norm.  H_h receives the (m+1) x m block
 * (row-major), k_h the achieved dimension, beta_h = ||b||. */
int airg_arnoldi(int n, const int32_t* p, const int32_t* c, const double* v, const double* b,
                 int m, double* H_h, int32_t* k_h, double* beta_h, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AIRG_H */
