/*
 * hodlr_b200.h -- C ABI of the B200-native HODLR hot path.
 *
 * Drop-in boundary for the compute path of hodlrkit 0.1.0
 * (/root/reference/pkg/src/hodlrkit).  The reference has no FFI of its own:
 * its boundary is the Python API re-exported by src/__init__.py:11-125.
 * Each entry point below names the reference function it replaces
 * (file:line, paths relative to pkg/src/hodlrkit/).  The Python package
 * paper_1403_5337_b200 binds these with ctypes (INTEGRATION.md shows the
 * binding); nothing here uses torch types.
 *
 * Conventions
 *   - All floating point is IEEE fp64.  Matrices passed in are ROW-MAJOR
 *     (C order, like the numpy arrays the reference passes around) unless a
 *     parameter says column-major.
 *   - Pointers named *_dev are device pointers; *_host are host pointers.
 *   - `stream` is a cudaStream_t passed as void*; NULL = legacy default stream.
 *   - Every function returns an hk_status; hk_last_error() gives a message.
 *   - A plan is used by one host thread at a time (SPEC: factorizations are
 *     immutable after factor; solve is re-entrant across rhs, not threads).
 */
#ifndef HODLR_B200_H
#define HODLR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* Status codes map 1:1 onto the reference exception classes (src/errors.py). */
typedef enum {
  HK_OK = 0,
  HK_ERR_VALUE = 1,              /* ValueError (bad config, non-finite input)       */
  HK_ERR_DIMENSION = 2,          /* DimensionMismatchError        errors.py:43       */
  HK_ERR_SINGULAR = 3,           /* SingularMatrixError           errors.py:8        */
  HK_ERR_SINGULAR_LEAF = 4,      /* SingularLeafError             errors.py:12       */
  HK_ERR_SINGULAR_SCHUR = 5,     /* SingularSchurError            errors.py:16       */
  HK_ERR_DEGENERATE = 6,         /* DegenerateSkeletonError       errors.py:32       */
  HK_ERR_BREAKDOWN = 7,          /* GmresBreakdownError           errors.py:39       */
  HK_ERR_EMPTY_SELECTION = 8,    /* EmptySelectionError           errors.py:28       */
  HK_ERR_CUDA = 20,              /* CUDA runtime failure / no device                 */
  HK_ERR_STATE = 21              /* call order violated (e.g. solve before factor)   */
} hk_status;

typedef enum { HK_SCHEME_SVD = 0, HK_SCHEME_ACA = 1, HK_SCHEME_BDLR = 2 } hk_scheme;

typedef struct hk_plan hk_plan;

/* Message of the last failing call on this thread. */
const char* hk_last_error(void);
/* Library version string "hodlr_b200 <semver> sm_100a". */
const char* hk_version(void);
/* Number of visible CUDA devices (0 on a host without a GPU; never fails). */
int hk_device_count(void);

/* ------------------------------------------------------------------------
 * Plans: one bisection tree (build_tree, hodlr.py:76-102) shared by `batch`
 * independent fronts of order n.  Front f lives at fronts_dev + f*front_stride.
 * ---------------------------------------------------------------------- */
hk_status hk_plan_create(int64_t n, int64_t leaf_threshold, int64_t batch, hk_plan** out);
hk_status hk_plan_destroy(hk_plan* plan);
/* Tree in preorder: level, lo, hi, left, right per node (left=-1 for a leaf).
 * Arrays must hold hk_plan_num_nodes() entries.  Mirrors HodlrTree.nodes. */
int64_t   hk_plan_num_nodes(const hk_plan* plan);
hk_status hk_plan_tree(const hk_plan* plan, int32_t* level, int64_t* lo, int64_t* hi,
                       int32_t* left, int32_t* right);

/* ------------------------------------------------------------------------
 * Build: compress both off-diagonal blocks of every internal node of every
 * front (factorize -> compress, hodlr.py:239-242; lowrank.py:353-359).
 * Blocks are numbered 2*k (upper, rows=left child, cols=right child) and
 * 2*k+1 (lower) for the k-th internal node in preorder.
 * ---------------------------------------------------------------------- */
/* ACA, lowrank.py:230-286.  tol2 = tol**2 computed by the caller (the
 * reference evaluates cfg.tol ** 2 in Python).  max_rank <= 0 = no cap.
 * record_trace != 0 keeps the per-block pivot trace (hk_get_aca_trace). */
hk_status hk_build_aca(hk_plan* plan, const double* fronts_dev, int64_t ld,
                       int64_t front_stride, double tol, double tol2, int64_t max_rank,
                       int record_trace, void* stream);
/* BDLR, lowrank.py:334-350 + graph.py:171-228.  One symmetric CSR graph in
 * front order (no self loops) shared by all fronts. */
hk_status hk_build_bdlr(hk_plan* plan, const double* fronts_dev, int64_t ld,
                        int64_t front_stride, double tol, int32_t depth, int64_t max_rank,
                        const int64_t* indptr_host, const int64_t* indices_host,
                        void* stream);
/* Externally computed factors (the parity-only svd scheme, lowrank.py:221-227):
 * declare the fronts, then set every block's factor from column-major device
 * buffers U (m x rank, ld_u) and V (n x rank, ld_v). */
hk_status hk_build_external_begin(hk_plan* plan, const double* fronts_dev, int64_t ld,
                                  int64_t front_stride, void* stream);
hk_status hk_set_block_factor(hk_plan* plan, int64_t front, int64_t block, int64_t rank,
                              const double* U_dev, int64_t ld_u, const double* V_dev,
                              int64_t ld_v, void* stream);

/* Ranks after a build, [batch][2*num_internal] (blocks as above). */
hk_status hk_get_ranks(hk_plan* plan, int32_t* ranks_host);
/* ACA trace of one block: rows read (in order) and columns read, as the
 * reference's BlockAccessor.row/.col see them (lowrank.py:253, :266). */
hk_status hk_get_aca_trace(hk_plan* plan, int64_t front, int64_t block, int32_t* rows_host,
                           int64_t* nrows, int32_t* cols_host, int64_t* ncols);
/* BDLR skeleton of one block: rank and the skeleton row/column positions
 * row_sel[row_perm[:r]], col_sel[col_perm[:r]] (lowrank.py:311, :317). */
hk_status hk_get_skeleton(hk_plan* plan, int64_t front, int64_t block, int64_t* rank,
                          int64_t* rows_host, int64_t* cols_host, int64_t cap);
/* Column-major factors of one block into host buffers (m x rank, n x rank). */
hk_status hk_get_block_factor(hk_plan* plan, int64_t front, int64_t block,
                              double* U_host, double* V_host);
/* Geometry of one block: m, n and the rank cap. */
hk_status hk_block_shape(const hk_plan* plan, int64_t block, int64_t* m, int64_t* n,
                         int64_t* cap);

/* ------------------------------------------------------------------------
 * Factor (factorize, hodlr.py:183-282): batched leaf LU, then one upward
 * level sweep of coupling assembly, coupling LU and correction.
 * ---------------------------------------------------------------------- */
hk_status hk_factor(hk_plan* plan, void* stream);
/* Factor with an external extension (HODLR-subtree sharding):
 * the plan covers one subtree of a larger front, and Zext (n x wext,
 * column-major, ld ldz, device) holds the U factors of the subtree's
 * top-level ancestors restricted to its rows, farthest ancestor first -- the
 * columns _factorize_node passes down as `ext` (hodlr.py:244-245, :280-282).
 * On return the extension holds K_T^{-1} Zext in its first wext columns.
 * batch must be 1.  hk_factor(plan) == hk_factor_ext(plan, NULL, 0, 0). */
hk_status hk_factor_ext(hk_plan* plan, const double* Zext, int64_t ldz, int64_t wext,
                        void* stream);
/* Device view of a front's extension buffer Y (n x width, column-major,
 * ld = n): columns [0, wext) after hk_factor_ext, then the d blocks of every
 * internal node (Coupling.d_left / d_right, hodlr.py:105-134). */
hk_status hk_get_extension(hk_plan* plan, int64_t front, double** Y, int64_t* ld,
                           int64_t* width);
/* Copy columns [col0, col0 + ncols) of a front's extension buffer into dst
 * (n x ncols, column-major, ld ldd, device). */
hk_status hk_copy_extension(hk_plan* plan, int64_t front, int64_t col0, int64_t ncols,
                            double* dst, int64_t ldd, void* stream);
/* C = alpha op(A) B + beta C on the FP64 tensor pipe (column-major; op(A) = A^T
 * when transa != 0) -- the `@` of the top-level coupling terms of a sharded
 * factorization (hodlr.py:131-134, :270-271). */
hk_status hk_dgemm(int transa, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                   int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                   void* stream);
/* Batched explicit inverses with implicit partial pivoting (Gauss-Jordan) --
 * the kernel behind every leaf and capacitance inverse of the factorization
 * (replaces lu_partial(...) of hodlr.py:225 and :273, dense.py:59-81;
 * singular iff min |pivot| < 1e-300 as dense.py:76-77).  A: `batch` row-major
 * n x n device matrices (leading dimension lda, matrix stride `stride`
 * elements); out: column-major device inverses, leading dimension n, stride
 * n*n; status_host[b] = 1 when matrix b is singular. */
hk_status hk_gj_inverse(const double* A, int64_t n, int64_t lda, int64_t batch, int64_t stride,
                        double* out, int32_t* status_host, void* stream);

/* In-place inverses of `batch` symmetric positive definite n x n matrices
 * (leading dimension lda, matrix stride `stride` elements) by block
 * Gauss-Jordan with 64 x 64 pivot blocks (128 for n > 2048) on the DMMA GEMM; status_host[b] = 1
 * if a pivot block of matrix b was singular.  Replaces torch.linalg.solve
 * (cuSOLVER) in the plane-by-plane front elimination (frontgen.py; the
 * reference's dense elimination src/frontgen.py:159-189). */
hk_status hk_spd_inverse(double* A, int64_t n, int64_t lda, int64_t batch, int64_t stride,
                         int32_t* status_host, void* stream);
/* Factor views for the test-visible attributes of HodlrFactorization
 * (hodlr.py:105-154): leaf LU (b x b row-major packed, LAPACK-style 0-based
 * swap indices `piv`) and per internal node d_left (na x r_u), d_right
 * (nb x r_l), Schur LU ((r_l+r_u)^2) -- all row-major host copies, computed on
 * demand by the partial-pivot LU kernel.  inv_host / schur_inv_host (may be
 * NULL) receive the row-major inverse, which PartialPivLU.solve applies. */
hk_status hk_get_leaf_lu(hk_plan* plan, int64_t front, int64_t node, double* lu_host,
                         int32_t* perm_host, double* inv_host);
hk_status hk_get_coupling(hk_plan* plan, int64_t front, int64_t node, double* d_left_host,
                          double* d_right_host, double* schur_lu_host, int32_t* schur_perm_host,
                          double* schur_inv_host);

/* ------------------------------------------------------------------------
 * Solve (solve, hodlr.py:285-306) in place on device right-hand sides of
 * every front: rhs front f = rhs_dev + f*rhs_stride, column-major n x nrhs
 * with leading dimension ld.
 * ---------------------------------------------------------------------- */
hk_status hk_solve(hk_plan* plan, double* rhs_dev, int64_t ld, int64_t nrhs,
                   int64_t rhs_stride, void* stream);
/* Solve for one front only (the GMRES preconditioner of that front). */
hk_status hk_solve_front(hk_plan* plan, int64_t front, double* rhs_dev, int64_t ld,
                         int64_t nrhs, void* stream);

/* ------------------------------------------------------------------------
 * GMRES (krylov.py:69-166): left preconditioned, no restart, MGS with one
 * conditional re-orthogonalisation, Givens, true-residual guard.
 * Operator: the dense row-major front A_dev, n x n with leading dimension
 * lda (cli.py:320-321 `dense @ v`).  precond: 0 = none, 1 = the plan's HODLR
 * solve for `front`, 2 = division by diag_dev (n entries, zeros already
 * replaced by 1: DiagonalPreconditioner, krylov.py:44-62).  n must equal the
 * plan's order (HK_ERR_DIMENSION otherwise: the reference's solve() raises
 * DimensionMismatchError, hodlr.py:291-293).
 * The whole iteration runs on the device: one CUDA graph whose conditional
 * WHILE node repeats GEMV -> preconditioner -> Arnoldi until every system has
 * converged; the host synchronises once, after the loop.
 * ---------------------------------------------------------------------- */
/* s (1..16) right-hand sides, s independent GMRES runs in lock step: one
 * s-column GEMV and one s-column HODLR solve per iteration, batched Arnoldi.
 * Per-system results equal s separate hk_gmres calls.  B, X: n x s (ld n),
 * device; iterations[s], history[s * max_iter] (row c = rhs c),
 * true_residual[s], flags[2s] (converged, breakdown per rhs), all host.
 * SURVEY.md §8(f)#3. */
hk_status hk_gmres_batch(hk_plan* plan, int64_t front, const double* A_dev, int64_t lda, int64_t n,
                         const double* B_dev, int64_t s, double tol, int64_t max_iter,
                         int precond, const double* diag_dev, double* X_dev, int64_t* iterations,
                         double* history, double* true_residual, int32_t* flags, void* stream);
/* One right-hand side: history_host holds max_iter doubles, flags_host[0] =
 * converged, [1] = breakdown. */
hk_status hk_gmres(hk_plan* plan, int64_t front, const double* A_dev, int64_t lda, int64_t n,
                   const double* b_dev, double tol, int64_t max_iter, int precond,
                   const double* diag_dev, double* x_dev, int64_t* iterations,
                   double* history_host, double* true_residual, int32_t* flags_host, void* stream);

/* Building blocks for GMRES with arbitrary operator callables. */
/* One Arnoldi/MGS/Givens column update for column j (krylov.py:110-145):
 * w_dev holds M^{-1} A v_j on entry.  basis n x (m+1) col-major (ld = n),
 * hess (m+1) x m col-major, cs/sn/g device arrays.  out_host: [0]=rel,
 * [1]=happy, [2]=breakdown.  beta = ||r0||. */
hk_status hk_arnoldi_step(int64_t n, int64_t j, int64_t mmax, double* basis_dev,
                          double* hess_dev, double* cs_dev, double* sn_dev, double* g_dev,
                          double* w_dev, double beta, double* out_host, void* stream);
/* s systems' column updates in one launch, device-only (no host sync): system
 * c lives at basis_dev + c*bstride, hess_dev + c*hstride, cs/sn/g_dev +
 * c*(mmax+1), w_dev + c*n, beta_dev[c]; out_dev[3c..3c+2] = rel, happy,
 * breakdown; systems with active_dev[c] == 0 are skipped.  Used by the
 * sharded (multi-GPU) GMRES, whose operator and preconditioner are
 * collectives, to advance all right-hand sides with one readback per step. */
hk_status hk_arnoldi_step_batch(int64_t n, int64_t j, int64_t mmax, double* basis_dev,
                                int64_t bstride, double* hess_dev, int64_t hstride, double* cs_dev,
                                double* sn_dev, double* g_dev, double* w_dev,
                                const double* beta_dev, double* out_dev, const int32_t* active_dev,
                                int64_t s, void* stream);
/* Back substitution + x = basis[:, :m] y (krylov.py:147-154). */
hk_status hk_gmres_combine(int64_t n, int64_t m, int64_t mmax, const double* basis_dev,
                           const double* hess_dev, const double* g_dev, double* x_dev,
                           void* stream);

/* ------------------------------------------------------------------------
 * Dense kernels (dense.py) and compression of a single block (lowrank.py).
 * ---------------------------------------------------------------------- */
/* dense @ x for row-major A (m x n) and column-major X (n x s): hodlr.py:309-316. */
/* Host -> device copy of `bytes` from pinned (UVA-mapped) host memory by a
 * `ctas`-CTA kernel with evict-first stores: streams the next batch of fronts
 * into HBM without displacing the L2 working set of the running build. */
hk_status hk_copy_h2d_streaming(const void* src_host, void* dst_dev, int64_t bytes, int ctas,
                                void* stream);
hk_status hk_gemv(const double* A_dev, int64_t lda, int64_t m, int64_t n, const double* x_dev,
                  int64_t ldx, int64_t s, double* y_dev, int64_t ldy, void* stream);
/* Complete-pivot LU (lu_full, dense.py:133-166), bit-exact pivot order.
 * a_dev row-major m x n (ld) is overwritten with the packed LU; perms 0-based;
 * pivots_dev receives |U_kk|; *npiv the number of pivots taken. */
hk_status hk_lu_full(double* a_dev, int64_t m, int64_t n, int64_t ld, int64_t* row_perm_dev,
                     int64_t* col_perm_dev, double* pivots_dev, int64_t* npiv, void* stream);
/* Partial-pivot LU (lu_partial, dense.py:59-81) with explicit inverse:
 * a_dev row-major n x n overwritten by the packed LU, perm 0-based row_perm,
 * inv_dev (may be NULL) receives A^{-1} row-major. HK_ERR_SINGULAR when
 * min|U_kk| < 1e-300. */
hk_status hk_lu_partial(double* a_dev, int64_t n, int64_t ld, int32_t* perm_dev,
                        double* inv_dev, void* stream);
/* ACA of one row-major block (compress_aca, lowrank.py:230-286). U, V are
 * column-major device buffers with room for `cap` columns. */
hk_status hk_aca_block(const double* a_dev, int64_t m, int64_t n, int64_t ld, double tol2,
                       int64_t cap, double* U_dev, double* V_dev, int64_t* rank,
                       int32_t* trace_rows_host, int64_t* nrows, int32_t* trace_cols_host,
                       int64_t* ncols, void* stream);

/* Pseudo-skeleton of one row-major block from given selections
 * (pseudo_skeleton, lowrank.py:289-331): complete-pivot LU of the skeleton
 * intersection, rank = #{|p_k| >= tol |p_0|} capped at cap, then
 * U = C U11^{-1} (m x rank) and V = (L11^{-1} R)^T (n x rank), column-major.
 * rows_out/cols_out (host, >= cap) receive the skeleton positions.
 * HK_ERR_DEGENERATE when rank 0 faces a numerically nonzero block. */
hk_status hk_skeleton_block(const double* a_dev, int64_t m, int64_t n, int64_t ld,
                            const int64_t* row_sel_host, int64_t k, const int64_t* col_sel_host,
                            int64_t kc, double tol, int64_t cap, double* U_dev, double* V_dev,
                            int64_t* rank, int64_t* rows_out, int64_t* cols_out, void* stream);

/* ------------------------------------------------------------------------
 * Graph selection (graph.py:171-228), host integer code, bit-exact.
 * ---------------------------------------------------------------------- */
/* Distances (graph.py:183-206) of `own` vertices to their boundary with
 * `other`, restricted to own; unreachable = -1. */
hk_status hk_graph_distance(int64_t nverts, const int64_t* indptr, const int64_t* indices,
                            const int64_t* own, int64_t n_own, const int64_t* other,
                            int64_t n_other, int64_t* dist_out);
/* select_by_depth (graph.py:209-228): positions ordered by (d, vertex id).
 * Returns HK_ERR_EMPTY_SELECTION when either side selects nothing. */
hk_status hk_select_by_depth(int64_t nverts, const int64_t* indptr, const int64_t* indices,
                             const int64_t* row_verts, int64_t n_rows, const int64_t* col_verts,
                             int64_t n_cols, int32_t depth, int64_t* row_sel, int64_t* n_row_sel,
                             int64_t* col_sel, int64_t* n_col_sel);

/* Timings of the last build/factor/solve on the plan's stream, in seconds
 * (keys of SolveReport.timings, hodlr.py:223-281): lowrank, leaf_lu, schur. */
hk_status hk_get_timings(hk_plan* plan, double* lowrank, double* leaf_lu, double* schur);

/* Device time of the last batched ACA launch alone (seconds), CUDA events
 * on the plan's stream around the single aca_kernel launch. */
hk_status hk_get_aca_time(hk_plan* plan, double* seconds);

/* Kernel launches issued by this library since load (evidence counter). */
int64_t hk_launch_count(void);

/* Task-extent validation (environment HK_VALIDATE=1, read once at first use):
 * every task array staged for a kernel is checked on the host against the
 * device allocations its matrix regions fall in (the substitute for
 * compute-sanitizer memcheck on this library's kernels; csrc/validate.cpp).
 * Returns the number of regions found outside their allocation since load;
 * *checked (optional) receives the number of regions checked.  No reference
 * counterpart (debugging aid). */
int64_t hk_debug_violations(int64_t* checked);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* HODLR_B200_H */
