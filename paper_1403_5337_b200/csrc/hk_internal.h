// Internal task descriptors and kernel launchers (host side of the .cu files).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// ---------------------------------------------------------------- ACA
struct AcaTask {
  const double* A;   // block origin in the row-major front: A[i*lda + j]
  const double* At;  // block origin in the transposed front: column j of the block = At + j*lda
  double* U;         // m x cap column-major, leading dimension 1 << ldu
  double* V;         // n x cap column-major, leading dimension 1 << ldv
  int32_t* rank;     // out
  int32_t* trace;    // optional: [0]=#rows, [1]=#cols, rows[m+cap+1], cols[cap+1]
  int64_t* clock;    // optional profiling probe: [start ns, end ns, smid]
  double* scratch;   // hk_aca_scratch_doubles(cap): per-warp dot partials
  int64_t lda;
  int32_t m, n, cap;
  int32_t ldu, ldv;  // log2 of the leading dimensions (6..13)
};

// ---------------------------------------------------------------- BDLR skeleton
struct SkelTask {
  const double* A;      // block origin (row-major, lda)
  int64_t lda;
  const int64_t* rsel;  // selected row positions (k)
  const int64_t* csel;  // selected column positions (kc)
  double* work;         // k x kc scratch (row-major, ld kc)
  int64_t* rperm;       // k
  int64_t* cperm;       // kc
  double* U;            // m x cap column-major, leading dimension ldu
  double* V;            // n x cap column-major, leading dimension ldv
  int32_t* rank;        // out
  int32_t* status;      // out: 0 ok, HK_ERR_DEGENERATE
  int32_t ldu, ldv;
  const int64_t* probe; // degenerate-check probe rows (nprobe)
  int32_t nprobe;
  int32_t m, n, k, kc, cap;
  double tol;
};

// ---------------------------------------------------------------- BDLR selection (select.cu)
struct SelTask {      // one side of one block: own range vs other range
  int64_t own0, oth0;
  int32_t n_own, n_oth;
  int64_t* out;       // capacity n_own: selected positions, (d, position) order
  int32_t* count;
};
cudaError_t hk_launch_select(const SelTask* tasks_dev, int ntasks, int max_own,
                             const int64_t* indptr_dev, const int64_t* indices_dev, int depth,
                             cudaStream_t st);

// ---------------------------------------------------------------- dense LU + inverse
// Partial-pivot LU of an N x N matrix assembled from a source, with explicit
// inverse.  mode 0: source is a row-major block (src, src_ld).  mode 1:
// Schur/coupling matrix S = I + off-diagonal blocks read from H (see lu.cu).
struct LuTask {
  const double* src;
  int64_t src_ld;
  double* lu;       // N x N column-major packed LU (ld N)
  int32_t* perm;    // N: row_perm (P A)[k] = A[perm[k]]
  int32_t* ipiv;    // N: LAPACK-style swap index of step k (0-based)
  double* inv;      // N x N column-major inverse (ld N), may be null
  int32_t* status;  // out: 0 ok, 1 singular
  int32_t N;
  int32_t mode;
  int32_t rl, ru;   // mode 1: ranks (S is (rl+ru)^2)
  int64_t h_col0;   // mode 1: first column of the coupling block in H (= w)
};

// ---------------------------------------------------------------- batched GEMM
// C(m x n) = alpha * op(A) * B + beta * C, all column-major.
// transA = 0: op(A)[i][l] = A[i + l*lda]; transA = 1: op(A)[i][l] = A[l + i*lda].
struct GemmTask {
  const double* A;
  const double* B;
  double* C;
  int64_t lda, ldb, ldc;
  int32_t m, n, k;
  int32_t transA;
  int32_t vec;      // 1: A, B 16-byte aligned with even leading dimensions (16-byte cp.async)
  int32_t pad_;
  double alpha, beta;
  double diag;      // added to C(i,i) after alpha*op(A)*B + beta*C
};

// ---------------------------------------------------------------- copies
struct CopyTask {  // dst(i, j) = src(i, j), element (i, j) at p[i*rs + j*cs]
  const double* src;
  double* dst;
  int64_t src_rs, src_cs, dst_rs, dst_cs;
  int32_t rows, cols;
};

// ---------------------------------------------------------------- small-s solve
struct MatVecTask {  // y(rows x s) (op)= M(rows x K) * x(K x s), all column-major
  const double* M;
  const double* x;
  double* y;
  int64_t ldm, ldx, ldy;
  int32_t rows, K;
  int32_t mode;     // 0: y = M x ; 1: y -= M x
  int32_t pad;
};
struct DotTask {     // y[k*ldy + c] = dot(M[:,k], x[:,c]) for k < cols, column-major M (rows x cols)
  const double* M;
  const double* x;
  double* y;
  int64_t ldm, ldx, ldy;
  int32_t rows, cols;
};

// Split skinny kernels of the few-RHS solve (s <= 16).  Work is cut into
// items small enough that every level of the sweep fills the GPU.
struct PdotTask {    // partial dots P[(c*cols + k)*s + r] = sum_{i in row chunk c} M[i,k] x[i,r]
  const double* M;   // rows x cols, column-major, ld ldm
  const double* x;   // rows x s, ld ldx
  double* P;         // [nchunks][cols][s]
  int64_t ldm, ldx;
  int32_t rows, cols;
};
struct SgemvTask {   // y[i,r] (op)= sum_k M[i,k] v[k,r] for i < rows, M column-major rows x K
  const double* M;
  int64_t ldm;
  // v: either direct (v0 = K x s, ld ldv) or the reduction of partial-dot
  // blocks: v[k] = sum_c PA[(c*KA + k)*s + r] for k < KA, then PB for the rest
  const double* v0;
  int64_t ldv;
  const double* PA;
  const double* PB;
  int32_t KA, nchA, nchB;
  int32_t mode;      // 0: y = M v ; 1: y -= M v
  double* y;
  int64_t ldy;
  int32_t rows, K;
};
constexpr int HK_PDOT_ROWS = 256;   // rows per partial-dot chunk
constexpr int HK_PDOT_COLS = 32;    // columns per partial-dot item
constexpr int HK_SGEMV_ROWS = 32;   // rows per sgemv item
cudaError_t hk_launch_pdot(const PdotTask* tasks, const int32_t* items, int nitems, int s,
                           cudaStream_t st);
cudaError_t hk_launch_sgemv(const SgemvTask* tasks, const int32_t* items, int nitems, int s,
                            int max_k, cudaStream_t st);

cudaError_t hk_launch_h2d_stream(const void* src_host, void* dst_dev, int64_t bytes, int ctas,
                                 cudaStream_t st);

// launchers (return cudaError_t)
cudaError_t hk_launch_transpose(const double* A, double* At, int64_t n, int64_t ld, int64_t batch,
                                int64_t stride, cudaStream_t st);
cudaError_t hk_launch_aca(const AcaTask* tasks_dev, int ntasks, int max_cap, int max_m,
                          double tol2, cudaStream_t st, int max_mn);
size_t hk_aca_scratch_doubles(int cap);
// cluster ACA for large blocks (one block per cluster of P CTAs)
int hk_aca_cluster_size(int m, int n);   // 1 = single-CTA size class
size_t hk_aca_scratch_doubles_cl(int cap, int P);
cudaError_t hk_launch_aca_cluster(const AcaTask* tasks_dev, int ntasks, int P, int max_cap,
                                  int max_m, double tol2, cudaStream_t st, int* started,
                                  int* max_active);
int hk_aca_class(int m, int n);   // 0..3 -> 512/256/128/64-thread CTAs
cudaError_t hk_launch_aca_classes(const AcaTask* tasks_dev, const int* class_begin,
                                  const int* class_max_cap, const int* class_max_m, double tol2,
                                  int* counters_dev, cudaStream_t* streams);
cudaError_t hk_launch_skeleton(const SkelTask* tasks_dev, int ntasks, int max_k, int max_kc,
                               int max_m, int max_n, cudaStream_t st);
cudaError_t hk_launch_lu(const LuTask* tasks_dev, int ntasks, int maxN, cudaStream_t st);
cudaError_t hk_launch_gemm(const GemmTask* tasks_dev, const int32_t* tilemap_dev, int ntiles,
                           cudaStream_t st);
cudaError_t hk_launch_copy(const CopyTask* tasks_dev, int ntasks, cudaStream_t st);
cudaError_t hk_launch_matvec(const MatVecTask* tasks_dev, int ntasks, int s, int max_rows,
                             cudaStream_t st, int max_k);
cudaError_t hk_launch_dot(const DotTask* tasks_dev, int ntasks, int s, int max_cols,
                          cudaStream_t st);
cudaError_t hk_launch_lu_full(double* a, int64_t m, int64_t n, int64_t ld, int64_t* rp,
                              int64_t* cp, double* piv, int64_t* npiv_dev, cudaStream_t st);
cudaError_t hk_launch_gemv_rowmajor(const double* A, int64_t lda, int64_t m, int64_t n,
                                    const double* x, int64_t ldx, int64_t s, double* y,
                                    int64_t ldy, cudaStream_t st);
cudaError_t hk_launch_fill(double* p, int64_t n, double v, cudaStream_t st);

// krylov helpers (krylov.cu)
cudaError_t hk_launch_arnoldi(int64_t n, int64_t j, int64_t mmax, double* basis, double* hess,
                              double* cs, double* sn, double* g, double* w, double beta,
                              double* out_dev, cudaStream_t st);
cudaError_t hk_launch_combine(int64_t n, int64_t m, int64_t mmax, const double* basis,
                              const double* hess, const double* g, double* x, double* y_scratch,
                              cudaStream_t st);
cudaError_t hk_launch_norm(const double* x, int64_t n, double* out, cudaStream_t st);
cudaError_t hk_launch_arnoldi_batch(int64_t n, int64_t j, int64_t mmax, double* basis,
                                    int64_t bstride, double* hess, int64_t hstride, double* cs,
                                    double* sn, double* g, double* w, const double* beta,
                                    double* out, const int32_t* active, int s, cudaStream_t st);
cudaError_t hk_launch_norms(const double* x, int64_t n, int64_t ld, int s, double* out,
                            cudaStream_t st);
cudaError_t hk_launch_scale(const double* x, int64_t n, const double* num, double* y,
                            int invert, cudaStream_t st);
cudaError_t hk_launch_axpby(const double* x, const double* y, double* z, int64_t n, double a,
                            double b, cudaStream_t st);
cudaError_t hk_launch_diag_scale(const double* A, int64_t lda, const double* x, double* y,
                                 int64_t n, cudaStream_t st);

void hk_count_launch(int k = 1);

// ---------------------------------------------------------------- device-resident GMRES
// State of up to HK_GM_MAXS systems advanced in lock step by one CUDA graph
// whose conditional WHILE node runs the Arnoldi iteration until every system
// has converged, broken down or hit the iteration cap (krylov.py:107-145):
// the host reads this struct once, after the loop.
constexpr int HK_GM_MAXS = 16;
struct GmState {
  int32_t k;          // iterations completed (the loop's k, 1-based after the first)
  int32_t cont;       // loop condition of the last control step
  int32_t finished;   // no active system left, or k == mmax
  int32_t counter;    // last-CTA-done counter of the Arnoldi / start kernels
  int32_t active[HK_GM_MAXS], m[HK_GM_MAXS], conv[HK_GM_MAXS], brk[HK_GM_MAXS];
  int32_t zero[HK_GM_MAXS];   // ||b|| == 0: x = 0, converged, 0 iterations (krylov.py:85-87)
  int32_t err[HK_GM_MAXS];    // preconditioned rhs exactly zero (krylov.py:91-92)
  double nb[HK_GM_MAXS], beta[HK_GM_MAXS], tres[HK_GM_MAXS];
  double out[3 * HK_GM_MAXS]; // rel, happy, breakdown of each system's last Arnoldi step
};
struct GmParams {
  int64_t n, cap, mmax, max_iter;   // cap: basis columns - 1 currently allocated
  int32_t s, pad_;
  double tol;
  double* basis;  int64_t bstride;  // system c: n x (cap+1), column-major, at basis + c*bstride
  double* hess;   int64_t hstride;  // (cap+1) x cap per system
  double *cs, *sn, *g;  int64_t vs; // cap+1 per system
  double* V;                        // n x s: the vector the next GEMV multiplies
  double* hist;                     // s x max_iter preconditioned residual history
  double* y;                        // s x vs back-substitution scratch
  GmState* st;
};
// start: per system, q0 = r0 / beta (r0 = column c of R0, n x s ld n), g[0] = beta,
// then the first loop-condition evaluation
cudaError_t hk_launch_gm_start(const GmParams& P, const double* R0, cudaGraphConditionalHandle h,
                               cudaStream_t st);
// one Arnoldi/MGS/Givens step of every active system on W (n x s, ld n), then
// (last CTA) the convergence bookkeeping and the loop condition
cudaError_t hk_launch_gm_arnoldi(const GmParams& P, double* W, cudaGraphConditionalHandle h,
                                 cudaStream_t st);
// x_c = basis_c y_c after back substitution (krylov.py:147-154), when finished
cudaError_t hk_launch_gm_combine(const GmParams& P, double* X, cudaStream_t st);
// true residuals ||b_c - (A x)_c|| / ||b_c|| (krylov.py:152-156), when finished
cudaError_t hk_launch_gm_resid(const GmParams& P, const double* B, const double* AX, cudaStream_t st);
// y[c*n + i] = x[c*n + i] / d[i] for s columns (DiagonalPreconditioner, krylov.py:58-62)
cudaError_t hk_launch_vdiv(const double* x, const double* d, double* y, int64_t n, int s,
                           cudaStream_t st);

// ---------------------------------------------------------------- Gauss-Jordan inverse
// In-place Gauss-Jordan with partial (row) pivoting -> explicit inverse.
// Pivots equal those of LU with partial pivoting (rows >= k see the same
// updates), so the singularity test min|pivot| < 1e-300 matches dense.py:76.
struct GjTask {
  const double* src;   // mode 0: row-major (src[i*ld + j]); mode 1: column-major (src[i + j*ld])
  int64_t src_ld;
  double* out;         // column-major inverse, leading dimension out_ld
  int64_t out_ld;
  double* scratch;     // hk_gj_scratch_bytes(N) used when N is too large for SMEM (else null)
  int32_t* status;     // 0 ok, 1 singular
  int32_t* near;       // optional: set to 1 when some |pivot| < HK_NEAR_PIVOT (not singular)
  int32_t N;
  int32_t mode;
};
// A Gauss-Jordan pivot below this (absolute) magnitude makes the factorization
// re-decide the coupling system's singularity with the reference's own
// partial-pivot LU of S (hodlr.py:272-277; api.cpp hk_factor_ext).
#define HK_NEAR_PIVOT 1e-8
cudaError_t hk_launch_gj(const GjTask* tasks_dev, int ntasks, int maxN, cudaStream_t st);
// leaf inverses (N <= 64, mode 0 blocks of the fronts) staged by the TMA; tmap is
// a CUtensorMap (128 bytes) from hk_gj_leaf_map over the same fronts
cudaError_t hk_launch_gj_leaf_tma(const GjTask* tasks_dev, int ntasks, const void* tmap,
                                  const double* base, int64_t lda, int64_t fstride,
                                  cudaStream_t st);
int hk_gj_leaf_map(void* out, const double* base, int64_t n, int64_t lda, int64_t fstride,
                   int64_t batch);   // 0 on success
size_t hk_gj_scratch_bytes(int N);     // 0 when N fits SMEM

// ---------------------------------------------------------------- validation (validate.cpp)
// HK_VALIDATE=1: every staged task's memory regions are checked against the
// device allocation that holds them, and the library's own buffers become
// plain cudaMalloc allocations (exact ranges); see validate.cpp.
bool hk_validate_enabled();
cudaError_t hk_dev_malloc_raw(void** p, size_t bytes, cudaStream_t st);
cudaError_t hk_dev_free(void* p, cudaStream_t st);
template <class T>
inline cudaError_t hk_dev_malloc(T** p, size_t bytes, cudaStream_t st) {
  return hk_dev_malloc_raw(reinterpret_cast<void**>(p), bytes, st);
}
void hk_validate(const GemmTask& t);
void hk_validate(const CopyTask& t);
void hk_validate(const AcaTask& t);
void hk_validate(const SkelTask& t);
void hk_validate(const GjTask& t);
void hk_validate(const LuTask& t);
void hk_validate(const PdotTask& t);
void hk_validate(const SgemvTask& t);
void hk_validate(const MatVecTask& t);
void hk_validate(const DotTask& t);
void hk_validate(const SelTask& t);
template <class T>
inline void hk_validate(const T&) {}   // index arrays and other plain data

