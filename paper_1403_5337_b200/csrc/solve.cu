// Few-right-hand-side kernels: the HODLR solve sweep (src/hodlr.py:285-306 ->
// Coupling.correct :129-134) and the dense operator GEMV (src/cli.py:320-321).
// These are HBM-bound: every stored factor byte is read once per application.
#include "hk_common.cuh"
#include "hk_internal.h"

namespace {

constexpr int MV_NT = 256;

// y(rows x s) = M x  or  y -= M x; M column-major rows x K; thread per row.
// x is staged in SMEM (K x s); launched with grid (row chunks, tasks).
__global__ void __launch_bounds__(MV_NT) matvec_kernel(const MatVecTask* __restrict__ tasks, int s) {
  const MatVecTask t = tasks[blockIdx.y];
  extern __shared__ double xs[];   // K * s
  const int K = t.K;
  for (int idx = threadIdx.x; idx < K * s; idx += MV_NT) {
    const int l = idx % K, c = idx / K;
    xs[idx] = t.x[l + (int64_t)c * t.ldx];
  }
  __syncthreads();
  const int i = blockIdx.x * MV_NT + threadIdx.x;
  if (i >= t.rows) return;
  const double* mrow = t.M + i;
  for (int c0 = 0; c0 < s; c0 += 4) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const int cs = s - c0 < 4 ? s - c0 : 4;
    const double* x0 = xs + (int64_t)c0 * K;
    for (int l = 0; l < K; ++l) {
      const double mv = mrow[(int64_t)l * t.ldm];
      a0 += mv * x0[l];
      if (cs > 1) a1 += mv * x0[l + K];
      if (cs > 2) a2 += mv * x0[l + 2 * K];
      if (cs > 3) a3 += mv * x0[l + 3 * K];
    }
    double acc[4] = {a0, a1, a2, a3};
    for (int c = 0; c < cs; ++c) {
      double* y = t.y + i + (int64_t)(c0 + c) * t.ldy;
      if (t.mode == 0) *y = acc[c];
      else *y -= acc[c];
    }
  }
}

// y[k + c*ldy] = M[:,k] . x[:,c], warp per column k; grid (k chunks, tasks).
__global__ void __launch_bounds__(MV_NT) dot_kernel(const DotTask* __restrict__ tasks, int s) {
  const DotTask t = tasks[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (MV_NT / 32) + (threadIdx.x >> 5);
  if (k >= t.cols) return;
  const double* mk = t.M + (int64_t)k * t.ldm;
  for (int c = 0; c < s; ++c) {
    const double* xc = t.x + (int64_t)c * t.ldx;
    double acc = 0.0;
    for (int i = lane; i < t.rows; i += 32) acc += mk[i] * xc[i];
    acc = warp_sum(acc);
    if (lane == 0) t.y[k + (int64_t)c * t.ldy] = acc;
  }
}

// y(m x s, col-major) = A(m x n, row-major) x(n x s, col-major); warp per row.
__global__ void __launch_bounds__(MV_NT) gemv_rm_kernel(const double* __restrict__ A, int64_t lda,
                                                        int64_t m, int64_t n,
                                                        const double* __restrict__ x, int64_t ldx,
                                                        int64_t s, double* __restrict__ y,
                                                        int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (MV_NT / 32) + (threadIdx.x >> 5);
  if (row >= m) return;
  const double* a = A + row * lda;
  for (int64_t c = 0; c < s; ++c) {
    const double* xc = x + c * ldx;
    double acc0 = 0.0, acc1 = 0.0;
    int64_t j = lane;
    for (; j + 32 < n; j += 64) {
      acc0 += a[j] * xc[j];
      acc1 += a[j + 32] * xc[j + 32];
    }
    for (; j < n; j += 32) acc0 += a[j] * xc[j];
    double acc = warp_sum(acc0 + acc1);
    if (lane == 0) y[row + c * ldy] = acc;
  }
}

}  // namespace

cudaError_t hk_launch_matvec(const MatVecTask* tasks_dev, int ntasks, int s, int max_rows,
                             cudaStream_t st, int max_k) {
  if (ntasks == 0 || max_rows == 0) return cudaSuccess;
  size_t smem = (size_t)max_k * s * 8;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(matvec_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((max_rows + MV_NT - 1) / MV_NT, ntasks);
  matvec_kernel<<<grid, MV_NT, smem, st>>>(tasks_dev, s);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_dot(const DotTask* tasks_dev, int ntasks, int s, int max_cols,
                          cudaStream_t st) {
  if (ntasks == 0 || max_cols == 0) return cudaSuccess;
  dim3 grid((max_cols + MV_NT / 32 - 1) / (MV_NT / 32), ntasks);
  dot_kernel<<<grid, MV_NT, 0, st>>>(tasks_dev, s);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_gemv_rowmajor(const double* A, int64_t lda, int64_t m, int64_t n,
                                    const double* x, int64_t ldx, int64_t s, double* y,
                                    int64_t ldy, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  int64_t blocks = (m + MV_NT / 32 - 1) / (MV_NT / 32);
  gemv_rm_kernel<<<(unsigned)blocks, MV_NT, 0, st>>>(A, lda, m, n, x, ldx, s, y, ldy);
  hk_count_launch();
  return cudaGetLastError();
}
