// Batched variable-size FP64 GEMM on the DMMA tensor pipe (mma.sync m8n8k4
// .f64 -> DMMA.8x8x4; tcgen05 has no f64 kind on sm_100a).
//
// Every contraction of the HODLR factorization is one of these tasks
// (SURVEY.md §2.3 K9/K11/K13): the coupling assembly V^T [c | d], the
// coupling solve S^{-1} rhs, the correction c -= d y, and the leaf solve
// K_leaf^{-1} Z.  One launch covers every node of a level across every front;
// each CTA computes one 64x64 tile of one task (tile list built on the host).
#include "hk_common.cuh"
#include "hk_internal.h"

namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 128, PAD = 4;

__global__ void __launch_bounds__(NT) gemm_kernel(const GemmTask* __restrict__ tasks,
                                                  const int32_t* __restrict__ tilemap) {
  const int task = tilemap[3 * blockIdx.x];
  const int tm = tilemap[3 * blockIdx.x + 1];
  const int tn = tilemap[3 * blockIdx.x + 2];
  const GemmTask t = tasks[task];
  __shared__ double As[2][BK][BM + PAD];
  __shared__ double Bs[2][BK][BN + PAD];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  const int m0 = tm * BM, n0 = tn * BN;
  const int M = t.m, N = t.n, K = t.k;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double ra[8], rb[8];
  auto load_regs = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = tid + NT * q;
      int i, l;
      if (!t.transA) { i = idx % BM; l = idx / BM; }
      else { i = idx / BK; l = idx % BK; }
      const int gi = m0 + i, gl = k0 + l;
      double v = 0.0;
      if (gi < M && gl < K)
        v = t.transA ? t.A[gl + (int64_t)gi * t.lda] : t.A[gi + (int64_t)gl * t.lda];
      ra[q] = v;
      const int l2 = idx % BK, j2 = idx / BK;
      const int gj = n0 + j2, gl2 = k0 + l2;
      rb[q] = (gj < N && gl2 < K) ? t.B[gl2 + (int64_t)gj * t.ldb] : 0.0;
    }
  };
  auto store_regs = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = tid + NT * q;
      int i, l;
      if (!t.transA) { i = idx % BM; l = idx / BM; }
      else { i = idx / BK; l = idx % BK; }
      As[buf][l][i] = ra[q];
      Bs[buf][idx % BK][idx / BK] = rb[q];
    }
  };

  const int nk = (K + BK - 1) / BK;
  if (nk > 0) {
    load_regs(0);
    store_regs(0);
  }
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load_regs((kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][kk + tig][wm * 32 + i * 8 + gid];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[buf][kk + tig][wn * 32 + j * 8 + gid];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    if (kt + 1 < nk) store_regs(buf ^ 1);
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + gid;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * 32 + j * 8 + 2 * tig + h;
        if (col >= N) continue;
        double* c = t.C + row + (int64_t)col * t.ldc;
        double v = t.alpha * acc[i][j][h];
        if (t.beta != 0.0) v += t.beta * (*c);
        if (row == col) v += t.diag;
        *c = v;
      }
    }
  }
}

__global__ void copy_kernel(const CopyTask* __restrict__ tasks) {
  const CopyTask t = tasks[blockIdx.y];
  const int64_t tot = (int64_t)t.rows * t.cols;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % t.rows), j = (int)(idx / t.rows);
    t.dst[i + (int64_t)j * t.ld_dst] = t.src[i + (int64_t)j * t.ld_src];
  }
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace

cudaError_t hk_launch_gemm(const GemmTask* tasks_dev, const int32_t* tilemap_dev, int ntiles,
                           cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  gemm_kernel<<<ntiles, NT, 0, st>>>(tasks_dev, tilemap_dev);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_copy(const CopyTask* tasks_dev, int ntasks, cudaStream_t st) {
  if (ntasks == 0) return cudaSuccess;
  copy_kernel<<<dim3(16, ntasks), 256, 0, st>>>(tasks_dev);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_fill(double* p, int64_t n, double v, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  fill_kernel<<<blocks, 256, 0, st>>>(p, n, v);
  hk_count_launch();
  return cudaGetLastError();
}
