// Few-right-hand-side kernels: the HODLR solve sweep (src/hodlr.py:285-306 ->
// Coupling.correct :129-134) and the dense operator GEMV (src/cli.py:320-321).
// These are HBM-bound: every stored factor byte is read once per application.
#include <stdlib.h>

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
// Columns are processed in groups of up to 4 per pass over the row, so the
// row of A is streamed from HBM once per 4 right-hand sides; per column the
// summation (two interleaved partial sums, then the warp tree) is the same as
// for s = 1, so a column's result does not depend on s.
template <int CG>
__device__ __forceinline__ void gemv_row_group(const double* __restrict__ a, const double* __restrict__ x,
                                               int64_t ldx, int64_t n, int lane, double (&res)[CG]) {
  double acc0[CG], acc1[CG];
#pragma unroll
  for (int c = 0; c < CG; ++c) acc0[c] = acc1[c] = 0.0;
  int64_t j = lane;
  for (; j + 32 < n; j += 64) {
    const double a0 = a[j], a1 = a[j + 32];
#pragma unroll
    for (int c = 0; c < CG; ++c) {
      acc0[c] += a0 * x[c * ldx + j];
      acc1[c] += a1 * x[c * ldx + j + 32];
    }
  }
  for (; j < n; j += 32) {
    const double a0 = a[j];
#pragma unroll
    for (int c = 0; c < CG; ++c) acc0[c] += a0 * x[c * ldx + j];
  }
#pragma unroll
  for (int c = 0; c < CG; ++c) res[c] = warp_sum(acc0[c] + acc1[c]);
}

__global__ void __launch_bounds__(MV_NT) gemv_rm_kernel(const double* __restrict__ A, int64_t lda,
                                                        int64_t m, int64_t n,
                                                        const double* __restrict__ x, int64_t ldx,
                                                        int64_t s, double* __restrict__ y,
                                                        int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (MV_NT / 32) + (threadIdx.x >> 5);
  if (row >= m) return;
  const double* a = A + row * lda;
  int64_t c0 = 0;
  for (; c0 + 4 <= s; c0 += 4) {
    double r[4];
    gemv_row_group<4>(a, x + c0 * ldx, ldx, n, lane, r);
    if (lane == 0)
      for (int c = 0; c < 4; ++c) y[row + (c0 + c) * ldy] = r[c];
  }
  for (; c0 < s; ++c0) {
    double r[1];
    gemv_row_group<1>(a, x + c0 * ldx, ldx, n, lane, r);
    if (lane == 0) y[row + c0 * ldy] = r[0];
  }
}

// ---------------------------------------------------------------------------
// Split skinny kernels (few-RHS solve sweep, s <= 16).
//
// pdot: item = (task, 256-row chunk, 32-column block); warp w owns 4 columns,
// each lane 8 rows of the chunk, so every thread keeps 32 independent
// coalesced loads in flight; x's chunk is staged in SMEM.  The per-(column,
// rhs) warp sums go to a partial array -- the reduction over row chunks
// happens in fixed order in the consumer (deterministic).
__device__ __forceinline__ void pdot_item(const PdotTask* __restrict__ tasks,
                                          const int32_t* __restrict__ items, int item, int s,
                                          double* __restrict__ xs) {
  const int ti = items[3 * item], ch = items[3 * item + 1], cb = items[3 * item + 2];
  const PdotTask t = tasks[ti];
  const int lane = threadIdx.x & 31, warp = uniform_warp_id();
  const int row0 = ch * HK_PDOT_ROWS;
  const int nr = min(HK_PDOT_ROWS, t.rows - row0);
  // the M loads go out first, so their latency overlaps the x staging
  const int k0 = cb * HK_PDOT_COLS + warp * 4;
  const int nk = max(0, min(4, t.cols - k0));
  double m[4][8];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = lane + 32 * u;
      m[j][u] = (j < nk && i < nr) ? t.M[row0 + i + (int64_t)(k0 + j) * t.ldm] : 0.0;
    }
  griddep_wait();                              // x is the previous phase's output
  for (int idx = threadIdx.x; idx < nr * s; idx += 256) {
    const int i = idx % nr, r = idx / nr;
    xs[r * HK_PDOT_ROWS + i] = t.x[row0 + i + (int64_t)r * t.ldx];
  }
  __syncthreads();
  if (nk == 0) return;
  for (int r = 0; r < s; ++r) {
    double xr[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = lane + 32 * u;
      xr[u] = i < nr ? xs[r * HK_PDOT_ROWS + i] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = fma(m[j][u], xr[u], acc);
      acc = warp_sum(acc);
      if (lane == 0 && j < nk) t.P[((int64_t)ch * t.cols + k0 + j) * s + r] = acc;
    }
  }
}

__global__ void __launch_bounds__(256) pdot_kernel(const PdotTask* __restrict__ tasks,
                                                   const int32_t* __restrict__ items, int s) {
  __shared__ double xs[HK_PDOT_ROWS * 16];
  griddep_launch();
  pdot_item(tasks, items, blockIdx.x, s, xs);
}

// sgemv: item = (task, 32-row block); warp q sums the columns k = q, q+8, ...
// of its 32 rows (each load a coalesced 256-byte row segment, 8 loads in
// flight per thread), the eight partial sums are combined in fixed order
// through SMEM.  v (K x s) is first staged in SMEM -- directly, or as the
// fixed-order reduction of partial-dot chunks.
__device__ __forceinline__ void sgemv_item(const SgemvTask* __restrict__ tasks,
                                           const int32_t* __restrict__ items, int item, int s,
                                           double* __restrict__ vs) {
  constexpr int QS = 256 / HK_SGEMV_ROWS;   // column residue classes (= warps)
  const int ti = items[2 * item], rb = items[2 * item + 1];
  const SgemvTask t = tasks[ti];
  // vs: v (K * s), then partials [QS][HK_SGEMV_ROWS][s]
  const int K = t.K;
  const int q = threadIdx.x >> 5, il = threadIdx.x & 31;
  const int i = rb * HK_SGEMV_ROWS + il;
  const bool live = i < t.rows;
  const double* mrow = t.M + i;
  // the first PF matrix entries of this thread go out before v is staged;
  // later chunks of PF are issued together (PF loads in flight per thread)
  constexpr int PF = 16;
  double mpre[PF];
#pragma unroll
  for (int u = 0; u < PF; ++u) {
    const int k = q + u * QS;
    mpre[u] = (live && k < K) ? mrow[(int64_t)k * t.ldm] : 0.0;
  }
  griddep_wait();                              // v / partials / y come from earlier phases
  // fixed-order sum over the partial-dot chunks, 8 independent loads at a time
  auto chunk_sum = [](const double* __restrict__ P, int nch, int64_t stride, int64_t off) {
    double v = 0.0;
    int c = 0;
    for (; c + 8 <= nch; c += 8) {
      double tt[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) tt[u] = P[(int64_t)(c + u) * stride + off];
#pragma unroll
      for (int u = 0; u < 8; ++u) v += tt[u];
    }
    for (; c < nch; ++c) v += P[(int64_t)c * stride + off];
    return v;
  };
  for (int idx = threadIdx.x; idx < K * s; idx += 256) {
    const int k = idx % K, r = idx / K;
    double v;
    if (t.v0) {
      v = t.v0[k + (int64_t)r * t.ldv];
    } else if (k < t.KA) {
      v = chunk_sum(t.PA, t.nchA, (int64_t)t.KA * s, (int64_t)k * s + r);
    } else {
      const int KB = K - t.KA, kb = k - t.KA;
      v = chunk_sum(t.PB, t.nchB, (int64_t)KB * s, (int64_t)kb * s + r);
    }
    vs[r * K + k] = v;
  }
  __syncthreads();
  double* part = vs + K * s;
  for (int r0 = 0; r0 < s; r0 += 4) {
    const int rs = min(4, s - r0);
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    if (live) {
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int k = q + u * QS;
        if (k < K) {
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (r < rs) a[r] = fma(mpre[u], vs[(r0 + r) * K + k], a[r]);
        }
      }
      for (int kk = q + PF * QS; kk < K; kk += PF * QS) {
        double mv[PF];
#pragma unroll
        for (int u = 0; u < PF; ++u) {
          const int k = kk + u * QS;
          mv[u] = k < K ? mrow[(int64_t)k * t.ldm] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PF; ++u) {
          const int k = kk + u * QS;
          if (k < K) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
              if (r < rs) a[r] = fma(mv[u], vs[(r0 + r) * K + k], a[r]);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (r < rs) part[(q * HK_SGEMV_ROWS + il) * s + r0 + r] = a[r];
  }
  __syncthreads();
  if (threadIdx.x < HK_SGEMV_ROWS && live) {
    for (int r = 0; r < s; ++r) {
      double v = 0.0;
#pragma unroll
      for (int qq = 0; qq < QS; ++qq) v += part[(qq * HK_SGEMV_ROWS + il) * s + r];
      double* y = t.y + i + (int64_t)r * t.ldy;
      if (t.mode == 0) *y = v;
      else *y -= v;
    }
  }
}

__global__ void __launch_bounds__(256) sgemv_kernel(const SgemvTask* __restrict__ tasks,
                                                    const int32_t* __restrict__ items, int s) {
  extern __shared__ double vs[];
  griddep_launch();
  sgemv_item(tasks, items, blockIdx.x, s, vs);
}

// Dense GEMV for the GMRES operator (src/cli.py:320-321): y(m x s) = A x with
// A row-major.  Each warp owns RW rows and walks them together with 16-byte
// loads (lane l covers columns 2l + 64t, 2l + 64t + 1), so every x chunk it
// loads is reused by RW rows; U chunks of A are issued before any is
// consumed (U * RW independent 16-byte loads in flight per lane).  Columns
// are processed in groups of up to 4.  Per (row, column) the summation order
// is fixed -- t ascending, two interleaved partials per lane, then the warp
// tree -- independent of s, RW and U, so every variant gives the same bits.
// RW = 4, U = 1 for the large fronts (one pass over A per 4 right-hand sides
// at the HBM roofline); RW = 1, U = 8 for small ones, where 4 rows per warp
// left too few warps and a 16-deep chain of dependent round trips per lane.
template <int RW, int CG, int U>
__device__ __forceinline__ void gemv_group(const double* __restrict__ A, int64_t lda, int64_t row0,
                                           int64_t m, int64_t n, const double* __restrict__ x,
                                           int64_t ldx, int lane, double (&res)[RW][CG],
                                           bool& waited) {
  double acc[RW][CG];
#pragma unroll
  for (int r = 0; r < RW; ++r)
#pragma unroll
    for (int c = 0; c < CG; ++c) acc[r][c] = 0.0;
  const double* a[RW];
#pragma unroll
  for (int r = 0; r < RW; ++r) a[r] = A + (row0 + r < m ? row0 + r : row0) * lda;
  for (int64_t j0 = 2 * lane; j0 < n; j0 += 64 * U) {
    double2 av[U][RW];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + 64 * u;
#pragma unroll
      for (int r = 0; r < RW; ++r)
        av[u][r] = j < n ? __ldcs(reinterpret_cast<const double2*>(a[r] + j)) : make_double2(0.0, 0.0);
    }
    if (!waited) {                     // the operator is independent of the previous kernel, x is not
      griddep_wait();
      waited = true;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + 64 * u;
      if (j >= n) break;
      double2 xv[CG];
#pragma unroll
      for (int c = 0; c < CG; ++c) xv[c] = *reinterpret_cast<const double2*>(x + c * ldx + j);
#pragma unroll
      for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int c = 0; c < CG; ++c)
          acc[r][c] = fma(av[u][r].y, xv[c].y, fma(av[u][r].x, xv[c].x, acc[r][c]));
    }
  }
#pragma unroll
  for (int r = 0; r < RW; ++r)
#pragma unroll
    for (int c = 0; c < CG; ++c) res[r][c] = warp_sum(acc[r][c]);
}

template <int RW, int U4, int U1>
__global__ void __launch_bounds__(MV_NT) gemv4_kernel(const double* __restrict__ A, int64_t lda,
                                                      int64_t m, int64_t n,
                                                      const double* __restrict__ x, int64_t ldx,
                                                      int64_t s, double* __restrict__ y, int64_t ldy) {
  griddep_launch();
  const int lane = threadIdx.x & 31;
  const int64_t row0 = ((int64_t)blockIdx.x * (MV_NT / 32) + (threadIdx.x >> 5)) * RW;
  bool waited = false;
  if (row0 < m) {
    int64_t c0 = 0;
    for (; c0 + 4 <= s; c0 += 4) {
      double r[RW][4];
      gemv_group<RW, 4, U4>(A, lda, row0, m, n, x + c0 * ldx, ldx, lane, r, waited);
      if (lane == 0)
        for (int q = 0; q < RW; ++q)
          if (row0 + q < m)
            for (int c = 0; c < 4; ++c) y[row0 + q + (c0 + c) * ldy] = r[q][c];
    }
    for (; c0 < s; ++c0) {
      double r[RW][1];
      gemv_group<RW, 1, U1>(A, lda, row0, m, n, x + c0 * ldx, ldx, lane, r, waited);
      if (lane == 0)
        for (int q = 0; q < RW; ++q)
          if (row0 + q < m) y[row0 + q + c0 * ldy] = r[q][0];
    }
  }
  if (!waited) griddep_wait();
}

// launch with programmatic dependent launch (HK_PDL=0 turns it off): the
// kernel may start while its predecessor in the stream drains and must
// griddep_wait() before reading the predecessor's output
static bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HK_PDL");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
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
  const bool vec = (n % 2 == 0) && (lda % 2 == 0) && (ldx % 2 == 0) &&
                   ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(x)) & 15) == 0;
  if (vec) {   // 16-byte loads
    cudaError_t e;
    if (m <= 8192) {            // one row per warp, 8 chunks in flight per lane
      const int64_t blocks = (m + MV_NT / 32 - 1) / (MV_NT / 32);
      e = launch_pdl(gemv4_kernel<1, 4, 8>, dim3((unsigned)blocks), dim3(MV_NT), 0, st, A, lda, m, n,
                     x, ldx, s, y, ldy);
    } else {                    // 4 rows per warp: x reuse, HBM-bound
      const int64_t rows_per_cta = (MV_NT / 32) * 4;
      const int64_t blocks = (m + rows_per_cta - 1) / rows_per_cta;
      e = launch_pdl(gemv4_kernel<4, 1, 1>, dim3((unsigned)blocks), dim3(MV_NT), 0, st, A, lda, m, n,
                     x, ldx, s, y, ldy);
    }
    hk_count_launch();
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  int64_t blocks = (m + MV_NT / 32 - 1) / (MV_NT / 32);
  gemv_rm_kernel<<<(unsigned)blocks, MV_NT, 0, st>>>(A, lda, m, n, x, ldx, s, y, ldy);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_pdot(const PdotTask* tasks, const int32_t* items, int nitems, int s,
                           cudaStream_t st) {
  if (nitems == 0) return cudaSuccess;
  const cudaError_t e = launch_pdl(pdot_kernel, dim3(nitems), dim3(256), 0, st, tasks, items, s);
  hk_count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t hk_launch_sgemv(const SgemvTask* tasks, const int32_t* items, int nitems, int s,
                            int max_k, cudaStream_t st) {
  if (nitems == 0) return cudaSuccess;
  const size_t smem = ((size_t)max_k * s + 256 * (size_t)s) * 8;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(sgemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  const cudaError_t e = launch_pdl(sgemv_kernel, dim3(nitems), dim3(256), smem, st, tasks, items, s);
  hk_count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

