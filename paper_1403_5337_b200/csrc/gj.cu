// Batched Gauss-Jordan inversion with partial pivoting (leaf blocks and the
// r x r Woodbury capacitance matrices I - Y X of the coupling systems).
//
// One CTA per matrix; the matrix lives in SMEM when it fits (N <= 165), else
// in a global scratch (L2 resident).  Each elimination step is one rank-1
// update of the whole N x N array, column-major with the row index fastest
// so SMEM accesses are conflict-free and global accesses coalesced.
#include "hk_common.cuh"
#include "hk_internal.h"

namespace {

constexpr int GJ_NT = 256;
constexpr size_t GJ_SMEM_CAP = 224 * 1024;

// workspace layout (SMEM or global scratch): W[N*N], colk[N], rowk[N] doubles,
// then piv[N], cperm[N] ints
__host__ __device__ inline size_t gj_bytes(int N) {
  return (size_t)N * N * 8 + (size_t)2 * N * 8 + (size_t)2 * N * 4;
}

// Register-resident Gauss-Jordan, N <= min(NW*CPW, 32*RPL).  The matrix is
// distributed column-cyclically: warp w holds columns j = w + NW*jj (jj < CPW),
// lane l holds rows i = l + 32*q (q < RPL), so W[i][j] lives in w_[jj][q] of
// warp j%NW / lane i%32.  Pivoting is implicit (no physical row swaps): step k
// takes the largest |W[i][k]| over rows not yet used as pivots (ties: lowest
// row), so the pivot magnitudes are those of LU with partial pivoting and the
// singularity test min|pivot| < 1e-300 is the reference's (dense.py:76-77).
// With pivot rows p_k the result satisfies A^{-1}[i][c] = W[p_i][q(c)],
// q = p^{-1}, applied by the final gather.  Per step: the owner warp of
// column k finds the pivot (shuffles), the lane holding row p publishes the
// scaled pivot row; every warp updates its columns in registers (one DFMA +
// one select per element).  Two barriers per step, double-buffered SMEM.
template <int NW, int CPW, int RPL>
__global__ void __launch_bounds__(NW * 32, 1) gj_reg_kernel(const GjTask* __restrict__ tasks) {
  constexpr int NT = NW * 32;
  const GjTask t = tasks[blockIdx.x];
  const int N = t.N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(16) double gsm[];   // stage N*N, colk[2][N], rowk[2][N]
  double* stage = gsm;
  double* colk = stage + N * N;
  double* rowk = colk + 2 * N;
  __shared__ int s_p[2], s_sing, pivrow[32 * RPL], invp[32 * RPL];
  __shared__ double s_rinv[2];
  __shared__ unsigned char usedrow[32 * RPL];
  if (N == 0) {
    if (tid == 0) *t.status = 0;
    return;
  }
  // load through SMEM (coalesced), then into registers
  if (t.mode == 0) {
    for (int i = warp; i < N; i += NW)
      for (int j = lane; j < N; j += 32) stage[i + j * N] = t.src[(int64_t)i * t.src_ld + j];
  } else {
    for (int j = warp; j < N; j += NW)
      for (int i = lane; i < N; i += 32) stage[i + j * N] = t.src[i + (int64_t)j * t.src_ld];
  }
  for (int i = tid; i < 32 * RPL; i += NT) usedrow[i] = 0;
  if (tid == 0) s_sing = 0;
  __syncthreads();
  double w_[CPW][RPL];
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q, j = warp + NW * jj;
      w_[jj][q] = (i < N && j < N) ? stage[i + j * N] : 0.0;
    }
  // k = w + NW*kk: the column slot kk of the owner warp is a compile-time
  // constant inside the unrolled kk loop (no register-array select chains)
#pragma unroll
  for (int kk = 0; kk < CPW; ++kk) {
    for (int w = 0; w < NW; ++w) {
      const int k = w + NW * kk;
      if (k >= N) break;
      const int buf = k & 1;
      double* ck_s = colk + buf * N;
      double* rk_s = rowk + buf * N;
      if (warp == w) {                // owner of column k: pivot over unused rows
        ArgMax a{0.0, -1};
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int i = lane + 32 * q;
          if (i < N) {
            ck_s[i] = w_[kk][q];
            if (!usedrow[i]) {
              const double av = fabs(w_[kk][q]);
              if (argmax_better(av, i, a.v, a.i)) { a.v = av; a.i = i; }
            }
          }
        }
        a = warp_argmax(a);
        if (lane == 0) {
          const int p = (int)a.i;
          s_p[buf] = p;
          if (!(a.v >= HK_PIVOT_FLOOR)) s_sing = 1;
          else {
            usedrow[p] = 1;
            pivrow[k] = p;
          }
        }
      }
      __syncthreads();
      if (s_sing) break;
      const int p = s_p[buf];
      const double rinv = 1.0 / ck_s[p];
      // pivot row of this warp's columns, published by the lane that holds row p
      const int qp = p >> 5;
      if (lane == (p & 31)) {
        switch (qp) {   // warp-uniform
#define HK_PUB(Q)                                                         \
  case Q:                                                                 \
    if (Q < RPL) {                                                        \
      _Pragma("unroll") for (int jj = 0; jj < CPW; ++jj) {               \
        const int j = warp + NW * jj;                                     \
        if (j < N) rk_s[j] = (j == k) ? rinv : w_[jj][Q < RPL ? Q : 0] * rinv; \
      }                                                                   \
    }                                                                     \
    break;
          HK_PUB(0) HK_PUB(1) HK_PUB(2) HK_PUB(3) HK_PUB(4) HK_PUB(5) HK_PUB(6) HK_PUB(7)
#undef HK_PUB
          default: break;
        }
      }
      __syncthreads();
      double ck[RPL];
      bool isp[RPL];
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        const int i = lane + 32 * q;
        ck[q] = (i < N) ? ck_s[i] : 0.0;
        isp[q] = (i == p);
      }
#pragma unroll
      for (int jj = 0; jj < CPW; ++jj) {
        const int j = warp + NW * jj;
        if (j >= N) break;
        const double rj = rk_s[j];
        if (jj == kk && warp == w) {
#pragma unroll
          for (int q = 0; q < RPL; ++q) w_[jj][q] = isp[q] ? rinv : -ck[q] * rinv;
        } else {
#pragma unroll
          for (int q = 0; q < RPL; ++q) {
            const double v = fma(-ck[q], rj, w_[jj][q]);
            w_[jj][q] = isp[q] ? rj : v;
          }
        }
      }
    }
  }
  if (tid == 0) *t.status = s_sing;
  if (s_sing) return;
  // ---- A^{-1}[i][c] = W[p_i][q(c)]
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q, j = warp + NW * jj;
      if (i < N && j < N) stage[i + j * N] = w_[jj][q];
    }
  for (int k = tid; k < N; k += NT) invp[pivrow[k]] = k;
  __syncthreads();
  for (int c = warp; c < N; c += NW) {
    const int qc = invp[c];
    double* dst = t.out + (int64_t)c * t.out_ld;
    for (int i = lane; i < N; i += 32) dst[i] = stage[pivrow[i] + qc * N];
  }
}

// SMEM-resident variant, N <= 32*MAXQ: every lane owns rows lane + 32q of the
// column its warp updates; the pivot column is cached in registers; all SMEM
// addressing is 32-bit.  Two barriers per elimination step.
template <int NT, int MAXQ>
__global__ void __launch_bounds__(NT) gj_smem_kernel(const GjTask* __restrict__ tasks) {
  const GjTask t = tasks[blockIdx.x];
  const int N = t.N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) double Ws[];   // N*N column-major, then rowk[N], colk[N]
  double* rowk = Ws + N * N;
  double* colk = rowk + N;
  __shared__ int piv[32 * MAXQ];
  __shared__ int cperm[32 * MAXQ];
  __shared__ int s_p, s_sing;
  __shared__ double s_rinv;
  if (N == 0) {
    if (tid == 0) *t.status = 0;
    return;
  }
  if (t.mode == 0) {
    for (int i = warp; i < N; i += NW)
      for (int j = lane; j < N; j += 32) Ws[i + j * N] = t.src[(int64_t)i * t.src_ld + j];
  } else {
    for (int j = warp; j < N; j += NW)
      for (int i = lane; i < N; i += 32) Ws[i + j * N] = t.src[i + (int64_t)j * t.src_ld];
  }
  __syncthreads();
  if (warp == 0) {
    ArgMax a{0.0, -1};
    for (int i = lane; i < N; i += 32) {
      const double v = fabs(Ws[i]);
      if (argmax_better(v, i, a.v, a.i)) { a.v = v; a.i = i; }
    }
    a = warp_argmax(a);
    if (lane == 0) {
      s_p = (int)a.i;
      s_sing = !(a.v >= HK_PIVOT_FLOOR);
    }
  }
  __syncthreads();
  for (int k = 0; k < N; ++k) {
    if (s_sing) break;
    const int p = s_p;
    for (int j = tid; j < N; j += NT) {
      const double wk = Ws[k + j * N];
      const double wp = Ws[p + j * N];
      rowk[j] = wp;
      if (p != k) Ws[p + j * N] = wk;
      if (j == k) s_rinv = 1.0 / wp;
    }
    for (int i = tid; i < N; i += NT) {
      double c;
      if (i == k) c = 0.0;
      else if (i == p) c = Ws[k + k * N];
      else c = Ws[i + k * N];
      colk[i] = c;
    }
    if (tid == 0) piv[k] = p;
    __syncthreads();
    const double rinv = s_rinv;
    double ck[MAXQ];
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int i = lane + 32 * q;
      ck[q] = (i < N) ? colk[i] : 0.0;
    }
    for (int j = warp; j < N; j += NW) {
      double* col = Ws + j * N;
      if (j == k) {
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
          const int i = lane + 32 * q;
          if (i < N) col[i] = (i == k) ? rinv : -ck[q] * rinv;
        }
        continue;
      }
      const double rj = rowk[j] * rinv;
      const bool nextcol = (j == k + 1);
      ArgMax a{0.0, -1};
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int i = lane + 32 * q;
        if (i < N) {
          const double v = (i == k) ? rj : col[i] - ck[q] * rj;
          col[i] = v;
          if (nextcol && i > k) {
            const double av = fabs(v);
            if (argmax_better(av, i, a.v, a.i)) { a.v = av; a.i = i; }
          }
        }
      }
      if (nextcol) {
        a = warp_argmax(a);
        if (lane == 0) {
          s_p = (int)a.i;
          s_sing = !(a.v >= HK_PIVOT_FLOOR);
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) *t.status = s_sing;
  if (s_sing) return;
  if (tid == 0) {
    for (int j = 0; j < N; ++j) cperm[j] = j;
    for (int k = N - 1; k >= 0; --k) {
      const int a = cperm[k];
      cperm[k] = cperm[piv[k]];
      cperm[piv[k]] = a;
    }
  }
  __syncthreads();
  for (int j = warp; j < N; j += NW) {
    const double* src = Ws + cperm[j] * N;
    double* dst = t.out + (int64_t)j * t.out_ld;
    for (int i = lane; i < N; i += 32) dst[i] = src[i];
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) gj_kernel(const GjTask* __restrict__ tasks, size_t smem_bytes) {
  const GjTask t = tasks[blockIdx.x];
  const int N = t.N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smraw[];
  const bool in_smem = gj_bytes(N) <= smem_bytes;
  double* W = in_smem ? reinterpret_cast<double*>(smraw) : t.scratch;
  double* colk = W + (size_t)N * N;
  double* rowk = colk + N;
  int* piv = reinterpret_cast<int*>(rowk + N);
  int* cperm = piv + N;
  __shared__ int s_p, s_sing;
  __shared__ double s_rinv;
  if (N == 0) {
    if (tid == 0) *t.status = 0;
    return;
  }
  if (t.mode == 0) {
    for (int i = warp; i < N; i += NW)                          // coalesced row-major read
      for (int j = lane; j < N; j += 32) W[i + (int64_t)j * N] = t.src[(int64_t)i * t.src_ld + j];
  } else {
    for (int j = warp; j < N; j += NW)
      for (int i = lane; i < N; i += 32) W[i + (int64_t)j * N] = t.src[i + (int64_t)j * t.src_ld];
  }
  __syncthreads();
  // pivot of step 0
  if (warp == 0) {
    ArgMax a{0.0, -1};
    for (int i = lane; i < N; i += 32) {
      const double v = fabs(W[i]);
      if (argmax_better(v, i, a.v, a.i)) { a.v = v; a.i = i; }
    }
    a = warp_argmax(a);
    if (lane == 0) {
      s_p = (int)a.i;
      s_sing = !(a.v >= HK_PIVOT_FLOOR);
    }
  }
  __syncthreads();
  for (int k = 0; k < N; ++k) {
    if (s_sing) break;
    const int p = s_p;
    // gather the swapped pivot row / column; move old row k into row p
    for (int j = tid; j < N; j += NT) {
      const double wk = W[k + (int64_t)j * N];
      const double wp = W[p + (int64_t)j * N];
      rowk[j] = wp;
      if (p != k) W[p + (int64_t)j * N] = wk;
      if (j == k) s_rinv = 1.0 / wp;
    }
    for (int i = tid; i < N; i += NT) {
      double c;
      if (i == k) c = 0.0;                          // unused: row k is rewritten below
      else if (i == p) c = W[k + (int64_t)k * N];
      else c = W[i + (int64_t)k * N];
      colk[i] = c;
    }
    if (tid == 0) piv[k] = p;
    __syncthreads();
    const double rinv = s_rinv;
    // rank-1 update (column j by warp, rows by lane); the warp owning column
    // k+1 also finds the next pivot while it writes that column
    for (int j = warp; j < N; j += NW) {
      double* col = W + (int64_t)j * N;
      if (j == k) {
        for (int i = lane; i < N; i += 32) col[i] = (i == k) ? rinv : -colk[i] * rinv;
        continue;
      }
      const double rj = rowk[j] * rinv;
      ArgMax a{0.0, -1};
      for (int i = lane; i < N; i += 32) {
        const double v = (i == k) ? rj : col[i] - colk[i] * rj;
        col[i] = v;
        if (j == k + 1 && i > k) {
          const double av = fabs(v);
          if (argmax_better(av, i, a.v, a.i)) { a.v = av; a.i = i; }
        }
      }
      if (j == k + 1) {
        a = warp_argmax(a);
        if (lane == 0) {
          s_p = (int)a.i;
          s_sing = !(a.v >= HK_PIVOT_FLOOR);
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) *t.status = s_sing;
  if (s_sing) return;
  // undo the row pivoting as a column gather: A^{-1}[:, j] = W[:, c(j)]
  if (tid == 0) {
    for (int j = 0; j < N; ++j) cperm[j] = j;
    for (int k = N - 1; k >= 0; --k) {
      const int a = cperm[k];
      cperm[k] = cperm[piv[k]];
      cperm[piv[k]] = a;
    }
  }
  __syncthreads();
  for (int j = warp; j < N; j += NW) {
    const double* src = W + (int64_t)cperm[j] * N;
    double* dst = t.out + (int64_t)j * t.out_ld;
    for (int i = lane; i < N; i += 32) dst[i] = src[i];
  }
}

}  // namespace

template <int NT, int MAXQ>
static cudaError_t launch_gj_smem(const GjTask* tasks_dev, int ntasks, int maxN, cudaStream_t st) {
  const size_t smem = (size_t)maxN * maxN * 8 + (size_t)2 * maxN * 8;
  cudaError_t e = cudaFuncSetAttribute(gj_smem_kernel<NT, MAXQ>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  gj_smem_kernel<NT, MAXQ><<<ntasks, NT, smem, st>>>(tasks_dev);
  hk_count_launch();
  return cudaGetLastError();
}

template <int NW, int CPW, int RPL>
static cudaError_t launch_gj_reg(const GjTask* tasks_dev, int ntasks, int maxN, cudaStream_t st) {
  const size_t smem = ((size_t)maxN * maxN + 4 * (size_t)maxN) * 8;
  cudaError_t e = cudaFuncSetAttribute(gj_reg_kernel<NW, CPW, RPL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  gj_reg_kernel<NW, CPW, RPL><<<ntasks, NW * 32, smem, st>>>(tasks_dev);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_gj(const GjTask* tasks_dev, int ntasks, int maxN, cudaStream_t st) {
  if (ntasks == 0) return cudaSuccess;
  if (maxN <= 64) return launch_gj_reg<8, 8, 2>(tasks_dev, ntasks, maxN, st);
  if (maxN <= 128) return launch_gj_reg<16, 8, 4>(tasks_dev, ntasks, maxN, st);
  if (maxN <= 160) return launch_gj_reg<16, 10, 5>(tasks_dev, ntasks, maxN, st);
  size_t need = gj_bytes(maxN);
  size_t smem = need <= GJ_SMEM_CAP ? need : 0;
  cudaError_t e;
  if (maxN > 80) {   // large systems: more warps per elimination step
    e = cudaFuncSetAttribute(gj_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)GJ_SMEM_CAP);
    if (e != cudaSuccess) return e;
    gj_kernel<1024><<<ntasks, 1024, smem, st>>>(tasks_dev, smem);
  } else {
    e = cudaFuncSetAttribute(gj_kernel<GJ_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)GJ_SMEM_CAP);
    if (e != cudaSuccess) return e;
    gj_kernel<GJ_NT><<<ntasks, GJ_NT, smem, st>>>(tasks_dev, smem);
  }
  hk_count_launch();
  return cudaGetLastError();
}

size_t hk_gj_scratch_bytes(int N) { return gj_bytes(N) <= GJ_SMEM_CAP ? 0 : gj_bytes(N); }
