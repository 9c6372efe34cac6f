// Batched adaptive cross approximation over every off-diagonal block of every
// front, one launch (reference src/lowrank.py:230-286).
//
// One CTA owns one block and runs the reference's serial pivot chain.  All
// compressions read only the original front (src/hodlr.py:240-241), so every
// block of every level of every front is an independent task of the same
// launch; tasks are ordered largest-first so the long root chains start at once.
//
// Bit-exactness: the residual row/column updates are evaluated in the
// reference's order (k = 0..r-1) with separate IEEE multiply and subtract
// (no FMA), the pivot scaling is an IEEE division, and both argmax searches
// break ties toward the lowest index, exactly as numpy does.  U and V are
// therefore bit-identical to the reference's; only the stopping estimate
// uses dot products whose summation order differs from OpenBLAS (measured
// decision margin >= 4.6e-3 relative).
//
// Layout: rows of the block come from the row-major front (coalesced along
// the row), columns from a transposed copy At (coalesced along the column);
// U (m x cap) and V (n x cap) are column-major so every cross vector u_k / v_k
// is contiguous and the k-loop of a sweep reads V[k*n + j] coalesced over j.
#include "hk_common.cuh"
#include "hk_internal.h"

namespace {

constexpr int ACA_NT = 256;

__global__ void transpose_kernel(const double* __restrict__ A, double* __restrict__ At,
                                 int64_t n, int64_t ld, int64_t stride) {
  __shared__ double tile[32][33];
  const int64_t f = blockIdx.z;
  const double* a = A + f * stride;
  double* at = At + f * stride;
  const int64_t bx = (int64_t)blockIdx.x * 32, by = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t i = by + r, j = bx + threadIdx.x;
    if (i < n && j < n) tile[r][threadIdx.x] = a[i * ld + j];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t j = bx + r, i = by + threadIdx.x;
    if (i < n && j < n) at[j * ld + i] = tile[threadIdx.x][r];
  }
}

// res[e] = src[e] - sum_k coef[k] * F[k*len + e], k in order; written to out.
// Returns nothing; callers fold their own reductions over the owned elements.

template <int NT>
__global__ void __launch_bounds__(NT) aca_kernel(const AcaTask* __restrict__ tasks, double tol2) {
  const AcaTask t = tasks[blockIdx.x];
  const int m = t.m, n = t.n, cap = t.cap;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(16) unsigned char smraw[];
  double* coef = reinterpret_cast<double*>(smraw);   // [cap]
  double* prod = coef + cap;                         // [cap]
  unsigned char* used = reinterpret_cast<unsigned char*>(prod + cap);  // [m]
  __shared__ double red_v[NT / 32];
  __shared__ int64_t red_i[NT / 32];
  __shared__ double red_s[2 * (NT / 32)];
  __shared__ int s_row;

  int32_t* trows = t.trace ? t.trace + 2 : nullptr;
  int32_t* tcols = t.trace ? t.trace + 2 + (m + cap + 1) : nullptr;
  int nrow_ev = 0, ncol_ev = 0;

  if (m == 0 || n == 0 || cap == 0) {
    if (tid == 0) {
      *t.rank = 0;
      if (t.trace) { t.trace[0] = 0; t.trace[1] = 0; }
    }
    return;
  }
  for (int i = tid; i < m; i += NT) used[i] = 0;
  __syncthreads();

  int rank = 0, row = 0, nused = 0;
  double fro2 = 0.0;
  const double* __restrict__ Ab = t.A;
  const double* __restrict__ Atb = t.At;
  double* __restrict__ U = t.U;
  double* __restrict__ V = t.V;

  while (rank < cap) {
    if (tid == 0) {
      used[row] = 1;
      if (trows) trows[nrow_ev] = row;
    }
    ++nrow_ev;
    ++nused;
    for (int k = tid; k < rank; k += NT) coef[k] = U[(int64_t)k * m + row];
    __syncthreads();

    // ---- residual row (lowrank.py:253-256)
    const double* src = Ab + (int64_t)row * t.lda;
    double* vout = V + (int64_t)rank * n;
    ArgMax best{0.0, -1};
    {
      int j = tid;
      for (; j + NT < n; j += 2 * NT) {
        double x0 = src[j], x1 = src[j + NT];
        const double* vp = V + j;
        for (int k = 0; k < rank; ++k) {
          const double c = coef[k];
          x0 = sub_rn(x0, mul_rn(c, vp[0]));
          x1 = sub_rn(x1, mul_rn(c, vp[NT]));
          vp += n;
        }
        vout[j] = x0;
        vout[j + NT] = x1;
        double a0 = fabs(x0), a1 = fabs(x1);
        if (argmax_better(a0, j, best.v, best.i)) { best.v = a0; best.i = j; }
        if (argmax_better(a1, j + NT, best.v, best.i)) { best.v = a1; best.i = j + NT; }
      }
      for (; j < n; j += NT) {
        double x0 = src[j];
        const double* vp = V + j;
        for (int k = 0; k < rank; ++k) {
          x0 = sub_rn(x0, mul_rn(coef[k], vp[0]));
          vp += n;
        }
        vout[j] = x0;
        double a0 = fabs(x0);
        if (argmax_better(a0, j, best.v, best.i)) { best.v = a0; best.i = j; }
      }
    }
    best = block_argmax<NT>(best, red_v, red_i);
    const int col = (int)best.i;
    const double delta = vout[col];
    if (delta == 0.0) {                 // zero residual row: restart (:258-264)
      if (nused == m) break;
      if (tid == 0) {
        int r = 0;
        while (used[r]) ++r;
        s_row = r;
      }
      __syncthreads();
      row = s_row;
      __syncthreads();
      continue;
    }
    // ---- v = res / delta (:265) and the column coefficients
    double vv = 0.0;
    for (int j = tid; j < n; j += NT) {
      double v = div_rn(vout[j], delta);
      vout[j] = v;
      vv += v * v;
    }
    for (int k = tid; k < rank; k += NT) coef[k] = V[(int64_t)k * n + col];
    if (tid == 0 && tcols) tcols[ncol_ev] = col;
    ++ncol_ev;
    __syncthreads();

    // ---- residual column (:266-268), plus next-row candidate (:283)
    const double* csrc = Atb + (int64_t)col * t.lda;
    double* uout = U + (int64_t)rank * m;
    double uu = 0.0;
    ArgMax nxt{0.0, -1};
    {
      int i = tid;
      for (; i + NT < m; i += 2 * NT) {
        double x0 = csrc[i], x1 = csrc[i + NT];
        const double* up = U + i;
        for (int k = 0; k < rank; ++k) {
          const double c = coef[k];
          x0 = sub_rn(x0, mul_rn(c, up[0]));
          x1 = sub_rn(x1, mul_rn(c, up[NT]));
          up += m;
        }
        uout[i] = x0;
        uout[i + NT] = x1;
        uu += x0 * x0 + x1 * x1;
        if (!used[i]) {
          double a = fabs(x0);
          if (argmax_better(a, i, nxt.v, nxt.i)) { nxt.v = a; nxt.i = i; }
        }
        if (!used[i + NT]) {
          double a = fabs(x1);
          if (argmax_better(a, i + NT, nxt.v, nxt.i)) { nxt.v = a; nxt.i = i + NT; }
        }
      }
      for (; i < m; i += NT) {
        double x0 = csrc[i];
        const double* up = U + i;
        for (int k = 0; k < rank; ++k) {
          x0 = sub_rn(x0, mul_rn(coef[k], up[0]));
          up += m;
        }
        uout[i] = x0;
        uu += x0 * x0;
        if (!used[i]) {
          double a = fabs(x0);
          if (argmax_better(a, i, nxt.v, nxt.i)) { nxt.v = a; nxt.i = i; }
        }
      }
    }
    nxt = block_argmax<NT>(nxt, red_v, red_i);
    block_sum2<NT>(uu, vv, red_s);

    // ---- stopping estimate (:269-275): cross terms 2 (u.u_k)(v.v_k), warp per k
    for (int k = warp; k < rank; k += NT / 32) {
      const double* uk = U + (int64_t)k * m;
      const double* vk = V + (int64_t)k * n;
      double su = 0.0, sv = 0.0;
      for (int i = lane; i < m; i += 32) su += uout[i] * uk[i];
      for (int j = lane; j < n; j += 32) sv += vout[j] * vk[j];
      su = warp_sum(su);
      sv = warp_sum(sv);
      if (lane == 0) prod[k] = 2.0 * su * sv;
    }
    __syncthreads();
    const double cross = uu * vv;
    double est = fro2 + cross;
    for (int k = 0; k < rank; ++k) est += prod[k];
    est = fmax(est, cross);
    if (cross <= tol2 * est) break;     // discard this cross and stop
    ++rank;
    fro2 = est;
    if (nused == m) break;              // row exhaustion (:279-282)
    row = (int)nxt.i;
    __syncthreads();
  }
  if (tid == 0) {
    *t.rank = rank;
    if (t.trace) { t.trace[0] = nrow_ev; t.trace[1] = ncol_ev; }
  }
}

}  // namespace

cudaError_t hk_launch_transpose(const double* A, double* At, int64_t n, int64_t ld, int64_t batch,
                                int64_t stride, cudaStream_t st) {
  if (n == 0 || batch == 0) return cudaSuccess;
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32), (unsigned)batch);
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(A, At, n, ld, stride);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_aca(const AcaTask* tasks_dev, int ntasks, int max_cap, int max_m,
                          double tol2, cudaStream_t st) {
  if (ntasks == 0) return cudaSuccess;
  size_t smem = (size_t)max_cap * 16 + (size_t)max_m + 16;
  cudaError_t e = cudaFuncSetAttribute(aca_kernel<ACA_NT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  aca_kernel<ACA_NT><<<ntasks, ACA_NT, smem, st>>>(tasks_dev, tol2);
  hk_count_launch();
  return cudaGetLastError();
}
