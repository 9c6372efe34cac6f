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

constexpr int ACA_NT = 128;

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

// ---------------------------------------------------------------------------
// Residual sweep: out[e] = src[e] - sum_{k<rank} coef[k] * F[k*len + e] for the
// two elements e0 = tid + base, e1 = e0 + NT owned by this thread, k in the
// reference order with separate IEEE multiply/subtract.  Loads are issued in
// batches of KB so each thread keeps 2*KB independent L2 requests in flight
// (the chain itself only depends on the arithmetic).
template <int NT, int KB>
__device__ __forceinline__ void sweep2(const double* __restrict__ F, int64_t len, int rank,
                                       const double* __restrict__ coef, int e0, bool has1,
                                       double& x0, double& x1) {
  // Register double buffering: the loads of chunk c+1 are in flight while the
  // subtract chain of chunk c runs.  The products c_k * F[k, e] do not depend
  // on the chain, so only the subtractions are serial.
  const double* p0 = F + e0;
  const int nfull = rank / KB;
  double a[KB], b[KB];
  if (nfull > 0) {
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      a[q] = p0[(int64_t)q * len];
      b[q] = has1 ? p0[(int64_t)q * len + NT] : 0.0;
    }
  }
  for (int c = 0; c < nfull; ++c) {
    const int k = c * KB;
    double pa[KB], pb[KB];
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      const double cc = coef[k + q];
      pa[q] = mul_rn(cc, a[q]);
      pb[q] = mul_rn(cc, b[q]);
    }
    if (c + 1 < nfull) {
#pragma unroll
      for (int q = 0; q < KB; ++q) {
        a[q] = p0[(int64_t)(k + KB + q) * len];
        b[q] = has1 ? p0[(int64_t)(k + KB + q) * len + NT] : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      x0 = sub_rn(x0, pa[q]);
      x1 = sub_rn(x1, pb[q]);
    }
  }
  for (int k = nfull * KB; k < rank; ++k) {
    const double cc = coef[k];
    x0 = sub_rn(x0, mul_rn(cc, p0[(int64_t)k * len]));
    if (has1) x1 = sub_rn(x1, mul_rn(cc, p0[(int64_t)k * len + NT]));
  }
}

// Lane l of the warp receives the warp-wide sum of a[l & 15] (butterfly
// reduce-scatter inside each half-warp, then one exchange between halves).
__device__ __forceinline__ double transpose_reduce16(double (&a)[16], int lane) {
#pragma unroll
  for (int s = 8; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double send = upper ? a[i] : a[i + s];
      const double keep = upper ? a[i + s] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return a[0] + __shfl_xor_sync(0xffffffffu, a[0], 16);
}

// du[k] = u . U[:, k] and dv[k] = v . V[:, k] for k < rank, with the sweep's
// access pattern: every thread owns elements e = tid + NT*q, loads 16 columns
// at a time (coalesced over e, 8 loads in flight per batch); the per-k sums
// are reduced by a warp transpose-reduce into per-warp SMEM partials, and
// after ONE barrier per DCH columns summed over warps in a fixed order
// (deterministic, independent of scheduling).
constexpr int DCH = 128;

template <int NT>
__device__ __forceinline__ void dot_chunk(const double* __restrict__ F, const double* __restrict__ x,
                                          int len, int k0, int kend, double* __restrict__ part) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int kb = k0; kb < kend; kb += 16) {
    double acc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = 0.0;
    for (int e = tid; e < len; e += NT) {
      const double xe = x[e];
      const double* p = F + e + (int64_t)kb * len;
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        double a[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = (kb + 8 * g + q < kend) ? p[(int64_t)(8 * g + q) * len] : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[8 * g + q] += xe * a[q];
      }
    }
    const double v = transpose_reduce16(acc, lane);
    if (lane < 16) part[warp * DCH + (kb - k0) + lane] = v;
  }
}

template <int NT>
__device__ __forceinline__ void dots_pass(const double* __restrict__ U, const double* __restrict__ u,
                                          int m, const double* __restrict__ V,
                                          const double* __restrict__ v, int n, int rank,
                                          double* __restrict__ du, double* __restrict__ dv,
                                          double* __restrict__ part) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x;
  for (int k0 = 0; k0 < rank; k0 += DCH) {
    const int kend = min(rank, k0 + DCH);
    dot_chunk<NT>(U, u, m, k0, kend, part);
    dot_chunk<NT>(V, v, n, k0, kend, part + NW * DCH);
    __syncthreads();
    for (int k = k0 + tid; k < kend; k += NT) {
      double su = 0.0, sv = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        su += part[w * DCH + (k - k0)];
        sv += part[NW * DCH + w * DCH + (k - k0)];
      }
      du[k] = su;
      dv[k] = sv;
    }
    __syncthreads();
  }
}

template <int NT>
__device__ void aca_block(const AcaTask& t, double tol2, int vec_in_smem);

// Persistent: CTAs pull tasks from a global counter in list order (largest
// blocks first), so the long root chains start at t = 0 whatever the hardware
// dispatch order of CTAs is.
template <int NT>
__global__ void __launch_bounds__(NT, 4) aca_kernel(const AcaTask* __restrict__ tasks, int ntasks,
                                                    int* __restrict__ counter, double tol2,
                                                    int vec_in_smem) {
  __shared__ int s_task;
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(counter, 1);
    __syncthreads();
    const int ti = s_task;
    __syncthreads();
    if (ti >= ntasks) break;
    aca_block<NT>(tasks[ti], tol2, vec_in_smem);
    __syncthreads();
  }
}

template <int NT>
__device__ void aca_block(const AcaTask& t, double tol2, int vec_in_smem) {
  const int m = t.m, n = t.n, cap = t.cap;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  uint64_t t_start = 0;
  if (t.clock && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  extern __shared__ __align__(16) unsigned char smraw[];
  double* coef = reinterpret_cast<double*>(smraw);   // [cap]
  double* du = coef + cap;                           // [cap]  u . u_k
  double* dv = du + cap;                             // [cap]  v . v_k
  double* part = dv + cap;                           // [2 * NW * DCH] dot partials
  double* svec = part + 2 * NW * DCH;                // [m + n] when vec_in_smem
  unsigned char* used = reinterpret_cast<unsigned char*>(svec + (vec_in_smem ? (m + n) : 0));
  __shared__ double red_v[NW], red_a[NW], red_b[NW];
  __shared__ int64_t red_i[NW];
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

    // ---- residual row (lowrank.py:253-256): V[:, rank] = A[row, :] - U[row, :] V^T
    const double* src = Ab + (int64_t)row * t.lda;
    double* vout = V + (int64_t)rank * n;
    ArgMax best{0.0, -1};
    for (int base = 0; base < n; base += 2 * NT) {
      const int e0 = base + tid;
      if (e0 >= n) break;
      const bool has1 = e0 + NT < n;
      double x0 = src[e0], x1 = has1 ? src[e0 + NT] : 0.0;
      sweep2<NT, 4>(V, n, rank, coef, e0, has1, x0, x1);
      vout[e0] = x0;
      double a0 = fabs(x0);
      if (argmax_better(a0, e0, best.v, best.i)) { best.v = a0; best.i = e0; }
      if (has1) {
        vout[e0 + NT] = x1;
        double a1 = fabs(x1);
        if (argmax_better(a1, e0 + NT, best.v, best.i)) { best.v = a1; best.i = e0 + NT; }
      }
    }
    best = block_argmax<NT, false>(best, red_v, red_i);
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
    double* vs = vec_in_smem ? svec + m : vout;
    for (int j = tid; j < n; j += NT) {
      const double v = div_rn(vout[j], delta);
      vout[j] = v;
      if (vec_in_smem) vs[j] = v;
      vv += v * v;
    }
    for (int k = tid; k < rank; k += NT) coef[k] = V[(int64_t)k * n + col];
    if (tid == 0 && tcols) tcols[ncol_ev] = col;
    ++ncol_ev;
    __syncthreads();

    // ---- residual column (:266-268) plus next-row candidate (:283)
    const double* csrc = Atb + (int64_t)col * t.lda;
    double* uout = U + (int64_t)rank * m;
    double* us = vec_in_smem ? svec : uout;
    double uu = 0.0;
    ArgMax nxt{0.0, -1};
    for (int base = 0; base < m; base += 2 * NT) {
      const int e0 = base + tid;
      if (e0 >= m) break;
      const bool has1 = e0 + NT < m;
      double x0 = csrc[e0], x1 = has1 ? csrc[e0 + NT] : 0.0;
      sweep2<NT, 4>(U, m, rank, coef, e0, has1, x0, x1);
      uout[e0] = x0;
      if (vec_in_smem) us[e0] = x0;
      uu += x0 * x0;
      if (!used[e0]) {
        const double a = fabs(x0);
        if (argmax_better(a, e0, nxt.v, nxt.i)) { nxt.v = a; nxt.i = e0; }
      }
      if (has1) {
        uout[e0 + NT] = x1;
        if (vec_in_smem) us[e0 + NT] = x1;
        uu += x1 * x1;
        if (!used[e0 + NT]) {
          const double a = fabs(x1);
          if (argmax_better(a, e0 + NT, nxt.v, nxt.i)) { nxt.v = a; nxt.i = e0 + NT; }
        }
      }
    }
    // one combined reduction: next-row argmax, ||u||^2, ||v||^2
    {
      nxt = warp_argmax(nxt);
      uu = warp_sum(uu);
      vv = warp_sum(vv);
      if (lane == 0) { red_v[warp] = nxt.v; red_i[warp] = nxt.i; red_a[warp] = uu; red_b[warp] = vv; }
      __syncthreads();
      if (warp == 0) {
        ArgMax b2;
        double a2 = 0.0, c2 = 0.0;
        if (lane < NW) { b2.v = red_v[lane]; b2.i = red_i[lane]; a2 = red_a[lane]; c2 = red_b[lane]; }
        else { b2.v = 0.0; b2.i = -1; }
        b2 = warp_argmax(b2);
        a2 = warp_sum(a2);
        c2 = warp_sum(c2);
        if (lane == 0) { red_v[0] = b2.v; red_i[0] = b2.i; red_a[0] = a2; red_b[0] = c2; }
      }
      // the dots below need every thread's u/v writes: this barrier covers both
      __syncthreads();
      nxt.i = red_i[0];
      uu = red_a[0];
      vv = red_b[0];
    }

    // ---- stopping estimate (:269-275): cross terms 2 (u.u_k)(v.v_k)
    dots_pass<NT>(U, us, m, V, vs, n, rank, du, dv, part);
    const double cross = uu * vv;
    double est = fro2 + cross;
    for (int k = 0; k < rank; ++k) est += 2.0 * du[k] * dv[k];
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
    if (t.clock) {
      uint64_t t_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      t.clock[0] = (int64_t)t_start;
      t.clock[1] = (int64_t)t_end;
      t.clock[2] = smid;
    }
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
                          double tol2, cudaStream_t st, int max_mn) {
  if (ntasks == 0) return cudaSuccess;
  // the new cross vectors are staged in SMEM for the dot products when that
  // keeps the CTA small enough for several CTAs per SM
  size_t base = (size_t)max_cap * 24 + 2 * (ACA_NT / 32) * DCH * 8 + (size_t)max_m + 16;
  int vec_in_smem = base + (size_t)max_mn * 8 <= 48 * 1024 ? 1 : 0;
  size_t smem = base + (vec_in_smem ? (size_t)max_mn * 8 : 0);
  cudaError_t e = cudaFuncSetAttribute(aca_kernel<ACA_NT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, aca_kernel<ACA_NT>, ACA_NT, smem);
  if (e != cudaSuccess) return e;
  int grid = sms * (per_sm > 0 ? per_sm : 1);
  if (grid > ntasks) grid = ntasks;
  int* counter = nullptr;
  e = cudaMallocAsync(&counter, sizeof(int), st);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(counter, 0, sizeof(int), st);
  aca_kernel<ACA_NT><<<grid, ACA_NT, smem, st>>>(tasks_dev, ntasks, counter, tol2, vec_in_smem);
  e = cudaGetLastError();
  cudaFreeAsync(counter, st);
  hk_count_launch();
  return e;
}
