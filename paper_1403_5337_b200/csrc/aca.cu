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

constexpr int KC = 8;     // columns per chunk (one transpose-reduce each)

// Lane l of the warp receives the warp-wide sum of a[l & 7] (butterfly
// reduce-scatter inside groups of 8 lanes, then two exchanges between groups).
__device__ __forceinline__ double transpose_reduce8(double (&a)[8], int lane) {
#pragma unroll
  for (int s = 4; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double send = upper ? a[i] : a[i + s];
      const double keep = upper ? a[i + s] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  double v = a[0];
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 16);
  return v;
}

// Fused residual sweep over one cross vector of length `len` (one element per
// thread, e = g0 + tid).  F is COLUMN-major with a power-of-two leading
// dimension LD = 1 << LDLOG (a template constant), so the eight loads of a
// column chunk are immediate offsets from one per-thread pointer and every
// warp-wide load is one coalesced 256-byte segment.
//   F[e, out_col] = src[e] - sum_{k<nk} coef[k] * F[e, k]   (reference k order,
//                   separate IEEE multiply and subtract: bit-exact)
// and, for k < ndot, the per-warp partial dot products
//   part[w*pld + k] = sum_{e owned by warp w} F[e, pend_col] * F[e, k]
// of the PREVIOUS cross with the accepted crosses: the stopping-test terms of
// the pending step ride along with the next step's sweep, so each cross vector
// is streamed once per step.  Chunks are software-pipelined (the next chunk's
// loads are in flight while the current chunk's subtract chain runs).
// Partial sums use a warp transpose-reduce and a fixed per-warp order
// (deterministic).  out_col < 0: dots only.  used != nullptr: column sweep
// (argmax over untouched entries + sum of squares); else row sweep.
template <int NT, int LDLOG>
__device__ __forceinline__ void fused_sweep_impl(const double* __restrict__ F, int len, int nk, int ndot,
                                         const double* __restrict__ coef,
                                         const double* __restrict__ src, int out_col, int pend_col,
                                         double* __restrict__ part, int pld,
                                         const unsigned char* __restrict__ used, ArgMax& best,
                                         double& sumsq, double& bestval) {
  constexpr int64_t LD = int64_t(1) << LDLOG;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  best.v = 0.0;
  best.i = -1;
  bestval = 0.0;
  sumsq = 0.0;
  double* mypart = part + warp * pld;
  for (int k = lane; k < ndot; k += 32) mypart[k] = 0.0;
  __syncwarp();
  const int kmax = nk > ndot ? nk : ndot;
  const int nchunks = (kmax + KC - 1) / KC;
#pragma unroll 1
  for (int g0 = 0; g0 < len; g0 += NT) {
    const int e = g0 + tid;
    const bool ok = e < len;
    const double* col = F + (ok ? e : 0);       // this element in column 0
    double x = (ok && src) ? src[e] : 0.0;
    const double pv = (ok && ndot > 0) ? __ldca(col + (int64_t)pend_col * LD) : 0.0;
    double cur[KC], nxt[KC];
    const double* pk = col;
    if (nchunks > 0) {
#pragma unroll
      for (int j = 0; j < KC; ++j) cur[j] = __ldca(pk + j * LD);
    }
#pragma unroll 1
    for (int c = 0; c < nchunks; ++c) {
      const int kb = c * KC;
      pk += KC * LD;
      if (c + 1 < nchunks) {
#pragma unroll
        for (int j = 0; j < KC; ++j) nxt[j] = __ldca(pk + j * LD);
      }
      if (kb < ndot) {                       // warp-uniform: dots first, then the chain
        double acc[KC];
#pragma unroll
        for (int j = 0; j < KC; ++j) acc[j] = (kb + j < ndot) ? pv * cur[j] : 0.0;
        const double v = transpose_reduce8(acc, lane);
        if (lane < KC && kb + lane < ndot) mypart[kb + lane] += v;
      }
      if (kb + KC <= nk) {
#pragma unroll
        for (int j = 0; j < KC; ++j) x = sub_rn(x, mul_rn(coef[kb + j], cur[j]));
      } else {
#pragma unroll
        for (int j = 0; j < KC; ++j)
          if (kb + j < nk) x = sub_rn(x, mul_rn(coef[kb + j], cur[j]));
      }
#pragma unroll
      for (int j = 0; j < KC; ++j) cur[j] = nxt[j];
    }
    if (out_col >= 0 && ok) {
      const_cast<double*>(col)[(int64_t)out_col * LD] = x;
      const double ax = fabs(x);
      if (used) {
        sumsq += x * x;
        if (!used[e] && argmax_better(ax, e, best.v, best.i)) { best.v = ax; best.i = e; bestval = x; }
      } else if (argmax_better(ax, e, best.v, best.i)) {
        best.v = ax;
        best.i = e;
        bestval = x;
      }
    }
  }
}

// One call target for the caller (keeps its register allocation small); the
// leading dimension is dispatched once, inside, to the specialised loop.
template <int NT>
__device__ __noinline__ void fused_sweep(int ldlog, const double* __restrict__ F, int len, int nk,
                                         int ndot, const double* __restrict__ coef,
                                         const double* __restrict__ src, int out_col, int pend_col,
                                         double* __restrict__ part, int pld,
                                         const unsigned char* __restrict__ used, ArgMax& best,
                                         double& sumsq, double& bestval) {
#define HK_SWEEP_CASE(L)                                                                         \
  case L:                                                                                        \
    fused_sweep_impl<NT, L>(F, len, nk, ndot, coef, src, out_col, pend_col, part, pld, used,   \
                            best, sumsq, bestval);                                               \
    return;
  switch (ldlog) {
    HK_SWEEP_CASE(6) HK_SWEEP_CASE(7) HK_SWEEP_CASE(8) HK_SWEEP_CASE(9) HK_SWEEP_CASE(10)
    HK_SWEEP_CASE(11) HK_SWEEP_CASE(12) HK_SWEEP_CASE(13)
    default: return;
  }
#undef HK_SWEEP_CASE
}

// Block argmax that also carries the signed value of the winner.
template <int NT>
__device__ __forceinline__ ArgMax block_argmax_val(ArgMax a, double val, double* sv, int64_t* si,
                                                   double* sval, double& out_val) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, a.v, off);
    const long long oi = __shfl_down_sync(0xffffffffu, (long long)a.i, off);
    const double ox = __shfl_down_sync(0xffffffffu, val, off);
    if (argmax_better(ov, oi, a.v, a.i)) { a.v = ov; a.i = oi; val = ox; }
  }
  if (lane == 0) { sv[warp] = a.v; si[warp] = a.i; sval[warp] = val; }
  __syncthreads();
  if (warp == 0) {
    ArgMax b;
    double bv = 0.0;
    if (lane < NT / 32) { b.v = sv[lane]; b.i = si[lane]; bv = sval[lane]; }
    else { b.v = 0.0; b.i = -1; }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, b.v, off);
      const long long oi = __shfl_down_sync(0xffffffffu, (long long)b.i, off);
      const double ox = __shfl_down_sync(0xffffffffu, bv, off);
      if (argmax_better(ov, oi, b.v, b.i)) { b.v = ov; b.i = oi; bv = ox; }
    }
    if (lane == 0) { sv[0] = b.v; si[0] = b.i; sval[0] = bv; }
  }
  __syncthreads();
  out_val = sval[0];
  return ArgMax{sv[0], si[0]};
}

// SMEM-resident sweep for small blocks (len <= NT): F column-major in SMEM with
// leading dimension ldf, src with element stride sstride.  Same arithmetic and
// dot-partial layout as fused_sweep_impl (bit-exact), no global traffic.
template <int NT>
__device__ __forceinline__ void smem_sweep(const double* __restrict__ F, int ldf, int len, int nk,
                                           int ndot, const double* __restrict__ coef,
                                           const double* __restrict__ src, int sstride,
                                           int out_col, int pend_col, double* __restrict__ part,
                                           int pld, const unsigned char* __restrict__ used,
                                           ArgMax& best, double& sumsq, double& bestval,
                                           double& xout) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  best.v = 0.0;
  best.i = -1;
  bestval = 0.0;
  sumsq = 0.0;
  double* mypart = part + warp * pld;
  for (int k = lane; k < ndot; k += 32) mypart[k] = 0.0;
  __syncwarp();
  const int e = tid;
  const bool ok = e < len;
  const double* col = F + (ok ? e : 0);
  double x = (ok && src) ? src[e * sstride] : 0.0;
  const double pv = (ok && ndot > 0) ? col[pend_col * ldf] : 0.0;
  const int kmax = nk > ndot ? nk : ndot;
  for (int kb = 0; kb < kmax; kb += KC) {
    double cur[KC];
#pragma unroll
    for (int j = 0; j < KC; ++j) cur[j] = (kb + j < kmax) ? col[(kb + j) * ldf] : 0.0;
    if (kb < ndot) {
      double acc[KC];
#pragma unroll
      for (int j = 0; j < KC; ++j) acc[j] = (kb + j < ndot) ? pv * cur[j] : 0.0;
      const double v = transpose_reduce8(acc, lane);
      if (lane < KC && kb + lane < ndot) mypart[kb + lane] += v;
    }
#pragma unroll
    for (int j = 0; j < KC; ++j)
      if (kb + j < nk) x = sub_rn(x, mul_rn(coef[kb + j], cur[j]));
  }
  xout = x;
  if (out_col >= 0 && ok) {
    const_cast<double*>(col)[out_col * ldf] = x;
    const double ax = fabs(x);
    if (used) {
      sumsq += x * x;
      if (!used[e] && argmax_better(ax, e, best.v, best.i)) { best.v = ax; best.i = e; bestval = x; }
    } else if (argmax_better(ax, e, best.v, best.i)) {
      best.v = ax;
      best.i = e;
      bestval = x;
    }
  }
}

// est = fro2 + cross + sum_k 2 (u.u_k)(v.v_k) over the per-warp partials,
// reduced in a fixed order; valid in every thread.
template <int NT>
__device__ __forceinline__ double stopping_estimate(const double* __restrict__ partU,
                                                    const double* __restrict__ partV, int pld,
                                                    int r, double fro2, double cross,
                                                    double* __restrict__ prod, double* s_est) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int k = tid; k < r; k += NT) {
    double du = 0.0, dv = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      du += partU[w * pld + k];
      dv += partV[w * pld + k];
    }
    prod[k] = 2.0 * du * dv;
  }
  __syncthreads();
  if (warp == 0) {
    double sacc = 0.0;
    for (int k = lane; k < r; k += 32) sacc += prod[k];
    sacc = warp_sum(sacc);
    if (lane == 0) *s_est = fmax(fro2 + cross + sacc, cross);
  }
  __syncthreads();
  return *s_est;
}

// Persistent: CTAs pull tasks from a global counter in list order (largest
// blocks first), so the long root chains start at t = 0 whatever the hardware
// dispatch order of CTAs is.
template <int NT>
__device__ void aca_block(const AcaTask& t, double tol2, int part_in_smem);

template <int NT>
__global__ void __launch_bounds__(NT, (NT >= 512 ? 1 : 512 / NT)) aca_kernel(const AcaTask* __restrict__ tasks, int ntasks,
                                                    int* __restrict__ counter, double tol2,
                                                    int part_in_smem) {
  __shared__ int s_task;
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(counter, 1);
    __syncthreads();
    const int ti = s_task;
    __syncthreads();
    if (ti >= ntasks) break;
    aca_block<NT>(tasks[ti], tol2, part_in_smem);
    __syncthreads();
  }
}

template <int NT>
__device__ void aca_block_smem(const AcaTask& t, double tol2);

template <int NT>
__global__ void __launch_bounds__(NT) aca_smem_kernel(const AcaTask* __restrict__ tasks, int ntasks,
                                                      int* __restrict__ counter, double tol2) {
  __shared__ int s_task;
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(counter, 1);
    __syncthreads();
    const int ti = s_task;
    __syncthreads();
    if (ti >= ntasks) break;
    aca_block_smem<NT>(tasks[ti], tol2);
    __syncthreads();
  }
}

template <int NT>
__device__ void aca_block(const AcaTask& t, double tol2, int part_in_smem) {
  const int m = t.m, n = t.n, cap = t.cap;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  uint64_t t_start = 0;
  if (t.clock && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  extern __shared__ __align__(16) unsigned char smraw[];
  // SMEM: coef[cap+KC]; when part_in_smem: partU/partV [NW*cap] and prod[cap]; used[m]
  double* coef = reinterpret_cast<double*>(smraw);
  const int pld = cap;
  double* partU = part_in_smem ? coef + cap + KC : t.scratch;
  double* partV = partU + NW * pld;
  double* prod = partV + NW * pld;
  unsigned char* used = reinterpret_cast<unsigned char*>(part_in_smem ? prod + cap : coef + cap + KC);
  __shared__ double red_v[NW], red_a[NW], red_b[NW], red_x[NW];
  __shared__ int64_t red_i[NW];
  __shared__ int s_row;
  __shared__ double s_est;

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
  // coef beyond the chain length is read (times 0) by the unrolled sweeps
  for (int k = tid; k < cap + KC; k += NT) coef[k] = 0.0;
  __syncthreads();

  const double* __restrict__ Ab = t.A;
  const double* __restrict__ Atb = t.At;
  double* __restrict__ U = t.U;      // column-major m x cap, leading dimension 2^ldu
  double* __restrict__ V = t.V;      // column-major n x cap, leading dimension 2^ldv
  const int ldlog = t.ldu;                   // U and V share one power-of-two leading dimension
  const int64_t LDU = int64_t(1) << ldlog, LDV = LDU;
  int r = 0, row = 0, nused = 0;
  bool pending = false;                       // column r holds an undecided cross
  double uu_p = 0.0, vv_p = 0.0, fro2 = 0.0;
  ArgMax best, nxt;
  double dummy, uu, bval;

  for (;;) {
    const int c = r + (pending ? 1 : 0);     // index of the new candidate
    const bool can_step = pending ? (c < cap && nused < m) : (c < cap);
    if (!can_step) {
      if (pending) {                          // decide the last cross: dots only
        fused_sweep<NT>(ldlog, U, m, 0, r, coef, nullptr, -1, r, partU, pld, nullptr, best, dummy, bval);
        fused_sweep<NT>(ldlog, V, n, 0, r, coef, nullptr, -1, r, partV, pld, nullptr, best, dummy, bval);
        __syncthreads();
        const double cross = uu_p * vv_p;
        const double est = stopping_estimate<NT>(partU, partV, pld, r, fro2, cross, prod, &s_est);
        if (!(cross <= tol2 * est)) ++r;
      }
      break;
    }
    // ---- next step (speculative when a cross is pending), lowrank.py:251-283
    if (tid == 0) {
      used[row] = 1;
      if (trows) trows[nrow_ev] = row;
    }
    ++nrow_ev;
    ++nused;
    for (int k = tid; k < c; k += NT) coef[k] = __ldca(U + row + (int64_t)k * LDU);
    __syncthreads();
    // residual row (:253-256) + the pending cross's v dots
    fused_sweep<NT>(ldlog, V, n, c, pending ? r : 0, coef, Ab + (int64_t)row * t.lda, c, r, partV, pld,
              nullptr, best, dummy, bval);
    double delta;
    best = block_argmax_val<NT>(best, bval, red_v, red_i, red_x, delta);
    const int col = (int)best.i;
    if (delta == 0.0) {                       // zero residual row (:258-264)
      if (pending) {
        fused_sweep<NT>(ldlog, U, m, 0, r, coef, nullptr, -1, r, partU, pld, nullptr, nxt, dummy, bval);
        __syncthreads();
        const double cross = uu_p * vv_p;
        const double est = stopping_estimate<NT>(partU, partV, pld, r, fro2, cross, prod, &s_est);
        if (cross <= tol2 * est) {            // reject: the reference never read this row
          --nrow_ev;
          break;
        }
        ++r;
        fro2 = est;
        pending = false;
      }
      if (nused == m) break;
      if (tid == 0) {
        int q = 0;
        while (used[q]) ++q;
        s_row = q;
      }
      __syncthreads();
      row = s_row;
      __syncthreads();
      continue;
    }
    // v = res / delta (:265) over own elements (same ownership as the sweep)
    double vv = 0.0;
    for (int e = tid; e < n; e += NT) {
      double* vp = V + e + (int64_t)c * LDV;
      const double v = div_rn(*vp, delta);
      *vp = v;
      vv += v * v;
    }
    for (int k = tid; k < c; k += NT) coef[k] = __ldca(V + col + (int64_t)k * LDV);
    if (tid == 0 && tcols) tcols[ncol_ev] = col;
    ++ncol_ev;
    __syncthreads();
    // residual column (:266-268) + next-row candidate (:283) + pending u dots
    fused_sweep<NT>(ldlog, U, m, c, pending ? r : 0, coef, Atb + (int64_t)col * t.lda, c, r, partU, pld,
              used, nxt, uu, bval);
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
      __syncthreads();
      nxt.i = red_i[0];
      uu = red_a[0];
      vv = red_b[0];
    }
    if (pending) {                            // stopping test of the pending cross (:269-275)
      const double cross = uu_p * vv_p;
      const double est = stopping_estimate<NT>(partU, partV, pld, r, fro2, cross, prod, &s_est);
      if (cross <= tol2 * est) {              // reject: drop the speculative step's reads
        --nrow_ev;
        --ncol_ev;
        break;
      }
      ++r;
      fro2 = est;
    }
    pending = true;                           // the new cross awaits its test
    uu_p = uu;
    vv_p = vv;
    row = (int)nxt.i;
    __syncthreads();
  }
  if (tid == 0) {
    *t.rank = r;
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

template <int NT>
__device__ void aca_block_smem(const AcaTask& t, double tol2) {
  const int m = t.m, n = t.n, cap = t.cap;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  uint64_t t_start = 0;
  if (t.clock && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  extern __shared__ __align__(16) unsigned char smraw[];
  // SMEM: Us[m x cap] (ld m), Vs[n x cap] (ld n), As[m x n] (ld n+1), coef[cap+KC],
  // partU/partV [NW*cap], prod[cap], used[m]
  const int ldus = m, ldvs = n, ldas = n + 1;
  double* Us = reinterpret_cast<double*>(smraw);
  double* Vs = Us + (size_t)m * cap;
  double* As = Vs + (size_t)n * cap;
  double* coef = As + (size_t)m * ldas;
  const int pld = cap;
  double* partU = coef + cap + KC;
  double* partV = partU + NW * pld;
  double* prod = partV + NW * pld;
  unsigned char* used = reinterpret_cast<unsigned char*>(prod + cap);
  __shared__ double red_v[NW], red_a[NW], red_b[NW], red_x[NW];
  __shared__ int64_t red_i[NW];
  __shared__ int s_row;
  __shared__ double s_est;

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
  for (int k = tid; k < cap + KC; k += NT) coef[k] = 0.0;
  for (int i = 0; i < m; ++i)
    for (int j = tid; j < n; j += NT) As[i * ldas + j] = t.A[(int64_t)i * t.lda + j];
  __syncthreads();

  const double* __restrict__ Ab = t.A;
  const double* __restrict__ Atb = t.At;
  double* __restrict__ U = Us;
  double* __restrict__ V = Vs;
  const int LDU = ldus, LDV = ldvs;
  double xreg = 0.0;
  int r = 0, row = 0, nused = 0;
  bool pending = false;                       // column r holds an undecided cross
  double uu_p = 0.0, vv_p = 0.0, fro2 = 0.0;
  ArgMax best, nxt;
  double dummy, uu, bval;

  for (;;) {
    const int c = r + (pending ? 1 : 0);     // index of the new candidate
    const bool can_step = pending ? (c < cap && nused < m) : (c < cap);
    if (!can_step) {
      if (pending) {                          // decide the last cross: dots only
        smem_sweep<NT>(U, ldus, m, 0, r, coef, nullptr, 1, -1, r, partU, pld, nullptr, best, dummy, bval, xreg);
        smem_sweep<NT>(V, ldvs, n, 0, r, coef, nullptr, 1, -1, r, partV, pld, nullptr, best, dummy, bval, xreg);
        __syncthreads();
        const double cross = uu_p * vv_p;
        const double est = stopping_estimate<NT>(partU, partV, pld, r, fro2, cross, prod, &s_est);
        if (!(cross <= tol2 * est)) ++r;
      }
      break;
    }
    // ---- next step (speculative when a cross is pending), lowrank.py:251-283
    if (tid == 0) {
      used[row] = 1;
      if (trows) trows[nrow_ev] = row;
    }
    ++nrow_ev;
    ++nused;
    for (int k = tid; k < c; k += NT) coef[k] = U[row + k * LDU];
    __syncthreads();
    // residual row (:253-256) + the pending cross's v dots
    smem_sweep<NT>(V, ldvs, n, c, pending ? r : 0, coef, As + row * ldas, 1, c, r, partV, pld,
                   nullptr, best, dummy, bval, xreg);
    double delta;
    best = block_argmax_val<NT>(best, bval, red_v, red_i, red_x, delta);
    const int col = (int)best.i;
    if (delta == 0.0) {                       // zero residual row (:258-264)
      if (pending) {
        smem_sweep<NT>(U, ldus, m, 0, r, coef, nullptr, 1, -1, r, partU, pld, nullptr, nxt, dummy, bval, xreg);
        __syncthreads();
        const double cross = uu_p * vv_p;
        const double est = stopping_estimate<NT>(partU, partV, pld, r, fro2, cross, prod, &s_est);
        if (cross <= tol2 * est) {            // reject: the reference never read this row
          --nrow_ev;
          break;
        }
        ++r;
        fro2 = est;
        pending = false;
      }
      if (nused == m) break;
      if (tid == 0) {
        int q = 0;
        while (used[q]) ++q;
        s_row = q;
      }
      __syncthreads();
      row = s_row;
      __syncthreads();
      continue;
    }
    // v = res / delta (:265) over own elements (same ownership as the sweep)
    double vv = 0.0;
    if (tid < n) {
      const double v = div_rn(xreg, delta);
      V[tid + c * LDV] = v;
      vv += v * v;
    }
    for (int k = tid; k < c; k += NT) coef[k] = V[col + k * LDV];
    if (tid == 0 && tcols) tcols[ncol_ev] = col;
    ++ncol_ev;
    __syncthreads();
    // residual column (:266-268) + next-row candidate (:283) + pending u dots
    smem_sweep<NT>(U, ldus, m, c, pending ? r : 0, coef, As + col, ldas, c, r, partU, pld, used,
                   nxt, uu, bval, xreg);
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
      __syncthreads();
      nxt.i = red_i[0];
      uu = red_a[0];
      vv = red_b[0];
    }
    if (pending) {                            // stopping test of the pending cross (:269-275)
      const double cross = uu_p * vv_p;
      const double est = stopping_estimate<NT>(partU, partV, pld, r, fro2, cross, prod, &s_est);
      if (cross <= tol2 * est) {              // reject: drop the speculative step's reads
        --nrow_ev;
        --ncol_ev;
        break;
      }
      ++r;
      fro2 = est;
    }
    pending = true;                           // the new cross awaits its test
    uu_p = uu;
    vv_p = vv;
    row = (int)nxt.i;
    __syncthreads();
  }
  {
    const int64_t LDG_ = int64_t(1) << t.ldu;
    for (int k = 0; k < r; ++k) {
      for (int i = tid; i < m; i += NT) t.U[i + k * LDG_] = Us[i + k * ldus];
      for (int j = tid; j < n; j += NT) t.V[j + k * LDG_] = Vs[j + k * ldvs];
    }
  }
  if (tid == 0) {
    *t.rank = r;
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

template <int NT>
static cudaError_t launch_class(const AcaTask* tasks_dev, int ntasks, int max_cap, int max_m,
                                double tol2, int* counter, cudaStream_t st) {
  const size_t part_bytes = (size_t)(2 * (NT / 32) + 1) * max_cap * 8;
  const size_t base = (size_t)(max_cap + KC) * 8 + (size_t)max_m + 16;
  const int part_in_smem = base + part_bytes <= 64 * 1024 ? 1 : 0;
  const size_t smem = base + (part_in_smem ? part_bytes : 0);
  cudaError_t e = cudaFuncSetAttribute(aca_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, aca_kernel<NT>, NT, smem);
  if (e != cudaSuccess) return e;
  int grid = sms * (per_sm > 0 ? per_sm : 1);
  if (grid > ntasks) grid = ntasks;
  aca_kernel<NT><<<grid, NT, smem, st>>>(tasks_dev, ntasks, counter, tol2, part_in_smem);
  hk_count_launch();
  return cudaGetLastError();
}

template <int NT>
static cudaError_t launch_smem_class(const AcaTask* tasks_dev, int ntasks, int max_cap, int max_m,
                                     double tol2, int* counter, cudaStream_t st) {
  // Us + Vs + As + coef + partials + prod + used, for m, n <= NT
  const size_t smem = (size_t)(2 * NT * max_cap + NT * (NT + 1) + max_cap + KC +
                               (2 * (NT / 32) + 1) * max_cap) * 8 + (size_t)max_m + 16;
  (void)max_m;
  cudaError_t e = cudaFuncSetAttribute(aca_smem_kernel<NT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, aca_smem_kernel<NT>, NT, smem);
  if (e != cudaSuccess) return e;
  int grid = sms * (per_sm > 0 ? per_sm : 1);
  if (grid > ntasks) grid = ntasks;
  aca_smem_kernel<NT><<<grid, NT, smem, st>>>(tasks_dev, ntasks, counter, tol2);
  hk_count_launch();
  return cudaGetLastError();
}

// Tasks arrive grouped by CTA size class (64/128/256/512 threads: one element
// of the longer cross vector per thread) and largest-first inside a class.
// Each class is one persistent launch; classes run concurrently on the given
// streams (caller forks/joins them).
cudaError_t hk_launch_aca_classes(const AcaTask* tasks_dev, const int* class_begin,
                                  const int* class_max_cap, const int* class_max_m, double tol2,
                                  int* counters_dev, cudaStream_t* streams) {
  static const int NTS[4] = {512, 256, 128, 64};
  for (int c = 0; c < 4; ++c) {
    const int nt = class_begin[c + 1] - class_begin[c];
    if (nt == 0) continue;
    const AcaTask* td = tasks_dev + class_begin[c];
    cudaError_t e;
    switch (NTS[c]) {
      case 512: e = launch_class<512>(td, nt, class_max_cap[c], class_max_m[c], tol2, counters_dev + c, streams[c]); break;
      case 256: e = launch_class<256>(td, nt, class_max_cap[c], class_max_m[c], tol2, counters_dev + c, streams[c]); break;
      case 128: e = launch_class<128>(td, nt, class_max_cap[c], class_max_m[c], tol2, counters_dev + c, streams[c]); break;
      default: e = launch_smem_class<64>(td, nt, class_max_cap[c], class_max_m[c], tol2, counters_dev + c, streams[c]); break;
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t hk_launch_aca(const AcaTask* tasks_dev, int ntasks, int max_cap, int max_m,
                          double tol2, cudaStream_t st, int max_mn) {
  // single class (the one-block API): 64..512 threads by the longer vector
  if (ntasks == 0) return cudaSuccess;
  int* counter = nullptr;
  cudaError_t e = cudaMallocAsync(&counter, sizeof(int), st);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(counter, 0, sizeof(int), st);
  const int L = max_mn;   // caller passes max(m, n) here
  if (L > 256) e = launch_class<512>(tasks_dev, ntasks, max_cap, max_m, tol2, counter, st);
  else if (L > 128) e = launch_class<256>(tasks_dev, ntasks, max_cap, max_m, tol2, counter, st);
  else if (L > 64) e = launch_class<128>(tasks_dev, ntasks, max_cap, max_m, tol2, counter, st);
  else e = launch_smem_class<64>(tasks_dev, ntasks, max_cap, max_m, tol2, counter, st);
  cudaFreeAsync(counter, st);
  return e;
}

int hk_aca_class(int m, int n) {
  const int L = m > n ? m : n;
  return L > 256 ? 0 : L > 128 ? 1 : L > 64 ? 2 : 3;
}

size_t hk_aca_scratch_doubles(int cap) { return (size_t)(2 * (512 / 32) + 1) * cap + KC; }
