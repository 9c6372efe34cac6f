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

#include <stdlib.h>

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

#ifndef HK_ACA_KC
#define HK_ACA_KC 8
#endif
constexpr int KC = HK_ACA_KC;   // columns per chunk (one transpose-reduce each): 8 or 16
#ifndef HK_ACA_KCY
#define HK_ACA_KCY 8
#endif
constexpr int KCY = HK_ACA_KCY;  // columns per chunk of the dot-free column sweep (sweep_y);
                                 // 16 measured slower (4.19 vs 3.96 ms: registers, occupancy)
constexpr int KPAD = 16;         // coefficient arrays are padded by this many entries

// Lane l of the warp receives the warp-wide sum of a[l & (KC-1)] (butterfly
// reduce-scatter inside groups of KC lanes, then exchanges between groups).
__device__ __forceinline__ double transpose_reduce(double (&a)[KC], int lane) {
#pragma unroll
  for (int s = KC / 2; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double send = upper ? a[i] : a[i + s];
      const double keep = upper ? a[i + s] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  double v = a[0];
#pragma unroll
  for (int o = KC; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// U/V column loads: plain weak loads, L1-cached (the CTA's own earlier stores
// are visible after its barriers; no other CTA writes this block's U/V)
#ifndef HK_ACA_UV_EL
#define HK_ACA_UV_EL 0
#endif
#ifndef HK_ACA_SRC_CS
#define HK_ACA_SRC_CS 0
#endif
__device__ __forceinline__ double ld_col(const double* p) {
#if HK_ACA_UV_EL
  // U/V are re-read every step: keep them in L2 ahead of the one-shot gathers
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
#else
  return *p;
#endif
}
// Row / column gathers of the front are read once per block: streaming loads
__device__ __forceinline__ double ld_src(const double* p) {
#if HK_ACA_SRC_CS
  return __ldcs(p);
#else
  return *p;
#endif
}

// Chunk helpers of the fused sweep (KC columns x EPT elements per thread).
//
// dots: part[w*pld + kb + j] += sum over the warp's elements of pv[e] * a[e][j]
// (EPT-sum in registers, then one transpose-reduce across the warp).  MASK
// zeroes the columns j with kb + j >= ndot (the chunk straddling ndot).
template <int EPT, bool MASK>
__device__ __forceinline__ void chunk_dots(const double (&a)[EPT][KC], const double (&pv)[EPT], int kb,
                                           int ndot, double* __restrict__ mypart, int lane) {
  double acc[KC];
#pragma unroll
  for (int j = 0; j < KC; ++j) {
    double sacc = 0.0;
#pragma unroll
    for (int q = 0; q < EPT; ++q) sacc = fma(pv[q], a[q][j], sacc);
    acc[j] = (!MASK || kb + j < ndot) ? sacc : 0.0;
  }
  const double v = transpose_reduce(acc, lane);
  if (lane < KC && (!MASK || kb + lane < ndot)) mypart[kb + lane] += v;
}

// residual update x[e] -= coef[k] * a[e][k] in k order (separate IEEE
// multiply and subtract: bit-exact with the reference); PART: only k < nk.
template <int EPT, bool PART, int KW>
__device__ __forceinline__ void chunk_sub(double (&x)[EPT], const double (&a)[EPT][KW],
                                          const double* __restrict__ coef, int kb, int nk) {
#pragma unroll
  for (int j = 0; j < KW; ++j) {
    const double c = coef[kb + j];
    if (!PART || kb + j < nk) {
#pragma unroll
      for (int q = 0; q < EPT; ++q) x[q] = sub_rn(x[q], mul_rn(c, a[q][j]));
    }
  }
}

// y[e] += sum_j a[e][j] * coef2[kb + j] (PART: only kb + j < n2): the U-side
// half of the stopping test as a coefficient sweep instead of dot products,
// sum_k (u.u_k)(v.v_k) = u . (U b) with b_k = v.v_k (no cross-lane reduction)
template <int EPT, bool PART, int KW>
__device__ __forceinline__ void chunk_y(double (&y)[EPT], const double (&a)[EPT][KW],
                                        const double* __restrict__ coef2, int kb, int n2) {
#pragma unroll
  for (int j = 0; j < KW; ++j) {
    const double c = coef2[kb + j];
    if (!PART || kb + j < n2) {
#pragma unroll
      for (int q = 0; q < EPT; ++q) y[q] = fma(a[q][j], c, y[q]);
    }
  }
}

template <int EPT, int LDLOG, int KW>
__device__ __forceinline__ void chunk_load_full(double (&a)[EPT][KW], const double* const (&pk)[EPT],
                                                int kb) {
  constexpr int64_t LD = int64_t(1) << LDLOG;
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    const double* p = pk[q] + (int64_t)kb * LD;
#pragma unroll
    for (int j = 0; j < KW; ++j) a[q][j] = ld_col(p + j * LD);
  }
}

// L1 prefetch of a whole chunk (issued one chunk ahead).  A warp's column
// segment is 32 consecutive doubles = two 128-byte lines, and prefetches are
// not coalesced across lanes, so only lanes 0 and 16 issue them (one request
// per line instead of 32: the ncu capture showed the per-lane prefetches as
// ~40% of the kernel's L2 sectors).
#ifndef HK_ACA_PF
#define HK_ACA_PF 1   // 0: no L1 prefetch (config-3 build 3.66 vs 3.46 ms, profiles/r02_aca_experiments.md)
#endif
template <int EPT, int LDLOG, int KW>
__device__ __forceinline__ void chunk_prefetch(const double* const (&pk)[EPT], int kb) {
  constexpr int64_t LD = int64_t(1) << LDLOG;
  if ((threadIdx.x & 15) != 0) return;
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    const double* p = pk[q] + (int64_t)kb * LD;
#pragma unroll
    for (int j = 0; j < KW; ++j) asm volatile("prefetch.global.L1 [%0];" ::"l"(p + j * LD));
  }
}

// Both halves of a full chunk's work; the chunk's column range is [kb, kb+KC).
template <int EPT, int KW>
__device__ __forceinline__ void chunk_process(double (&x)[EPT], const double (&a)[EPT][KW],
                                              const double (&pv)[EPT], const double* __restrict__ coef,
                                              int kb, int nk, int ndot, double* __restrict__ mypart,
                                              int lane, double (&y)[EPT],
                                              const double* __restrict__ coef2, int n2) {
  if constexpr (KW == KC) {
    if (kb < ndot) {                             // warp-uniform
      if (kb + KC <= ndot) chunk_dots<EPT, false>(a, pv, kb, ndot, mypart, lane);
      else chunk_dots<EPT, true>(a, pv, kb, ndot, mypart, lane);
    }
  }
  if (kb < n2) {                                 // warp-uniform
    if (kb + KW <= n2) chunk_y<EPT, false, KW>(y, a, coef2, kb, n2);
    else chunk_y<EPT, true, KW>(y, a, coef2, kb, n2);
  }
  if (kb + KW <= nk) chunk_sub<EPT, false, KW>(x, a, coef, kb, nk);
  else if (kb < nk) chunk_sub<EPT, true, KW>(x, a, coef, kb, nk);
}

// ---------------------------------------------------------------------------
// Fused residual sweep over one cross vector of length `len`.  F is COLUMN-major
// with power-of-two leading dimension LD = 1 << LDLOG (compile time, so every
// column load is an immediate offset from a per-element pointer).  Each thread
// owns EPT elements e = g0 + tid + q*NT (coalesced for every q):
//   F[e, out_col] = src[e] - sum_{k<nk} coef[k] * F[e, k]   (reference k order,
//                   separate IEEE multiply and subtract: bit-exact)
// and, for k < ndot, the per-warp partial dot products
//   part[w*pld + k] = sum_{e owned by warp w} F[e, pend_col] * F[e, k]
// of the PREVIOUS cross with the accepted crosses -- the stopping-test terms
// of the pending step ride along with the next step's sweep, so each cross
// vector is streamed once per step.  A chunk of KC columns issues EPT*KC
// independent loads; chunks that lie entirely inside the block are loaded
// unpredicated, with the next chunk prefetched into L1 while the current one
// is reduced; the ragged tail goes through a predicated path.  The dot partials of a chunk are summed over the thread's
// EPT elements first and then over the warp with one transpose-reduce.  Fixed
// reduction order (deterministic).  out_col < 0: dots only.  used != nullptr:
// column sweep (argmax over untouched entries + sum of squares); else row sweep.
template <int NT, int EPT, int LDLOG, int DB, int KW>
__device__ __forceinline__ void sweep_impl(const double* __restrict__ F, int len, int nk, int ndot,
                                           const double* __restrict__ coef,
                                           const double* __restrict__ src, int sstride,
                                           int out_col, bool store, int pend_col,
                                           double* __restrict__ part,
                                           int pld, const unsigned char* __restrict__ used,
                                           ArgMax& best, double& sumsq, double& bestval,
                                           double* __restrict__ xout,
                                           const double* __restrict__ coef2, int n2, double& ydot) {
  constexpr int64_t LD = int64_t(1) << LDLOG;
  const int tid = threadIdx.x, lane = tid & 31, warp = uniform_warp_id();
  // call arguments are not provably uniform across the call boundary
  len = __shfl_sync(0xffffffffu, len, 0);
  nk = __shfl_sync(0xffffffffu, nk, 0);
  ndot = __shfl_sync(0xffffffffu, ndot, 0);
  n2 = __shfl_sync(0xffffffffu, n2, 0);
  out_col = __shfl_sync(0xffffffffu, out_col, 0);
  ydot = 0.0;
  best.v = 0.0;
  best.i = -1;
  bestval = 0.0;
  sumsq = 0.0;
  double* mypart = part + warp * pld;
  for (int k = lane; k < ndot; k += 32) mypart[k] = 0.0;
  __syncwarp();
  const int kmax = nk > ndot ? nk : ndot;
#pragma unroll 1
  for (int g0 = 0; g0 < len; g0 += NT * EPT) {
    double x[EPT], pv[EPT], y[EPT];
    const double* pk[EPT];
    bool ok[EPT];
    // Chunks whose KC columns all lie inside the block load unpredicated even
    // in a ragged element group: a thread past `len` reads element 0 of the
    // column (always valid), its pv is 0 and its x is never stored, so it
    // contributes nothing.  (Blocks of 288/144/72 entries and the cluster
    // slices took the predicated path before: 2-3x slower sweeps.)
    constexpr bool gfull = true;
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
      const int e = g0 + tid + q * NT;
      ok[q] = e < len;
      pk[q] = F + (ok[q] ? e : 0);
      x[q] = (ok[q] && src) ? ld_src(src + (int64_t)e * sstride) : 0.0;
      pv[q] = (ok[q] && (ndot > 0 || n2 > 0)) ? pk[q][(int64_t)pend_col * LD] : 0.0;
      y[q] = 0.0;
    }
    int kb = 0;
    if (gfull) {
      const int kfull = (kmax / KW) * KW;
      if constexpr (DB != 0) {
      // register double buffer: chunk kb+KC is in flight while chunk kb is reduced
      if (kfull > 0) {
        double a0[EPT][KW], a1[EPT][KW];
        chunk_load_full<EPT, LDLOG, KW>(a0, pk, 0);
#pragma unroll 1
        for (; kb + 2 * KW <= kfull; kb += 2 * KW) {
          chunk_load_full<EPT, LDLOG, KW>(a1, pk, kb + KW);
          if (HK_ACA_PF == 1 && kb + 2 * KW < kfull) chunk_prefetch<EPT, LDLOG, KW>(pk, kb + 2 * KW);
          chunk_process<EPT, KW>(x, a0, pv, coef, kb, nk, ndot, mypart, lane, y, coef2, n2);
          if (kb + 2 * KW < kfull) chunk_load_full<EPT, LDLOG, KW>(a0, pk, kb + 2 * KW);
          chunk_process<EPT, KW>(x, a1, pv, coef, kb + KW, nk, ndot, mypart, lane, y, coef2, n2);
        }
        if (kb < kfull) {
          chunk_process<EPT, KW>(x, a0, pv, coef, kb, nk, ndot, mypart, lane, y, coef2, n2);
          kb += KW;
        }
      }
      } else {
#pragma unroll 1
      for (; kb < kfull; kb += KW) {
        double a[EPT][KW];
        chunk_load_full<EPT, LDLOG, KW>(a, pk, kb);
        // the next chunk's lines are pulled into L1 while this one is reduced
        // (prefetch distance 1 measured best: 2..4 thrash L1)
        if (HK_ACA_PF == 1 && kb + KW < kfull) chunk_prefetch<EPT, LDLOG, KW>(pk, kb + KW);
        chunk_process<EPT, KW>(x, a, pv, coef, kb, nk, ndot, mypart, lane, y, coef2, n2);
      }
      }
    }
#pragma unroll 1
    for (; kb < kmax; kb += KW) {                 // ragged tail (predicated loads)
      double a[EPT][KW];
#pragma unroll
      for (int q = 0; q < EPT; ++q)
#pragma unroll
        for (int j = 0; j < KW; ++j)
          a[q][j] = (ok[q] && kb + j < kmax) ? ld_col(pk[q] + (int64_t)(kb + j) * LD) : 0.0;
      chunk_process<EPT, KW>(x, a, pv, coef, kb, nk, ndot, mypart, lane, y, coef2, n2);
    }
    if (n2 > 0) {
#pragma unroll
      for (int q = 0; q < EPT; ++q) ydot = fma(pv[q], y[q], ydot);
    }
    if (out_col >= 0) {
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        if (!ok[q]) continue;
        const int e = g0 + tid + q * NT;
        // store == false: the caller keeps the residual in registers (xout) and
        // writes the scaled cross itself, so this store would be overwritten
        if (store) const_cast<double*>(F)[e + (int64_t)out_col * LD] = x[q];
        xout[q] = x[q];
        const double ax = fabs(x[q]);
        if (used) {
          sumsq += x[q] * x[q];
          if (!used[e] && argmax_better(ax, e, best.v, best.i)) { best.v = ax; best.i = e; bestval = x[q]; }
        } else if (argmax_better(ax, e, best.v, best.i)) {
          best.v = ax;
          best.i = e;
          bestval = x[q];
        }
      }
    }
  }
}

// One call target per (NT, EPT) for the caller (keeps its register allocation
// small); the leading dimension is dispatched once, inside.  The results come
// back BY VALUE (a struct of <= 64 bytes returns in registers): with reference
// out-parameters every call spilled them through the thread's stack, and those
// local-memory stores were 85% of the kernel's L2 write sectors (ncu:
// 3.8M of 4.45M write sectors per class-0 launch at 8 fronts).
template <int EPT>
struct SweepOut {
  double bv, sumsq, bestval, ydot;
  int bi;
  double x[EPT];
};

template <int NT, int EPT, int DB>
__device__ __noinline__ SweepOut<EPT> sweep_r(int ldlog, const double* __restrict__ F, int len, int nk,
                                              int ndot, const double* __restrict__ coef,
                                              const double* __restrict__ src, int sstride, int out_col,
                                              bool store, int pend_col, double* __restrict__ part,
                                              int pld, const unsigned char* __restrict__ used) {
  SweepOut<EPT> o;
  ArgMax best;
  best.v = 0.0;
  best.i = -1;
  o.sumsq = o.bestval = o.ydot = 0.0;
#pragma unroll
  for (int q = 0; q < EPT; ++q) o.x[q] = 0.0;
#define HK_SWEEP_CASE(L)                                                                       \
  case L:                                                                                      \
    sweep_impl<NT, EPT, L, DB, KC>(F, len, nk, ndot, coef, src, sstride, out_col, store, pend_col, part, pld, \
                           used, best, o.sumsq, o.bestval, o.x, nullptr, 0, o.ydot);           \
    break;
  switch (ldlog) {
    HK_SWEEP_CASE(6) HK_SWEEP_CASE(7) HK_SWEEP_CASE(8) HK_SWEEP_CASE(9) HK_SWEEP_CASE(10)
    HK_SWEEP_CASE(11) HK_SWEEP_CASE(12) HK_SWEEP_CASE(13)
    default: break;
  }
#undef HK_SWEEP_CASE
  o.bv = best.v;
  o.bi = (int)best.i;
  return o;
}

template <int NT, int EPT, int DB>
__device__ __forceinline__ void sweep(int ldlog, const double* __restrict__ F, int len, int nk, int ndot,
                                      const double* __restrict__ coef, const double* __restrict__ src,
                                      int sstride, int out_col, int pend_col, double* __restrict__ part,
                                      int pld, const unsigned char* __restrict__ used, ArgMax& best,
                                      double& sumsq, double& bestval, double* xout, bool store = true) {
  const SweepOut<EPT> o = sweep_r<NT, EPT, DB>(ldlog, F, len, nk, ndot, coef, src, sstride, out_col, store,
                                               pend_col, part, pld, used);
  best.v = o.bv;
  best.i = o.bi;
  sumsq = o.sumsq;
  bestval = o.bestval;
#pragma unroll
  for (int q = 0; q < EPT; ++q) xout[q] = o.x[q];
}

// The column sweep of the main ACA step with the coefficient sweep of the
// stopping test (y = U b, ydot = u_r . y), a separate call target so the
// other sweeps keep their register allocation.
template <int NT, int EPT, int DB>
__device__ __noinline__ SweepOut<EPT> sweep_y_r(int ldlog, const double* __restrict__ F, int len, int nk,
                                                const double* __restrict__ coef,
                                                const double* __restrict__ src, int sstride, int out_col,
                                                int pend_col, const unsigned char* __restrict__ used,
                                                const double* __restrict__ coef2, int n2) {
  SweepOut<EPT> o;
  ArgMax best;
  best.v = 0.0;
  best.i = -1;
  o.sumsq = o.bestval = o.ydot = 0.0;
#pragma unroll
  for (int q = 0; q < EPT; ++q) o.x[q] = 0.0;
#define HK_SWEEP_CASE(L)                                                                       \
  case L:                                                                                      \
    sweep_impl<NT, EPT, L, DB, KCY>(F, len, nk, 0, coef, src, sstride, out_col, true, pend_col, nullptr, 0, \
                           used, best, o.sumsq, o.bestval, o.x, coef2, n2, o.ydot);            \
    break;
  switch (ldlog) {
    HK_SWEEP_CASE(6) HK_SWEEP_CASE(7) HK_SWEEP_CASE(8) HK_SWEEP_CASE(9) HK_SWEEP_CASE(10)
    HK_SWEEP_CASE(11) HK_SWEEP_CASE(12) HK_SWEEP_CASE(13)
    default: break;
  }
#undef HK_SWEEP_CASE
  o.bv = best.v;
  o.bi = (int)best.i;
  return o;
}

template <int NT, int EPT, int DB>
__device__ __forceinline__ void sweep_y(int ldlog, const double* __restrict__ F, int len, int nk,
                                        const double* __restrict__ coef, const double* __restrict__ src,
                                        int sstride, int out_col, int pend_col,
                                        const unsigned char* __restrict__ used, ArgMax& best,
                                        double& sumsq, double& bestval, double* xout,
                                        const double* __restrict__ coef2, int n2, double& ydot) {
  const SweepOut<EPT> o =
      sweep_y_r<NT, EPT, DB>(ldlog, F, len, nk, coef, src, sstride, out_col, pend_col, used, coef2, n2);
  best.v = o.bv;
  best.i = o.bi;
  sumsq = o.sumsq;
  bestval = o.bestval;
  ydot = o.ydot;
#pragma unroll
  for (int q = 0; q < EPT; ++q) xout[q] = o.x[q];
}

// Block argmax of |x| (lowest index on ties) that also returns the signed
// value of the winner, in every thread and provably warp-uniform.  Thread
// candidates: (a.v = |x|, a.i = index or -1, val = signed x).  The element e
// of a sweep is owned by thread e % NT, so the winning lane of a warp is
// e & 31.  Warp stage: three REDUX reductions (warp_argmax_idx); block stage:
// the NW warp winners through SMEM, reduced the same way by every warp.
template <int NT>
__device__ __forceinline__ ArgMax block_argmax_val(ArgMax a, double val, double* sv, int64_t* si,
                                                   double* sval, double& out_val) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31;
  const int wi = warp_argmax_idx(a.v, a.i >= 0, (int)a.i);
  const int wl = wi & 31;
  const double wv = __shfl_sync(0xffffffffu, a.v, wl);
  const double wx = __shfl_sync(0xffffffffu, val, wl);
  if (NW == 1) {
    out_val = wx;
    return ArgMax{wv, (int64_t)wi};
  }
  const int warp = uniform_warp_id();
  if (lane == 0) { sv[warp] = wv; si[warp] = wi; sval[warp] = wx; }
  __syncthreads();
  const bool ok = lane < NW && si[lane < NW ? lane : 0] >= 0;
  const double cv = lane < NW ? sv[lane] : 0.0;
  const int ci = lane < NW ? (int)si[lane] : -1;
  const double cx = lane < NW ? sval[lane] : 0.0;
  const int bi = warp_argmax_idx(cv, ok, ci);
  // winner's warp slot: the smallest slot holding index bi (indices are unique)
  const unsigned mask = __ballot_sync(0xffffffffu, ok && ci == bi);
  const int slot = mask ? __ffs(mask) - 1 : 0;
  out_val = __shfl_sync(0xffffffffu, cx, slot);
  const double bv = __shfl_sync(0xffffffffu, cv, slot);
  // sv/si/sval are next written after the caller's next block barrier
  return ArgMax{bv, (int64_t)bi};
}

template <int NT>
__device__ __forceinline__ void bar() {
  if (NT == 32) __syncwarp();
  else __syncthreads();
}

// est = max(fro2 + cross + sum_k 2 (u.u_k)(v.v_k), cross) from the per-warp
// partials, fixed reduction order; valid in every thread.
template <int NT>
__device__ __forceinline__ double stopping_estimate(const double* __restrict__ partU,
                                                    const double* __restrict__ partV, int pld,
                                                    int r, double fro2, double cross,
                                                    double* __restrict__ prod, double* s_est) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = uniform_warp_id();
  for (int k = tid; k < r; k += NT) {
    double du = 0.0, dv = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      du += partU[w * pld + k];
      dv += partV[w * pld + k];
    }
    prod[k] = 2.0 * du * dv;
  }
  bar<NT>();
  if (warp == 0) {
    double sacc = 0.0;
    for (int k = lane; k < r; k += 32) sacc += prod[k];
    sacc = warp_sum(sacc);
    if (lane == 0) *s_est = fmax(fro2 + cross + sacc, cross);
  }
  bar<NT>();
  const double v = __shfl_sync(0xffffffffu, *s_est, 0);
  bar<NT>();
  return v;
}

// One block's ACA pivot chain (lowrank.py:230-286) as a speculative pipeline:
// the sweeps of step s+1 (which assume cross s is accepted) also accumulate
// cross s's stopping-test dot products; cross s is decided after them, and the
// speculative step (and its trace events) is discarded on rejection.
template <int NT, int EPT, int DB>
__device__ __forceinline__ void aca_block(const AcaTask& t, double tol2, int part_in_smem) {
  // task scalars and every control value below are provably warp-uniform
  // (shuffles from lane 0), so no shuffle compiles to the divergent fallback
  const int m = __shfl_sync(0xffffffffu, t.m, 0), n = __shfl_sync(0xffffffffu, t.n, 0);
  const int cap = __shfl_sync(0xffffffffu, t.cap, 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = uniform_warp_id();
  constexpr int NW = NT / 32;
  uint64_t t_start = 0;
  if (t.clock && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  extern __shared__ __align__(16) unsigned char smraw[];
  const int ldlog = __shfl_sync(0xffffffffu, t.ldu, 0);   // U and V share one power-of-two LD
  const int64_t LD = int64_t(1) << ldlog;
  // SMEM layout: coef[cap+KC], bv[cap+KC], partU/partV[NW*cap], prod[cap]
  // (or global scratch when they do not fit), used[m]
  double* sbase = reinterpret_cast<double*>(smraw);
  double* U = t.U;
  double* V = t.V;
  double* coef = sbase;
  const int pld = cap;
  const bool pin = part_in_smem;
  double* bv = coef + cap + KPAD;     // b_k = v_r . v_k of the pending cross (stopping test)
  double* partU = pin ? bv + cap + KPAD : t.scratch;
  double* partV = partU + NW * pld;
  double* prod = partV + NW * pld;
  unsigned char* used = reinterpret_cast<unsigned char*>(pin ? prod + cap : bv + cap + KPAD);
  __shared__ double red_v[NW > 0 ? NW : 1], red_a[NW > 0 ? NW : 1], red_b[NW > 0 ? NW : 1],
      red_x[NW > 0 ? NW : 1];
  __shared__ int64_t red_i[NW > 0 ? NW : 1];
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
  for (int k = tid; k < cap + KPAD; k += NT) coef[k] = bv[k] = 0.0;
  __syncthreads();

  const double* rowsrc_base = t.A;
  const int64_t rowsrc_ld = t.lda;
  int r = 0, row = 0, nused = 0;
  bool pending = false;                       // column r holds an undecided cross
  double uu_p = 0.0, vv_p = 0.0, fro2 = 0.0;
  ArgMax best, nxt;
  double dummy, uu, bval;
  double xv[EPT];

  for (;;) {
    const int c = r + (pending ? 1 : 0);     // index of the new candidate
    const bool can_step = pending ? (c < cap && nused < m) : (c < cap);
    if (!can_step) {
      if (pending) {                          // decide the last cross: dots only
        sweep<NT, EPT, DB>(ldlog, U, m, 0, r, coef, nullptr, 1, -1, r, partU, pld, nullptr, best, dummy, bval, xv);
        sweep<NT, EPT, DB>(ldlog, V, n, 0, r, coef, nullptr, 1, -1, r, partV, pld, nullptr, best, dummy, bval, xv);
        bar<NT>();
        const double cross = uu_p * vv_p;
        const double est = stopping_estimate<NT>(partU, partV, pld, r, fro2, cross, prod, &s_est);
        if (!(cross <= tol2 * est)) ++r;
      }
      break;
    }
    if (tid == 0) {
      used[row] = 1;
      if (trows) trows[nrow_ev] = row;
    }
    ++nrow_ev;
    ++nused;
    for (int k = tid; k < c; k += NT) coef[k] = U[row + (int64_t)k * LD];
    bar<NT>();
    // residual row (:253-256) + the pending cross's v dots
    sweep<NT, EPT, DB>(ldlog, V, n, c, pending ? r : 0, coef, rowsrc_base + (int64_t)row * rowsrc_ld, 1,
                   c, r, partV, pld, nullptr, best, dummy, bval, xv, n > NT * EPT);
    double delta;
    best = block_argmax_val<NT>(best, bval, red_v, red_i, red_x, delta);
    const int col = (int)best.i;
    if (delta == 0.0) {                       // zero residual row (:258-264)
      if (pending) {
        sweep<NT, EPT, DB>(ldlog, U, m, 0, r, coef, nullptr, 1, -1, r, partU, pld, nullptr, nxt, dummy, bval, xv);
        bar<NT>();
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
      bar<NT>();
      row = __shfl_sync(0xffffffffu, s_row, 0);
      bar<NT>();
      continue;
    }
    // b = V^T v_r of the pending cross (the row sweep's dots), fixed warp
    // order; the U side of the stopping test becomes a coefficient sweep
    if (pending) {
      if (NT == 32) __syncwarp();
      for (int k = tid; k < r; k += NT) {
        double sb = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) sb += partV[w * pld + k];
        bv[k] = sb;
      }
    }
    // v = res / delta (:265) over own elements
    double vv = 0.0;
    if (n <= NT * EPT) {
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        const int e = tid + q * NT;
        if (e < n) {
          const double v = div_rn(xv[q], delta);
          V[e + (int64_t)c * LD] = v;
          vv += v * v;
        }
      }
    } else {
      for (int e = tid; e < n; e += NT) {
        double* vp = V + e + (int64_t)c * LD;
        const double v = div_rn(*vp, delta);
        *vp = v;
        vv += v * v;
      }
    }
    for (int k = tid; k < c; k += NT) coef[k] = V[col + (int64_t)k * LD];
    if (tid == 0 && tcols) tcols[ncol_ev] = col;
    ++ncol_ev;
    bar<NT>();
    // residual column (:266-268) + next-row candidate (:283) + pending u dots
    // column gather: the transposed copy (coalesced) or, without one, the
    // row-major front itself with stride lda
    const double* csrc = t.At ? t.At + (int64_t)col * t.lda : t.A + col;
    const int cstride = t.At ? 1 : (int)t.lda;
    double ydot = 0.0;
    sweep_y<NT, EPT, DB>(ldlog, U, m, c, coef, csrc, cstride, c, r, used, nxt, uu, bval, xv, bv,
                         pending ? r : 0, ydot);
    {
      // next row = argmax over untouched rows; uu = |u|^2, vv = |v|^2 (fixed
      // summation order: warp tree, then the warp partials in warp order)
      const int wi = warp_argmax_idx(nxt.v, nxt.i >= 0, (int)nxt.i);
      uu = warp_sum(uu);
      vv = warp_sum(vv);
      ydot = warp_sum(ydot);
      if (NT == 32) {
        nxt.i = wi;
        uu = __shfl_sync(0xffffffffu, uu, 0);
        vv = __shfl_sync(0xffffffffu, vv, 0);
        ydot = __shfl_sync(0xffffffffu, ydot, 0);
      } else {
        const double wv = __shfl_sync(0xffffffffu, nxt.v, wi & 31);
        if (lane == 0) {
          red_v[warp] = wv; red_i[warp] = wi; red_a[warp] = uu; red_b[warp] = vv; red_x[warp] = ydot;
        }
        __syncthreads();
        const bool ok = lane < NW && red_i[lane < NW ? lane : 0] >= 0;
        const double cv = lane < NW ? red_v[lane] : 0.0;
        const int ci = lane < NW ? (int)red_i[lane] : -1;
        double a2 = lane < NW ? red_a[lane] : 0.0;
        double c2 = lane < NW ? red_b[lane] : 0.0;
        double y2 = lane < NW ? red_x[lane] : 0.0;
        nxt.i = warp_argmax_idx(cv, ok, ci);
        a2 = warp_sum(a2);
        c2 = warp_sum(c2);
        y2 = warp_sum(y2);
        uu = __shfl_sync(0xffffffffu, a2, 0);
        vv = __shfl_sync(0xffffffffu, c2, 0);
        ydot = __shfl_sync(0xffffffffu, y2, 0);
        // red_* are next written after the next step's first block barrier
      }
    }
    if (pending) {                            // stopping test of the pending cross (:269-275)
      // sum_k 2 (u_r.u_k)(v_r.v_k) = 2 u_r . (U b): the column sweep's ydot
      const double cross = uu_p * vv_p;
      const double est = fmax(fro2 + cross + 2.0 * ydot, cross);
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
    bar<NT>();
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

// Persistent: CTAs pull tasks from a global counter in list order (largest
// blocks first), so the long root chains start at t = 0 whatever the hardware
// dispatch order of CTAs is.
// HK_ACA_REGCAP: registers of the single-CTA classes capped through the
// minimum-blocks launch bound, so more pivot chains are co-resident per SM
// (measured same-run A/B on config 3: 128 -> ACA 3.88 ms, uncapped 160-168
// registers -> 4.28 ms, 96 -> 4.40 ms; config 4 build 6.5 vs 7.2 ms)
#ifndef HK_ACA_REGCAP
#define HK_ACA_REGCAP 128
#endif
#ifndef HK_ACA_REGCAP_BIG
#define HK_ACA_REGCAP_BIG HK_ACA_REGCAP   // classes 0 and 1 (NT >= 128)
#endif
constexpr int aca_cap(int nt) { return nt >= 128 ? HK_ACA_REGCAP_BIG : HK_ACA_REGCAP; }
constexpr int aca_minb(int nt) {
  return aca_cap(nt) ? (65536 / (nt * aca_cap(nt)) > 0 ? 65536 / (nt * aca_cap(nt)) : 1) : 1;
}

template <int NT, int EPT, int DB>
__global__ void __launch_bounds__(NT, aca_minb(NT)) aca_kernel(const AcaTask* __restrict__ tasks, int ntasks,
                                                 int* __restrict__ counter, double tol2,
                                                 int part_in_smem) {
  __shared__ int s_task;
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(counter, 1);
    __syncthreads();
    const int ti = __shfl_sync(0xffffffffu, s_task, 0);
    __syncthreads();
    if (ti >= ntasks) break;
    aca_block<NT, EPT, DB>(tasks[ti], tol2, part_in_smem);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Cluster ACA: one block's pivot chain run by a thread-block cluster of P CTAs.
//
// A single CTA sweeps all m (n) entries of every cross vector; for the large
// blocks of a big front (config 4: 4608 x 4608 at rank 227) that chain ran on
// one SM for 53 ms while the rest of the GPU idled.  Here CTA q of the cluster
// owns the 16-aligned slice [q*S, (q+1)*S) of the entries of both U and V, so
// each sweep streams only its slice; the decisions that couple the slices go
// through distributed shared memory, two cluster barriers per step:
//   BAR1  row-sweep argmax -> pivot column and delta (R slots); per-CTA
//         b = V^T v_r partials, summed over the cluster for the column sweep
//   BAR2  column-sweep argmax -> next row, |u|^2, |v|^2 and the per-CTA
//         u_r . (U b) of the stopping test (C slots)
// (the rare paths -- zero residual row, last step -- still decide through
// explicit dot partials and the E slots)
// Every CTA evaluates every decision from the same slots in the same order,
// so control stays cluster-uniform.  The residual entries are computed
// exactly as in aca_block (reference k order, separate multiply/subtract), so
// U, V, pivots and ranks are bit-identical to the single-CTA kernel's; only
// the summation order of the stopping-test dots changes (decision margins,
// SURVEY.md Appendix C).  Coefficient rows U[row, 0:c] / V[col, 0:c] written
// by other CTAs are read from global memory after the release/acquire
// cluster barriers; slices are 16-aligned so no 128-byte line is written by
// two CTAs.
struct ClSlot {
  double v, val, a, b;
  int idx;
  int pad;
};

// Cluster argmax over the P slots (lowest index on ties); idx, val and the
// slot's a/b sums in fixed slot order.  Valid in every lane of every warp.
__device__ __forceinline__ int cl_argmax(const ClSlot* slot, unsigned P, double& val, double& sa,
                                         double& sb) {
  const int lane = threadIdx.x & 31;
  double v = 0.0, x = 0.0, a = 0.0, b = 0.0;
  int i = -1;
  if (lane < (int)P) {
    const ClSlot* s = cl_map(slot, (unsigned)lane);
    v = s->v;
    x = s->val;
    a = s->a;
    b = s->b;
    i = s->idx;
  }
  const int bi = warp_argmax_idx(v, i >= 0, i);
  const unsigned mask = __ballot_sync(0xffffffffu, i >= 0 && i == bi);
  const int sl = mask ? __ffs(mask) - 1 : 0;
  val = __shfl_sync(0xffffffffu, x, sl);
  // fixed order sums over the slots (lane p holds slot p; shfl_down tree)
  sa = warp_sum(a);
  sb = warp_sum(b);
  sa = __shfl_sync(0xffffffffu, sa, 0);
  sb = __shfl_sync(0xffffffffu, sb, 0);
  return bi;
}

// CTA-level sums of the per-warp dot partials into cpart (k < r).
template <int NT>
__device__ __forceinline__ void cl_reduce_parts(const double* __restrict__ partU,
                                                const double* __restrict__ partV, int pld, int r,
                                                double* __restrict__ cpU, double* __restrict__ cpV) {
  constexpr int NW = NT / 32;
  for (int k = threadIdx.x; k < r; k += NT) {
    double du = 0.0, dv = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      du += partU[w * pld + k];
      dv += partV[w * pld + k];
    }
    cpU[k] = du;
    cpV[k] = dv;
  }
}

// After a cluster barrier that published cpart: this CTA's share of
// sum_k 2 (u.u_k)(v.v_k) over k in its range, written to its E slot by warp 0.
__device__ __forceinline__ void cl_est_share(const double* cpU, const double* cpV, int r,
                                             unsigned q, unsigned P, double* slE) {
  if (uniform_warp_id() != 0) return;
  const int lane = threadIdx.x & 31;
  const int per = (r + (int)P - 1) / (int)P;
  const int k0 = (int)q * per, k1 = min(r, k0 + per);
  double s = 0.0;
  for (int k = k0 + lane; k < k1; k += 32) {
    double du = 0.0, dv = 0.0;
    for (unsigned p = 0; p < P; ++p) {
      du += *cl_map(cpU + k, p);
      dv += *cl_map(cpV + k, p);
    }
    s += 2.0 * du * dv;
  }
  s = warp_sum(s);
  if (lane == 0) *slE = s;
}

__device__ __forceinline__ double cl_est_total(const double* slE, unsigned P) {
  const int lane = threadIdx.x & 31;
  double s = lane < (int)P ? *cl_map(slE, (unsigned)lane) : 0.0;
  s = warp_sum(s);
  return __shfl_sync(0xffffffffu, s, 0);
}

template <int NT, int EPT, int DB>
__global__ void __maxnreg__(200) aca_cluster_kernel(const AcaTask* __restrict__ tasks,
                                                         double tol2, int part_in_smem,
                                                         int* started) {
  constexpr int NW = NT / 32;
  const unsigned P = cl_nrank(), q = cl_rank();
  // residency signal for the host (mapped pinned memory): the launches that
  // follow wait until the largest clusters hold their SMs (see hk_build_aca)
  if (started && q == 0 && threadIdx.x == 0) atomicAdd_system(started, 1);
  const AcaTask& t = tasks[blockIdx.x / P];
  const int m = __shfl_sync(0xffffffffu, t.m, 0), n = __shfl_sync(0xffffffffu, t.n, 0);
  const int cap = __shfl_sync(0xffffffffu, t.cap, 0);
  const int tid = threadIdx.x;
  uint64_t t_start = 0;
  if (t.clock && tid == 0 && q == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  extern __shared__ __align__(16) unsigned char smraw[];
  const int ldlog = __shfl_sync(0xffffffffu, t.ldu, 0);
  const int64_t LD = int64_t(1) << ldlog;
  // entry slices (16-aligned: no 128-byte line of U/V is written by two CTAs)
  const int slm = (((m + (int)P - 1) / (int)P) + 15) & ~15;
  const int sln = (((n + (int)P - 1) / (int)P) + 15) & ~15;
  const int mu0 = min(m, (int)q * slm), mlen = min(m, mu0 + slm) - mu0;
  const int nv0 = min(n, (int)q * sln), nlen = min(n, nv0 + sln) - nv0;
  // SMEM: coef[cap+KC], cpU[cap], cpV[cap], bvc[cap+KC], (partU, partV [NW*cap] each), used[m]
  double* coef = reinterpret_cast<double*>(smraw);
  double* cpU = coef + cap + KPAD;
  double* cpV = cpU + cap;
  double* bvc = cpV + cap;          // b_k = v_r . v_k over the whole cluster (stopping test)
  const int pld = cap;
  double* partU = part_in_smem ? bvc + cap + KPAD : t.scratch + (size_t)q * 2 * NW * cap;
  double* partV = partU + NW * pld;
  unsigned char* used =
      reinterpret_cast<unsigned char*>(part_in_smem ? partV + NW * pld : bvc + cap + KPAD);
  __shared__ double red_v[NW], red_a[NW], red_b[NW], red_x[NW];
  __shared__ int64_t red_i[NW];
  __shared__ ClSlot slR, slC;
  __shared__ double slE;
  __shared__ int s_row;

  const bool lead = q == 0;
  int32_t* trows = (t.trace && lead) ? t.trace + 2 : nullptr;
  int32_t* tcols = (t.trace && lead) ? t.trace + 2 + (m + cap + 1) : nullptr;
  int nrow_ev = 0, ncol_ev = 0;
  if (m == 0 || n == 0 || cap == 0) {
    if (tid == 0 && lead) {
      *t.rank = 0;
      if (t.trace) { t.trace[0] = 0; t.trace[1] = 0; }
    }
    cluster_bar();
    return;
  }
  for (int i = tid; i < m; i += NT) used[i] = 0;
  for (int k = tid; k < cap + KPAD; k += NT) coef[k] = bvc[k] = 0.0;
  cluster_bar();

  double* Us = t.U + mu0;
  double* Vs = t.V + nv0;
  // column gathers: column col of the slice starts at cbase + col * cstep
  const double* cbase = t.At ? t.At + mu0 : t.A + (int64_t)mu0 * t.lda;
  const int64_t cstep = t.At ? t.lda : 1;
  const int cstride = t.At ? 1 : (int)t.lda;
  int r = 0, row = 0, nused = 0;
  bool pending = false;
  double uu_p = 0.0, vv_p = 0.0, fro2 = 0.0;
  ArgMax best, nxt;
  double dummy, uu, bval;
  double xv[EPT];

  // decide the pending cross from partials already in partU/partV (rare paths)
  auto decide_pending = [&](void) -> bool {   // true = accept
    bar<NT>();
    cl_reduce_parts<NT>(partU, partV, pld, r, cpU, cpV);
    cluster_bar();
    cl_est_share(cpU, cpV, r, q, P, &slE);
    cluster_bar();
    const double cross = uu_p * vv_p;
    const double est = fmax(fro2 + cross + cl_est_total(&slE, P), cross);
    const bool acc = !(cross <= tol2 * est);
    if (acc) fro2 = est;
    return acc;
  };

  for (;;) {
    const int c = r + (pending ? 1 : 0);
    const bool can_step = pending ? (c < cap && nused < m) : (c < cap);
    if (!can_step) {
      if (pending) {
        sweep<NT, EPT, DB>(ldlog, Us, mlen, 0, r, coef, nullptr, 1, -1, r, partU, pld, nullptr, best, dummy, bval, xv);
        sweep<NT, EPT, DB>(ldlog, Vs, nlen, 0, r, coef, nullptr, 1, -1, r, partV, pld, nullptr, best, dummy, bval, xv);
        if (decide_pending()) ++r;
      }
      break;
    }
    if (tid == 0) {
      used[row] = 1;
      if (trows) trows[nrow_ev] = row;
    }
    ++nrow_ev;
    ++nused;
    for (int k = tid; k < c; k += NT) coef[k] = __ldcg(t.U + row + (int64_t)k * LD);
    bar<NT>();
    // residual row slice + the pending cross's v dots
    sweep<NT, EPT, DB>(ldlog, Vs, nlen, c, pending ? r : 0, coef,
                       t.A + (int64_t)row * t.lda + nv0, 1, c, r, partV, pld, nullptr, best, dummy,
                       bval, xv, nlen > NT * EPT);
    {
      double lval;
      ArgMax lb = block_argmax_val<NT>(best, bval, red_v, red_i, red_x, lval);
      if (tid == 0) {
        slR.v = lb.v;
        slR.val = lval;
        slR.idx = lb.i >= 0 ? (int)lb.i + nv0 : -1;
        slR.a = slR.b = 0.0;
      }
      // this CTA's share of b = V^T v_r (its warps' partials, fixed order)
      if (pending)
        for (int k = tid; k < r; k += NT) {
          double sb = 0.0;
#pragma unroll
          for (int w = 0; w < NW; ++w) sb += partV[w * pld + k];
          cpV[k] = sb;
        }
    }
    cluster_bar();                                             // BAR1
    double delta, sa, sb;
    const int col = cl_argmax(&slR, P, delta, sa, sb);
    if (delta == 0.0) {                       // zero residual row (:258-264)
      if (pending) {
        sweep<NT, EPT, DB>(ldlog, Us, mlen, 0, r, coef, nullptr, 1, -1, r, partU, pld, nullptr, nxt, dummy, bval, xv);
        if (!decide_pending()) {
          --nrow_ev;
          break;
        }
        ++r;
        pending = false;
      }
      if (nused == m) break;
      if (tid == 0) {
        int qq = 0;
        while (used[qq]) ++qq;
        s_row = qq;
      }
      // cluster barrier: every CTA has read this step's R slots before the
      // next step's row sweep overwrites them
      cluster_bar();
      row = __shfl_sync(0xffffffffu, s_row, 0);
      bar<NT>();
      continue;
    }
    // v = res / delta over the own slice
    double vv = 0.0;
    if (nlen <= NT * EPT) {
#pragma unroll
      for (int qq = 0; qq < EPT; ++qq) {
        const int e = tid + qq * NT;
        if (e < nlen) {
          const double v = div_rn(xv[qq], delta);
          Vs[e + (int64_t)c * LD] = v;
          vv += v * v;
        }
      }
    } else {
      for (int e = tid; e < nlen; e += NT) {
        double* vp = Vs + e + (int64_t)c * LD;
        const double v = div_rn(*vp, delta);
        *vp = v;
        vv += v * v;
      }
    }
    // b over the cluster (slot order), the coefficients of the U-side sweep
    if (pending)
      for (int k = tid; k < r; k += NT) {
        double sb = 0.0;
        for (unsigned pp = 0; pp < P; ++pp) sb += *cl_map(cpV + k, pp);
        bvc[k] = sb;
      }
    for (int k = tid; k < c; k += NT) coef[k] = __ldcg(t.V + col + (int64_t)k * LD);
    if (tid == 0 && tcols) tcols[ncol_ev] = col;
    ++ncol_ev;
    bar<NT>();
    // residual column slice + next-row candidate + y = U b for the pending cross
    double ydot = 0.0;
    sweep_y<NT, EPT, DB>(ldlog, Us, mlen, c, coef, cbase + (int64_t)col * cstep, cstride, c, r,
                         used + mu0, nxt, uu, bval, xv, bvc, pending ? r : 0, ydot);
    {
      const int lane = tid & 31, warp = uniform_warp_id();
      const int wi = warp_argmax_idx(nxt.v, nxt.i >= 0, (int)nxt.i);
      uu = warp_sum(uu);
      vv = warp_sum(vv);
      ydot = warp_sum(ydot);
      const double wv = __shfl_sync(0xffffffffu, nxt.v, wi & 31);
      if (lane == 0) {
        red_v[warp] = wv; red_i[warp] = wi; red_a[warp] = uu; red_b[warp] = vv; red_x[warp] = ydot;
      }
      __syncthreads();
      const bool ok = lane < NW && red_i[lane < NW ? lane : 0] >= 0;
      const double cv = lane < NW ? red_v[lane] : 0.0;
      const int ci = lane < NW ? (int)red_i[lane] : -1;
      double a2 = lane < NW ? red_a[lane] : 0.0;
      double c2 = lane < NW ? red_b[lane] : 0.0;
      double y2 = lane < NW ? red_x[lane] : 0.0;
      const int bi = warp_argmax_idx(cv, ok, ci);
      a2 = warp_sum(a2);
      c2 = warp_sum(c2);
      y2 = warp_sum(y2);
      const unsigned mask = __ballot_sync(0xffffffffu, ok && ci == bi);
      const double bv = __shfl_sync(0xffffffffu, cv, mask ? __ffs(mask) - 1 : 0);
      if (tid == 0) {
        slC.v = bv;
        slC.idx = bi >= 0 ? bi + mu0 : -1;
        slC.val = y2;                     // this CTA's u_r . (U b)
        slC.a = a2;
        slC.b = c2;
      }
    }
    cluster_bar();                                             // BAR2
    double dum;
    const int nrow = cl_argmax(&slC, P, dum, uu, vv);
    if (pending) {                            // stopping test of the pending cross (:269-275)
      // sum_k 2 (u_r.u_k)(v_r.v_k) = 2 u_r . (U b), summed over the slots in order
      const int lane = tid & 31;
      double ys = lane < (int)P ? cl_map(&slC, (unsigned)lane)->val : 0.0;
      ys = warp_sum(ys);
      ys = __shfl_sync(0xffffffffu, ys, 0);
      const double cross = uu_p * vv_p;
      const double est = fmax(fro2 + cross + 2.0 * ys, cross);
      if (cross <= tol2 * est) {
        --nrow_ev;
        --ncol_ev;
        break;
      }
      ++r;
      fro2 = est;
    }
    pending = true;
    uu_p = uu;
    vv_p = vv;
    row = nrow;
  }
  if (tid == 0 && lead) {
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
  cluster_bar();   // no CTA leaves while another may still read its SMEM
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

// Size classes by the longer cross vector L = max(m, n); every class runs
// 2 elements per thread (measured best against 1 and 4 on config 3):
//   class 0: L > 256         256 threads
//   class 1: 128 < L <= 256  128 threads
//   class 2: 64 < L <= 128    64 threads
//   class 3: L <= 64          32 threads (one warp, no block barriers)
int hk_aca_class(int m, int n) {
  const int L = m > n ? m : n;
  return L > 256 ? 0 : L > 128 ? 1 : L > 64 ? 2 : 3;
}

// Per-warp dot partials live in SMEM when the CTA's whole footprint stays
// under this bound (2 CTAs per SM still fit); otherwise in global scratch.
#ifndef HK_ACA_PART_SMEM
#define HK_ACA_PART_SMEM (112 * 1024)
#endif

template <int NT, int EPT, int DB>
static cudaError_t launch_cls(const AcaTask* tasks_dev, int ntasks, int max_cap, int max_m,
                              double tol2, int* counter, cudaStream_t st) {
  const size_t part_bytes = (size_t)(2 * (NT / 32) + 1) * max_cap * 8;
  const size_t base = (size_t)2 * (max_cap + KPAD) * 8 + (size_t)max_m + 16;   // coef, bv, used
  const int part_in_smem = (base + part_bytes <= HK_ACA_PART_SMEM) ? 1 : 0;
  const size_t smem = base + (part_in_smem ? part_bytes : 0);
  cudaError_t e = cudaFuncSetAttribute(aca_kernel<NT, EPT, DB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, aca_kernel<NT, EPT, DB>, NT, smem);
  if (e != cudaSuccess) return e;
  int grid = sms * (per_sm > 0 ? per_sm : 1);
  if (grid > ntasks) grid = ntasks;
  aca_kernel<NT, EPT, DB><<<grid, NT, smem, st>>>(tasks_dev, ntasks, counter, tol2, part_in_smem);
  hk_count_launch();
  return cudaGetLastError();
}

// Register double-buffered sweeps per class (HK_ACA_Dc = 1): faster steps
// (fewer exposed L2 round trips) at more registers, i.e. fewer resident CTAs.
#ifndef HK_ACA_D0
#define HK_ACA_D0 0
#endif
#ifndef HK_ACA_D1
#define HK_ACA_D1 1
#endif
#ifndef HK_ACA_D2
#define HK_ACA_D2 1
#endif
#ifndef HK_ACA_D3
#define HK_ACA_D3 1
#endif

// CTA shape (threads x elements per thread) of each size class.
#ifndef HK_ACA_T0
#define HK_ACA_T0 256
#define HK_ACA_E0 2
#define HK_ACA_T1 128
#define HK_ACA_E1 2
#define HK_ACA_T2 64
#define HK_ACA_E2 2
#define HK_ACA_T3 32
#define HK_ACA_E3 2
#endif

static cudaError_t launch_class_id(int cls, const AcaTask* td, int nt, int max_cap, int max_m,
                                   double tol2, int* counter, cudaStream_t st) {
  switch (cls) {
    case 0: return launch_cls<HK_ACA_T0, HK_ACA_E0, HK_ACA_D0>(td, nt, max_cap, max_m, tol2, counter, st);
    case 1: return launch_cls<HK_ACA_T1, HK_ACA_E1, HK_ACA_D1>(td, nt, max_cap, max_m, tol2, counter, st);
    case 2: return launch_cls<HK_ACA_T2, HK_ACA_E2, HK_ACA_D2>(td, nt, max_cap, max_m, tol2, counter, st);
    default: return launch_cls<HK_ACA_T3, HK_ACA_E3, HK_ACA_D3>(td, nt, max_cap, max_m, tol2, counter, st);
  }
}

// Tasks arrive grouped by size class and largest-first inside a class; each
// class is one persistent launch; classes run concurrently on the given
// streams (the caller forks/joins them).
cudaError_t hk_launch_aca_classes(const AcaTask* tasks_dev, const int* class_begin,
                                  const int* class_max_cap, const int* class_max_m, double tol2,
                                  int* counters_dev, cudaStream_t* streams) {
  for (int c = 0; c < 4; ++c) {
    const int nt = class_begin[c + 1] - class_begin[c];
    if (nt == 0) continue;
    cudaError_t e = launch_class_id(c, tasks_dev + class_begin[c], nt, class_max_cap[c],
                                    class_max_m[c], tol2, counters_dev + c, streams[c]);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t hk_launch_aca(const AcaTask* tasks_dev, int ntasks, int max_cap, int max_m,
                          double tol2, cudaStream_t st, int max_mn) {
  // single-block API: the class of the block (max_mn = max(m, n))
  if (ntasks == 0) return cudaSuccess;
  const int P = hk_aca_cluster_size(max_mn, max_mn);
  if (P > 1) return hk_launch_aca_cluster(tasks_dev, ntasks, P, max_cap, max_m, tol2, st, nullptr,
                                          nullptr);
  int* counter = nullptr;
  cudaError_t e = hk_dev_malloc(&counter, sizeof(int), st);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(counter, 0, sizeof(int), st);
  e = launch_class_id(hk_aca_class(max_mn, max_mn), tasks_dev, ntasks, max_cap, max_m, tol2, counter, st);
  hk_dev_free(counter, st);
  return e;
}

size_t hk_aca_scratch_doubles(int cap) { return (size_t)(2 * (512 / 32) + 1) * cap + 16; }

// ---------------------------------------------------------------- cluster ACA
#ifndef HK_ACA_CLNT
#define HK_ACA_CLNT 160   // threads per cluster CTA: 2 entries each -> 320-entry slices
#endif
#ifndef HK_ACA_CLDB
#define HK_ACA_CLDB 1
#endif
constexpr int kClNT = HK_ACA_CLNT, kClEPT = 2;

// Blocks whose longer side exceeds HK_ACA_CLMIN (default 512) run on a
// cluster of P = pow2ceil(ceil(L / 320)) CTAs (at most 16), so that every CTA
// sweeps one <= 320-entry slice in a single pass; smaller blocks stay on the
// single-CTA size classes.  Returns 1 for a single-CTA block.
int hk_aca_cluster_size(int m, int n) {
  static int clmin = -1;
  if (clmin < 0) {
    const char* e = getenv("HK_ACA_CLMIN");
    clmin = e ? atoi(e) : 512;
  }
  const int L = m > n ? m : n;
  if (L <= clmin) return 1;
  static int pmax = -1;
  if (pmax < 0) {
    const char* e = getenv("HK_ACA_PMAX");
    pmax = e ? atoi(e) : 16;
  }
  const int need = (L + kClNT * kClEPT - 1) / (kClNT * kClEPT);
  int P = 2;
  while (P < need && P < pmax) P <<= 1;
  return P;
}

size_t hk_aca_scratch_doubles_cl(int cap, int P) {
  return (size_t)P * 2 * (kClNT / 32) * cap + 16;
}

cudaError_t hk_launch_aca_cluster(const AcaTask* tasks_dev, int ntasks, int P, int max_cap,
                                  int max_m, double tol2, cudaStream_t st, int* started,
                                  int* max_active) {
  if (ntasks == 0) return cudaSuccess;
  auto kern = aca_cluster_kernel<kClNT, kClEPT, HK_ACA_CLDB>;
  constexpr int NW = kClNT / 32;
  const size_t base = (size_t)2 * (max_cap + KPAD) * 8 + (size_t)2 * max_cap * 8 + (size_t)max_m + 16;
  const size_t part_bytes = (size_t)2 * NW * max_cap * 8;
  const int part_in_smem = (base + part_bytes <= 200 * 1024) ? 1 : 0;
  const size_t smem = base + (part_in_smem ? part_bytes : 0);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (P > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  cfg.blockDim = dim3(kClNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // largest cluster the device can co-schedule with this footprint (the
  // slices follow the runtime cluster size, so any P >= 1 is correct)
  for (;;) {
    at[0].val.clusterDim.x = (unsigned)P;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(P * ntasks));
    int ncl = 0;
    e = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
    if (e == cudaSuccess && ncl >= 1) {
      if (max_active) *max_active = ncl;
      break;
    }
    (void)cudaGetLastError();
    if (P == 1) return e != cudaSuccess ? e : cudaErrorLaunchOutOfResources;
    P >>= 1;
  }
  e = cudaLaunchKernelEx(&cfg, kern, tasks_dev, tol2, part_in_smem, started);
  hk_count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}
