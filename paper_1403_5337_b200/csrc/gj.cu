// Batched Gauss-Jordan inversion with partial pivoting (leaf blocks and the
// r x r Woodbury capacitance matrices I - Y X of the coupling systems).
//
// One CTA per matrix.  N <= 160: the matrix is held in registers, distributed
// over the warps by column blocks (gj_df_kernel / gj_blk_kernel below).
// Larger N (config 4's top levels): gj_kernel keeps the matrix in SMEM or a
// global scratch and applies one rank-1 update per elimination step.  Pivoting
// is partial (largest |entry| among rows not yet used, lowest row on ties), so
// the singularity test min|pivot| < 1e-300 is the reference's
// (src/dense.py:76-77).
#include <cuda.h>

#include "hk_common.cuh"
#include "hk_internal.h"

#include <stdlib.h>

namespace {

// One pivot step applied to CPW register columns (rows lane + 32 q): for
// every column but `skip`, rj = W[p][j] / pivot (through rinv), W[i][j] -=
// ck[i] rj for i != p and W[p][j] = rj -- the arithmetic of the loop this
// replaces, so the bits are unchanged.  QP = p >> 5 is warp-uniform, so the
// caller dispatches it once per step (switch) and the pivot row's register is
// a compile-time index: no per-element selects (the select-based form spent
// 85% of the kernel's instructions on FSEL/LOP3/ISETP).
template <int CPW, int RPL, int QP>
__device__ __forceinline__ void gj_apply_step(double (&w)[CPW][RPL], const double (&ck)[RPL],
                                              double rinv, int lp, int lane, int skip) {
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj) {
    if (jj == skip) continue;
    const double rj = __shfl_sync(0xffffffffu, w[jj][QP], lp) * rinv;
#pragma unroll
    for (int q = 0; q < RPL; ++q) w[jj][q] = fma(-ck[q], rj, w[jj][q]);
    if (lane == lp) w[jj][QP] = rj;
  }
}
template <int CPW, int RPL>
__device__ __forceinline__ void gj_apply_step_dyn(double (&w)[CPW][RPL], const double (&ck)[RPL],
                                                  double rinv, int qp, int lp, int lane, int skip) {
  static_assert(RPL <= 8, "RPL <= 8");
  switch (qp) {
    case 0: gj_apply_step<CPW, RPL, 0>(w, ck, rinv, lp, lane, skip); break;
    case 1: if constexpr (RPL > 1) gj_apply_step<CPW, RPL, (RPL > 1 ? 1 : 0)>(w, ck, rinv, lp, lane, skip); break;
    case 2: if constexpr (RPL > 2) gj_apply_step<CPW, RPL, (RPL > 2 ? 2 : 0)>(w, ck, rinv, lp, lane, skip); break;
    case 3: if constexpr (RPL > 3) gj_apply_step<CPW, RPL, (RPL > 3 ? 3 : 0)>(w, ck, rinv, lp, lane, skip); break;
    case 4: if constexpr (RPL > 4) gj_apply_step<CPW, RPL, (RPL > 4 ? 4 : 0)>(w, ck, rinv, lp, lane, skip); break;
    case 5: if constexpr (RPL > 5) gj_apply_step<CPW, RPL, (RPL > 5 ? 5 : 0)>(w, ck, rinv, lp, lane, skip); break;
    case 6: if constexpr (RPL > 6) gj_apply_step<CPW, RPL, (RPL > 6 ? 6 : 0)>(w, ck, rinv, lp, lane, skip); break;
    default: if constexpr (RPL > 7) gj_apply_step<CPW, RPL, (RPL > 7 ? 7 : 0)>(w, ck, rinv, lp, lane, skip); break;
  }
}



constexpr int GJ_NT = 256;
constexpr size_t GJ_SMEM_CAP = 224 * 1024;

// workspace layout (SMEM or global scratch): W[N*N], colk[N], rowk[N] doubles,
// then piv[N], cperm[N] ints
__host__ __device__ inline size_t gj_bytes(int N) {
  return (size_t)N * N * 8 + (size_t)2 * N * 8 + (size_t)2 * N * 4;
}

// Panel-blocked Gauss-Jordan (same implicit partial pivoting, same per-element
// arithmetic and order as the unblocked elimination, so bit-identical results).  Warp w
// owns the CPW consecutive columns j = w*CPW + jj; lane l holds rows
// l + 32q.  Panel P is the column block of warp P: that warp alone runs the CPW
// pivot steps of its panel (warp-synchronous, no CTA barrier), saving for every
// step the pre-step pivot column and 1/pivot in SMEM; after ONE CTA barrier
// every other warp replays the CPW steps on its own columns (pivot-row entries
// broadcast by shuffle from the lane that holds the row).  N/CPW barriers per
// matrix instead of N.  Per pivot step: the used-row mask lives in registers
// (every warp sees every pivot), the search is three REDUX reductions
// (warp_argmax_idx), and each lane computes the reciprocal of its own
// candidate while the reduction runs.  Every branch is on values ptxas can
// prove warp-uniform, so no shuffle takes the divergent-warp fallback.
template <int NW, int CPW, int RPL>
__global__ void __launch_bounds__(NW * 32, 1) gj_blk_kernel(const GjTask* __restrict__ tasks) {
  constexpr int NT = NW * 32;
  constexpr int NR = 32 * RPL;
  const GjTask t = tasks[blockIdx.x];
  const int N = __shfl_sync(0xffffffffu, t.N, 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = uniform_warp_id();
  __shared__ double ckbuf[2][CPW][NR];
  __shared__ double rinvbuf[2][CPW];
  __shared__ int pbuf[2][CPW];
  __shared__ int s_sing, pivrow[NR], invp[NR];
  if (N == 0) {
    if (tid == 0) *t.status = 0;
    return;
  }
  double w_[CPW][RPL];
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q, j = warp * CPW + jj;
      const bool in = i < N && j < N;
      const int64_t off = t.mode == 0 ? (int64_t)i * t.src_ld + j : i + (int64_t)j * t.src_ld;
      w_[jj][q] = in ? t.src[off] : 0.0;
    }
  unsigned used = 0;                     // bit q: row lane + 32q already a pivot row
  if (tid == 0) s_sing = 0;
  __syncthreads();
  const int npan = (N + CPW - 1) / CPW;
  for (int P = 0; P < npan; ++P) {
    const int buf = P & 1;
    const int nl = min(CPW, N - P * CPW);
    if (warp == P) {
      int sing = 0;
#pragma unroll
      for (int l = 0; l < CPW; ++l) {
        if (l >= nl) break;
        const int c = P * CPW + l;
        // lane-local best over its unused rows (lowest q on ties), its
        // reciprocal computed while the warp reduction runs
        double bv = 0.0, bw = 1.0;
        int bi = 0x7fffffff;
        bool have = false;
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int i = lane + 32 * q;
          const double av = fabs(w_[l][q]);
          if (i < N && !((used >> q) & 1u) && (!have || av > bv)) {
            bv = av; bw = w_[l][q]; bi = i; have = true;
          }
        }
        const double myrinv = __drcp_rn(bw);
        const int p = warp_argmax_idx(bv, have, bi);
        const int lp = p & 31, qp = p >> 5;
        const double pivabs = __shfl_sync(0xffffffffu, bv, lp);
        if (t.near && lane == 0 && pivabs < HK_NEAR_PIVOT) *t.near = 1;
        if (!(pivabs >= HK_PIVOT_FLOOR)) { sing = 1; break; }
        const double rinv = __shfl_sync(0xffffffffu, myrinv, lp);
        double ck[RPL];
        bool isp[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int i = lane + 32 * q;
          ck[q] = w_[l][q];
          isp[q] = i == p;
          if (i < N) ckbuf[buf][l][i] = ck[q];
        }
        if (lane == lp) used |= 1u << qp;
        if (lane == 0) {
          rinvbuf[buf][l] = rinv;
          pbuf[buf][l] = p;
          pivrow[c] = p;
        }
        gj_apply_step_dyn<CPW, RPL>(w_, ck, rinv, qp, lp, lane, l);
#pragma unroll
        for (int q = 0; q < RPL; ++q) w_[l][q] = isp[q] ? rinv : -ck[q] * rinv;
      }
      if (sing && lane == 0) s_sing = 1;
    }
    __syncthreads();
    if (__shfl_sync(0xffffffffu, s_sing, 0)) break;
    if (warp != P) {
#pragma unroll 1
      for (int l = 0; l < nl; ++l) {
        const int p = __shfl_sync(0xffffffffu, pbuf[buf][l], 0);
        const double rinv = rinvbuf[buf][l];
        const int qp = p >> 5, lp = p & 31;
        if (lane == lp) used |= 1u << qp;
        double ck[RPL];
        bool isp[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int i = lane + 32 * q;
          ck[q] = (i < N) ? ckbuf[buf][l][i] : 0.0;
          isp[q] = i == p;
        }
        gj_apply_step_dyn<CPW, RPL>(w_, ck, rinv, qp, lp, lane, -1);
      }
    }
  }
  const int singular = __shfl_sync(0xffffffffu, s_sing, 0);
  if (tid == 0) *t.status = singular;
  if (singular) return;
  for (int k = tid; k < N; k += NT) invp[pivrow[k]] = k;
  __syncthreads();
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int r = lane + 32 * q, j = warp * CPW + jj;
      if (r < N && j < N) t.out[invp[r] + (int64_t)pivrow[j] * t.out_ld] = w_[jj][q];
    }
}

// Dataflow Gauss-Jordan (no CTA barrier inside the elimination).  Same
// distribution, pivoting and per-element arithmetic as gj_blk_kernel (bit-
// identical results).  Every pivot step c is published once -- the pre-step
// pivot column, the pivot row and 1/pivot, in SMEM slots that are never
// reused -- followed by a release store of the step counter.  Each warp walks
// the steps in order: the owner of column c runs the pivot step on its
// registers and publishes it, every other warp waits for the counter (acquire)
// and replays the step on its own columns.  The owner of the next panel is
// therefore never more than one step behind, and the critical path is one
// pivot search + update per step instead of a CTA barrier per panel.
#ifndef HK_GJ_MBAR
#define HK_GJ_MBAR 1
#endif
#ifndef HK_GJ_LAZY
#define HK_GJ_LAZY 0
#endif
#ifndef HK_GJ_SPIN_NS
#define HK_GJ_SPIN_NS 0
#endif
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

// Leaf tiles through the TMA: with a tensor map of the batch of row-major
// fronts ([batch][n][n], box 64 x 64 x 1), the CTA stages its leaf block
// K = A[lo:lo+N, lo:lo+N] into SMEM with one cp.async.bulk.tensor.3d (rows
// beyond n are zero-filled by the TMA unit) and fills its registers from there,
// instead of 32 row-strided global loads per warp instruction.  The block's
// coordinates follow from its source pointer: src = A + f*fstride + lo*lda + lo.
struct GjLeafMap {
  const double* base;
  int64_t lda, fstride;
};

template <int NW, int CPW, int RPL, bool TMA>
__global__ void __launch_bounds__(NW * 32, 1) gj_df_kernel(const GjTask* __restrict__ tasks,
                                                           const __grid_constant__ CUtensorMap tmap,
                                                           GjLeafMap lm) {
  constexpr int NT = NW * 32;
  constexpr int NR = 32 * RPL;
  const GjTask t = tasks[blockIdx.x];
  const int N = __shfl_sync(0xffffffffu, t.N, 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = uniform_warp_id();
  extern __shared__ __align__(16) double ckall[];   // [N][NR] pre-step pivot columns
  __shared__ double rinv_s[NR];
  __shared__ int p_s[NR], invp[NR];
  __shared__ int s_pub;                             // number of published steps
#if HK_GJ_MBAR
  // one mbarrier per step (never reused): waiters sleep in try_wait instead of
  // spinning on s_pub, so the owner's pivot chain keeps the issue slots
  __shared__ __align__(8) uint64_t stepbar[NR];
#endif
  if (N == 0) {
    if (tid == 0) *t.status = 0;
    return;
  }
  double w_[CPW][RPL];
  if constexpr (TMA) {
    // the 64 x 64 box lands in ckall (sized for it); ckall is rewritten only
    // after every warp has moved the box into registers (barrier below)
    __shared__ __align__(8) uint64_t bar;
    // bulk tensor copies need a 128-byte aligned destination (launch adds 128 B)
    double* stage = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ckall) + 127) & ~uintptr_t(127));
    if (tid == 0) {
      const int64_t off = t.src - lm.base;
      const int f = (int)(off / lm.fstride);
      const int64_t rem = off - (int64_t)f * lm.fstride;
      const int row = (int)(rem / lm.lda), col = (int)(rem - (int64_t)row * lm.lda);
      mbar_init(&bar, 1);
      mbar_init_fence();
      mbar_arrive_tx(&bar, 64 * 64 * 8);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(stage)),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(col), "r"(row), "r"(f), "r"(smem_u32(&bar))
          : "memory");
    }
    __syncthreads();
    mbar_wait(&bar, 0);
#pragma unroll
    for (int jj = 0; jj < CPW; ++jj)
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        const int i = lane + 32 * q, j = warp * CPW + jj;
        w_[jj][q] = (i < N && j < N) ? stage[i * 64 + j] : 0.0;
      }
    __syncthreads();
  } else {
#pragma unroll
    for (int jj = 0; jj < CPW; ++jj)
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        const int i = lane + 32 * q, j = warp * CPW + jj;
        const bool in = i < N && j < N;
        const int64_t off = t.mode == 0 ? (int64_t)i * t.src_ld + j : i + (int64_t)j * t.src_ld;
        w_[jj][q] = in ? t.src[off] : 0.0;
      }
  }
  unsigned used = 0;
  if (tid == 0) s_pub = 0;
#if HK_GJ_MBAR
  if (tid == 0) {
    for (int k = 0; k < N; ++k) mbar_init(&stepbar[k], 1);
    mbar_init_fence();
  }
#endif
  __syncthreads();
  bool singular = false;
  // walk every step in order (panel-major, so the column slot l is a compile-
  // time constant for the owner's register accesses)
  const int npan = (N + CPW - 1) / CPW;
  for (int P = 0; P < npan; ++P) {
    if (__shfl_sync(0xffffffffu, (int)singular, 0)) break;
#pragma unroll
    for (int l = 0; l < CPW; ++l) {
      const int c = P * CPW + l;
      if (c >= N) break;
      double* ck_s = ckall + (size_t)c * NR;
      if (warp == P) {
        double bv = 0.0, bw = 1.0;
        int bi = 0x7fffffff;
        bool have = false;
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int i = lane + 32 * q;
          const double av = fabs(w_[l][q]);
          if (i < N && !((used >> q) & 1u) && (!have || av > bv)) {
            bv = av; bw = w_[l][q]; bi = i; have = true;
          }
        }
        const double myrinv = __drcp_rn(bw);
        const int p = warp_argmax_idx(bv, have, bi);
        const int lp = p & 31, qp = p >> 5;
        const double pivabs = __shfl_sync(0xffffffffu, bv, lp);
        if (t.near && lane == 0 && pivabs < HK_NEAR_PIVOT) *t.near = 1;
        if (__any_sync(0xffffffffu, !(pivabs >= HK_PIVOT_FLOOR))) {
          if (lane == 0) {
            p_s[c] = -1;
            // release every waiter, lazy ones included: they stop at step c
            st_release_cta(&s_pub, HK_GJ_LAZY ? N + 1 : c + 1);
#if HK_GJ_MBAR
            mbar_arrive(&stepbar[c]);
#endif
          }
          singular = true;
          break;
        }
        const double rinv = __shfl_sync(0xffffffffu, myrinv, lp);
        double ck[RPL];
        bool isp[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int i = lane + 32 * q;
          ck[q] = w_[l][q];
          isp[q] = i == p;
          if (i < N) ck_s[i] = ck[q];
        }
        if (lane == lp) used |= 1u << qp;
        if (lane == 0) {
          rinv_s[c] = rinv;
          p_s[c] = p;
        }
        __syncwarp();
#if HK_GJ_MBAR
        if (lane == 0) mbar_arrive(&stepbar[c]);   // release: the step's SMEM slots are visible
#else
        if (lane == 0) st_release_cta(&s_pub, c + 1);
#endif
        gj_apply_step_dyn<CPW, RPL>(w_, ck, rinv, qp, lp, lane, l);
#pragma unroll
        for (int q = 0; q < RPL; ++q) w_[l][q] = isp[q] ? rinv : -ck[q] * rinv;
      } else {
        // every lane acquires the publication itself (a value read by lane 0
        // alone would not order the other lanes' reads of the step's data).
        // Lazy replay: only the next panel's owner follows the owner step by
        // step; every other warp waits for the whole panel and then replays its
        // steps in the same order (same arithmetic, same bits), so the owner's
        // pivot chain no longer shares its SM sub-partition's issue slots with
        // NW-2 warps replaying every step.
#if HK_GJ_MBAR
        mbar_wait(&stepbar[c], 0);                  // acquire
#else
        const int need = (!HK_GJ_LAZY || warp == P + 1) ? c : min(N, (P + 1) * CPW) - 1;
        while (ld_acquire_cta(&s_pub) <= need) {
#if HK_GJ_SPIN_NS
          __nanosleep(HK_GJ_SPIN_NS);   // back off: the spinning warps share the MIO pipe with the owner
#endif
        }
#endif
        __syncwarp();
        const int p = __shfl_sync(0xffffffffu, lane == 0 ? p_s[c] : 0, 0);
        if (p < 0) {
          singular = true;
          break;
        }
        const double rinv = rinv_s[c];
        const int qp = p >> 5, lp = p & 31;
        if (lane == lp) used |= 1u << qp;
        double ck[RPL];
        bool isp[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int i = lane + 32 * q;
          ck[q] = (i < N) ? ck_s[i] : 0.0;
          isp[q] = i == p;
        }
        gj_apply_step_dyn<CPW, RPL>(w_, ck, rinv, qp, lp, lane, -1);
      }
    }
  }
  __syncthreads();
  if (singular) {
    if (tid == 0) *t.status = 1;
    return;
  }
  if (tid == 0) *t.status = 0;
  for (int k = tid; k < N; k += NT) invp[p_s[k]] = k;
  __syncthreads();
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int r = lane + 32 * q, j = warp * CPW + jj;
      if (r < N && j < N) t.out[invp[r] + (int64_t)p_s[j] * t.out_ld] = w_[jj][q];
    }
}

// Cluster Gauss-Jordan for 160 < N <= 256 (config 4's capacitance matrices,
// r up to 227): the matrix no longer fits one SM's registers, so it is spread
// over a cluster of P = ceil(N / (NW*CPW)) CTAs, still register-resident.
// Global warp g = cta*NW + warp owns columns g*CPW + jj; panel g is that
// warp's column block.  Per panel, exactly as gj_blk_kernel: the owner runs
// its CPW pivot steps warp-synchronously and leaves the pre-step pivot columns,
// pivot rows and reciprocals in its CTA's SMEM (double-buffered by panel
// parity); one cluster barrier; every other warp of every CTA reads them
// through DSMEM and replays the steps on its own columns.  Same pivoting and
// per-element arithmetic as gj_blk_kernel / gj_df_kernel, so the inverse is
// bit-identical to theirs.
template <int NW, int CPW, int RPL>
__global__ void __launch_bounds__(NW * 32, 1) gj_cl_kernel(const GjTask* __restrict__ tasks) {
  constexpr int NT = NW * 32;
  constexpr int NR = 32 * RPL;
  const unsigned P = cl_nrank(), cta = cl_rank();
  const GjTask t = tasks[blockIdx.x / P];
  const int N = __shfl_sync(0xffffffffu, t.N, 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = uniform_warp_id();
  const int gw = (int)cta * NW + warp;   // global warp = panel index it owns
  __shared__ double ckbuf[2][CPW][NR];
  __shared__ double rinvbuf[2][CPW];
  __shared__ int pbuf[2][CPW];
  __shared__ int s_sing, pivrow[NR], invp[NR];
  if (N == 0) {
    if (tid == 0 && cta == 0) *t.status = 0;
    cluster_bar();
    return;
  }
  double w_[CPW][RPL];
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q, j = gw * CPW + jj;
      const bool in = i < N && j < N;
      const int64_t off = t.mode == 0 ? (int64_t)i * t.src_ld + j : i + (int64_t)j * t.src_ld;
      w_[jj][q] = in ? t.src[off] : 0.0;
    }
  unsigned used = 0;                     // bit q: row lane + 32q already a pivot row
  if (tid == 0) s_sing = 0;
  cluster_bar();
  const int npan = (N + CPW - 1) / CPW;
  int singular = 0;
  for (int Pn = 0; Pn < npan; ++Pn) {
    const int buf = Pn & 1;
    const int nl = min(CPW, N - Pn * CPW);
    const unsigned oc = (unsigned)(Pn / NW);     // owner CTA
    if (gw == Pn) {
      int sing = 0;
#pragma unroll
      for (int l = 0; l < CPW; ++l) {
        if (l >= nl) break;
        const int c = Pn * CPW + l;
        double bv = 0.0, bw = 1.0;
        int bi = 0x7fffffff;
        bool have = false;
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int i = lane + 32 * q;
          const double av = fabs(w_[l][q]);
          if (i < N && !((used >> q) & 1u) && (!have || av > bv)) {
            bv = av; bw = w_[l][q]; bi = i; have = true;
          }
        }
        const double myrinv = __drcp_rn(bw);
        const int p = warp_argmax_idx(bv, have, bi);
        const int lp = p & 31, qp = p >> 5;
        const double pivabs = __shfl_sync(0xffffffffu, bv, lp);
        if (t.near && lane == 0 && pivabs < HK_NEAR_PIVOT) *t.near = 1;
        if (!(pivabs >= HK_PIVOT_FLOOR)) { sing = 1; break; }
        const double rinv = __shfl_sync(0xffffffffu, myrinv, lp);
        double ck[RPL];
        bool isp[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int i = lane + 32 * q;
          ck[q] = w_[l][q];
          isp[q] = i == p;
          if (i < N) ckbuf[buf][l][i] = ck[q];
        }
        if (lane == lp) used |= 1u << qp;
        if (lane == 0) {
          rinvbuf[buf][l] = rinv;
          pbuf[buf][l] = p;
          pivrow[c] = p;
        }
        gj_apply_step_dyn<CPW, RPL>(w_, ck, rinv, qp, lp, lane, l);
#pragma unroll
        for (int q = 0; q < RPL; ++q) w_[l][q] = isp[q] ? rinv : -ck[q] * rinv;
      }
      if (sing && lane == 0) s_sing = 1;
    }
    cluster_bar();
    singular = __shfl_sync(0xffffffffu, *cl_map(&s_sing, oc), 0);
    if (singular) break;
    if (gw != Pn) {
      const int* pb = cl_map(&pbuf[buf][0], oc);
      const double* rb = cl_map(&rinvbuf[buf][0], oc);
      const double* cb = cl_map(&ckbuf[buf][0][0], oc);
#pragma unroll 1
      for (int l = 0; l < nl; ++l) {
        const int p = __shfl_sync(0xffffffffu, pb[l], 0);
        const double rinv = rb[l];
        if (cta != oc && tid == 0) pivrow[Pn * CPW + l] = p;
        const int qp = p >> 5, lp = p & 31;
        if (lane == lp) used |= 1u << qp;
        double ck[RPL];
        bool isp[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int i = lane + 32 * q;
          ck[q] = (i < N) ? cb[l * NR + i] : 0.0;
          isp[q] = i == p;
        }
        gj_apply_step_dyn<CPW, RPL>(w_, ck, rinv, qp, lp, lane, -1);
      }
    }
  }
  if (tid == 0 && cta == 0) *t.status = singular;
  // every CTA has read every other CTA's panel buffers and recorded all pivots
  cluster_bar();
  if (singular) return;
  for (int k = tid; k < N; k += NT) invp[pivrow[k]] = k;
  __syncthreads();
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int r = lane + 32 * q, j = gw * CPW + jj;
      if (r < N && j < N) t.out[invp[r] + (int64_t)pivrow[j] * t.out_ld] = w_[jj][q];
    }
}

// Dataflow variant of the cluster Gauss-Jordan (no cluster barrier inside the
// elimination): the warp owning column c runs pivot step c on its registers,
// leaves the pre-step pivot column, pivot row and 1/pivot in its CTA's SMEM
// slot for that step (slots are never reused: each CTA owns NW*CPW steps),
// and publishes it with a cluster-scope release store of its CTA's step
// counter.  Every other warp of every CTA waits for that counter (lane 0
// polls, then every lane acquires), reads the step through DSMEM and replays
// it on its own columns.  The critical path per step is one pivot search plus
// one DSMEM publication instead of a cluster barrier per panel.  Same
// distribution, pivoting and per-element arithmetic as gj_cl_kernel (bit-
// identical inverses).
__device__ __forceinline__ unsigned cl_shared_addr(const void* p, unsigned rank) {
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(ra) : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(rank));
  return ra;
}
__device__ __forceinline__ int ld_acquire_cluster(unsigned addr) {
  int v;
  asm volatile("ld.acquire.cluster.shared::cluster.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_cluster(unsigned addr) {
  int v;
  asm volatile("ld.relaxed.cluster.shared::cluster.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cluster(int* p, int v) {
  asm volatile("st.release.cluster.shared::cta.b32 [%0], %1;"
               ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

template <int NW, int CPW, int RPL>
__global__ void __launch_bounds__(NW * 32, 1) gj_cldf_kernel(const GjTask* __restrict__ tasks) {
  constexpr int NT = NW * 32;
  constexpr int NR = 32 * RPL;
  constexpr int COLS = NW * CPW;                    // steps owned by one CTA
  const unsigned P = cl_nrank(), cta = cl_rank();
  const GjTask t = tasks[blockIdx.x / P];
  const int N = __shfl_sync(0xffffffffu, t.N, 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = uniform_warp_id();
  const int gw = (int)cta * NW + warp;
  extern __shared__ __align__(16) double ckall[];   // [COLS][NR] pre-step pivot columns
  __shared__ double rinv_s[COLS];
  __shared__ int p_s[COLS];
  __shared__ int s_pub;                             // steps of this CTA published
  __shared__ int pivrow[NR], invp[NR];
  double w_[CPW][RPL];
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q, j = gw * CPW + jj;
      const bool in = i < N && j < N;
      const int64_t off = t.mode == 0 ? (int64_t)i * t.src_ld + j : i + (int64_t)j * t.src_ld;
      w_[jj][q] = in ? t.src[off] : 0.0;
    }
  unsigned used = 0;
  if (tid == 0) s_pub = 0;
  cluster_bar();                                    // every counter is 0 before anyone polls
  bool singular = false;
  for (int c = 0; c < N; ++c) {
    const unsigned oc = (unsigned)(c / COLS);
    const int lc = c - (int)oc * COLS;
    const int ow = lc / CPW, l = lc - ow * CPW;
    if (cta == oc && warp == ow) {
      double bv = 0.0, bw = 1.0;
      int bi = 0x7fffffff;
      bool have = false;
      double colv[RPL];
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        double x = w_[0][q];
#pragma unroll
        for (int jj = 1; jj < CPW; ++jj) x = (jj == l) ? w_[jj][q] : x;
        colv[q] = x;
        const int i = lane + 32 * q;
        const double av = fabs(x);
        if (i < N && !((used >> q) & 1u) && (!have || av > bv)) {
          bv = av; bw = x; bi = i; have = true;
        }
      }
      const double myrinv = __drcp_rn(bw);
      const int p = warp_argmax_idx(bv, have, bi);
      const int lp = p & 31, qp = p >> 5;
      const double pivabs = __shfl_sync(0xffffffffu, bv, lp);
      if (t.near && lane == 0 && pivabs < HK_NEAR_PIVOT) *t.near = 1;
      if (!(pivabs >= HK_PIVOT_FLOOR)) {
        if (lane == 0) {
          p_s[lc] = -1;
          st_release_cluster(&s_pub, lc + 1);
        }
        singular = true;
        break;
      }
      const double rinv = __shfl_sync(0xffffffffu, myrinv, lp);
      double* ck_s = ckall + (size_t)lc * NR;
      bool isp[RPL];
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        const int i = lane + 32 * q;
        isp[q] = i == p;
        if (i < N) ck_s[i] = colv[q];
      }
      if (lane == lp) used |= 1u << qp;
      if (lane == 0) {
        rinv_s[lc] = rinv;
        p_s[lc] = p;
        pivrow[c] = p;
      }
      __syncwarp();
      if (lane == 0) st_release_cluster(&s_pub, lc + 1);
#pragma unroll
      for (int jj = 0; jj < CPW; ++jj) {
        if (jj == l) {
#pragma unroll
          for (int q = 0; q < RPL; ++q) w_[jj][q] = isp[q] ? rinv : -colv[q] * rinv;
        } else {
          double src = w_[jj][0];
#pragma unroll
          for (int q = 1; q < RPL; ++q) src = (qp == q) ? w_[jj][q] : src;
          const double rj = __shfl_sync(0xffffffffu, src, lp) * rinv;
#pragma unroll
          for (int q = 0; q < RPL; ++q) {
            const double v = fma(-colv[q], rj, w_[jj][q]);
            w_[jj][q] = isp[q] ? rj : v;
          }
        }
      }
    } else {
      const unsigned fa = cl_shared_addr(&s_pub, oc);
      if (lane == 0)
        while (ld_relaxed_cluster(fa) <= lc) {
        }
      __syncwarp();
      (void)ld_acquire_cluster(fa);               // every lane orders its own reads
      const int p = __shfl_sync(0xffffffffu, lane == 0 ? *cl_map(&p_s[lc], oc) : 0, 0);
      if (p < 0) {
        singular = true;
        break;
      }
      const double rinv = *cl_map(&rinv_s[lc], oc);
      if (cta != oc && warp == 0 && lane == 0) pivrow[c] = p;
      const int qp = p >> 5, lp = p & 31;
      if (lane == lp) used |= 1u << qp;
      const double* ckr = cl_map(ckall + (size_t)lc * NR, oc);
      double ck[RPL];
      bool isp[RPL];
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        const int i = lane + 32 * q;
        ck[q] = (i < N) ? ckr[i] : 0.0;
        isp[q] = i == p;
      }
        gj_apply_step_dyn<CPW, RPL>(w_, ck, rinv, qp, lp, lane, -1);
    }
  }
  const int sing = __any_sync(0xffffffffu, singular) ? 1 : 0;
  __shared__ int s_sing;
  if (tid == 0) s_sing = 0;
  __syncthreads();
  if (sing && lane == 0) atomicOr(&s_sing, 1);
  cluster_bar();                                    // all DSMEM reads done; s_sing complete
  const int any_sing = s_sing;
  if (tid == 0 && cta == 0) *t.status = any_sing;
  if (any_sing) return;
  for (int k = tid; k < N; k += NT) invp[pivrow[k]] = k;
  __syncthreads();
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int r = lane + 32 * q, j = gw * CPW + jj;
      if (r < N && j < N) t.out[invp[r] + (int64_t)pivrow[j] * t.out_ld] = w_[jj][q];
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
      if (t.near && a.v < HK_NEAR_PIVOT) *t.near = 1;
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
          if (t.near && a.v < HK_NEAR_PIVOT) *t.near = 1;
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

template <int NW, int CPW, int RPL>
static cudaError_t launch_gj_reg(const GjTask* tasks_dev, int ntasks, int maxN, cudaStream_t st) {
  if constexpr (CPW * RPL > 32 && NW > 8) {   // 512 threads x 128 registers: the dataflow variant would spill
    gj_blk_kernel<NW, CPW, RPL><<<ntasks, NW * 32, 0, st>>>(tasks_dev);
  } else {
    const size_t smem = (size_t)maxN * 32 * RPL * 8;
    static bool attr = false;   // one attribute call per instantiation
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(gj_df_kernel<NW, CPW, RPL, false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)((size_t)NW * CPW * 32 * RPL * 8));
      if (e != cudaSuccess) return e;
      attr = true;
    }
    CUtensorMap none{};
    gj_df_kernel<NW, CPW, RPL, false><<<ntasks, NW * 32, smem, st>>>(tasks_dev, none, GjLeafMap{});
  }
  hk_count_launch();
  return cudaGetLastError();
}

// 160 < N <= 256: cluster of P = ceil(N / 64) CTAs (8 warps x 8 columns each; 4
// columns per warp measured 20% slower on config 4, 2 columns 2x slower: every
// panel costs a cluster barrier, and it grows with the cluster size)
#ifndef HK_GJ_CL_CPW
#define HK_GJ_CL_CPW 8
#endif
constexpr int kGjClNW = 8, kGjClCPW = HK_GJ_CL_CPW, kGjClRPL = 8, kGjClRows = 32 * kGjClRPL;
static cudaError_t launch_gj_cluster(const GjTask* tasks_dev, int ntasks, int maxN, cudaStream_t st) {
  const int cols = kGjClNW * kGjClCPW;
  const int P = (maxN + cols - 1) / cols;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)P;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)(P * ntasks));
  cfg.blockDim = dim3(kGjClNW * 32);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static int df = -1;
  if (df < 0) {
    // opt-in: measured no faster than the panel version on config 4 (the per-
    // step DSMEM round trips cost what the per-panel barrier did)
    const char* ev = getenv("HK_GJ_CLUSTER_DF");
    df = ev ? atoi(ev) : 0;
  }
  cudaError_t e;
  if (P > 8) {
    e = cudaFuncSetAttribute(gj_cl_kernel<kGjClNW, kGjClCPW, kGjClRPL>,
                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(gj_cldf_kernel<kGjClNW, kGjClCPW, kGjClRPL>,
                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  if (df) {
    auto kern = gj_cldf_kernel<kGjClNW, kGjClCPW, kGjClRPL>;
    const size_t smem = (size_t)kGjClNW * kGjClCPW * 32 * kGjClRPL * 8;
    static bool attr = false;
    if (!attr) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    cfg.dynamicSmemBytes = smem;
    e = cudaLaunchKernelEx(&cfg, kern, tasks_dev);
  } else {
    e = cudaLaunchKernelEx(&cfg, gj_cl_kernel<kGjClNW, kGjClCPW, kGjClRPL>, tasks_dev);
  }
  hk_count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t hk_launch_gj(const GjTask* tasks_dev, int ntasks, int maxN, cudaStream_t st) {
  if (ntasks == 0) return cudaSuccess;
  if (maxN <= 64) return launch_gj_reg<8, 8, 2>(tasks_dev, ntasks, maxN, st);
// HK_GJ128_NW: warps of the N <= 128 dataflow kernel (8 warps x 16 columns measured
// slower: factor 3.5 vs 2.95 ms on config 3)
#ifndef HK_GJ128_NW
#define HK_GJ128_NW 16
#endif
  if (maxN <= 128) return launch_gj_reg<HK_GJ128_NW, 128 / HK_GJ128_NW, 4>(tasks_dev, ntasks, maxN, st);
  if (maxN <= 160) return launch_gj_reg<16, 10, 5>(tasks_dev, ntasks, maxN, st);
  if (maxN <= kGjClRows) return launch_gj_cluster(tasks_dev, ntasks, maxN, st);
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

// Leaf Gauss-Jordan inverses (N <= 64, row-major blocks of the fronts) with
// the blocks staged by the TMA (tensor map built by the caller, hk_gj_leaf_map).
cudaError_t hk_launch_gj_leaf_tma(const GjTask* tasks_dev, int ntasks, const void* tmap,
                                  const double* base, int64_t lda, int64_t fstride,
                                  cudaStream_t st) {
  if (ntasks == 0) return cudaSuccess;
  constexpr size_t smem = (size_t)64 * 64 * 8 + 128;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gj_df_kernel<8, 8, 2, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  gj_df_kernel<8, 8, 2, true><<<ntasks, 256, smem, st>>>(
      tasks_dev, *static_cast<const CUtensorMap*>(tmap), GjLeafMap{base, lda, fstride});
  hk_count_launch();
  return cudaGetLastError();
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda
// at link time): a [batch][n][n] row-major fp64 tensor, box 64 x 64 x 1.
int hk_gj_leaf_map(void* out, const double* base, int64_t n, int64_t lda, int64_t fstride,
                   int64_t batch) {
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                               const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                               const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  if (!fn) return 1;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (lda * 8) % 16 || (fstride * 8) % 16) return 1;
  const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)lda * 8, (cuuint64_t)fstride * 8};
  const cuuint32_t box[3] = {64, 64, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(static_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                        const_cast<double*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 1;
}

size_t hk_gj_scratch_bytes(int N) {
  return (N <= kGjClRows || gj_bytes(N) <= GJ_SMEM_CAP) ? 0 : gj_bytes(N);
}
