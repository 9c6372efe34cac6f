// Dense factorizations on the HODLR path.
//
//  * lu_inv_kernel   -- batched partial-pivot LU + explicit inverse.  Used for
//    every leaf block (src/hodlr.py:222-232 -> dense.py:59-81) and every
//    coupling (Schur) system (src/hodlr.py:269-277).  The inverse turns the
//    leaf Z-solve and the coupling solves into plain GEMMs.
//  * cpiv_kernel     -- complete-pivot LU with numpy's exact pivot order
//    (src/dense.py:133-166): argmax over the row-major flattened, currently
//    permuted trailing block, first occurrence; division then separate
//    multiply/subtract.  Bit-exact with the reference.
//  * skeleton_kernel -- BDLR pseudo-skeleton of one block per CTA
//    (src/lowrank.py:289-331): gather, complete-pivot LU, rank, degenerate
//    check, and the two triangular solves.
#include "hk_common.cuh"
#include "hk_internal.h"

namespace {

constexpr int LU_NT = 512;
constexpr int CP_NT = 1024;
constexpr size_t LU_SMEM_CAP = 200 * 1024;   // in-SMEM working matrix up to N = 160

// ------------------------------------------------------------------ partial pivoting
template <int NT>
__global__ void __launch_bounds__(NT) lu_inv_kernel(const LuTask* __restrict__ tasks,
                                                    size_t smem_bytes) {
  const LuTask t = tasks[blockIdx.x];
  const int N = t.N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(16) unsigned char smraw[];
  const bool in_smem = (size_t)N * N * 8 <= smem_bytes;
  double* W = in_smem ? reinterpret_cast<double*>(smraw) : t.lu;   // column-major ld N
  __shared__ int s_piv;
  __shared__ int s_sing;
  if (tid == 0) s_sing = 0;

  // assemble
  if (t.mode == 0) {
    for (int64_t idx = tid; idx < (int64_t)N * N; idx += NT) {
      int i = (int)(idx / N), j = (int)(idx % N);
      W[i + (int64_t)j * N] = t.src[(int64_t)i * t.src_ld + j];
    }
  } else {
    // S = [[I, S12], [S21, I]]: S12 = H[0:rl, w:w+ru], S21 = H[rl:, w:w+rl]
    // with H column-major (ld = N = rl+ru), h_col0 = w.
    const int rl = t.rl;
    const double* H = t.src;
    const int64_t ldh = t.src_ld;
    for (int64_t idx = tid; idx < (int64_t)N * N; idx += NT) {
      int i = (int)(idx % N), j = (int)(idx / N);
      double v = (i == j) ? 1.0 : 0.0;
      if (i < rl && j >= rl) v = H[i + (t.h_col0 + (j - rl)) * ldh];
      else if (i >= rl && j < rl) v = H[i + (t.h_col0 + j) * ldh];
      W[i + (int64_t)j * N] = v;
    }
  }
  for (int i = tid; i < N; i += NT) t.perm[i] = i;
  __syncthreads();

  for (int k = 0; k < N; ++k) {
    if (warp == 0) {
      ArgMax a{0.0, -1};
      for (int i = k + lane; i < N; i += 32) {
        double v = fabs(W[i + (int64_t)k * N]);
        if (argmax_better(v, i, a.v, a.i)) { a.v = v; a.i = i; }
      }
      a = warp_argmax(a);
      if (lane == 0) s_piv = (int)a.i;
    }
    __syncthreads();
    const int p = s_piv;
    if (p != k) {
      for (int j = tid; j < N; j += NT) {
        double a = W[k + (int64_t)j * N];
        W[k + (int64_t)j * N] = W[p + (int64_t)j * N];
        W[p + (int64_t)j * N] = a;
      }
      if (tid == 0) {
        int a = t.perm[k];
        t.perm[k] = t.perm[p];
        t.perm[p] = a;
      }
    }
    if (tid == 0) t.ipiv[k] = p;
    __syncthreads();
    const double piv = W[k + (int64_t)k * N];
    if (fabs(piv) < HK_PIVOT_FLOOR) {
      if (tid == 0) s_sing = 1;
    }
    if (piv != 0.0) {
      for (int i = k + 1 + tid; i < N; i += NT) W[i + (int64_t)k * N] = W[i + (int64_t)k * N] / piv;
    }
    __syncthreads();
    const int rem = N - k - 1;
    if (rem > 0) {
      const int64_t tot = (int64_t)rem * rem;
      for (int64_t idx = tid; idx < tot; idx += NT) {
        int i = k + 1 + (int)(idx % rem), j = k + 1 + (int)(idx / rem);
        W[i + (int64_t)j * N] -= W[i + (int64_t)k * N] * W[k + (int64_t)j * N];
      }
    }
    __syncthreads();
  }
  if (in_smem) {
    for (int64_t idx = tid; idx < (int64_t)N * N; idx += NT) t.lu[idx] = W[idx];
  }
  if (tid == 0) *t.status = s_sing;
  __syncthreads();
  if (s_sing || t.inv == nullptr) return;

  // explicit inverse: thread per column c of A^{-1}, first stored row-major
  // as inv[i*N + c] (coalesced over c), then transposed in place to column
  // major.  A^{-1} e_c = U^{-1} L^{-1} P e_c.
  for (int c = tid; c < N; c += NT) {
    int kc = 0;
    for (int k = 0; k < N; ++k)
      if (t.perm[k] == c) kc = k;
    double* X = t.inv;
    for (int i = 0; i < kc; ++i) X[(int64_t)i * N + c] = 0.0;
    X[(int64_t)kc * N + c] = 1.0;
    for (int i = kc + 1; i < N; ++i) {          // unit lower forward
      double s = 0.0;
      for (int l = kc; l < i; ++l) s += W[i + (int64_t)l * N] * X[(int64_t)l * N + c];
      X[(int64_t)i * N + c] = -s;
    }
    for (int i = N - 1; i >= 0; --i) {          // upper backward
      double s = X[(int64_t)i * N + c];
      for (int l = i + 1; l < N; ++l) s -= W[i + (int64_t)l * N] * X[(int64_t)l * N + c];
      X[(int64_t)i * N + c] = s / W[i + (int64_t)i * N];
    }
  }
  __syncthreads();
  for (int64_t idx = tid; idx < (int64_t)N * N; idx += NT) {
    const int i = (int)(idx / N), j = (int)(idx % N);
    if (i < j) {
      double a = t.inv[(int64_t)i * N + j];
      t.inv[(int64_t)i * N + j] = t.inv[(int64_t)j * N + i];
      t.inv[(int64_t)j * N + i] = a;
    }
  }
}

// ------------------------------------------------------------------ complete pivoting
// Works on a row-major k x kc matrix W (ld = ldw, SMEM or global).  Returns
// the number of pivots taken; perms and |pivots| written to rp, cp, piv.
//
// Warp w owns rows s+1+w, s+1+w+NW, ...; lanes stride the columns (coalesced,
// no index divisions).  The argmax of step s+1 is fused into the rank-1 update
// of step s: the updated trailing entries are exactly the next step's search
// set, and the flattened index (i-s-1)*(kc-s-1) + (j-s-1) keeps numpy's
// row-major first-occurrence tie-break.  The multiplier of row i is computed
// once (lane 0, IEEE division) and broadcast, so every entry is
// w[i][j] - (l_i * w[s][j]) with a separate multiply and subtract, exactly as
// dense.py:147-165 / the oracle (bit-identical packed LU and pivots).
// Block argmax of |x| >= 0 with the lowest flattened index on ties, valid in
// every thread after ONE barrier: REDUX-based warp stage (warp_argmax_idx),
// the NW warp winners through SMEM, reduced again by every warp.  The caller
// must pass another barrier before the next call reuses sv/si.
template <int NT>
__device__ __forceinline__ ArgMax block_argmax1(ArgMax a, double* sv, int64_t* si) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool ok = a.i >= 0;
  const int wi = warp_argmax_idx(a.v, ok, ok ? (int)a.i : 0);
  const unsigned m = __ballot_sync(0xffffffffu, ok && (int)a.i == wi);
  const double wv = __shfl_sync(0xffffffffu, a.v, m ? __ffs(m) - 1 : 0);
  if (lane == 0) { sv[warp] = wv; si[warp] = m ? wi : -1; }
  __syncthreads();
  const bool ok2 = lane < NW && si[lane < NW ? lane : 0] >= 0;
  const double cv = lane < NW ? sv[lane] : 0.0;
  const int ci = lane < NW ? (int)si[lane] : 0;
  const int bi = warp_argmax_idx(cv, ok2, ci);
  const unsigned m2 = __ballot_sync(0xffffffffu, ok2 && ci == bi);
  const double bv = __shfl_sync(0xffffffffu, cv, m2 ? __ffs(m2) - 1 : 0);
  return ArgMax{bv, m2 ? (int64_t)bi : (int64_t)-1};
}

template <int NT>
__device__ int complete_pivot_lu(double* Wsm, double* Wg, int ksm, int k, int kc, int64_t ldw,
                                 int64_t* rp, int64_t* cp, double* piv, double* red_v,
                                 int64_t* red_i) {
  constexpr int NW = NT / 32;
  // rows [0, ksm) live in SMEM, the rest in global memory (same row stride)
  auto R = [&](int i) -> double* { return (i < ksm ? Wsm : Wg) + (int64_t)i * ldw; };
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < k; i += NT) rp[i] = i;
  for (int j = tid; j < kc; j += NT) cp[j] = j;
  ArgMax a{0.0, -1};
  for (int i = warp; i < k; i += NW)
    for (int j = lane; j < kc; j += 32) {
      const double v = fabs(R(i)[j]);
      const int64_t idx = (int64_t)i * kc + j;
      if (argmax_better(v, idx, a.v, a.i)) { a.v = v; a.i = idx; }
    }
  a = block_argmax1<NT>(a, red_v, red_i);
  const int steps = k < kc ? k : kc;
  int taken = 0;
  for (int s = 0; s < steps; ++s) {
    if (a.i < 0 || !(a.v != 0.0)) break;
    const int cc = kc - s;
    const int pr = s + (int)(a.i / cc), pc = s + (int)(a.i % cc);
    if (pr != s) {
      double* rs_ = R(s);
      double* rr_ = R(pr);
      for (int j = tid; j < kc; j += NT) {
        const double x = rs_[j];
        rs_[j] = rr_[j];
        rr_[j] = x;
      }
      if (tid == 0) {
        const int64_t x = rp[s]; rp[s] = rp[pr]; rp[pr] = x;
      }
      __syncthreads();   // the column swap below reads the swapped rows
    }
    if (pc != s) {
      for (int i = tid; i < k; i += NT) {
        double* ri = R(i);
        const double x = ri[s];
        ri[s] = ri[pc];
        ri[pc] = x;
      }
      if (tid == 0) {
        const int64_t x = cp[s]; cp[s] = cp[pc]; cp[pc] = x;
      }
    }
    __syncthreads();
    const double* ps = R(s);
    const double p = ps[s];
    if (tid == 0) piv[s] = fabs(p);
    ++taken;
    a = ArgMax{0.0, -1};
    if (s + 1 < k) {
      const int c2 = kc - s - 1;
      for (int i = s + 1 + warp; i < k; i += NW) {
        double* ri = R(i);
        double l = 0.0;
        if (lane == 0) {
          l = div_rn(ri[s], p);
          ri[s] = l;
        }
        l = __shfl_sync(0xffffffffu, l, 0);
        const int64_t rbase = (int64_t)(i - s - 1) * c2;
        for (int j = s + 1 + lane; j < kc; j += 32) {
          const double v = sub_rn(ri[j], mul_rn(l, ps[j]));
          ri[j] = v;
          const int64_t idx = rbase + (j - s - 1);
          if (argmax_better(fabs(v), idx, a.v, a.i)) { a.v = fabs(v); a.i = idx; }
        }
      }
    }
    // its barrier also orders this step's updates before the next swaps; the
    // next write of sv/si comes after the next step's swap barrier
    a = block_argmax1<NT>(a, red_v, red_i);
  }
  return taken;
}

template <int NT>
__global__ void __launch_bounds__(NT) cpiv_kernel(double* W, int k, int kc, int64_t ldw,
                                                  int64_t* rp, int64_t* cp, double* piv,
                                                  int64_t* npiv) {
  __shared__ double red_v[NT / 32];
  __shared__ int64_t red_i[NT / 32];
  int taken = complete_pivot_lu<NT>(W, W, 0, k, kc, ldw, rp, cp, piv, red_v, red_i);
  if (threadIdx.x == 0) *npiv = taken;
}

// ------------------------------------------------------------------ BDLR skeleton
template <int NT>
__global__ void __launch_bounds__(NT) skeleton_kernel(const SkelTask* __restrict__ tasks,
                                                      double* pivbuf, int64_t pivstride,
                                                      size_t smem_bytes) {
  const SkelTask t = tasks[blockIdx.x];
  const int tid = threadIdx.x;
  __shared__ double red_v[NT / 32];
  __shared__ int64_t red_i[NT / 32];
  __shared__ int s_rank;
  extern __shared__ double wsm[];
  double* piv = pivbuf + (int64_t)blockIdx.x * pivstride;
  const int k = t.k, kc = t.kc, n = t.n;
  // working matrix: its first ksm rows in SMEM (all of it when it fits), the
  // rest in t.work; SMEM rows are written back to t.work after the LU
  const int ksm = kc > 0 ? (int)min((size_t)k, smem_bytes / ((size_t)kc * 8)) : k;
  auto R = [&](int i) -> double* { return (i < ksm ? wsm : t.work) + (int64_t)i * kc; };
  // gather A-hat = A[rsel, csel] (row-major k x kc), warp per row
  double amax = 0.0;   // max|A-hat| for the degenerate check, before the LU overwrites it
  for (int a = tid >> 5; a < k; a += NT / 32) {
    const double* arow = t.A + t.rsel[a] * t.lda;
    double* w = R(a);
    for (int b = tid & 31; b < kc; b += 32) {
      const double v = arow[t.csel[b]];
      w[b] = v;
      amax = fmax(amax, fabs(v));
    }
  }
  __syncthreads();
  {
    ArgMax a{amax, 0};
    a = block_argmax<NT>(a, red_v, red_i);
    amax = a.v;
  }
  const int taken = complete_pivot_lu<NT>(wsm, t.work, ksm, k, kc, kc, t.rperm, t.cperm, piv,
                                          red_v, red_i);
  for (int64_t idx = tid; idx < (int64_t)ksm * kc; idx += NT) t.work[idx] = wsm[idx];
  if (tid == 0) {
    int r = 0;
    if (taken > 0) {
      const double lim = t.tol * piv[0];
      for (int s = 0; s < taken; ++s) r += (piv[s] >= lim) ? 1 : 0;
    }
    if (r > t.cap) r = t.cap;
    s_rank = r;
  }
  __syncthreads();
  const int r = s_rank;
  if (tid == 0) { *t.rank = r; *t.status = 0; }
  if (r == 0) {
    // _check_degenerate, lowrank.py:322-331
    double smax = 0.0;
    for (int64_t idx = tid; idx < (int64_t)t.nprobe * n; idx += NT) {
      int p = (int)(idx / n), c = (int)(idx % n);
      smax = fmax(smax, fabs(t.A[t.probe[p] * t.lda + c]));
    }
    ArgMax a{smax, 0};
    a = block_argmax<NT>(a, red_v, red_i);
    if (tid == 0 && a.v > t.tol * amax) *t.status = HK_STATUS_DEGENERATE;
    return;
  }
}

// C~ = C U11^{-1} (thread per row of the block) and R~ = L11^{-1} R[rperm[:r]]
// (thread per column), V = R~^T -- one CTA per (task, 64-row or 64-column
// chunk), so the triangular solves of a block spread over many SMs and each
// CTA's rows of U stay in its L1 (the single-CTA version ran them on the SM
// that did the LU, whose L1 was mostly carved out as SMEM).  Same per-entry
// arithmetic and order as before (lowrank.py:315-318).
template <int NT>
__global__ void __launch_bounds__(NT) skeleton_trsm_kernel(const SkelTask* __restrict__ tasks) {
  const SkelTask t = tasks[blockIdx.x];
  const int r = *t.rank;
  if (r == 0) return;
  const int kc = t.kc;
  const double* W = t.work;   // packed LU, row-major ld kc
  const int nrc = (t.m + NT - 1) / NT;
  int chunk = blockIdx.y;
  if (chunk < nrc) {
    const int i = chunk * NT + threadIdx.x;
    if (i >= t.m) return;
    double* x = t.U + i;                      // row i of U (column-major, ld ldu)
    for (int l = 0; l < r; ++l) {
      double s = t.A[(int64_t)i * t.lda + t.csel[t.cperm[l]]];
      for (int p = 0; p < l; ++p) s -= x[(int64_t)p * t.ldu] * W[(int64_t)p * kc + l];
      x[(int64_t)l * t.ldu] = s / W[(int64_t)l * kc + l];
    }
    return;
  }
  chunk -= nrc;
  const int c = chunk * NT + threadIdx.x;
  if (c >= t.n) return;
  double* z = t.V + c;                        // row c of V (column-major, ld ldv)
  for (int a = 0; a < r; ++a) {
    double s = t.A[t.rsel[t.rperm[a]] * t.lda + c];
    for (int p = 0; p < a; ++p) s -= W[(int64_t)a * kc + p] * z[(int64_t)p * t.ldv];
    z[(int64_t)a * t.ldv] = s;
  }
}

}  // namespace

cudaError_t hk_launch_lu(const LuTask* tasks_dev, int ntasks, int maxN, cudaStream_t st) {
  if (ntasks == 0) return cudaSuccess;
  size_t need = (size_t)maxN * maxN * 8;
  size_t smem = need <= LU_SMEM_CAP ? need : 0;
  cudaError_t e = cudaFuncSetAttribute(lu_inv_kernel<LU_NT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)LU_SMEM_CAP);
  if (e != cudaSuccess) return e;
  // every task decides in_smem from its own N; give all tasks the max buffer
  lu_inv_kernel<LU_NT><<<ntasks, LU_NT, smem ? smem : 16, st>>>(tasks_dev, smem);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_lu_full(double* a, int64_t m, int64_t n, int64_t ld, int64_t* rp,
                              int64_t* cp, double* piv, int64_t* npiv_dev, cudaStream_t st) {
  cpiv_kernel<CP_NT><<<1, CP_NT, 0, st>>>(a, (int)m, (int)n, ld, rp, cp, piv, npiv_dev);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_skeleton(const SkelTask* tasks_dev, int ntasks, int max_k, int max_kc,
                               int max_m, int max_n, cudaStream_t st) {
  if (ntasks == 0) return cudaSuccess;
  double* pivbuf = nullptr;
  int64_t pstride = (max_k < max_kc ? max_k : max_kc) + 1;
  cudaError_t e = hk_dev_malloc(&pivbuf, (size_t)ntasks * pstride * 8, st);
  if (e != cudaSuccess) return e;
  // every task whose working matrix fits takes the SMEM path (1024-thread
  // CTAs run one per SM anyway); larger ones work in global memory
  const size_t need = (size_t)max_k * max_kc * 8;
  const size_t smem = need <= LU_SMEM_CAP ? need : LU_SMEM_CAP;
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(skeleton_kernel<CP_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return e;
  }
  skeleton_kernel<CP_NT><<<ntasks, CP_NT, smem, st>>>(tasks_dev, pivbuf, pstride, smem);
  hk_count_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  constexpr int TR_NT = 64;
  const int chunks = (max_m + TR_NT - 1) / TR_NT + (max_n + TR_NT - 1) / TR_NT;
  if (chunks > 0) {
    skeleton_trsm_kernel<TR_NT><<<dim3((unsigned)ntasks, (unsigned)chunks), TR_NT, 0, st>>>(tasks_dev);
    hk_count_launch();
    e = cudaGetLastError();
  }
  hk_dev_free(pivbuf, st);
  return e;
}
