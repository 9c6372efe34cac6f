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

// Measured alternatives (config 3 factor, 64 fronts): 3 stages / 3 CTAs per SM
// and 2 stages / 4 CTAs per SM spill at the implied register caps (3.9-4.1 ms
// vs 3.46 ms); a persistent CTA walking its tiles through one cp.async ring
// was ~20% slower than one tile per CTA with two CTAs per SM.
#ifndef HK_GEMM_BK
#define HK_GEMM_BK 16
#endif
#ifndef HK_GEMM_STAGES
#define HK_GEMM_STAGES 4
#endif
constexpr int BM = 64, BN = 64, BK = HK_GEMM_BK, NT = 256, STAGES = HK_GEMM_STAGES;
constexpr int QV = BM * BK / 2 / NT;   // 16-byte pair copies per thread per operand and stage
constexpr int QS = BM * BK / NT;       // 8-byte copies per thread per operand and stage
constexpr int SA = BM + 4;   // k-major A rows (transA = 0): conflict-free DMMA fragment loads
constexpr int ST = BK + 4;   // m/n-major rows (transA = 1 and B)

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// One 64x64 tile of C = alpha op(A) B + beta C (+ diag on C's diagonal).
// 8 warps (2 along m x 4 along n), each owning a 32x16 sub-tile of 4x2 DMMA
// 8x8 accumulators.  Four-stage cp.async pipeline (global -> SMEM without
// register staging) so the L2 latency of the next k-tiles overlaps the DMMA
// work of the current one; for beta != 0 the C values are fetched into
// registers before the k loop so the epilogue does not wait on memory.
template <int TRANSA, int VEC>
__device__ __forceinline__ void gemm_tile(const GemmTask& t, int tm, int tn, double* smem) {
  constexpr int A_STAGE = TRANSA ? BM * ST : BK * SA;
  constexpr int B_STAGE = BN * ST;
  double* As = smem;
  double* Bs = smem + STAGES * A_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;       // 2 x 4 warps
  const int m0 = tm * BM, n0 = tn * BN;
  const int M = t.m, N = t.n, K = t.k;
  const double* __restrict__ Ag = t.A;
  const double* __restrict__ Bg = t.B;

  // C prefetch (beta != 0): the 16 values this thread will update
#ifndef HK_GEMM_CPRE
#define HK_GEMM_CPRE 1   // 0: read C in the epilogue (32 fewer registers: 3 CTAs per SM fit)
#endif
#ifndef HK_GEMM_MINB
#define HK_GEMM_MINB 2
#endif
  double cpre[HK_GEMM_CPRE ? 4 : 1][2][2];
  if (HK_GEMM_CPRE && t.beta != 0.0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = m0 + wm * 32 + i * 8 + gid;
          const int col = n0 + wn * 16 + j * 8 + 2 * tig + h;
          cpre[i][j][h] = (row < M && col < N) ? t.C[row + (int64_t)col * t.ldc] : 0.0;
        }
  }

  auto load_stage = [&](int kt, int stage) {
    const int k0 = kt * BK;
    double* as = As + stage * A_STAGE;
    double* bs = Bs + stage * B_STAGE;
    if constexpr (VEC != 0) {
      // 16-byte copies of element pairs along the contiguous dimension (pairs
      // start at even offsets, so a pair straddling the edge copies 8 bytes
      // and zero-fills the rest); half the cp.async instructions
#pragma unroll
      for (int q = 0; q < QV; ++q) {
        const int idx = tid + NT * q;
        if (!TRANSA) {
          const int i = 2 * (idx % (BM / 2)), l = idx / (BM / 2);
          const int rem = M - (m0 + i);
          const int nb = (k0 + l < K) ? (rem >= 2 ? 16 : rem == 1 ? 8 : 0) : 0;
          const double* src = nb ? Ag + (m0 + i) + (int64_t)(k0 + l) * t.lda : Ag;
          cp_async16(as + l * SA + i, src, nb);
        } else {
          const int l = 2 * (idx % (BK / 2)), i = idx / (BK / 2);
          const int rem = K - (k0 + l);
          const int nb = (m0 + i < M) ? (rem >= 2 ? 16 : rem == 1 ? 8 : 0) : 0;
          const double* src = nb ? Ag + (k0 + l) + (int64_t)(m0 + i) * t.lda : Ag;
          cp_async16(as + i * ST + l, src, nb);
        }
        const int l = 2 * (idx % (BK / 2)), j = idx / (BK / 2);
        const int remb = K - (k0 + l);
        const int nbb = (n0 + j < N) ? (remb >= 2 ? 16 : remb == 1 ? 8 : 0) : 0;
        const double* srcb = nbb ? Bg + (k0 + l) + (int64_t)(n0 + j) * t.ldb : Bg;
        cp_async16(bs + j * ST + l, srcb, nbb);
      }
    } else {
#pragma unroll
    for (int q = 0; q < QS; ++q) {
      const int idx = tid + NT * q;
      if (!TRANSA) {
        const int i = idx % BM, l = idx / BM;
        const bool ok = (m0 + i < M) && (k0 + l < K);
        const double* src = ok ? Ag + (m0 + i) + (int64_t)(k0 + l) * t.lda : Ag;
        cp_async8(as + l * SA + i, src, ok ? 8 : 0);
      } else {
        const int l = idx % BK, i = idx / BK;
        const bool ok = (m0 + i < M) && (k0 + l < K);
        const double* src = ok ? Ag + (k0 + l) + (int64_t)(m0 + i) * t.lda : Ag;
        cp_async8(as + i * ST + l, src, ok ? 8 : 0);
      }
      const int l = idx % BK, j = idx / BK;
      const bool okb = (n0 + j < N) && (k0 + l < K);
      const double* srcb = okb ? Bg + (k0 + l) + (int64_t)(n0 + j) * t.ldb : Bg;
      cp_async8(bs + j * ST + l, srcb, okb ? 8 : 0);
    }
    }
  };

  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int stage = kt % STAGES;
    const double* as = As + stage * A_STAGE;
    const double* bs = Bs + stage * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = wm * 32 + i * 8 + gid;
        a[i] = TRANSA ? as[r * ST + kk + tig] : as[(kk + tig) * SA + r];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = bs[(wn * 16 + j * 8 + gid) * ST + kk + tig];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    const int nxt = kt + STAGES - 1;
    if (nxt < nk) load_stage(nxt, nxt % STAGES);
    cp_async_commit();
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + gid;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * 16 + j * 8 + 2 * tig + h;
        if (col >= N) continue;
        double v = t.alpha * acc[i][j][h];
        if (t.beta != 0.0)
          v += t.beta * (HK_GEMM_CPRE ? cpre[HK_GEMM_CPRE ? i : 0][j][h] : t.C[row + (int64_t)col * t.ldc]);
        if (row == col) v += t.diag;
        t.C[row + (int64_t)col * t.ldc] = v;
      }
    }
  }
}

constexpr size_t GEMM_SMEM = (size_t)STAGES * (BM * ST + BN * ST) * 8;   // >= transA=0 layout

__global__ void __launch_bounds__(NT, HK_GEMM_MINB) gemm_kernel(const GemmTask* __restrict__ tasks,
                                                     const int32_t* __restrict__ tilemap) {
  extern __shared__ __align__(16) double gsmem[];
  const int task = tilemap[3 * blockIdx.x];
  const int tm = tilemap[3 * blockIdx.x + 1];
  const int tn = tilemap[3 * blockIdx.x + 2];
  const GemmTask t = tasks[task];
  if (t.vec) {
    if (t.transA) gemm_tile<1, 1>(t, tm, tn, gsmem);
    else gemm_tile<0, 1>(t, tm, tn, gsmem);
  } else {
    if (t.transA) gemm_tile<1, 0>(t, tm, tn, gsmem);
    else gemm_tile<0, 0>(t, tm, tn, gsmem);
  }
}

// dst(i, j) = src(i, j).  Column-major destinations (the Z gather of the
// factorization) walk columns across CTAs and rows across threads, so both
// sides are coalesced when the source is column-major too; otherwise rows
// across CTAs and columns across threads.  No per-element index division.
__global__ void __launch_bounds__(256) copy_kernel(const CopyTask* __restrict__ tasks) {
  const CopyTask t = tasks[blockIdx.y];
  if (t.dst_rs == 1 && t.src_rs == 1) {
    // both column-major (the Z gather): the 256 threads tile rt rows x ct columns
    // (rt = the power of two covering the rows, 32..256) and keep U columns in
    // flight per thread.  One column per CTA pass with 64-row blocks left 3/4 of
    // the threads idle and one load in flight each: 209 us for 387 MB on config 3.
    constexpr int U = 4;
    int rt = 32;
    while (rt < t.rows && rt < 256) rt <<= 1;
    const int ct = 256 / rt;
    const int tx = threadIdx.x & (rt - 1), ty = threadIdx.x / rt;
    const int jstep = gridDim.x * ct;
    for (int j0 = blockIdx.x * ct + ty; j0 < t.cols; j0 += U * jstep) {
      for (int i = tx; i < t.rows; i += rt) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + u * jstep;
          v[u] = j < t.cols ? t.src[i + (int64_t)j * t.src_cs] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + u * jstep;
          if (j < t.cols) t.dst[i + (int64_t)j * t.dst_cs] = v[u];
        }
      }
    }
  } else if (t.dst_rs == 1) {
    for (int j = blockIdx.x; j < t.cols; j += gridDim.x) {
      const double* s = t.src + (int64_t)j * t.src_cs;
      double* d = t.dst + (int64_t)j * t.dst_cs;
      for (int i = threadIdx.x; i < t.rows; i += blockDim.x) d[i] = s[(int64_t)i * t.src_rs];
    }
  } else {
    for (int i = blockIdx.x; i < t.rows; i += gridDim.x) {
      const double* s = t.src + (int64_t)i * t.src_rs;
      double* d = t.dst + (int64_t)i * t.dst_rs;
      for (int j = threadIdx.x; j < t.cols; j += blockDim.x) d[(int64_t)j * t.dst_cs] = s[(int64_t)j * t.src_cs];
    }
  }
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}


// Host -> device staging copy run by a few SMs: 16-byte loads straight from
// pinned (UVA-mapped) host memory, evict-first (.cs) stores into HBM, so the
// streamed fronts of the next batch do not flush the L2 working set of the
// batch being compressed (a copy-engine DMA write-allocates in L2 and slowed
// the concurrent ACA build ~3x).
__global__ void __launch_bounds__(256) h2d_stream_kernel(const double2* __restrict__ src,
                                                         double2* __restrict__ dst, int64_t n2) {
  constexpr int U = 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(dst + i + u * stride, v[u]);
  }
  for (; i < n2; i += stride) __stcs(dst + i, __ldcs(src + i));
}
}  // namespace

cudaError_t hk_launch_gemm(const GemmTask* tasks_dev, const int32_t* tilemap_dev, int ntiles,
                           cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;

  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)GEMM_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  gemm_kernel<<<ntiles, NT, GEMM_SMEM, st>>>(tasks_dev, tilemap_dev);
  hk_count_launch();
  return cudaGetLastError();
}

cudaError_t hk_launch_copy(const CopyTask* tasks_dev, int ntasks, cudaStream_t st) {
  if (ntasks == 0) return cudaSuccess;
  copy_kernel<<<dim3(8, ntasks), 256, 0, st>>>(tasks_dev);
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

cudaError_t hk_launch_h2d_stream(const void* src_host, void* dst_dev, int64_t bytes, int ctas,
                                 cudaStream_t st) {
  if (bytes <= 0) return cudaSuccess;
  const int64_t n2 = bytes / 16;
  if (n2 > 0)
    h2d_stream_kernel<<<ctas, 256, 0, st>>>((const double2*)src_host, (double2*)dst_dev, n2);
  const int64_t tail = bytes - n2 * 16;
  if (tail) {
    cudaError_t e = cudaMemcpyAsync((char*)dst_dev + n2 * 16, (const char*)src_host + n2 * 16, tail,
                                    cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
  }
  hk_count_launch();
  return cudaGetLastError();
}
