// Shared device helpers for the HODLR B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define HK_PIVOT_FLOOR 1e-300   // src/dense.py:19 PIVOT_UNDERFLOW
#define HK_STATUS_DEGENERATE 6  // == HK_ERR_DEGENERATE in include/hodlr_b200.h

// Exact IEEE operations that numpy performs elementwise.  Using the _rn
// intrinsics keeps nvcc from contracting a*b - c into an FMA, which would
// change the last bit and with it the pivot decisions.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// (value, index) argmax with numpy's tie-break: larger value wins, equal
// values -> smaller index wins.  Values are magnitudes (>= 0); index -1 = none.
struct ArgMax {
  double v;
  int64_t i;
};

__device__ __forceinline__ bool argmax_better(double va, int64_t ia, double vb, int64_t ib) {
  // is (va, ia) better than (vb, ib)?
  if (ia < 0) return false;
  if (ib < 0) return true;
  if (va > vb) return true;
  if (va < vb) return false;
  return ia < ib;
}

__device__ __forceinline__ ArgMax warp_argmax(ArgMax a) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double ov = __shfl_down_sync(0xffffffffu, a.v, off);
    long long oi = __shfl_down_sync(0xffffffffu, (long long)a.i, off);
    if (argmax_better(ov, oi, a.v, a.i)) { a.v = ov; a.i = oi; }
  }
  return a;
}

// Warp index that ptxas can prove warp-uniform (a shuffle from a constant
// lane), so shuffles inside `if (warp == w)` branches compile without the
// divergent-warp collective fallback (measured: 413 -> 322 cycles for a
// 5-round reduction).
__device__ __forceinline__ int uniform_warp_id() {
  return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
}

// Same, result valid in every lane (butterfly; the (value, lowest index) order
// is total, so the result does not depend on the combination order).
__device__ __forceinline__ ArgMax warp_argmax_all(ArgMax a) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, a.v, off);
    long long oi = __shfl_xor_sync(0xffffffffu, (long long)a.i, off);
    if (argmax_better(ov, oi, a.v, a.i)) { a.v = ov; a.i = oi; }
  }
  return a;
}

// Warp argmax of non-negative doubles with lowest-index tie break, in every
// lane, by three 32-bit REDUX reductions instead of five shuffle rounds:
// for v >= 0 the IEEE bit pattern is monotonic, so (v, idx) compares as the
// 64-bit key bits(v)+1 (0 = no candidate) and then the smallest idx.
// Returns the winning index (or -1 if no lane had a candidate) in every lane.
__device__ __forceinline__ int warp_argmax_idx(double v, bool valid, int idx) {
  const unsigned long long key = valid ? (unsigned long long)__double_as_longlong(v) + 1ull : 0ull;
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const bool win = hi == mhi && lo == mlo && key != 0ull;
  return (int)__reduce_min_sync(0xffffffffu, win ? (unsigned)idx : 0xffffffffu);
}

// Block-wide argmax; result valid in all threads.  scratch needs 2*nwarps slots.
// TAIL_SYNC=false drops the trailing barrier when the caller separates the
// next use of the scratch by another barrier anyway.
template <int NT, bool TAIL_SYNC = true>
__device__ __forceinline__ ArgMax block_argmax(ArgMax a, double* sv, int64_t* si) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_argmax(a);
  if (lane == 0) { sv[warp] = a.v; si[warp] = a.i; }
  __syncthreads();
  if (warp == 0) {
    ArgMax b;
    if (lane < NT / 32) { b.v = sv[lane]; b.i = si[lane]; } else { b.v = 0.0; b.i = -1; }
    b = warp_argmax(b);
    if (lane == 0) { sv[0] = b.v; si[0] = b.i; }
  }
  __syncthreads();
  ArgMax r{sv[0], si[0]};
  if (TAIL_SYNC) __syncthreads();
  return r;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
  return x;
}

// Block sum of two values; result valid in all threads. scratch: 2*nwarps.
template <int NT>
__device__ __forceinline__ void block_sum2(double& a, double& b, double* s) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) { s[2 * warp] = a; s[2 * warp + 1] = b; }
  __syncthreads();
  if (warp == 0) {
    double x = lane < NT / 32 ? s[2 * lane] : 0.0;
    double y = lane < NT / 32 ? s[2 * lane + 1] : 0.0;
    x = warp_sum(x);
    y = warp_sum(y);
    if (lane == 0) { s[0] = x; s[1] = y; }
  }
  __syncthreads();
  a = s[0];
  b = s[1];
  __syncthreads();
}

template <int NT>
__device__ __forceinline__ double block_sum(double a, double* s) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  if (lane == 0) s[warp] = a;
  __syncthreads();
  if (warp == 0) {
    double x = lane < NT / 32 ? s[lane] : 0.0;
    x = warp_sum(x);
    if (lane == 0) s[0] = x;
  }
  __syncthreads();
  double r = s[0];
  __syncthreads();
  return r;
}

// ---- thread-block clusters: barrier, rank, distributed-shared-memory mapping
__device__ __forceinline__ void cluster_bar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_nrank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
// generic address of the same shared variable in CTA `rank` of the cluster
template <class T>
__device__ __forceinline__ const T* cl_map(const T* p, unsigned rank) {
  uint64_t out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(p), "r"(rank));
  return reinterpret_cast<const T*>(out);
}

// ---- programmatic dependent launch: a kernel launched with the
// programmatic-stream-serialization attribute may start while its predecessor
// drains; it must call griddep_wait() before reading anything the predecessor
// writes (independent loads -- stored factors -- go out before the wait).
// Both are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- mbarriers (completion of the TMA tensor loads, gj.cu)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// arm the barrier's current phase with `bytes` of expected transactions (+1 arrival)
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// FP64 tensor-core MMA (DMMA.8x8x4 on sm_100a; tcgen05 has no f64 kind).
// Fragment layout (PTX ISA, mma.m8n8k4 .f64): gid = lane>>2, tig = lane&3;
//   A (8x4, row):  a  = A[gid][tig]
//   B (4x8, col):  b  = B[tig][gid]
//   C (8x8):       c0 = C[gid][2*tig], c1 = C[gid][2*tig+1]
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
