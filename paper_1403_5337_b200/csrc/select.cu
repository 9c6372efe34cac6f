// BDLR skeleton selection on the GPU (src/graph.py:171-228):
// for one side of an off-diagonal block -- the own vertex range [own0,
// own0+n_own) against the other range [oth0, oth0+n_oth) -- the boundary is
// the own vertices with a neighbour on the other side (distance 0), distances
// grow by level-synchronous BFS inside the own range up to `depth`, and the
// selection is every position with d <= depth ordered by (d, vertex id).
// HODLR blocks are contiguous index ranges in front order, so membership is a
// range test.  BFS distances do not depend on visiting order, and the output
// order is fixed, so the selection is bit-identical to the host's
// (graph.cpp) and the reference's.
#include "hk_common.cuh"
#include "hk_internal.h"

namespace {

constexpr int SEL_NT = 512;

// block-wide exclusive prefix sum of one int per thread; *total gets the sum
__device__ __forceinline__ int block_exscan(int v, int* warp_tot, int* total) {
  constexpr int NW = SEL_NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < NW ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NW) warp_tot[lane] = w;            // inclusive warp totals
    if (lane == NW - 1) *total = w;
  }
  __syncthreads();
  const int before = warp > 0 ? warp_tot[warp - 1] : 0;
  const int r = before + x - v;
  __syncthreads();                                 // warp_tot reused by the next call
  return r;
}

__global__ void __launch_bounds__(SEL_NT) select_kernel(const SelTask* __restrict__ tasks,
                                                        const int64_t* __restrict__ indptr,
                                                        const int64_t* __restrict__ indices,
                                                        int depth) {
  const SelTask t = tasks[blockIdx.x];
  extern __shared__ short dist[];
  __shared__ int warp_tot[SEL_NT / 32];
  __shared__ int s_total;
  const int n = t.n_own;
  const int64_t o0 = t.own0, o1 = t.own0 + t.n_own, b0 = t.oth0, b1 = t.oth0 + t.n_oth;
  for (int v = threadIdx.x; v < n; v += SEL_NT) {
    short d = -1;
    const int64_t gv = o0 + v;
    for (int64_t e = indptr[gv]; e < indptr[gv + 1]; ++e) {
      const int64_t u = indices[e];
      if (u >= b0 && u < b1) { d = 0; break; }
    }
    dist[v] = d;
  }
  __syncthreads();
  for (int lev = 0; lev < depth; ++lev) {
    // a vertex set to lev+1 in this pass is never read as a level-lev source
    for (int v = threadIdx.x; v < n; v += SEL_NT) {
      if (dist[v] != -1) continue;
      const int64_t gv = o0 + v;
      for (int64_t e = indptr[gv]; e < indptr[gv + 1]; ++e) {
        const int64_t u = indices[e];
        if (u >= o0 && u < o1 && ((volatile short*)dist)[u - o0] == lev) {
          dist[v] = (short)(lev + 1);
          break;
        }
      }
    }
    __syncthreads();
  }
  // level-major, position-ordered compaction; thread t owns a contiguous run
  const int per = (n + SEL_NT - 1) / SEL_NT;
  const int p0 = min(n, (int)threadIdx.x * per), p1 = min(n, p0 + per);
  int offset = 0;
  for (int lev = 0; lev <= depth; ++lev) {
    int c = 0;
    for (int v = p0; v < p1; ++v) c += dist[v] == lev;
    const int pre = block_exscan(c, warp_tot, &s_total);
    int w = offset + pre;
    for (int v = p0; v < p1; ++v)
      if (dist[v] == lev) t.out[w++] = v;
    offset += s_total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *t.count = offset;
}

}  // namespace

cudaError_t hk_launch_select(const SelTask* tasks_dev, int ntasks, int max_own,
                             const int64_t* indptr_dev, const int64_t* indices_dev, int depth,
                             cudaStream_t st) {
  if (ntasks == 0) return cudaSuccess;
  const size_t smem = (size_t)max_own * sizeof(short) + 16;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  select_kernel<<<ntasks, SEL_NT, smem, st>>>(tasks_dev, indptr_dev, indices_dev, depth);
  hk_count_launch();
  return cudaGetLastError();
}
