// Per-SM streaming probe for the ACA sweep's access pattern: each CTA (one
// per SM, 128 CTAs) re-streams its own L2-resident 512 x 64 column-major
// panel (256 KB, like a class-0 block's U at rank 64) chunk by chunk (8
// columns = 32 KB), the way one ACA sweep does, and reduces it.  Variants:
//   0  plain loads, 16 per thread in flight (the register-prefetched sweep)
//   1  TMA bulk copy, one 32 KB copy per chunk, S-stage ring (mbarriers)
//   2  TMA bulk copy, 8 x 4 KB column copies per chunk
//   3  cp.async (LDGSTS) 16-byte per-thread copies, S-stage ring (wait_group)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/build/stream_probe tools/stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int NT = 256, G = 512, KC = 8, NCOL = 64, NCH = NCOL / KC, S = 4;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_tx(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, unsigned n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}

template <int V>
__global__ void __launch_bounds__(NT, 1) probe(const double* __restrict__ P, int sweeps, double* out) {
  extern __shared__ __align__(16) double ring[];
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const double* F = P + (size_t)blockIdx.x * G * NCOL;
  const int tid = threadIdx.x, lane = tid & 31;
  double acc0 = 0, acc1 = 0;
  if (V == 1 || V == 2) {
    if (tid == 0) {
      for (int s = 0; s < S; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], NT / 32); }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  int seq = 0;
  for (int it = 0; it < sweeps; ++it) {
    if (V == 0) {
      for (int c = 0; c < NCH; ++c) {
        double a[2][KC];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int j = 0; j < KC; ++j) a[q][j] = F[(size_t)(c * KC + j) * G + tid + q * NT];
#pragma unroll
        for (int j = 0; j < KC; ++j) { acc0 = acc0 * 0.999 + a[0][j]; acc1 = acc1 * 0.999 + a[1][j]; }
      }
    } else if (V == 1 || V == 2) {
      auto issue = [&](int c, int g) {
        const int s = g % S;
        if (g >= S) mb_wait(&empty[s], ((g / S) - 1) & 1);
        double* dst = ring + (size_t)s * KC * G;
        mb_tx(&full[s], KC * G * 8);
        if (V == 1) bulk(dst, F + (size_t)c * KC * G, KC * G * 8, &full[s]);
        else for (int j = 0; j < KC; ++j) bulk(dst + j * G, F + (size_t)(c * KC + j) * G, G * 8, &full[s]);
      };
      const int g0 = seq;
      if (tid == 0) for (int c = 0; c < S - 1 && c < NCH; ++c) issue(c, g0 + c);
      for (int c = 0; c < NCH; ++c) {
        const int g = g0 + c, s = g % S;
        if (tid == 0 && c + S - 1 < NCH) issue(c + S - 1, g + S - 1);
        mb_wait(&full[s], (g / S) & 1);
        const double* st = ring + (size_t)s * KC * G + tid;
        double a[2][KC];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int j = 0; j < KC; ++j) a[q][j] = st[j * G + q * NT];
        __syncwarp();
        if (lane == 0) mb_arrive(&empty[s]);
#pragma unroll
        for (int j = 0; j < KC; ++j) { acc0 = acc0 * 0.999 + a[0][j]; acc1 = acc1 * 0.999 + a[1][j]; }
      }
      seq = g0 + NCH;
    } else {
      // per-thread LDGSTS: thread owns rows 2*tid, 2*tid+1 (16 bytes per column)
      auto issue = [&](int c) {
        double* dst = ring + (size_t)(c % S) * KC * G;
#pragma unroll
        for (int j = 0; j < KC; ++j)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + j * G + 2 * tid)),
                       "l"(F + (size_t)(c * KC + j) * G + 2 * tid) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      for (int c = 0; c < S - 1; ++c) issue(c);
      for (int c = 0; c < NCH; ++c) {
        if (c + S - 1 < NCH) issue(c + S - 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
        const double* st = ring + (size_t)(c % S) * KC * G + 2 * tid;
#pragma unroll
        for (int j = 0; j < KC; ++j) {
          const double2 v = *reinterpret_cast<const double2*>(st + j * G);
          acc0 = acc0 * 0.999 + v.x;
          acc1 = acc1 * 0.999 + v.y;
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
  }
  if (acc0 + acc1 == 1234.5) out[0] = acc0;
}

template <int V>
static int run(const double* P, int ctas, double* out, const char* name) {
  const size_t smem = (V == 0) ? 0 : (size_t)S * KC * G * 8;
  CK(cudaFuncSetAttribute(probe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int sweeps = 200;
  probe<V><<<ctas, NT, smem>>>(P, 2, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<V><<<ctas, NT, smem>>>(P, sweeps, out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)ctas * sweeps * NCOL * G * 8;
  printf("{\"variant\": \"%s\", \"ctas\": %d, \"us_per_sweep\": %.3f, \"gbs_per_cta\": %.1f, \"total_gbs\": %.0f}\n",
         name, ctas, ms * 1e3 / sweeps, bytes / ctas / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9);
  return 0;
}

int main() {
  double* P;
  double* out;
  const int ctas = 128;
  CK(cudaMalloc(&P, (size_t)ctas * G * NCOL * 8));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(P, 0, (size_t)ctas * G * NCOL * 8));
  for (int c : {1, 128}) {
    run<0>(P, c, out, "plain_loads");
    run<1>(P, c, out, "tma_32KB");
    run<2>(P, c, out, "tma_8x4KB");
    run<3>(P, c, out, "ldgsts16");
  }
  return 0;
}
