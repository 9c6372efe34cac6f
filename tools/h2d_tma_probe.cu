// H2D copy probe: pinned host memory -> HBM through the TMA (cp.async.bulk load into a
// shared-memory ring, cp.async.bulk store with an L2 evict-first hint), against the
// 16-byte-load copy kernel and the copy engine.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o oracle/_ref/h2d_tma_probe tools/h2d_tma_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

template <int CHUNK, int STAGES>
__global__ void __launch_bounds__(32) tma_copy(const char* __restrict__ src, char* __restrict__ dst, size_t bytes) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  const size_t nchunk = bytes / CHUNK;   // bytes is a multiple of CHUNK in the probe
  for (int s = 0; s < STAGES; ++s) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(b));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const size_t first = blockIdx.x, step = gridDim.x;
  auto issue = [&](size_t c, int s) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(ring + (size_t)s * CHUNK);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"((uint32_t)CHUNK) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(src + c * CHUNK), "r"((uint32_t)CHUNK), "r"(b) : "memory");
  };
  // prologue
  size_t c_issue = first;
  for (int s = 0; s < STAGES && c_issue < nchunk; ++s, c_issue += step) issue(c_issue, s);
  int s = 0;
  uint32_t phase = 0;
  for (size_t c = first; c < nchunk; c += step) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(b), "r"(phase) : "memory");
    const uint32_t sm = (uint32_t)__cvta_generic_to_shared(ring + (size_t)s * CHUNK);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                 ::"l"(dst + c * CHUNK), "r"(sm), "r"((uint32_t)CHUNK), "l"(pol) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // the stage may be refilled once its store has read the shared memory
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (c_issue < nchunk) { issue(c_issue, s); c_issue += step; }
    if (++s == STAGES) { s = 0; phase ^= 1; }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(256) ld_copy(const double2* __restrict__ src, double2* __restrict__ dst, size_t n2) {
  constexpr int U = 8;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(dst + i + u * stride, v[u]);
  }
}

template <class F>
static double bw(F f, size_t bytes) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int r = 0; r < 5; ++r) f();
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  return 5.0 * bytes / (ms * 1e-3) / 1e9;
}

int main() {
  const size_t bytes = (size_t)512 << 20;
  char *h, *d;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocDefault));
  CK(cudaMalloc(&d, bytes));
  for (size_t i = 0; i < bytes / 8; ++i) ((double*)h)[i] = (double)(i % 977);
  printf("copy engine       : %.1f GB/s\n", bw([&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, 0); }, bytes));
  printf("16-byte loads 4x256: %.1f GB/s\n", bw([&] { ld_copy<<<4, 256>>>((const double2*)h, (double2*)d, bytes / 16); }, bytes));
#define RUN(CH, ST, G) { CK(cudaFuncSetAttribute(tma_copy<CH, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * ST)); \
  printf("TMA %5d B x %d stages, %2d CTAs: %.1f GB/s\n", CH, ST, G, \
         bw([&] { tma_copy<CH, ST><<<G, 32, CH * ST>>>(h, d, bytes); }, bytes)); CK(cudaGetLastError()); }
  RUN(16384, 4, 4) RUN(16384, 4, 8) RUN(16384, 8, 8) RUN(32768, 4, 8) RUN(4096, 8, 16) RUN(65536, 3, 8)
  // verify the last copy
  CK(cudaMemset(d, 0, bytes));
  tma_copy<16384, 4><<<8, 32, 16384 * 4>>>(h, d, bytes);
  CK(cudaDeviceSynchronize());
  double* chk = (double*)malloc(1 << 20);
  CK(cudaMemcpy(chk, d + bytes - (1 << 20), 1 << 20, cudaMemcpyDeviceToHost));
  size_t bad = 0;
  for (size_t i = 0; i < (1 << 20) / 8; ++i) bad += chk[i] != ((double*)h)[(bytes - (1 << 20)) / 8 + i];
  printf("verify tail: %zu mismatches\n", bad);
  return 0;
}
