// L2 read-bandwidth probe (the second roofline of the ACA build, whose
// O(r^2 (m+n)) re-streaming of earlier crosses is L2 traffic).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o oracle/_ref/l2_peak tools/l2_peak.cu
//   ./l2_peak  -> one JSON line
//
// Full chip: every SM streams a buffer that fits in L2 (8..64 MB) with 16-byte
// L1-bypassing loads (ld.global.cg), many passes, CUDA-event timed; the HBM
// line streams 4 GB the same way.  Per SM: CTAs on a few SMs only, so the
// per-SM L1<-L2 path is the limit (what one ACA pivot chain can pull).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void read_kernel(const double2* __restrict__ p, size_t n2, int passes, double* sink) {
  double acc = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int it = 0; it < passes; ++it) {
    // rotate the start so consecutive passes do not hit the same lines in step
    const size_t off = ((size_t)it * 4099 * blockDim.x) % n2;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 4
    for (; i < n2; i += stride) {
      size_t j = i + off;
      if (j >= n2) j -= n2;
      double2 v;
      asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p + j));
      acc += v.x + v.y;
    }
  }
  if (acc == 12345.678) *sink = acc;
}

static float run(const double2* p, size_t n2, int passes, int grid, int block, double* sink) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  read_kernel<<<grid, block>>>(p, n2, 1, sink);           // warm (fills L2)
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(a));
    read_kernel<<<grid, block>>>(p, n2, passes, sink);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms);
  }
  CK(cudaEventDestroy(a));
  CK(cudaEventDestroy(b));
  return best;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t big = size_t(4) << 30;
  double2* buf;
  double* sink;
  CK(cudaMalloc(&buf, big));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(buf, 0, big));
  printf("{\"sms\": %d, \"l2_full_chip\": [", sms);
  const size_t sizes_mb[] = {8, 16, 32, 64};
  double best_l2 = 0;
  for (int k = 0; k < 4; ++k) {
    const size_t bytes = sizes_mb[k] << 20, n2 = bytes / 16;
    const int passes = (int)std::max<size_t>(4, (size_t(16) << 30) / bytes);
    const float ms = run(buf, n2, passes, sms * 4, 512, sink);
    const double gbs = (double)bytes * passes / (ms * 1e-3) / 1e9;
    best_l2 = std::max(best_l2, gbs);
    printf("%s{\"mb\": %zu, \"gbs\": %.1f}", k ? ", " : "", sizes_mb[k], gbs);
  }
  printf("], \"l2_gbs\": %.1f", best_l2);
  // working sets past the L2 (the ACA re-streams a 100-300 MB U/V pool): the
  // blend of L2 hits and HBM fills a streaming kernel actually gets
  printf(", \"l2_overflow\": [");
  const size_t over_mb[] = {96, 128, 192, 256, 384};
  for (int k = 0; k < 5; ++k) {
    const size_t bytes = over_mb[k] << 20, n2 = bytes / 16;
    const int passes = (int)std::max<size_t>(4, (size_t(16) << 30) / bytes);
    const float ms = run(buf, n2, passes, sms * 4, 512, sink);
    printf("%s{\"mb\": %zu, \"gbs\": %.1f}", k ? ", " : "", over_mb[k],
           (double)bytes * passes / (ms * 1e-3) / 1e9);
  }
  printf("]");
  {
    const float ms = run(buf, big / 16, 1, sms * 4, 512, sink);
    printf(", \"hbm_read_gbs\": %.1f", (double)big / (ms * 1e-3) / 1e9);
  }
  // per-SM: `nsm` CTAs of 512 threads (one per SM) over an 8 MB L2-resident buffer
  printf(", \"l2_per_sm\": [");
  const int nsms[] = {1, 8, 32};
  for (int k = 0; k < 3; ++k) {
    const size_t bytes = size_t(8) << 20, n2 = bytes / 16;
    const int passes = 8 / (k + 1);
    const float ms = run(buf, n2, passes, nsms[k], 1024, sink);
    const double gbs = (double)bytes * passes / (ms * 1e-3) / 1e9;
    printf("%s{\"ctas\": %d, \"gbs_per_sm\": %.1f}", k ? ", " : "", nsms[k], gbs / nsms[k]);
  }
  int clk = 0;
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("], \"sm_clock_khz_attr\": %d}\n", clk);
  return 0;
}
