"""Measure the FP64 denominators for the roofline on this B200 (MEASURED_PEAKS.json has
only HBM and bf16): cuBLAS DGEMM 8192^3 (burst, best of 10) and a register-only
DMMA.8x8x4 / DFMA issue microbenchmark.  Writes profiles/fp64_peak.json."""

import json
import subprocess
import sys
import tempfile
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent

KERNEL = r'''
#include <cstdio>
__global__ void dmma_loop(double* out, int iters) {
  double c[8][2] = {};
  double a = threadIdx.x * 1e-9, b = blockIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
  if (s == 12345.0) out[0] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double x[8]; for (int q = 0; q < 8; ++q) x[q] = threadIdx.x + q;
  const double a = 1.0000001, b = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = fma(x[q], a, b);
  double s = 0; for (int q = 0; q < 8; ++q) s += x[q];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, blocks = sms * 8, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    dmma_loop<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e0); dmma_loop<<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (blocks * threads / 32);
    if (rep) printf("dmma_tflops %.3f\n", flops / ms / 1e9);
    dfma_loop<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8.0 * iters * blocks * threads;
    if (rep) printf("dfma_tflops %.3f\n", flops / ms / 1e9);
  }
  return 0;
}
'''


def main():
    out = {}
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out["cublas_dgemm_tflops"] = 2 * n ** 3 / (best * 1e-3) / 1e12
    with tempfile.TemporaryDirectory() as td:
        src = Path(td) / "p.cu"
        src.write_text(KERNEL)
        exe = Path(td) / "p"
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", str(src),
                        "-o", str(exe)], check=True)
        r = subprocess.run([str(exe)], capture_output=True, text=True, check=True)
        for line in r.stdout.splitlines():
            k, v = line.split()
            out[k] = float(v)
    out["device"] = torch.cuda.get_device_name(0)
    (ROOT / "profiles").mkdir(exist_ok=True)
    (ROOT / "profiles" / "fp64_peak.json").write_text(json.dumps(out, indent=1))
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
