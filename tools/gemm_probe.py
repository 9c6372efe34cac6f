"""Throughput of the batched DMMA GEMM (hk_dgemm, one task) on a few shapes,
CUDA events over 20 launches: python tools/gemm_probe.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1403_5337_b200 import _native as N

shapes = [(4096, 4096, 4096), (2048, 2048, 64), (2048, 2048, 128), (4096, 384, 64), (1024, 1024, 1024),
          (216, 384, 216), (512, 512, 512)]
for (m, n, k) in shapes:
    A = torch.randn(k, m, dtype=torch.float64, device="cuda")   # column-major m x k: ld m
    A = torch.randn(m * k, dtype=torch.float64, device="cuda")
    B = torch.randn(k * n, dtype=torch.float64, device="cuda")
    C = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    st = N.stream_handle()
    f = lambda: N.check(N.lib().hk_dgemm(0, m, n, k, 1.0, N.ptr(A), m, N.ptr(B), k, 0.0, N.ptr(C), m, st))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ref = (A.view(k, m).t() @ B.view(n, k).t())
    err = (C.view(n, m).t() - ref).abs().max().item() / ref.abs().max().item()
    print(f"m={m:5d} n={n:5d} k={k:5d}  {ms*1e3:9.1f} us  {2*m*n*k/ms/1e9:7.2f} TFLOP/s  relerr={err:.1e}")
