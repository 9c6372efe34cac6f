"""Per-op solve-sweep times (HK_HOST_PROFILE=1: CUDA events between the
kernels, so each line is one kernel plus its launch gap):
    HK_HOST_PROFILE=1 python tools/solve_ops.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_1403_5337_b200 as hk
from paper_1403_5337_b200 import frontgen as fg
from paper_1403_5337_b200.hodlr import HodlrBatch

d = (32, 32, 32)
f = fg.layered_grid_front(d, 2, 16, conductivity=fg.cell_conductivity(d, 0), device="cuda",
                          return_torch=True).contiguous()
b = HodlrBatch(1024, 64, 1).factorize(f[None].contiguous(), hk.CompressionConfig(scheme="aca", tol=1e-6))
fact = b.factorization(0)
W = torch.randn(1, 1024, dtype=torch.float64, device="cuda")
for _ in range(3):
    fact.solve_device(W)
torch.cuda.synchronize()
print("---- cfg4", file=sys.stderr)
f4 = fg.layered_grid_front((96, 96, 96), "z", 48, device="cuda", return_torch=True).contiguous()
b4 = HodlrBatch(9216, 72, 1).factorize(f4[None], hk.CompressionConfig(scheme="aca", tol=1e-4))
fact4 = b4.factorization(0)
W4 = torch.randn(4, 9216, dtype=torch.float64, device="cuda")
for _ in range(3):
    fact4.solve_device(W4)
torch.cuda.synchronize()
