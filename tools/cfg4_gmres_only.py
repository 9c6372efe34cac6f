"""Config-4 GMRES only (front built once, HODLR factored once, then the 4-rhs
batched GMRES twice) -- a short command for ncu launch lists of the GMRES kernels."""
import os, sys, time, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_5337_b200 as hk
from paper_1403_5337_b200.frontgen import layered_grid_front
from paper_1403_5337_b200.hodlr import HodlrBatch
front = layered_grid_front((96, 96, 96), "z", 48, device="cuda", return_torch=True).contiguous()
n = front.shape[0]
batch = HodlrBatch(n, 72, 1).factorize(front[None], hk.CompressionConfig("aca", tol=1e-4))
fact = batch.factorization(0)
op = hk.DenseOperator(front)
B = np.random.default_rng(3).standard_normal((n, 4))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(2):
    t0 = time.perf_counter()
    res = hk.gmres_batch(op, B, hk.GmresConfig(tol=1e-10), preconditioner=fact)
    torch.cuda.synchronize()
    print("gmres 4rhs ms", (time.perf_counter() - t0) * 1e3, [r.iterations for r in res])
torch.cuda.cudart().cudaProfilerStop()
