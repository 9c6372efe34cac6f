"""Config-4 factorize() timing, standalone or after a config-3 batch has run
in the same process (--after-cfg3): the bench's line item runs in the latter
context."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_5337_b200 as hk
from paper_1403_5337_b200.frontgen import layered_grid_front, cell_conductivity
from paper_1403_5337_b200.hodlr import HodlrBatch
if "--after-cfg3" in sys.argv:
    fr = torch.stack([layered_grid_front((32, 32, 32), "z", 16, conductivity=cell_conductivity((32, 32, 32), s),
                                         device="cuda", return_torch=True) for s in range(64)]).contiguous()
    b3 = HodlrBatch(1024, 64, 64)
    for _ in range(3):
        b3.factorize(fr, hk.CompressionConfig("aca", tol=1e-6))
    torch.cuda.synchronize()
    if "--free" in sys.argv:
        del b3, fr
        torch.cuda.synchronize()
pad = None
for a in sys.argv:
    if a.startswith("--pad-mb="):
        pad = torch.empty(int(a.split("=")[1]) * 131072, dtype=torch.float64, device="cuda")
front = layered_grid_front((96, 96, 96), "z", 48, device="cuda", return_torch=True).contiguous()
cfg = hk.CompressionConfig("aca", tol=1e-4)
b = HodlrBatch(9216, 72, 1)
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for i in range(4):
    torch.cuda.synchronize()
    e[0].record(); b.build_only(front[None], cfg); e[1].record(); b.factor_only(); e[2].record()
    torch.cuda.synchronize()
    print(f"rep {i}: build {e[0].elapsed_time(e[1]):.2f} ms factor {e[1].elapsed_time(e[2]):.2f} ms")
