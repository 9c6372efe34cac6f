"""GPU front generation with this library's block Gauss-Jordan (hk_spd_inverse)
against the cuSOLVER path on the same recipe: relative difference and time.
    python tools/frontgen_check.py"""
import os
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1403_5337_b200 import frontgen as fg

for dims, plane, seed in [((32, 32, 32), 16, 0), ((48, 48, 48), 24, 1)]:
    out = {}
    for solver in ("torch", "hk", "torch", "hk"):
        os.environ["HK_FRONTGEN"] = solver
        kc = fg.cell_conductivity(dims, seed)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A = fg.layered_grid_front(dims, 2, plane, conductivity=kc, device="cuda", return_torch=True)
        torch.cuda.synchronize()
        out[solver] = (A, time.perf_counter() - t0)
    d = (out["hk"][0] - out["torch"][0]).abs().max().item() / out["torch"][0].abs().max().item()
    print(f"{dims}: n={out['hk'][0].shape[0]} max rel diff hk vs cuSOLVER {d:.2e}; "
          f"time hk {out['hk'][1]*1e3:.1f} ms, cuSOLVER {out['torch'][1]*1e3:.1f} ms")

# a batch of config-3 fronts eliminated together (one hk_spd_inverse per plane step)
os.environ["HK_FRONTGEN"] = "hk"
dims = (32, 32, 32)
kcs = [fg.cell_conductivity(dims, s) for s in range(64)]
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Fb = fg.layered_grid_fronts(dims, 2, 16, kcs, device="cuda")
    torch.cuda.synchronize()
    tb = time.perf_counter() - t0
one = fg.layered_grid_front(dims, 2, 16, conductivity=kcs[5], device="cuda", return_torch=True)
print(f"64 fronts batched: {tb*1e3:.1f} ms ({tb/64*1e3:.2f} ms/front); front 5 batched == single: "
      f"{bool(torch.equal(Fb[5], one))}")

# config 4's front (n = 9216): both solvers
for solver in ("hk", "torch"):
    os.environ["HK_FRONTGEN"] = solver
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    F4 = fg.layered_grid_front((96, 96, 96), "z", 48, device="cuda", return_torch=True)
    torch.cuda.synchronize()
    print(f"cfg4 front via {solver}: {time.perf_counter() - t0:.2f} s")
    if solver == "hk":
        F4h = F4
print("cfg4 max rel diff", float((F4h - F4).abs().max() / F4.abs().max()))
