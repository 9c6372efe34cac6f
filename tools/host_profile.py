import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_1403_5337_b200 as hk
from paper_1403_5337_b200.frontgen import layered_grid_front, cell_conductivity
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
fr = torch.stack([layered_grid_front((32,32,32), 'z', 16, conductivity=cell_conductivity((32,32,32), s), device='cuda', return_torch=True) for s in range(B)]).contiguous()
cfg = hk.CompressionConfig('aca', tol=1e-6)
b = hk.HodlrBatch(1024, 64, B)
rhs = torch.randn(B, 1024, dtype=torch.float64, device='cuda')
for it in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    b.build_only(fr, cfg); t1 = time.perf_counter()
    b.factor_only(); t2 = time.perf_counter()
    b.solve_(rhs.clone()); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"wall build {1e3*(t1-t0):.3f} factor {1e3*(t2-t1):.3f} solve {1e3*(t3-t2):.3f} ms; gpu t={b.plan.timings()}", file=sys.stderr)
