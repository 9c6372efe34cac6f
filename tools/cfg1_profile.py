import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_1403_5337_b200 as hk
from paper_1403_5337_b200 import frontgen as fg
from paper_1403_5337_b200.hodlr import HodlrBatch
kc = fg.cell_conductivity((48, 48, 48), 1)
A = fg.layered_grid_front((48, 48, 48), 2, 24, conductivity=kc, device='cuda')
g = fg.grid_graph(fg.GridSpec((48, 48, 48)), 2, 24)
csr = (np.asarray(g.indptr, dtype=np.int64), np.asarray(g.indices, dtype=np.int64))
Ad = torch.from_numpy(A).cuda()
b = HodlrBatch(2304, 64, 1)
cfg = hk.CompressionConfig('bdlr', tol=1e-4, depth=3)
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    b.build_only(Ad[None], cfg, graph=csr); torch.cuda.synchronize(); t1 = time.perf_counter()
    b.factor_only(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"build {1e3*(t1-t0):.3f} factor {1e3*(t2-t1):.3f}", file=sys.stderr)
