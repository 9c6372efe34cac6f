"""Experiment: one 64-front plan vs G plans of 64/G fronts driven by G host
threads on G streams (the ACA of one group overlapping another's factor)."""
import os, sys, time, threading, torch
sys.path.insert(0, os.getcwd())
import paper_1403_5337_b200 as hk
from paper_1403_5337_b200.frontgen import layered_grid_front, cell_conductivity
from paper_1403_5337_b200.hodlr import HodlrBatch
B = 64
fr = torch.stack([layered_grid_front((32,32,32), 'z', 16, conductivity=cell_conductivity((32,32,32), s), device='cuda', return_torch=True) for s in range(B)]).contiguous()
cfg = hk.CompressionConfig('aca', tol=1e-6)
rhs = torch.randn(B, 1024, dtype=torch.float64, device='cuda')
for G in [1, 2, 4]:
    per = B // G
    plans = [HodlrBatch(1024, 64, per) for _ in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]
    def work(g, delay):
        with torch.cuda.stream(streams[g]):
            if delay: time.sleep(delay)
            plans[g].build_only(fr[g*per:(g+1)*per], cfg)
            plans[g].factor_only()
            plans[g].solve_(rhs[g*per:(g+1)*per].clone())
    for delay in ([0.0] if G == 1 else [0.0, 0.0015]):
        ts = []
        for it in range(8):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            th = [threading.Thread(target=work, args=(g, delay * g)) for g in range(G)]
            for t in th: t.start()
            for t in th: t.join()
            torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        print(f"G={G} delay={delay*1e3:.1f}ms step {1e3*min(ts[2:]):.3f} ms (median {1e3*sorted(ts[2:])[3]:.3f})", flush=True)
