"""GMRES time-to-tol breakdown: the public call vs the bare native call vs
the graph alone, on config-3 front 0 and config 4 (4 rhs).

    python tools/gmres_profile.py [--cfg 3|4|both] [--reps 20]
"""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1403_5337_b200 as hk  # noqa: E402
from paper_1403_5337_b200 import _native as N  # noqa: E402
from paper_1403_5337_b200 import frontgen as fg  # noqa: E402
from paper_1403_5337_b200.hodlr import HodlrBatch  # noqa: E402


def ev_time(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        t0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
    a = np.array(out)
    return float(np.median(a[:, 0])), float(np.median(a[:, 1]))


def run(front, leaf, tol, B, reps, label):
    n = front.shape[0]
    batch = HodlrBatch(n, leaf, 1).factorize(front[None].contiguous(), hk.CompressionConfig(scheme="aca", tol=tol))
    fact = batch.factorization(0)
    op = hk.DenseOperator(front)
    s = B.shape[1]
    cfg = hk.GmresConfig(tol=1e-10)
    if s == 1:
        pub = lambda: hk.gmres(op, B[:, 0], cfg, preconditioner=fact)
    else:
        pub = lambda: hk.gmres_batch(op, B, cfg, preconditioner=fact)
    res = pub()
    its = [res.iterations] if s == 1 else [r.iterations for r in res]
    bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    xd = torch.zeros_like(bd)
    its_h = np.zeros(s, dtype=np.int64)
    hist = np.zeros((s, cfg.max_iter))
    tres = np.zeros(s)
    flags = np.zeros(2 * s, dtype=np.int32)

    def native():
        N.check(N.lib().hk_gmres_batch(batch.plan.h, 0, N.ptr(op.dev), n, n, N.ptr(bd), s, cfg.tol,
                                       cfg.max_iter, 1, None, N.ptr(xd), N.arr_ptr(its_h, N.I64),
                                       N.arr_ptr(hist, N.D), N.arr_ptr(tres, N.D),
                                       N.arr_ptr(flags, N.I32), N.stream_handle()))
    W = bd.clone()

    def solve():
        fact.solve_device(W)

    def gemv():
        N.check(N.lib().hk_gemv(N.ptr(op.dev), n, n, n, N.ptr(bd), n, s, N.ptr(W), n, N.stream_handle()))
    t_pub = ev_time(pub, reps)
    t_nat = ev_time(native, reps)
    t_sol = ev_time(solve, reps)
    t_gmv = ev_time(gemv, reps)
    print(f"{label}: n={n} s={s} its={its}")
    print(f"  public call     {t_pub[0]:8.3f} ms (events)  {t_pub[1]:8.3f} ms (wall)")
    print(f"  native call     {t_nat[0]:8.3f} ms (events)  {t_nat[1]:8.3f} ms (wall)")
    print(f"  one solve       {t_sol[0]:8.3f} ms   one gemv {t_gmv[0]:8.3f} ms")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="both")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    if a.cfg in ("3", "both"):
        d = (32, 32, 32)
        f = fg.layered_grid_front(d, 2, 16, conductivity=fg.cell_conductivity(d, 0), device="cuda",
                                  return_torch=True).contiguous()
        b = np.random.default_rng(0).standard_normal((f.shape[0], 1))
        run(f, 64, 1e-6, b, a.reps, "cfg3 front 0")
    if a.cfg in ("4", "both"):
        f = fg.layered_grid_front((96, 96, 96), "z", 48, device="cuda", return_torch=True).contiguous()
        B = np.random.default_rng(3).standard_normal((f.shape[0], 4))
        run(f, 72, 1e-4, B, a.reps, "cfg4")


if __name__ == "__main__":
    main()
