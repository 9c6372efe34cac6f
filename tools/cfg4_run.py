"""BASELINE config 4 on one GPU: the 96^3 constant-coefficient front (n = 9216),
HODLR depth 7 / leaf 72 / ACA 1e-4, GMRES to 1e-10 on 4 N(0,1) right-hand
sides (seed 3).  Prints one JSON line with the phase timings, the max rank per
level and the GMRES iteration counts; the reference's own values measured in
this container are SURVEY.md §6.3 (ranks 227,227,227,195,193,98,53; 10,11,11,10
iterations; build+factor 20.2 s and GMRES 4.76 s single-threaded).

    python tools/cfg4_run.py [--grid 96] [--reps 3]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=96)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--nrhs", type=int, default=4)
    args = ap.parse_args()
    import torch
    import paper_1403_5337_b200 as hk
    from paper_1403_5337_b200.frontgen import layered_grid_front

    g = args.grid
    t0 = time.perf_counter()
    front = layered_grid_front((g, g, g), "z", g // 2, device="cuda", return_torch=True)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    n = front.shape[0]
    front = front.contiguous()
    cfg = hk.CompressionConfig("aca", tol=1e-4)
    batch = hk.HodlrBatch(n, 72, 1)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    build_ms, factor_ms = [], []
    for _ in range(args.reps):
        ev[0].record()
        batch.build_only(front[None], cfg)
        ev[1].record()
        batch.factor_only()
        ev[2].record()
        torch.cuda.synchronize()
        build_ms.append(ev[0].elapsed_time(ev[1]))
        factor_ms.append(ev[1].elapsed_time(ev[2]))
    fact = batch.factorization(0)
    rep = batch.report(0)
    op = hk.DenseOperator(front)
    B = np.random.default_rng(3).standard_normal((n, args.nrhs))
    its, tres, gm_ms = [], [], []
    for _k in range(2):                        # warm, then timed
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        res_all = hk.gmres_batch(op, B, hk.GmresConfig(tol=1e-10), preconditioner=fact)
        torch.cuda.synchronize()
    gm_ms.append((time.perf_counter() - t1) * 1e3)
    for res in res_all:
        its.append(res.iterations)
        tres.append(res.true_residual)
    # direct solve of the 4 rhs at once and its residual through the dense front
    Bd = torch.from_numpy(B).cuda()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    X = hk.solve(fact, Bd)
    torch.cuda.synchronize()
    solve_ms = (time.perf_counter() - t2) * 1e3
    rel = float(torch.linalg.norm(front @ X - Bd) / torch.linalg.norm(Bd))
    print(json.dumps({
        "config": "cfg4", "n": n, "frontgen_s": round(t_gen, 2),
        "build_ms": [round(x, 2) for x in build_ms], "factor_ms": [round(x, 2) for x in factor_ms],
        "max_rank_per_level": [lv["max_rank"] for lv in rep.ranks_per_level],
        "gmres_iterations": its, "gmres_true_residual": tres,
        "gmres_batch_wall_ms": [round(x, 2) for x in gm_ms],
        "hodlr_solve_4rhs_ms": round(solve_ms, 3), "hodlr_solve_rel_residual": rel,
        "aca_seconds": batch.plan.aca_seconds(),
    }))


if __name__ == "__main__":
    main()
