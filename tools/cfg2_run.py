"""BASELINE config 2 on one GPU: 200k uniform points (seed 2), symmetrised
8-NN graph Laplacian + 1e-3 I, slab |x - 1/2| <= h (0.005 -> ~2k dofs, 0.01 ->
~4k), front = Schur complement eliminating every
non-slab vertex jointly (block CG on the GPU), RCB ordering, leaf 64; HODLR
with ACA and with BDLR at 1e-4 as GMRES preconditioners to 1e-10.  Prints one
JSON line: generation diagnostics, per scheme the max rank per level,
build / factor times (CUDA events, warm), GMRES iterations and time, and --
with --oracle -- the parity checks against the CPU oracle on the same front.

    python tools/cfg2_run.py [--points 200000] [--h 0.005] [--oracle]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
import warnings

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.filterwarnings("ignore", message=".*[Ss]parse.*")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=200000)
    ap.add_argument("--h", type=float, default=0.005)
    ap.add_argument("--depth", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--oracle", action="store_true")
    args = ap.parse_args()
    import torch
    import paper_1403_5337_b200 as hk
    from paper_1403_5337_b200 import frontgen as fg
    from paper_1403_5337_b200.hodlr import HodlrBatch, _graph_in_front_order, _FrontGraph

    t0 = time.perf_counter()
    kf = fg.knn_front(args.points, h=args.h, leaf=64, device="cuda", solver="cg")
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    A = kf.front
    n = A.shape[0]
    acc = kf.accessor()
    graph = _graph_in_front_order(_FrontGraph(acc))
    Ad = torch.from_numpy(A).cuda().contiguous()
    b = np.random.default_rng(2).standard_normal(n)
    out = {"config": "cfg2", "n": n, "generation_s": round(gen_s, 2), "gen": kf.info}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for scheme in ("aca", "bdlr"):
        cfg = hk.CompressionConfig(scheme, tol=1e-4, depth=args.depth)
        batch = HodlrBatch(n, 64, 1)
        bms, fms = [], []
        for _ in range(args.reps):
            ev[0].record()
            batch.build_only(Ad[None], cfg, graph=graph if scheme == "bdlr" else None)
            ev[1].record()
            batch.factor_only()
            ev[2].record()
            torch.cuda.synchronize()
            bms.append(ev[0].elapsed_time(ev[1]))
            fms.append(ev[1].elapsed_time(ev[2]))
        fact = batch.factorization(0)
        rep = batch.report(0)
        op = hk.DenseOperator(Ad)
        gm = []
        for _ in range(2):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            res = hk.gmres(op, b, hk.GmresConfig(tol=1e-10), preconditioner=fact)
            torch.cuda.synchronize()
            gm.append((time.perf_counter() - t1) * 1e3)
        d = {"max_rank_per_level": [lv["max_rank"] for lv in rep.ranks_per_level],
             "build_ms": [round(x, 3) for x in bms], "factor_ms": [round(x, 3) for x in fms],
             "gmres_iterations": res.iterations, "gmres_true_residual": res.true_residual,
             "gmres_ms": round(min(gm), 3), "converged": res.converged}
        if args.oracle:
            from oracle import hodlr_oracle as O
            t2 = time.perf_counter()
            of = O.factorize(A, 64, scheme, 1e-4, args.depth, None, (kf.graph.indptr, kf.graph.indices))
            d["oracle_build_factor_s"] = round(time.perf_counter() - t2, 2)
            d["oracle_max_rank_per_level"] = [e["max_rank"] for e in O.ranks_per_level(of)]
            x = hk.solve(fact, b)
            xo = O.solve(of, b)
            d["solve_rel_diff_vs_oracle"] = float(np.linalg.norm(x - xo) / np.linalg.norm(xo))
            ores = O.gmres(lambda v: A @ v, b, 1e-10, 1000, lambda r: O.solve(of, r))
            d["oracle_gmres_iterations"] = ores["iterations"]
            d["gmres_x_rel_diff_vs_oracle"] = float(np.linalg.norm(res.x - ores["x"]) /
                                                    np.linalg.norm(ores["x"]))
        out[scheme] = d
    print(json.dumps(out))


if __name__ == "__main__":
    main()
