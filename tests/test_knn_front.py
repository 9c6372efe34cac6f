"""BASELINE config 2 (unstructured-graph front): generator properties on the
CPU, and GPU parity of ACA and BDLR on a reduced-size instance (the 200k-point
case runs in tools/cfg2_run.py; its front generation is a block CG on the GPU).

The reference has no generator for this config: the
front is manufactured here, and parity is GPU path vs the oracle on the same
front bits, to the same bars as the other configs."""

import warnings

import numpy as np
import pytest

from oracle import hodlr_oracle as O
import paper_1403_5337_b200 as hk
from paper_1403_5337_b200 import frontgen as fg

warnings.filterwarnings("ignore", message=".*[Ss]parse.*")


def test_rcb_order_matches_build_tree_splits():
    pts = fg.knn_points(1000, seed=7)
    order = fg.rcb_order(pts, 64)
    assert np.array_equal(np.sort(order), np.arange(1000))
    tree = O.bisection_tree(1000, 64)
    # every internal node's two children are the two halves of one RCB cut:
    # separated along the node's widest coordinate
    for level, lo, hi, left, right in tree:
        if left < 0:
            continue
        a = pts[order[lo:tree[left][2]]]
        b = pts[order[tree[right][1]:hi]]
        ext = np.vstack([a, b])
        ax = int(np.argmax(ext.max(0) - ext.min(0)))
        assert a.shape[0] == (hi - lo + 1) // 2
        assert a[:, ax].max() <= b[:, ax].min()


def test_knn_graph_symmetric_and_exact():
    pts = fg.knn_points(3000, seed=3)
    g = fg.knn_graph(pts, 8)
    # symmetric, no self loops, every vertex has its 8 exact nearest neighbours
    dense = np.zeros((3000, 3000), dtype=bool)
    for v in range(3000):
        nb = g.neighbors(v)
        assert v not in nb
        dense[v, nb] = True
    assert np.array_equal(dense, dense.T)
    d2 = ((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(d2, np.inf)
    nn = np.argsort(d2, axis=1, kind="stable")[:, :8]
    assert dense[np.repeat(np.arange(3000), 8), nn.ravel()].all()
    assert np.diff(g.indptr).min() >= 8


def test_knn_front_direct_vs_block_cg():
    kd = fg.knn_front(4000, h=0.03, leaf=32)
    kc = fg.knn_front(4000, h=0.03, leaf=32, solver="cg", device="cpu", cg_tol=1e-13)
    assert kd.info["n"] == kc.info["n"] > 100
    assert np.linalg.norm(kc.front - kd.front) <= 1e-12 * np.linalg.norm(kd.front)
    # SPD front of an M-matrix Schur complement: symmetric to rounding, positive
    A = kd.front
    assert np.abs(A - A.T).max() <= 1e-13 * np.abs(A).max()
    assert np.linalg.eigvalsh((A + A.T) / 2)[0] > 0
    # the slab is not a separator: some edges cross it
    assert kd.info["crossing_directed_edges"] > 0
    assert np.array_equal(np.sort(kd.ordering), np.flatnonzero(np.abs(fg.knn_points(4000)[:, 0] - 0.5) <= 0.03))


@pytest.fixture(scope="module")
def cfg2_small():
    return fg.knn_front(20000, h=0.01, leaf=64)


def _internal(nodes):
    return [s for s, nd in enumerate(nodes) if nd[3] >= 0]


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,depth", [("aca", 1), ("bdlr", 1), ("bdlr", 3)])
def test_cfg2_reduced_parity(cfg2_small, scheme, depth):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1403_5337_b200.hodlr import factorize_traced
    kf = cfg2_small
    A, graph = kf.front, kf.graph
    n = A.shape[0]
    acc = hk.BlockAccessor.from_matrix(A, pattern=graph)
    tree = hk.build_tree(n, 64)
    cfg = hk.CompressionConfig(scheme=scheme, tol=1e-4, depth=depth)
    fact, report, recs = factorize_traced(acc, tree, cfg)
    ofact = O.factorize(A, 64, scheme, 1e-4, depth, None, (graph.indptr, graph.indices))
    for k, s in enumerate(_internal(ofact.nodes)):
        for side in (0, 1):
            b = 2 * k + side
            rows, cols = recs[b]
            if scheme == "aca":
                tr = ofact.traces[s][side]
                assert np.array_equal(rows, [v for kk, v in tr if kk == "r"]), b
                assert np.array_equal(cols, [v for kk, v in tr if kk == "c"]), b
                U, V = fact.block_factor(b)
                assert np.array_equal(U, ofact.factors[s][side][0]), b
                assert np.array_equal(V, ofact.factors[s][side][1]), b
            else:
                info = ofact.skeletons[s][side]
                if info is None:
                    assert rows.size == 0
                    continue
                assert np.array_equal(rows, info["rows"]) and np.array_equal(cols, info["cols"]), b
    assert [e["max_rank"] for e in report.ranks_per_level] == \
        [e["max_rank"] for e in O.ranks_per_level(ofact)]
    b0 = np.random.default_rng(2).standard_normal(n)
    x = hk.solve(fact, b0)
    xo = O.solve(ofact, b0)
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
    E = hk.solve(fact, A) - np.eye(n)
    Eo = O.solve(ofact, A) - np.eye(n)
    assert np.linalg.norm(E - Eo) <= 1e-10 * np.linalg.norm(Eo)
    res = hk.gmres(hk.DenseOperator(A), b0, hk.GmresConfig(tol=1e-10), preconditioner=fact)
    ores = O.gmres(lambda v: A @ v, b0, 1e-10, 1000, lambda r: O.solve(ofact, r))
    assert res.converged and abs(res.iterations - ores["iterations"]) <= 1
    assert np.linalg.norm(res.x - ores["x"]) <= 1e-10 * np.linalg.norm(ores["x"])


@pytest.mark.gpu
@pytest.mark.parametrize("npts,h,leaf,depth", [(3000, 0.05, 16, 0), (3000, 0.05, 16, 2),
                                               (6000, 0.02, 32, 1), (1500, 0.1, 8, 4)])
def test_bdlr_small_knn_fronts_edge_depths(npts, h, leaf, depth):
    """BDLR on small unstructured fronts with shallow/deep selections and small
    leaves: GPU skeletons (GPU BFS selection + complete-pivot LU) identical to
    the oracle's, ranks equal, solves within 1e-10."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1403_5337_b200.hodlr import factorize_traced
    kf = fg.knn_front(npts, h=h, leaf=leaf)
    A, graph = kf.front, kf.graph
    n = A.shape[0]
    cfg = hk.CompressionConfig(scheme="bdlr", tol=1e-4, depth=depth)
    try:
        ofact = O.factorize(A, leaf, "bdlr", 1e-4, depth, None, (graph.indptr, graph.indices))
    except Exception as exc:                       # the reference raises -> so must we
        with pytest.raises(type(exc)):
            factorize_traced(hk.BlockAccessor.from_matrix(A, pattern=graph), hk.build_tree(n, leaf), cfg)
        return
    fact, report, recs = factorize_traced(hk.BlockAccessor.from_matrix(A, pattern=graph),
                                          hk.build_tree(n, leaf), cfg)
    for k, sl in enumerate(_internal(ofact.nodes)):
        for side in (0, 1):
            rows, cols = recs[2 * k + side]
            info = ofact.skeletons[sl][side]
            if info is None:
                assert rows.size == 0
                continue
            assert np.array_equal(rows, info["rows"]) and np.array_equal(cols, info["cols"])
    assert [e["max_rank"] for e in report.ranks_per_level] == \
        [e["max_rank"] for e in O.ranks_per_level(ofact)]
    b0 = np.random.default_rng(5).standard_normal(n)
    x = hk.solve(fact, b0)
    xo = O.solve(ofact, b0)
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)

