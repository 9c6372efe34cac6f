"""GPU parity: the CUDA path against the oracle and the reference's golden
vectors on identical inputs.

Bars (BASELINE north_star): ACA pivot traces, ranks and U/V factors
bit-exact; BDLR skeleton indices and ranks bit-exact; factor / solve within
1e-10 relative (solve(fact, b) and E = solve(fact, A) - I, as
||E_gpu - E_oracle||_F / ||E_oracle||_F); GMRES iteration counts within +-1.
"""

import numpy as np
import pytest

from conftest import SMALL_FRONTS, golden
from oracle import hodlr_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_1403_5337_b200 as hk  # noqa: E402
from paper_1403_5337_b200.hodlr import HodlrBatch, factorize_traced  # noqa: E402

SOLVE_RTOL = 1e-10   # stated tolerance for floating-point agreement


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _internal(nodes):
    return [s for s, nd in enumerate(nodes) if nd[3] >= 0]


def _otrace(tr):
    return (np.array([v for k, v in tr if k == "r"], dtype=np.int64),
            np.array([v for k, v in tr if k == "c"], dtype=np.int64))


# ------------------------------------------------------------------ kernels vs goldens
def test_aca_kernel_bit_exact_on_golden_blocks():
    g = golden("aca_blocks")
    for name in g["names"]:
        name = str(name)
        mr = int(g[f"{name}_maxrank"]) or None
        cfg = hk.CompressionConfig(scheme="aca", tol=float(g[f"{name}_tol"]), max_rank=mr)
        tr = {}
        f = hk.compress_aca(hk.BlockAccessor(g[f"{name}_A"]), cfg, trace=tr)
        assert np.array_equal(tr["rows"], g[f"{name}_rows"]), name
        assert np.array_equal(tr["cols"], g[f"{name}_cols"]), name
        assert np.array_equal(f.u, g[f"{name}_U"]), name
        assert np.array_equal(f.v, g[f"{name}_V"]), name


def test_aca_cluster_path_bit_exact():
    """Every block forced onto the thread-block-cluster ACA (HK_ACA_CLMIN=0, read
    once per process, hence the subprocess): pivots, ranks and U/V stay
    bit-identical to the reference's goldens and to a config-0-style front's
    single-CTA factors."""
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.');"
        "import test_gpu_parity as T; T.test_aca_kernel_bit_exact_on_golden_blocks();"
        "T.test_baseline_aca_front_parity(0, 'cfg0'); print('ok')")
    env = dict(os.environ, HK_ACA_CLMIN="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]


def test_complete_pivot_kernel_bit_exact():
    g = golden("lu_full")
    for name in g["names"]:
        name = str(name)
        f = hk.lu_full(g[f"{name}_A"])
        assert np.array_equal(f.lu, g[f"{name}_lu"]), name
        assert np.array_equal(f.row_perm, g[f"{name}_rp"]), name
        assert np.array_equal(f.col_perm, g[f"{name}_cp"]), name
        assert np.array_equal(f.pivot_magnitudes, g[f"{name}_piv"]), name


def test_partial_pivot_lu_and_inverse(rng):
    for n in (1, 5, 36, 64, 72, 150, 200):
        a = rng.standard_normal((n, n)) + n * np.eye(n)
        f = hk.lu_partial(a)
        low = np.tril(f.lu, -1) + np.eye(n)
        up = np.triu(f.lu)
        assert np.linalg.norm(a[f.row_perm] - low @ up) <= 1e-13 * np.linalg.norm(a)
        assert np.linalg.norm(a @ f.inverse - np.eye(n)) <= 1e-12 * n
        b = rng.standard_normal((n, 3))
        assert np.linalg.norm(a @ f.solve(b) - b) <= 1e-10 * np.linalg.norm(b)
    with pytest.raises(hk.SingularMatrixError):
        hk.lu_partial(np.zeros((3, 3)))


def test_gj_inverse_all_kernel_shapes(rng):
    """Every Gauss-Jordan variant (register dataflow N<=128, panel N<=160, the
    thread-block-cluster kernel 160<N<=256, the global-memory one above)
    against numpy's inverse, including batches of mixed conditioning and a
    singular member."""
    from paper_1403_5337_b200.dense import gj_inverse
    for n in (1, 17, 64, 100, 128, 150, 160, 161, 190, 227, 255, 256, 300):
        a = rng.standard_normal((3, n, n)) + 0.5 * np.sqrt(n) * np.eye(n)
        a[1] = a[1][rng.permutation(n)]          # pivoting must find the diagonal
        inv = gj_inverse(a)
        for b in range(3):
            ref = np.linalg.inv(a[b])
            assert np.linalg.norm(inv[b] - ref) <= 1e-11 * np.linalg.norm(ref), (n, b)
    a = rng.standard_normal((2, 200, 200))
    a[1, :, 7] = 0.0
    with pytest.raises(hk.SingularMatrixError):
        gj_inverse(a)


# ------------------------------------------------------------------ HODLR on golden fronts
@pytest.mark.parametrize("front", SMALL_FRONTS)
@pytest.mark.parametrize("cname,scheme,tol,depth", [("aca6", "aca", 1e-6, 1), ("aca3", "aca", 1e-3, 1),
                                                     ("bdlr1", "bdlr", 1e-1, 1),
                                                     ("bdlr3", "bdlr", 1e-3, 3)])
def test_hodlr_small_fronts_vs_reference_goldens(front, cname, scheme, tol, depth):
    fr = golden("fronts")
    h = golden("hodlr_small")
    key = f"{front}_{cname}_"
    A = fr[f"{front}_front"]
    pat = hk.SparsePattern(fr[f"{front}_indptr"], fr[f"{front}_indices"])
    acc = hk.BlockAccessor.from_matrix(A, pattern=pat)
    leaf = int(h[f"{key}leaf"])
    tree = hk.build_tree(A.shape[0], leaf)
    cfg = hk.CompressionConfig(scheme=scheme, tol=tol, depth=depth)
    fact, report, recs = factorize_traced(acc, tree, cfg)
    nb = int(h[f"{key}nblocks"])
    assert len(recs) == nb
    for b in range(nb):
        r = int(h[f"{key}b{b}_rank"])
        if scheme == "aca":
            rows, cols = recs[b]
            assert np.array_equal(rows, h[f"{key}b{b}_rows"]), b
            assert np.array_equal(cols, h[f"{key}b{b}_cols"]), b
            U, V = fact.block_factor(b)
            assert np.array_equal(U, h[f"{key}b{b}_U"]), b
            assert np.array_equal(V, h[f"{key}b{b}_V"]), b
        else:
            rows, cols = recs[b]
            assert rows.size == r, b
            if r:
                assert np.array_equal(rows, h[f"{key}b{b}_srows"]), b
                assert np.array_equal(cols, h[f"{key}b{b}_scols"]), b
    assert [e["max_rank"] for e in report.ranks_per_level] == list(h[f"{key}maxranks"])
    x = hk.solve(fact, fr[f"{front}_rhs"])
    want = h[f"{key}x"]
    assert np.linalg.norm(x - want) <= SOLVE_RTOL * np.linalg.norm(want)


@pytest.mark.parametrize("front", SMALL_FRONTS)
def test_gmres_small_fronts_vs_reference(front):
    fr = golden("fronts")
    g = golden("gmres_small")
    A = fr[f"{front}_front"]
    pat = hk.SparsePattern(fr[f"{front}_indptr"], fr[f"{front}_indices"])
    acc = hk.BlockAccessor.from_matrix(A, pattern=pat)
    fact, _ = hk.factorize(acc, hk.build_tree(A.shape[0], 32),
                           hk.CompressionConfig(scheme="bdlr", tol=1e-1, depth=1))
    rhs = fr[f"{front}_rhs"]
    cfg = hk.GmresConfig(tol=1e-10, max_iter=1000)
    dev = hk.gmres(hk.DenseOperator(acc), rhs, cfg, preconditioner=fact)
    assert abs(dev.iterations - int(g[f"{front}_its"])) <= 1
    assert dev.converged
    want = g[f"{front}_x"]
    assert np.linalg.norm(dev.x - want) <= SOLVE_RTOL * np.linalg.norm(want)
    # reference-style callables go through the same device Arnoldi kernel
    cb = hk.gmres(lambda v: A @ v, rhs, cfg, preconditioner=lambda r: hk.solve(fact, r))
    assert abs(cb.iterations - int(g[f"{front}_its"])) <= 1
    dia = hk.gmres(hk.DenseOperator(acc), rhs, cfg, preconditioner=hk.diagonal_preconditioner(acc))
    assert abs(dia.iterations - int(g[f"{front}_diag_its"])) <= 1


# ------------------------------------------------------------------ BASELINE fronts, oracle on the same bits
def _cfg_front(cfg):
    from paper_1403_5337_b200 import frontgen as fg
    if cfg == 0:
        return fg.layered_grid_front((32, 32, 32), 2, 16, device="cuda")
    if cfg == 3:
        kc = fg.cell_conductivity((32, 32, 32), 0)
        return fg.layered_grid_front((32, 32, 32), 2, 16, conductivity=kc, device="cuda")
    kc = fg.cell_conductivity((48, 48, 48), 1)
    return fg.layered_grid_front((48, 48, 48), 2, 24, conductivity=kc, device="cuda")


@pytest.mark.parametrize("cfgid,gname", [(0, "cfg0"), (3, "cfg3_front0")])
def test_baseline_aca_front_parity(cfgid, gname):
    g = golden(gname)
    A = _cfg_front(cfgid)
    assert np.abs(A[g["rows_sample_idx"]] - g["rows_sample"]).max() <= 1e-12 * np.abs(g["rows_sample"]).max()
    acc = hk.BlockAccessor.from_matrix(A)
    tree = hk.build_tree(A.shape[0], 64)
    cfg = hk.CompressionConfig(scheme="aca", tol=1e-6)
    fact, report, recs = factorize_traced(acc, tree, cfg)
    ofact = O.factorize(A, 64, "aca", 1e-6)
    internal = _internal(ofact.nodes)
    for k, s in enumerate(internal):
        for side in (0, 1):
            b = 2 * k + side
            rows, cols = recs[b]
            orow, ocol = _otrace(ofact.traces[s][side])
            # bit-exact against the oracle on identical bits ...
            assert np.array_equal(rows, orow) and np.array_equal(cols, ocol), b
            U, V = fact.block_factor(b)
            assert np.array_equal(U, ofact.factors[s][side][0]), b
            assert np.array_equal(V, ofact.factors[s][side][1]), b
            # ... and against the reference's own run on its own front
            assert np.array_equal(rows, g[f"b{b}_rows"]) and np.array_equal(cols, g[f"b{b}_cols"]), b
    assert [e["max_rank"] for e in report.ranks_per_level] == list(g["maxranks"])
    b0 = np.random.default_rng(0).standard_normal((A.shape[0], 1))[:, 0]
    x = hk.solve(fact, b0)
    xo = O.solve(ofact, b0)
    assert np.linalg.norm(x - xo) <= SOLVE_RTOL * np.linalg.norm(xo)
    # ||HODLR^{-1} A - I|| behaviour
    E = hk.solve(fact, A) - np.eye(A.shape[0])
    Eo = O.solve(ofact, A) - np.eye(A.shape[0])
    assert np.linalg.norm(E - Eo) <= SOLVE_RTOL * np.linalg.norm(Eo)
    tol = 1e-12 if cfgid == 0 else 1e-10
    res = hk.gmres(hk.DenseOperator(A), b0, hk.GmresConfig(tol=tol, max_iter=1000), preconditioner=fact)
    assert res.converged
    assert abs(res.iterations - int(g["gmres_its"])) <= 1
    ores = O.gmres(lambda v: A @ v, b0, tol, 1000, lambda r: O.solve(ofact, r))
    assert np.linalg.norm(res.x - ores["x"]) <= SOLVE_RTOL * np.linalg.norm(ores["x"])


def test_baseline_cfg1_bdlr_parity():
    g = golden("cfg1")
    from paper_1403_5337_b200 import frontgen as fg
    A = _cfg_front(1)
    assert np.abs(A[g["rows_sample_idx"]] - g["rows_sample"]).max() <= 1e-12 * np.abs(g["rows_sample"]).max()
    graph = fg.grid_graph(fg.GridSpec((48, 48, 48)), 2, 24)
    acc = hk.BlockAccessor.from_matrix(A, pattern=graph)
    tree = hk.build_tree(A.shape[0], 64)
    cfg = hk.CompressionConfig(scheme="bdlr", tol=1e-4, depth=3)
    fact, report, recs = factorize_traced(acc, tree, cfg)
    ofact = O.factorize(A, 64, "bdlr", 1e-4, 3, None, (graph.indptr, graph.indices))
    internal = _internal(ofact.nodes)
    for k, s in enumerate(internal):
        for side in (0, 1):
            b = 2 * k + side
            rows, cols = recs[b]
            info = ofact.skeletons[s][side]
            if info is None:
                assert rows.size == 0
                continue
            assert np.array_equal(rows, info["rows"]) and np.array_equal(cols, info["cols"]), b
            r = int(g[f"b{b}_rank"])
            assert rows.size == r
            if r:
                assert np.array_equal(rows, g[f"b{b}_srows"]) and np.array_equal(cols, g[f"b{b}_scols"])
    assert [e["max_rank"] for e in report.ranks_per_level] == list(g["maxranks"])
    b1 = np.random.default_rng(0).standard_normal((A.shape[0], 1))[:, 0]
    x = hk.solve(fact, b1)
    xo = O.solve(ofact, b1)
    assert np.linalg.norm(x - xo) <= SOLVE_RTOL * np.linalg.norm(xo)
    res = hk.gmres(hk.DenseOperator(A), b1, hk.GmresConfig(tol=1e-10), preconditioner=fact)
    assert res.converged and abs(res.iterations - int(g["gmres_its"])) <= 1


# ------------------------------------------------------------------ batching / determinism
def test_batched_fronts_bit_identical_to_single():
    from paper_1403_5337_b200 import frontgen as fg
    fronts = np.stack([fg.layered_grid_front((16, 16, 16), 2, 8,
                                             conductivity=fg.cell_conductivity((16, 16, 16), s))
                       for s in range(6)])
    n = fronts.shape[1]
    cfg = hk.CompressionConfig(scheme="aca", tol=1e-6)
    batch = HodlrBatch(n, 32, fronts.shape[0]).factorize(torch.from_numpy(fronts), cfg, trace=True)
    rhs = np.random.default_rng(5).standard_normal((fronts.shape[0], n))
    xb = batch.solve_(torch.from_numpy(rhs).cuda().contiguous()).cpu().numpy()
    for f in range(fronts.shape[0]):
        single, _ = hk.factorize(hk.BlockAccessor.from_matrix(fronts[f]), hk.build_tree(n, 32), cfg)
        xs = hk.solve(single, rhs[f])
        assert np.array_equal(xs, xb[f]), f
        assert np.array_equal(batch.ranks[f], single._ranks)
    # a second run gives identical bits
    xb2 = batch.factorize(torch.from_numpy(fronts), cfg).solve_(
        torch.from_numpy(rhs).cuda().contiguous()).cpu().numpy()
    assert np.array_equal(xb, xb2)


# ------------------------------------------------------------------ error contract
def test_error_contract():
    a = np.eye(8)
    a[2:4, 2:4] = 0.0
    with pytest.raises(hk.SingularLeafError):
        hk.factorize(hk.BlockAccessor.from_matrix(a), hk.build_tree(8, 2),
                     hk.CompressionConfig(scheme="svd", tol=1e-12))
    with pytest.raises(hk.SingularSchurError):
        hk.factorize(hk.BlockAccessor.from_matrix(np.ones((2, 2))), hk.build_tree(2, 1),
                     hk.CompressionConfig(scheme="svd", tol=1e-12))
    with pytest.raises(hk.SingularSchurError):
        hk.factorize(hk.BlockAccessor.from_matrix(np.ones((2, 2))), hk.build_tree(2, 1),
                     hk.CompressionConfig(scheme="aca", tol=1e-12))
    n = 10
    z = np.zeros((n, n))
    z[:, -1] = 1.0
    pat = hk.SparsePattern.from_edges(n, np.arange(n - 1), np.arange(1, n))
    blk = hk.BlockAccessor(z, pattern=pat).block(np.arange(5), np.arange(5, n))
    with pytest.raises(hk.DegenerateSkeletonError):
        hk.compress_bdlr(blk, hk.CompressionConfig(scheme="bdlr", tol=1e-2, depth=0))
    fact, _ = hk.factorize(hk.BlockAccessor.from_matrix(np.eye(16) * 3), hk.build_tree(16, 8),
                           hk.CompressionConfig(scheme="aca", tol=1e-6))
    with pytest.raises(hk.DimensionMismatchError):
        hk.solve(fact, np.ones(17))
    with pytest.raises(hk.DimensionMismatchError):
        hk.factorize(hk.BlockAccessor.from_matrix(np.eye(16)), hk.build_tree(15, 8),
                     hk.CompressionConfig(scheme="aca"))


@pytest.mark.parametrize("n,leaf,max_rank", [(1, 1, None), (2, 1, None), (3, 8, None), (17, 4, None),
                                              (65, 8, 1), (65, 8, 3), (100, 100, None),
                                              (129, 16, None), (257, 32, 5)])
def test_edge_shapes_vs_oracle(n, leaf, max_rank):
    """Ragged trees, a single leaf, n = 1, and rank caps: ranks equal to the oracle's,
    solves within 1e-10, on a perturbed kernel matrix (test_acceptance.py:66-71 style)."""
    from paper_1403_5337_b200 import frontgen as fg
    rng = np.random.default_rng(n * 7 + leaf)
    A = fg.kernel_matrix(n, "exp-decay", shift=2.0) + 1e-3 * rng.standard_normal((n, n))
    cfg = hk.CompressionConfig(scheme="aca", tol=1e-8, max_rank=max_rank)
    fact, report = hk.factorize(hk.BlockAccessor.from_matrix(A), hk.build_tree(n, leaf), cfg)
    ofact = O.factorize(A, leaf, "aca", 1e-8, 1, max_rank)
    assert [e["max_rank"] for e in report.ranks_per_level] == \
        [e["max_rank"] for e in O.ranks_per_level(ofact)]
    b = rng.standard_normal(n)
    x = hk.solve(fact, b)
    xo = O.solve(ofact, b)
    assert np.linalg.norm(x - xo) <= SOLVE_RTOL * max(np.linalg.norm(xo), 1e-300)
    B = rng.standard_normal((n, 3))
    X = hk.solve(fact, B)
    assert X.shape == (n, 3)
    assert np.linalg.norm(X - O.solve(ofact, B)) <= SOLVE_RTOL * np.linalg.norm(O.solve(ofact, B))


# ------------------------------------------------------------------ BASELINE config 4 (n = 9216)
# The reference's own numbers on this front, measured in this container by running it
# (SURVEY.md §6.3): max rank per level 227,227,227,195,193,98,53; GMRES to 1e-10 on
# default_rng(3).standard_normal((9216, 4)) takes 10, 11, 11, 10 iterations.
CFG4_RANKS = [227, 227, 227, 195, 193, 98, 53]
CFG4_ITERS = [10, 11, 11, 10]


def test_config4_large_front():
    from paper_1403_5337_b200.frontgen import layered_grid_front
    front = layered_grid_front((96, 96, 96), "z", 48, device="cuda", return_torch=True).contiguous()
    n = front.shape[0]
    assert n == 9216
    cfg = hk.CompressionConfig(scheme="aca", tol=1e-4)
    batch = HodlrBatch(n, 72, 1).factorize(front[None], cfg)
    rep = batch.report(0)
    assert [lv["max_rank"] for lv in rep.ranks_per_level] == CFG4_RANKS
    fact = batch.factorization(0)
    # the two root blocks (4608 x 4608, rank 227) bit-exact against the oracle's ACA
    A = front.cpu().numpy()
    h = n // 2
    for blk, (rs, cs) in enumerate(((slice(0, h), slice(h, n)), (slice(h, n), slice(0, h)))):
        U, V = fact.block_factor(blk)
        Uo, Vo = O.aca(A[rs, cs], 1e-4)
        assert np.array_equal(U, Uo), blk
        assert np.array_equal(V, Vo), blk
    op = hk.DenseOperator(front)
    B = np.random.default_rng(3).standard_normal((n, 4))
    for j in range(4):
        res = hk.gmres(op, B[:, j], hk.GmresConfig(tol=1e-10), preconditioner=fact)
        assert res.converged
        assert abs(res.iterations - CFG4_ITERS[j]) <= 1, (j, res.iterations)
        assert res.true_residual <= 1e-9


# ------------------------------------------------------------------ subtree sharding (§8(e), config 4 path)
@pytest.mark.parametrize("G", [2, 4])
def test_subtree_sharded_matches_single_gpu(G):
    """ShardedHodlr over G emulated ranks on one device (GpuBackend: the rank's
    subtree plan with hk_factor_ext, hk_aca_block for the shared top blocks,
    hk_dgemm / hk_lu_partial for the top-level coupling terms) against the
    single-plan factorization of the same front: the top-level blocks are the
    same bit-exact ACA factors, only partial-sum order differs."""
    from paper_1403_5337_b200 import subtree as ST
    from paper_1403_5337_b200.frontgen import cell_conductivity, layered_grid_front
    dims = (32, 32, 32)
    front = layered_grid_front(dims, "z", 16, conductivity=cell_conductivity(dims, 0), device="cuda",
                               return_torch=True).contiguous()
    n = front.shape[0]
    cfg = hk.CompressionConfig(scheme="aca", tol=1e-6)
    single = HodlrBatch(n, 64, 1).factorize(front[None], cfg)
    fact = single.factorization(0)
    sh = ST.ShardedHodlr(front, 64, ST.EmulatedRanks(G))
    sh.factorize(cfg)
    b = torch.from_numpy(np.random.default_rng(11).standard_normal(n)).cuda()
    x_sh = sh.solve(b)
    x_1 = hk.solve(fact, b.cpu().numpy())
    rel = np.linalg.norm(x_sh.cpu().numpy() - x_1) / np.linalg.norm(x_1)
    assert rel < SOLVE_RTOL, rel
    assert torch.allclose(sh.apply(b), front @ b, rtol=1e-13, atol=1e-12)
    res_sh = sh.gmres(b, hk.GmresConfig(tol=1e-10))
    res_1 = hk.gmres(hk.DenseOperator(front), b.cpu().numpy(), hk.GmresConfig(tol=1e-10),
                     preconditioner=fact)
    assert res_sh.converged and res_1.converged
    assert abs(res_sh.iterations - res_1.iterations) <= 1
    assert np.linalg.norm(res_sh.x - res_1.x) / np.linalg.norm(res_1.x) < 1e-9
    # 3 right-hand sides in lock step (one sharded GEMV + solve per iteration)
    B = np.random.default_rng(12).standard_normal((n, 3))
    bat_sh = sh.gmres_batch(torch.from_numpy(B).cuda(), hk.GmresConfig(tol=1e-10))
    bat_1 = hk.gmres_batch(hk.DenseOperator(front), B, hk.GmresConfig(tol=1e-10), preconditioner=fact)
    for c in range(3):
        assert bat_sh[c].converged and abs(bat_sh[c].iterations - bat_1[c].iterations) <= 1
        assert np.linalg.norm(bat_sh[c].x - bat_1[c].x) / np.linalg.norm(bat_1[c].x) < 1e-9
    Xs = sh.solve_batch(torch.from_numpy(B.T.copy()).cuda()).cpu().numpy()
    X1 = hk.solve(fact, B).T
    assert np.linalg.norm(Xs - X1) / np.linalg.norm(X1) < SOLVE_RTOL


def test_gmres_batch_matches_single_rhs_runs():
    """hk_gmres_batch advances s systems together; each column's iterations,
    flags and iterates equal the single-rhs gmres() on that column."""
    from paper_1403_5337_b200.frontgen import cell_conductivity, layered_grid_front
    dims = (24, 24, 24)
    front = layered_grid_front(dims, "z", 12, conductivity=cell_conductivity(dims, 2))
    n = front.shape[0]
    fact, _ = hk.factorize(hk.BlockAccessor.from_matrix(front), hk.build_tree(n, 32),
                           hk.CompressionConfig(scheme="aca", tol=1e-4))
    op = hk.DenseOperator(front)
    B = np.random.default_rng(9).standard_normal((n, 4))
    cfg = hk.GmresConfig(tol=1e-10)
    batch = hk.gmres_batch(op, B, cfg, preconditioner=fact)
    for c in range(4):
        single = hk.gmres(op, B[:, c], cfg, preconditioner=fact)
        assert batch[c].iterations == single.iterations, c
        assert batch[c].converged == single.converged
        assert np.array_equal(batch[c].x, single.x), c
        assert batch[c].residual_history == single.residual_history
