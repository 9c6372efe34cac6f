"""GPU tests of the public paths around the hot path, each against the oracle
or against the device path it must reproduce:

* the end-to-end host-streaming batch path behind bench.py's e2e headline
  (``HodlrBatch.run_host_stream``);
* the device-resident GMRES loop (one CUDA graph with a conditional WHILE
  node): Krylov-capacity growth past 64 vectors, zero columns, repeat calls,
  the diagonal preconditioner's own diagonal, shape errors;
* the raise/no-raise decision of near-singular coupling systems
  (src/hodlr.py:272-277);
* the factor views the reference's tests read (``leaf_lus[s].lu``,
  ``couplings[s].d_left/.d_right/.schur_lu``; pkg/tests/test_hodlr.py:158-196).
"""

import numpy as np
import pytest

from oracle import hodlr_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_1403_5337_b200 as hk  # noqa: E402
from paper_1403_5337_b200.hodlr import HodlrBatch  # noqa: E402

RTOL = 1e-10


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _cfg3_fronts(seeds, dims=(32, 32, 32)):
    from paper_1403_5337_b200 import frontgen as fg
    return torch.stack([fg.layered_grid_front(dims, 2, dims[2] // 2,
                                              conductivity=fg.cell_conductivity(dims, s),
                                              device="cuda", return_torch=True) for s in seeds])


# ------------------------------------------------------------------ e2e streaming path
def test_run_host_stream_bit_identical_to_device_path_and_oracle():
    """Three items through the two device buffers (item 1 unpinned, so both
    copy paths run): every output equals factorize() + solve_() on the same
    fronts bit for bit, and the oracle's solve within 1e-10."""
    B = 4
    fronts = _cfg3_fronts(range(3 * B))                       # n = 1024: every ACA size class
    n = fronts.shape[1]
    rhs = torch.from_numpy(np.random.default_rng(7).standard_normal((3 * B, n))).cuda()
    cfg = hk.CompressionConfig(scheme="aca", tol=1e-6)
    hf, hr = fronts.cpu(), rhs.cpu()
    items = []
    for i in range(3):
        f = hf[i * B:(i + 1) * B].contiguous()
        r = hr[i * B:(i + 1) * B].contiguous()
        out = torch.empty((B, n), dtype=torch.float64)
        if i != 1:
            f, r, out = f.pin_memory(), r.pin_memory(), out.pin_memory()
        items.append((f, r, out))
    batch = HodlrBatch(n, 64, B)
    batch.run_host_stream(items, cfg)
    for i in range(3):
        batch.factorize(fronts[i * B:(i + 1) * B], cfg)
        w = rhs[i * B:(i + 1) * B].clone()
        batch.solve_(w)
        assert torch.equal(items[i][2], w.cpu()), i
    for f in (0, 5, 11):                                      # oracle on one front per item
        A = hf[f].numpy()
        of = O.factorize(A, 64, "aca", 1e-6)
        xo = O.solve(of, hr[f].numpy())
        x = items[f // B][2][f % B].numpy()
        assert np.linalg.norm(x - xo) <= RTOL * np.linalg.norm(xo), f


def test_solve_batch_argument_validation():
    fronts = _cfg3_fronts([0, 1], dims=(12, 12, 12))
    n = fronts.shape[1]
    batch = HodlrBatch(n, 32, 2).factorize(fronts, hk.CompressionConfig(scheme="aca", tol=1e-6))
    with pytest.raises(hk.DimensionMismatchError):
        batch.solve_(torch.zeros((2, n + 1), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        batch.solve_(torch.zeros((2, n), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        batch.solve_(torch.zeros((n, 2), dtype=torch.float64, device="cuda").t())
    x = torch.ones((2, 3, n), dtype=torch.float64, device="cuda")
    batch.solve_(x)                                           # (batch, s, n) is accepted
    assert torch.isfinite(x).all()


# ------------------------------------------------------------------ device-resident GMRES
def test_gmres_device_loop_grows_krylov_capacity():
    """~250 iterations (the basis starts with room for 64 vectors): the loop
    stops at the capacity, the host grows the buffers and resumes.  Iterations
    within +-1 of the oracle, the same history to rounding, x within 1e-8."""
    n = 400
    rng = np.random.default_rng(3)
    A = np.eye(n) + 0.9 * rng.standard_normal((n, n)) / np.sqrt(n)
    b = rng.standard_normal(n)
    cfg = hk.GmresConfig(tol=1e-12, max_iter=n)
    res = hk.gmres(hk.DenseOperator(A), b, cfg)
    ores = O.gmres(lambda v: A @ v, b, 1e-12, n)
    assert ores["iterations"] > 128
    assert res.converged == ores["converged"]
    assert abs(res.iterations - ores["iterations"]) <= 1
    h, ho = np.array(res.residual_history), np.array(ores["history"])
    k = min(h.size, ho.size)
    assert np.all(np.abs(h[:k] - ho[:k]) <= 1e-6 * ho[:k] + 1e-15)
    assert np.linalg.norm(res.x - ores["x"]) <= 1e-8 * np.linalg.norm(ores["x"])
    # not converged within max_iter: iterations == max_iter exactly
    short = hk.gmres(hk.DenseOperator(A), b, hk.GmresConfig(tol=1e-12, max_iter=100))
    assert not short.converged and short.iterations == 100


def test_gmres_batch_zero_column_and_repeat_calls():
    fronts = _cfg3_fronts([3], dims=(16, 16, 16))
    A = fronts[0]
    n = A.shape[0]
    fact, _ = hk.factorize(hk.BlockAccessor.from_matrix(A.cpu().numpy()), hk.build_tree(n, 32),
                           hk.CompressionConfig(scheme="aca", tol=1e-4))
    op = hk.DenseOperator(A)
    B = np.random.default_rng(1).standard_normal((n, 3))
    B[:, 1] = 0.0
    cfg = hk.GmresConfig(tol=1e-10)
    r1 = hk.gmres_batch(op, B, cfg, preconditioner=fact)
    assert r1[1].converged and r1[1].iterations == 0 and not np.any(r1[1].x)
    r2 = hk.gmres_batch(op, B, cfg, preconditioner=fact)      # cached graph: same bits
    Ah = A.cpu().numpy()
    of = O.factorize(Ah, 32, "aca", 1e-4)
    for c in (0, 2):
        single = hk.gmres(op, B[:, c], cfg, preconditioner=fact)
        assert r1[c].iterations == single.iterations
        assert np.array_equal(r1[c].x, single.x) and np.array_equal(r2[c].x, r1[c].x)
        ores = O.gmres(lambda v: Ah @ v, B[:, c], 1e-10, 1000, lambda r: O.solve(of, r))
        assert abs(r1[c].iterations - ores["iterations"]) <= 1
        assert np.linalg.norm(r1[c].x - ores["x"]) <= RTOL * np.linalg.norm(ores["x"])


def test_diagonal_preconditioner_uses_its_own_diagonal():
    """The device path divides by the preconditioner's diagonal (krylov.py:58-62),
    not by the operator's: a preconditioner built from 2A + I gives the
    oracle's iterations and iterate for that preconditioner."""
    rng = np.random.default_rng(4)
    n = 96
    A = np.diag(np.linspace(1.0, 50.0, n)) + 0.05 * rng.standard_normal((n, n))
    P = 2.0 * A + np.eye(n)
    b = rng.standard_normal(n)
    pre = hk.diagonal_preconditioner(P)
    res = hk.gmres(hk.DenseOperator(A), b, hk.GmresConfig(tol=1e-10), preconditioner=pre)
    ores = O.gmres(lambda v: A @ v, b, 1e-10, 1000, O.diagonal_scaling(P))
    assert res.iterations == ores["iterations"]
    assert np.linalg.norm(res.x - ores["x"]) <= RTOL * np.linalg.norm(ores["x"])


def test_gmres_shape_errors():
    A = np.eye(64) * 3.0
    fact, _ = hk.factorize(hk.BlockAccessor.from_matrix(A), hk.build_tree(64, 16),
                           hk.CompressionConfig(scheme="aca", tol=1e-6))
    with pytest.raises(hk.DimensionMismatchError):           # solve() of a 64-front on 65 rows
        hk.gmres(hk.DenseOperator(np.eye(65)), np.ones(65), hk.GmresConfig(), preconditioner=fact)
    with pytest.raises(ValueError):                           # `dense @ v` with the wrong size
        hk.gmres(hk.DenseOperator(np.eye(65)), np.ones(64), hk.GmresConfig(), preconditioner=fact)
    with pytest.raises(ValueError):
        hk.gmres_batch(hk.DenseOperator(A), np.ones((64, 17)), hk.GmresConfig(), preconditioner=fact)


# ------------------------------------------------------------------ singular coupling systems
def _planted(y, x):
    """2x2 front with leaves of 1: S = [[1, x], [y, 1]] exactly (hodlr.py:269-271)."""
    return np.array([[1.0, x], [y, 1.0]])


_CASES = [
    ("ones", np.ones((2, 2))),                                # S exactly singular
    ("y3", _planted(3.0, 1.0 / 3.0)),                         # LU(S) pivot and I - YX both 0
    ("y49", _planted(49.0, 1.0 / 49.0)),                      # LU(S) pivot 0, I - YX = 5.6e-17
    ("y10", _planted(10.0, 1.0 / 10.0)),
    ("y7", _planted(7.0, 1.0 / 7.0)),
    ("subnormal", _planted(1e300, np.nextafter(1.0 / 1e300, 1.0))),   # LU(S) pivot 1.7e-316
    ("tiny_ok", _planted(0.5, 2.0 * (1.0 - 1e-12))),          # pivot 1e-12: regular
    ("neg", _planted(-4.0, np.nextafter(-0.25, 0.0))),
]


@pytest.mark.parametrize("name,A", _CASES, ids=[c[0] for c in _CASES])
@pytest.mark.parametrize("scheme", ["aca", "svd"])
def test_near_singular_coupling_decision_matches_oracle(name, A, scheme):
    """SingularSchurError is raised exactly when the reference's partial-pivot
    LU of S has a pivot below 1e-300 (hodlr.py:272-277, dense.py:76-77)."""
    try:
        O.factorize(A, 1, scheme, 1e-12)
        want = None
    except O.SingularSchur:
        want = "schur"
    except O.SingularLeaf:
        want = "leaf"
    tree = hk.build_tree(2, 1)
    got = None
    try:
        hk.factorize(hk.BlockAccessor.from_matrix(A), tree, hk.CompressionConfig(scheme=scheme, tol=1e-12))
    except hk.SingularSchurError:
        got = "schur"
    except hk.SingularLeafError:
        got = "leaf"
    assert got == want, (name, got, want)


def test_near_singular_coupling_inside_a_larger_tree():
    """A planted exactly-singular 2x2 coupling at a depth-2 node of an 8x8
    front raises; the same front with a regular coupling does not."""
    base = np.eye(8) * 4.0 + 0.01
    bad = base.copy()
    bad[0:2, 0:2] = _planted(49.0, 1.0 / 49.0)
    bad[0, 2:] = bad[1, 2:] = bad[2:, 0] = bad[2:, 1] = 0.0
    for A, raises in ((base, False), (bad, True)):
        try:
            O.factorize(A, 1, "aca", 1e-12)
            want = False
        except O.SingularSchur:
            want = True
        assert want == raises
        if raises:
            with pytest.raises(hk.SingularSchurError):
                hk.factorize(hk.BlockAccessor.from_matrix(A), hk.build_tree(8, 1),
                             hk.CompressionConfig(scheme="aca", tol=1e-12))
        else:
            hk.factorize(hk.BlockAccessor.from_matrix(A), hk.build_tree(8, 1),
                         hk.CompressionConfig(scheme="aca", tol=1e-12))


# ------------------------------------------------------------------ test-visible factor views
@pytest.mark.parametrize("scheme,tol,depth", [("aca", 1e-6, 1), ("bdlr", 1e-3, 2)])
def test_factor_views_match_oracle(scheme, tol, depth):
    """leaf_lus[s].lu / .piv and couplings[s].{v_upper, v_lower, d_left,
    d_right, schur_lu.lu, schur_lu.piv} against the oracle's (which keeps the
    reference's getrf outputs, hodlr.py:222-232, :264-277)."""
    from paper_1403_5337_b200 import frontgen as fg
    dims = (12, 12, 12)
    A = fg.layered_grid_front(dims, 2, 6, conductivity=fg.cell_conductivity(dims, 4))
    graph = fg.grid_graph(fg.GridSpec(dims), 2, 6)
    n = A.shape[0]
    fact, _ = hk.factorize(hk.BlockAccessor.from_matrix(A, pattern=graph), hk.build_tree(n, 24),
                           hk.CompressionConfig(scheme=scheme, tol=tol, depth=depth))
    of = O.factorize(A, 24, scheme, tol, depth, None, (graph.indptr, graph.indices))
    nleaf = ncpl = 0
    for slot, nd in enumerate(fact.tree.nodes):
        if nd.is_leaf:
            lu = fact.leaf_lus[slot]
            olu, opiv = of.leaf[slot]
            assert np.array_equal(np.asarray(lu.piv), opiv), slot
            assert np.linalg.norm(lu.lu - olu) <= 1e-12 * np.linalg.norm(olu), slot
            assert fact.couplings[slot] is None
            nleaf += 1
            continue
        c = fact.couplings[slot]
        oc = of.cpl[slot]
        assert fact.leaf_lus[slot] is None
        assert c.d_left.shape[1] == c.v_upper.shape[1] and c.d_right.shape[1] == c.v_lower.shape[1]
        assert c.schur_lu.n == c.rank_upper + c.rank_lower
        if scheme == "aca":                                   # bit-exact factors
            assert np.array_equal(c.v_upper, oc["v_up"]) and np.array_equal(c.v_lower, oc["v_low"])
        for mine, ref in ((c.d_left, oc["d_left"]), (c.d_right, oc["d_right"]), (c.schur_lu.lu, oc["lu"])):
            assert mine.shape == ref.shape
            assert np.linalg.norm(mine - ref) <= RTOL * max(np.linalg.norm(ref), 1e-300), slot
        assert np.array_equal(np.asarray(c.schur_lu.piv), oc["piv"]), slot
        ncpl += 1
    assert nleaf and ncpl
    # Coupling.correct on the host views reproduces the oracle's correction
    slot = fact.tree.internal_nodes()[-1]
    c, oc = fact.couplings[slot], of.cpl[slot]
    na, nb = c.d_left.shape[0], c.d_right.shape[0]
    rng = np.random.default_rng(0)
    top, bot = rng.standard_normal((na, 2)), rng.standard_normal((nb, 2))
    t1, b1 = c.correct(top, bot)
    t2, b2 = O._correct(oc, top, bot)
    assert np.linalg.norm(t1 - t2) <= RTOL * np.linalg.norm(t2)
    assert np.linalg.norm(b1 - b2) <= RTOL * np.linalg.norm(b2)
