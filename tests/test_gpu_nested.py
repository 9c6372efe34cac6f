"""Forward/back substitution across the one-level elimination tree of a grid
(nested.PlaneNestedSolver): the whole grid problem solved
through its separator front, against a sparse direct solve of the same
operator and through the residual of the block-tridiagonal operator."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_1403_5337_b200 as hk  # noqa: E402
from paper_1403_5337_b200 import frontgen as fg  # noqa: E402
from paper_1403_5337_b200.nested import PlaneNestedSolver  # noqa: E402


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _sparse_operator(solver):
    """The full operator assembled from the plane blocks (scipy CSR)."""
    import scipy.sparse as sp
    op = solver.op
    ext, nl = solver.ext, solver.nl
    blocks = [[None] * ext for _ in range(ext)]
    for t in range(ext):
        blocks[t][t] = sp.csr_matrix(op.layer_matrix(t)[0].cpu().numpy())
        if t > 0:
            c = op.coupling(t)[0].cpu().numpy()
            blocks[t][t - 1] = sp.diags(-c)
            blocks[t - 1][t] = sp.diags(-c)
    return sp.bmat(blocks, format="csr")


@pytest.mark.parametrize("dims,plane,seed", [((10, 10, 10), 5, 1), ((12, 12, 9), 4, 3)])
def test_nested_solve_matches_sparse_direct(dims, plane, seed):
    import scipy.sparse.linalg as spla
    kc = fg.cell_conductivity(dims, seed)
    s = PlaneNestedSolver(dims, 2, plane, conductivity=kc, leaf=16,
                          cfg=hk.CompressionConfig(scheme="aca", tol=1e-8))
    b = np.random.default_rng(seed).standard_normal((s.ext, s.nl))
    x, res = s.solve(b, hk.GmresConfig(tol=1e-13))
    assert res.converged
    L = _sparse_operator(s)
    xr = spla.spsolve(L.tocsc(), b.ravel()).reshape(b.shape)
    assert np.linalg.norm(x - xr) <= 1e-10 * np.linalg.norm(xr)
    # the front the solver factors is the generator's front, bit for bit
    F = fg.layered_grid_front(dims, 2, plane, conductivity=kc, device="cuda", return_torch=True)
    assert torch.equal(F, s.front)


def test_nested_solve_constant_coefficients_vs_reference_operator():
    """Constant coefficients: the plane operator is the reference's grid
    operator (src/frontgen.py:90-123) reordered plane-major, and the nested
    solve matches a sparse direct solve of it."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    dims = (8, 8, 8)
    s = PlaneNestedSolver(dims, 2, 4, leaf=16, cfg=hk.CompressionConfig(scheme="aca", tol=1e-9))
    g = hk.grid_operator(hk.GridSpec(dims))
    n = g.n
    A = sp.csr_matrix((np.asarray(g.edge_values), np.asarray(g.indices), np.asarray(g.indptr)),
                      shape=(n, n)) + sp.diags(np.asarray(g.diagonal))
    # plane-major order along axis 2: plane t, then the (x, y) nodes row-major
    perm = np.arange(n).reshape(dims).transpose(2, 0, 1).ravel()
    Ap = A[perm][:, perm]
    assert abs(Ap - _sparse_operator(s)).max() == 0.0
    b = np.random.default_rng(0).standard_normal((s.ext, s.nl))
    x, res = s.solve(b, hk.GmresConfig(tol=1e-13))
    assert res.converged
    xr = spla.spsolve(Ap.tocsc(), b.ravel()).reshape(b.shape)
    assert np.linalg.norm(x - xr) <= 1e-10 * np.linalg.norm(xr)


def test_nested_solve_cfg3_front_residual():
    """Config 3's grid (32^3, variable k, seed 0): the whole-grid solve through
    the HODLR-preconditioned separator GMRES, checked by its residual."""
    dims = (32, 32, 32)
    s = PlaneNestedSolver(dims, 2, 16, conductivity=fg.cell_conductivity(dims, 0), leaf=64,
                          cfg=hk.CompressionConfig(scheme="aca", tol=1e-6))
    b = np.random.default_rng(0).standard_normal((s.ext, s.nl))
    x, res = s.solve(b, hk.GmresConfig(tol=1e-12))
    assert res.converged and res.iterations <= 6
    r = s.apply(x) - b
    assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(b)
