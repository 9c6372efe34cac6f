"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only; these make the oracle trustworthy
as the checker of the GPU path."""

import numpy as np
import pytest

from conftest import SMALL_FRONTS, golden
from oracle import hodlr_oracle as O


def _trace_arrays(tr):
    rows = np.array([v for k, v in tr if k == "r"], dtype=np.int64)
    cols = np.array([v for k, v in tr if k == "c"], dtype=np.int64)
    return rows, cols


def test_aca_blocks_bit_exact():
    g = golden("aca_blocks")
    for name in g["names"]:
        name = str(name)
        mr = int(g[f"{name}_maxrank"]) or None
        tr = []
        u, v = O.aca(g[f"{name}_A"], float(g[f"{name}_tol"]), mr, trace=tr)
        rows, cols = _trace_arrays(tr)
        assert np.array_equal(rows, g[f"{name}_rows"]), name
        assert np.array_equal(cols, g[f"{name}_cols"]), name
        assert np.array_equal(u, g[f"{name}_U"]), name
        assert np.array_equal(v, g[f"{name}_V"]), name


def test_complete_pivot_lu_bit_exact():
    g = golden("lu_full")
    for name in g["names"]:
        name = str(name)
        lu, rp, cp, piv = O.complete_pivot_lu(g[f"{name}_A"])
        assert np.array_equal(lu, g[f"{name}_lu"]), name
        assert np.array_equal(rp, g[f"{name}_rp"]), name
        assert np.array_equal(cp, g[f"{name}_cp"]), name
        assert np.array_equal(piv, g[f"{name}_piv"]), name


def test_known_full_pivot():
    # test_dense.py: first complete pivot of [[1,2],[3,4]] is 4
    _, rp, cp, piv = O.complete_pivot_lu(np.array([[1.0, 2.0], [3.0, 4.0]]))
    assert piv[0] == 4.0 and rp[0] == 1 and cp[0] == 1


def test_graph_distance_and_selection():
    g = golden("graph")
    t = 0
    while f"g{t}_n" in g:
        n = int(g[f"g{t}_n"])
        ip, ix = g[f"g{t}_indptr"], g[f"g{t}_indices"]
        rv, cv = g[f"g{t}_rv"], g[f"g{t}_cv"]
        assert np.array_equal(O.side_distances(ip, ix, rv, cv, n), g[f"g{t}_drow"])
        assert np.array_equal(O.side_distances(ip, ix, cv, rv, n), g[f"g{t}_dcol"])
        for depth in (0, 1, 3):
            sel = O.depth_selection(ip, ix, rv, cv, depth, n)
            want_r, want_c = g[f"g{t}_d{depth}_rs"], g[f"g{t}_d{depth}_cs"]
            if sel is None:
                assert want_r.size == 1 and want_r[0] == -1
            else:
                assert np.array_equal(sel[0], want_r) and np.array_equal(sel[1], want_c)
        t += 1
    assert t >= 10


def _internal(nodes):
    return [s for s, nd in enumerate(nodes) if nd[3] >= 0]


@pytest.mark.parametrize("front", SMALL_FRONTS)
@pytest.mark.parametrize("cname,scheme,tol,depth", [("aca6", "aca", 1e-6, 1), ("aca3", "aca", 1e-3, 1),
                                                     ("bdlr1", "bdlr", 1e-1, 1),
                                                     ("bdlr3", "bdlr", 1e-3, 3)])
def test_hodlr_small_fronts(front, cname, scheme, tol, depth):
    fr = golden("fronts")
    h = golden("hodlr_small")
    key = f"{front}_{cname}_"
    A = fr[f"{front}_front"]
    graph = (fr[f"{front}_indptr"], fr[f"{front}_indices"])
    fact = O.factorize(A, int(h[f"{key}leaf"]), scheme, tol, depth, None, graph)
    internal = _internal(fact.nodes)
    assert 2 * len(internal) == int(h[f"{key}nblocks"])
    for k, s in enumerate(internal):
        for side in (0, 1):
            b = 2 * k + side
            uv = fact.factors[s][side]
            assert uv[0].shape[1] == int(h[f"{key}b{b}_rank"])
            if scheme == "aca":
                rows, cols = _trace_arrays(fact.traces[s][side])
                assert np.array_equal(rows, h[f"{key}b{b}_rows"])
                assert np.array_equal(cols, h[f"{key}b{b}_cols"])
                assert np.array_equal(uv[0], h[f"{key}b{b}_U"])
                assert np.array_equal(uv[1], h[f"{key}b{b}_V"])
            else:
                info = fact.skeletons[s][side]
                r = int(h[f"{key}b{b}_rank"])
                if r:
                    assert np.array_equal(info["rows"], h[f"{key}b{b}_srows"])
                    assert np.array_equal(info["cols"], h[f"{key}b{b}_scols"])
    x = O.solve(fact, fr[f"{front}_rhs"])
    want = h[f"{key}x"]
    assert np.linalg.norm(x - want) <= 1e-12 * np.linalg.norm(want)
    ml = [e["max_rank"] for e in O.ranks_per_level(fact)]
    assert ml == list(h[f"{key}maxranks"])


@pytest.mark.parametrize("front", SMALL_FRONTS)
def test_gmres_small_fronts(front):
    fr = golden("fronts")
    g = golden("gmres_small")
    A = fr[f"{front}_front"]
    graph = (fr[f"{front}_indptr"], fr[f"{front}_indices"])
    fact = O.factorize(A, 32, "bdlr", 1e-1, 1, None, graph)
    rhs = fr[f"{front}_rhs"]
    res = O.gmres(lambda v: A @ v, rhs, 1e-10, 1000, lambda r: O.solve(fact, r))
    assert res["iterations"] == int(g[f"{front}_its"])
    assert np.linalg.norm(res["x"] - g[f"{front}_x"]) <= 1e-10 * np.linalg.norm(g[f"{front}_x"])
    dia = O.gmres(lambda v: A @ v, rhs, 1e-10, 1000, O.diagonal_scaling(A))
    assert dia["iterations"] == int(g[f"{front}_diag_its"])
    # criterion 5: the HODLR preconditioner halves the iteration count
    assert res["iterations"] < 0.5 * dia["iterations"]


def test_cfg0_traces_on_generated_front():
    """BASELINE config 0: the oracle on this package's generated 32^3 front
    reproduces the reference's pivot traces and ranks recorded on the
    reference's own front."""
    from paper_1403_5337_b200 import frontgen
    g = golden("cfg0")
    A = frontgen.layered_grid_front((32, 32, 32), 2, 16)
    rows_idx = g["rows_sample_idx"]
    assert np.abs(A[rows_idx] - g["rows_sample"]).max() <= 1e-13 * np.abs(g["rows_sample"]).max()
    fact = O.factorize(A, 64, "aca", 1e-6)
    internal = _internal(fact.nodes)
    for k, s in enumerate(internal):
        for side in (0, 1):
            rows, cols = _trace_arrays(fact.traces[s][side])
            assert np.array_equal(rows, g[f"b{2 * k + side}_rows"])
            assert np.array_equal(cols, g[f"b{2 * k + side}_cols"])
    assert [e["max_rank"] for e in O.ranks_per_level(fact)] == list(g["maxranks"])
