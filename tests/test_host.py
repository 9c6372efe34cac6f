"""CPU tests of the host side: the C ABI loads and exports every declared
symbol, host-only native code (tree, graph selection) is bit-exact, configs
validate like the reference, and the compute path refuses to run without a
GPU (no CPU fallback)."""

import re

import numpy as np
import pytest

from conftest import ROOT, SMALL_FRONTS, golden
from oracle import hodlr_oracle as O
import paper_1403_5337_b200 as hk
from paper_1403_5337_b200 import _native as N


def declared_symbols():
    text = (ROOT / "include" / "hodlr_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = N.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(N.SIGNATURES), "ctypes table out of sync with the header"


def test_version_and_device_count():
    assert N.lib().hk_version().decode().startswith("hodlr_b200")
    assert N.device_count() >= 0


@pytest.mark.parametrize("n,leaf", [(1, 1), (8, 8), (8, 2), (7, 3), (97, 10), (100, 30),
                                    (1024, 64), (2304, 64), (9216, 72), (333, 17)])
def test_native_tree_matches_reference_rule(n, leaf):
    h = N.P()
    N.check(N.lib().hk_plan_create(n, leaf, 1, N.C.byref(h)))
    k = N.lib().hk_plan_num_nodes(h)
    lvl = np.zeros(k, np.int32)
    lo = np.zeros(k, np.int64)
    hi = np.zeros(k, np.int64)
    le = np.zeros(k, np.int32)
    ri = np.zeros(k, np.int32)
    N.check(N.lib().hk_plan_tree(h, N.arr_ptr(lvl, N.I32), N.arr_ptr(lo, N.I64), N.arr_ptr(hi, N.I64),
                                 N.arr_ptr(le, N.I32), N.arr_ptr(ri, N.I32)))
    N.lib().hk_plan_destroy(h)
    native = [(int(a), int(b), int(c), int(d), int(e)) for a, b, c, d, e in zip(lvl, lo, hi, le, ri)]
    oracle = [tuple(x) for x in O.bisection_tree(n, leaf)]
    py = [(t.level, t.lo, t.hi, t.left, t.right) for t in hk.build_tree(n, leaf).nodes]
    assert native == oracle == py


def test_tree_shapes_like_reference_tests():
    tree = hk.build_tree(100, 30)
    root = tree.nodes[0]
    assert (tree.nodes[root.left].size, tree.nodes[root.right].size) == (50, 50)
    t7 = hk.build_tree(7, 3)
    assert t7.nodes[t7.nodes[0].left].size == 4
    assert hk.build_tree(9216, 72).depth == 7
    assert sum(nd.is_leaf for nd in hk.build_tree(9216, 72).nodes) == 128
    with pytest.raises(ValueError):
        hk.build_tree(0, 4)
    with pytest.raises(ValueError):
        hk.build_tree(4, 0)


def test_native_graph_selection_matches_golden():
    g = golden("graph")
    t = 0
    while f"g{t}_n" in g:
        n = int(g[f"g{t}_n"])
        pat = hk.SparsePattern(g[f"g{t}_indptr"], g[f"g{t}_indices"])
        view = hk.BlockGraphView(pat, g[f"g{t}_rv"], g[f"g{t}_cv"])
        assert np.array_equal(hk.distance_index(view, "row"), g[f"g{t}_drow"])
        assert np.array_equal(hk.distance_index(view, "col"), g[f"g{t}_dcol"])
        for depth in (0, 1, 3):
            want_r = g[f"g{t}_d{depth}_rs"]
            if want_r.size == 1 and want_r[0] == -1:
                with pytest.raises(hk.EmptySelectionError):
                    hk.select_by_depth(view, depth)
            else:
                rs, cs = hk.select_by_depth(view, depth)
                assert np.array_equal(rs, want_r)
                assert np.array_equal(cs, g[f"g{t}_d{depth}_cs"])
        t += 1
        del n


def test_graph_small_known_answers():
    # path 0-1-2-3-4 split [0,1,2] | [3,4]  (test_graph.py style)
    pat = hk.SparsePattern.from_edges(5, [0, 1, 2, 3], [1, 2, 3, 4])
    view = hk.BlockGraphView(pat, [0, 1, 2], [3, 4])
    assert list(hk.boundary_vertices(view, "row")) == [2]
    assert list(hk.distance_index(view, "row")) == [2.0, 1.0, 0.0]
    rs, cs = hk.select_by_depth(view, 1)
    assert list(rs) == [2, 1] and list(cs) == [0, 1]
    disc = hk.SparsePattern.from_edges(4, [0, 2], [1, 3])
    with pytest.raises(hk.EmptySelectionError):
        hk.select_by_depth(hk.BlockGraphView(disc, [0, 1], [2, 3]), 2)
    with pytest.raises(ValueError):
        hk.BlockGraphView(pat, [0, 1], [1, 2])


def test_sparse_pattern_from_edges_semantics():
    p = hk.SparsePattern.from_edges(4, [0, 1, 1, 2, 3], [1, 0, 1, 3, 2], [5.0, 5.0, 7.0, 2.0, 2.0])
    assert list(p.indptr) == [0, 1, 2, 3, 4]
    assert list(p.indices) == [1, 0, 3, 2]
    assert list(p.edge_values) == [5.0, 5.0, 2.0, 2.0]
    assert p.diagonal[1] == 7.0
    with pytest.raises(ValueError):
        hk.SparsePattern.from_edges(3, [0, 1], [1, 0], [1.0, 2.0])
    with pytest.raises(ValueError):
        hk.SparsePattern.from_edges(3, [0], [3])


@pytest.mark.parametrize("front", SMALL_FRONTS)
def test_generated_fronts_match_reference_fronts(front):
    """frontgen (layered elimination) vs the reference's dense grid_front."""
    cases = {"3d-9": ((9, 9, 9), 0, 4, "laplacian"), "2d-100": ((100, 21), 1, 10, "laplacian"),
             "3d-12": ((12, 12, 12), 0, 6, "laplacian"),
             "3d-vec-7": ((7, 7, 7), 0, 3, "vector-laplacian"),
             "3d-15": ((15, 15, 15), 2, 7, "laplacian"), "3d-16": ((16, 16, 16), 0, 8, "laplacian")}
    dims, axis, plane, stencil = cases[front]
    fr = golden("fronts")
    p = hk.grid_front(hk.GridSpec(dims, stencil=stencil), axis, plane)
    want = fr[f"{front}_front"]
    assert np.abs(p.front - want).max() <= 1e-14 * np.abs(want).max()
    assert np.array_equal(p.graph.indptr, fr[f"{front}_indptr"])
    assert np.array_equal(p.graph.indices, fr[f"{front}_indices"])
    assert np.array_equal(p.rhs[:, 0], fr[f"{front}_rhs"])


def test_variable_coefficient_generator_reduces_to_constant():
    a = hk.layered_grid_front((9, 9, 9), 0, 4)
    b = hk.layered_grid_front((9, 9, 9), 0, 4, conductivity=np.ones((10, 10, 10)))
    assert np.abs(a - b).max() <= 1e-14
    # the schur_front path on the same operator agrees too
    spec = hk.GridSpec((5, 5, 5))
    op = hk.grid_operator(spec)
    sep, left, right = hk.planar_separator(spec, 2, 2)
    c = hk.schur_front(op, sep, left, right).front
    d = hk.layered_grid_front((5, 5, 5), 2, 2)
    assert np.abs(c - d).max() <= 1e-14


def test_config_validation():
    with pytest.raises(ValueError):
        hk.CompressionConfig(scheme="nope")
    with pytest.raises(ValueError):
        hk.CompressionConfig(tol=1.0)
    with pytest.raises(ValueError):
        hk.CompressionConfig(depth=-1)
    with pytest.raises(ValueError):
        hk.CompressionConfig(max_rank=0)
    assert hk.CompressionConfig(max_rank=5).rank_cap(10, 20) == 5
    with pytest.raises(ValueError):
        hk.GmresConfig(tol=0.0)
    with pytest.raises(ValueError):
        hk.GmresConfig(max_iter=0)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    acc = hk.BlockAccessor.from_matrix(np.eye(8))
    with pytest.raises(RuntimeError, match="CUDA"):
        hk.factorize(acc, hk.build_tree(8, 4), hk.CompressionConfig(scheme="aca"))
    with pytest.raises(RuntimeError, match="CUDA"):
        hk.lu_full(np.eye(3))


def test_aca_kernels_keep_their_sweep_results_in_registers():
    """The ACA sweeps return their results by value.  With reference out-parameters
    every call went through the thread's stack, and those local-memory stores were
    85% of the kernel's L2 write sectors (profiles/r02_aca_experiments.md §5): a
    regression shows up as hundreds of STL instructions in the aca kernels' SASS."""
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not shutil.which(cuobjdump):
        pytest.skip("cuobjdump not available")
    if not N.LIB_PATH.exists():
        pytest.skip("library not built")
    sass = subprocess.run([cuobjdump, "-sass", str(N.LIB_PATH)], capture_output=True, text=True,
                          check=True).stdout
    stl, fn = {}, None
    for line in sass.splitlines():
        if "Function :" in line:
            fn = line.split("Function :")[1].strip()
            stl.setdefault(fn, 0)
        elif fn and " STL" in line:
            stl[fn] += 1
    aca = {k: v for k, v in stl.items() if "aca_kernel" in k or "aca_cluster_kernel" in k}
    assert len(aca) >= 5, sorted(stl)
    assert max(aca.values()) <= 16, aca
