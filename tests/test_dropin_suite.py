"""The reference's own test suite, restated against this package imported
under the reference's name (``import paper_1403_5337_b200 as hodlrkit``).

Every test below restates one test of /root/reference/pkg/tests (cited as
file:line) with the same inputs, the same property and the same tolerance,
so a user switching packages keeps the guarantees the reference's suite
gives.  The reference suite itself cannot run here: it imports the
off-path CLI / Matrix Market / report modules and, on the GPU box, the
reference tree is absent.  Graph selection and tree
construction are host integer code and run without a GPU; everything else
computes on the device (``-m gpu``).
"""

import functools

import numpy as np
import pytest

import paper_1403_5337_b200 as hodlrkit
from paper_1403_5337_b200.graph import BlockGraphView

torch = pytest.importorskip("torch")
gpu = pytest.mark.gpu


def _has_gpu():
    return torch.cuda.is_available()


@pytest.fixture
def need_gpu():
    if not _has_gpu():
        pytest.skip("needs a CUDA device")


@functools.lru_cache(maxsize=None)
def front_of(dims, axis, plane):
    """pkg/tests/conftest.py:9-12 (fronts are deterministic: share them)."""
    return hodlrkit.grid_front(hodlrkit.GridSpec(dims), axis, plane)


def low_rank(rng, m, n, r):
    return rng.standard_normal((m, r)) @ rng.standard_normal((r, n))


# =================================================================== test_hodlr.py
class TestTree:
    def test_single_leaf(self):                                   # test_hodlr.py:24-27
        t = hodlrkit.build_tree(8, 8)
        assert len(t.nodes) == 1 and t.nodes[0].is_leaf

    def test_power_of_two(self):                                  # :30-35
        t = hodlrkit.build_tree(8, 2)
        assert len(t.nodes) == 7 and t.depth == 2
        assert {nd.size for nd in t.nodes if nd.is_leaf} == {2}

    def test_halving(self):                                       # :38-44
        t = hodlrkit.build_tree(100, 30)
        left, right = t.nodes[t.nodes[0].left], t.nodes[t.nodes[0].right]
        assert (left.size, right.size) == (50, 50)
        assert max(nd.size for nd in t.nodes if nd.is_leaf) <= 30
        assert t.nodes[left.left].size == t.nodes[left.right].size == 25

    def test_odd_split_smaller_child_last(self):                  # :47-51
        t = hodlrkit.build_tree(7, 3)
        assert (t.nodes[t.nodes[0].left].size, t.nodes[t.nodes[0].right].size) == (4, 3)

    def test_contiguous_partition(self):                          # :54-62
        t = hodlrkit.build_tree(97, 10)
        for nd in t.nodes:
            if not nd.is_leaf:
                a, b = t.nodes[nd.left], t.nodes[nd.right]
                assert a.lo == nd.lo and b.hi == nd.hi and a.hi == b.lo
                assert abs(a.size - b.size) <= 1


@gpu
@pytest.mark.usefixtures("need_gpu")
class TestHodlr:
    def test_block_diagonal_rank_zero(self, rng):                 # :65-77
        blocks = [rng.standard_normal((16, 16)) + 16 * np.eye(16) for _ in range(4)]
        a = np.zeros((64, 64))
        for k, blk in enumerate(blocks):
            a[16 * k:16 * k + 16, 16 * k:16 * k + 16] = blk
        fact, rep = hodlrkit.factorize(hodlrkit.BlockAccessor.from_matrix(a), hodlrkit.build_tree(64, 16),
                                       hodlrkit.CompressionConfig(scheme="svd", tol=1e-10))
        assert all(e["max_rank"] == 0 for e in rep.ranks_per_level)
        b = rng.standard_normal((64, 2))
        want = np.vstack([np.linalg.solve(blk, b[16 * k:16 * k + 16]) for k, blk in enumerate(blocks)])
        assert np.linalg.norm(hodlrkit.solve(fact, b) - want) <= 1e-12 * np.linalg.norm(want)

    def test_shifted_kernel_residual(self, rng):                  # :80-87
        a = np.eye(64) + 0.1 * hodlrkit.kernel_matrix(64, "inv-distance")
        acc = hodlrkit.BlockAccessor.from_matrix(a)
        fact, _ = hodlrkit.factorize(acc, hodlrkit.build_tree(64, 16),
                                     hodlrkit.CompressionConfig(scheme="svd", tol=1e-12))
        b = rng.standard_normal((64, 1))
        assert hodlrkit.residual_norm(acc, hodlrkit.solve(fact, b), b) <= 1e-10

    def test_bdlr_regimes(self):                                  # :90-97
        prob = front_of((12, 12, 12), 0, 6)
        tree = hodlrkit.build_tree(prob.n, 32)
        for tol, depth in ((1e-1, 1), (1e-3, 3), (1e-5, 5)):
            fact, _ = hodlrkit.factorize(prob.accessor(), tree,
                                         hodlrkit.CompressionConfig(scheme="bdlr", tol=tol, depth=depth))
            assert np.isfinite(hodlrkit.solve(fact, prob.rhs)).all()

    def test_identity(self, rng):                                 # :100-104
        fact, _ = hodlrkit.factorize(hodlrkit.BlockAccessor.from_matrix(np.eye(40)),
                                     hodlrkit.build_tree(40, 8),
                                     hodlrkit.CompressionConfig(scheme="svd", tol=1e-10))
        b = rng.standard_normal((40, 3))
        assert np.abs(hodlrkit.solve(fact, b) - b).max() <= 1e-13

    def test_matches_dense_lu(self, rng):                         # :107-114
        acc = hodlrkit.BlockAccessor.from_matrix(hodlrkit.kernel_matrix(256, "inv-distance", shift=5.0))
        fact, _ = hodlrkit.factorize(acc, hodlrkit.build_tree(256, 64),
                                     hodlrkit.CompressionConfig(scheme="svd", tol=1e-12))
        b = rng.standard_normal((256, 2))
        want = np.linalg.solve(acc.materialize(), b)
        assert np.linalg.norm(hodlrkit.solve(fact, b) - want) <= 1e-9 * np.linalg.norm(want)

    def test_vector_and_matrix_rhs(self, rng):                    # :117-123
        acc = hodlrkit.BlockAccessor.from_matrix(hodlrkit.kernel_matrix(48, "inv-distance", shift=5.0))
        fact, _ = hodlrkit.factorize(acc, hodlrkit.build_tree(48, 16),
                                     hodlrkit.CompressionConfig(scheme="svd", tol=1e-13))
        b = rng.standard_normal(48)
        assert hodlrkit.solve(fact, b).shape == (48,)
        assert hodlrkit.solve(fact, b[:, None]).shape == (48, 1)

    def test_dimension_mismatch(self, rng):                       # :126-130
        acc = hodlrkit.BlockAccessor.from_matrix(hodlrkit.kernel_matrix(16, "inv-distance", shift=5.0))
        fact, _ = hodlrkit.factorize(acc, hodlrkit.build_tree(16, 8),
                                     hodlrkit.CompressionConfig(scheme="svd", tol=1e-13))
        with pytest.raises(hodlrkit.DimensionMismatchError):
            hodlrkit.solve(fact, rng.standard_normal(17))

    def test_exact_compression_equivalence(self, rng):           # :133-143
        for n in (96, 200, 512):
            a = hodlrkit.kernel_matrix(n, "exp-decay", shift=3.0)
            e = rng.standard_normal((n, n))
            a = a + 0.01 * (e + e.T) + 0.05 * n * np.eye(n)
            fact, _ = hodlrkit.factorize(hodlrkit.BlockAccessor.from_matrix(a), hodlrkit.build_tree(n, 64),
                                         hodlrkit.CompressionConfig(scheme="svd", tol=1e-14))
            b = rng.standard_normal(n)
            want = np.linalg.solve(a, b)
            assert np.linalg.norm(hodlrkit.solve(fact, b) - want) <= 1e-9 * np.linalg.norm(want), n

    def test_report_residual(self):                               # :146-155
        prob = front_of((9, 9, 9), 0, 4)
        acc = prob.accessor()
        fact, rep = hodlrkit.factorize(acc, hodlrkit.build_tree(prob.n, 16),
                                       hodlrkit.CompressionConfig(scheme="bdlr", tol=1e-3, depth=3))
        x = hodlrkit.solve(fact, prob.rhs)
        rep.residual = hodlrkit.residual_norm(acc, x, prob.rhs)
        want = np.linalg.norm(prob.front @ x - prob.rhs) / np.linalg.norm(prob.rhs)
        assert abs(rep.residual - want) <= 1e-13

    def test_d_block_shapes(self):                                # :158-166
        prob = front_of((100, 21), 1, 10)
        fact, _ = hodlrkit.factorize(prob.accessor(), hodlrkit.build_tree(prob.n, 16),
                                     hodlrkit.CompressionConfig(scheme="svd", tol=1e-8))
        for slot in fact.tree.internal_nodes():
            c = fact.couplings[slot]
            assert c.d_left.shape[1] == c.v_upper.shape[1]
            assert c.d_right.shape[1] == c.v_lower.shape[1]
            assert c.schur_lu.n == c.rank_upper + c.rank_lower

    def test_rank_decay(self):                                    # :169-176
        prob = front_of((16, 16, 16), 0, 8)
        _, rep = hodlrkit.factorize(prob.accessor(), hodlrkit.build_tree(prob.n, 16),
                                    hodlrkit.CompressionConfig(scheme="svd", tol=1e-6))
        mx = [e["max_rank"] for e in sorted(rep.ranks_per_level, key=lambda e: e["level"])]
        pairs = list(zip(mx, mx[1:]))
        assert sum(a >= b for a, b in pairs) >= 0.8 * len(pairs)

    def test_threads_bit_identical(self):                         # :179-196
        prob = front_of((100, 21), 1, 10)
        tree = hodlrkit.build_tree(prob.n, 16)
        cfg = hodlrkit.CompressionConfig(scheme="bdlr", tol=1e-3, depth=3)
        fa, _ = hodlrkit.factorize(prob.accessor(), tree, cfg, threads=1)
        fb, _ = hodlrkit.factorize(prob.accessor(), tree, cfg, threads=4)
        for slot in range(len(tree.nodes)):
            ca, cb = fa.couplings[slot], fb.couplings[slot]
            assert (ca is None) == (cb is None)
            if ca is not None:
                for x, y in ((ca.d_left, cb.d_left), (ca.d_right, cb.d_right),
                             (ca.schur_lu.lu, cb.schur_lu.lu)):
                    assert np.array_equal(x, y)
            la, lb = fa.leaf_lus[slot], fb.leaf_lus[slot]
            assert (la is None) == (lb is None)
            if la is not None:
                assert np.array_equal(la.lu, lb.lu)

    def test_singular_leaf(self):                                 # :199-204
        a = np.eye(8)
        a[2:4, 2:4] = 0.0
        with pytest.raises(hodlrkit.SingularLeafError):
            hodlrkit.factorize(hodlrkit.BlockAccessor.from_matrix(a), hodlrkit.build_tree(8, 2),
                               hodlrkit.CompressionConfig(scheme="svd", tol=1e-12))

    def test_singular_schur(self):                                # :207-210
        with pytest.raises(hodlrkit.SingularSchurError):
            hodlrkit.factorize(hodlrkit.BlockAccessor.from_matrix(np.ones((2, 2))), hodlrkit.build_tree(2, 1),
                               hodlrkit.CompressionConfig(scheme="svd", tol=1e-12))

    def test_apply(self, rng):                                    # :213-224
        a = rng.standard_normal((32, 32))
        acc = hodlrkit.BlockAccessor.from_matrix(a)
        assert np.array_equal(hodlrkit.apply(hodlrkit.BlockAccessor.from_matrix(np.eye(5)), np.ones((5, 2))),
                              np.ones((5, 2)))
        assert np.array_equal(hodlrkit.apply(hodlrkit.BlockAccessor.from_matrix(np.zeros((4, 4))), np.ones(4)),
                              np.zeros(4))
        e3 = np.eye(32)[3]
        assert np.array_equal(hodlrkit.apply(acc, e3), a[:, 3])
        with pytest.raises(hodlrkit.DimensionMismatchError):
            hodlrkit.apply(acc, np.ones(31))


# =================================================================== test_krylov.py
@gpu
@pytest.mark.usefixtures("need_gpu")
class TestKrylov:
    def test_identity_one_iteration(self, rng):                   # test_krylov.py:17-21
        b = rng.standard_normal(12)
        r = hodlrkit.gmres(lambda v: v, b, hodlrkit.GmresConfig())
        assert r.iterations == 1 and r.converged and np.allclose(r.x, b)

    def test_diagonal_makes_identity(self, rng):                  # :24-30
        a = np.diag(np.arange(1.0, 101.0))
        b = rng.standard_normal(100)
        for op in (lambda v: a @ v, hodlrkit.DenseOperator(a)):   # callable and device paths
            r = hodlrkit.gmres(op, b, hodlrkit.GmresConfig(), preconditioner=hodlrkit.diagonal_preconditioner(a))
            assert r.iterations == 1 and r.converged
            assert np.linalg.norm(a @ r.x - b) <= 1e-10 * np.linalg.norm(b)

    def test_diagonal_values(self, rng):                          # :33-41
        m = hodlrkit.diagonal_preconditioner(np.diag([2.0, 4.0]))
        assert np.allclose(m(np.array([2.0, 4.0])), [1.0, 1.0])
        g = rng.standard_normal((16, 16))
        spd = g @ g.T + 16 * np.eye(16)
        b = rng.standard_normal(16)
        assert np.allclose(hodlrkit.diagonal_preconditioner(spd)(b), b / np.diag(spd))

    def test_zero_diagonal(self):                                 # :44-48
        m = hodlrkit.diagonal_preconditioner(np.diag([1.0, 0.0, 3.0]))
        assert m.flagged and m.zero_count == 1
        assert np.allclose(m(np.array([1.0, 5.0, 3.0])), [1.0, 5.0, 1.0])

    def test_monotone_history(self, rng):                         # :51-56
        a = hodlrkit.kernel_matrix(96, "inv-distance", shift=2.0)
        b = rng.standard_normal(96)
        for op in (lambda v: a @ v, hodlrkit.DenseOperator(a)):
            h = hodlrkit.gmres(op, b, hodlrkit.GmresConfig(tol=1e-12, max_iter=96)).residual_history
            assert all(x >= y - 1e-15 for x, y in zip(h, h[1:]))

    def test_true_residual_guard(self, rng):                      # :59-65
        a = hodlrkit.kernel_matrix(64, "inv-distance", shift=2.0)
        b = rng.standard_normal(64)
        r = hodlrkit.gmres(hodlrkit.DenseOperator(a), b, hodlrkit.GmresConfig(tol=1e-10))
        assert r.converged and r.true_residual <= 1e-9

    def test_exact_preconditioner(self):                          # :67-76
        prob = front_of((9, 9, 9), 0, 4)
        acc = prob.accessor()
        fact, _ = hodlrkit.factorize(acc, hodlrkit.build_tree(prob.n, 32),
                                     hodlrkit.CompressionConfig(scheme="svd", tol=1e-14))
        dense = acc.materialize()
        b = prob.rhs[:, 0]
        r = hodlrkit.gmres(lambda v: dense @ v, b, hodlrkit.GmresConfig(tol=1e-10),
                           preconditioner=lambda x: hodlrkit.solve(fact, x))
        assert r.converged and r.iterations <= 3
        r2 = hodlrkit.gmres(hodlrkit.DenseOperator(dense), b, hodlrkit.GmresConfig(tol=1e-10),
                            preconditioner=fact)
        assert r2.converged and r2.iterations <= 3

    def test_loose_beats_diagonal(self):                          # :79-92
        prob = front_of((9, 9, 9), 0, 4)
        acc = prob.accessor()
        fact, _ = hodlrkit.factorize(acc, hodlrkit.build_tree(prob.n, 32),
                                     hodlrkit.CompressionConfig(scheme="bdlr", tol=1e-1, depth=1))
        op = hodlrkit.DenseOperator(acc)
        cfg = hodlrkit.GmresConfig(tol=1e-10, max_iter=1000)
        b = prob.rhs[:, 0]
        wf = hodlrkit.gmres(op, b, cfg, preconditioner=fact)
        wd = hodlrkit.gmres(op, b, cfg, preconditioner=hodlrkit.diagonal_preconditioner(acc))
        assert wf.converged and wd.converged and wf.iterations < wd.iterations

    def test_nonconvergence(self, rng):                           # :95-100
        a = hodlrkit.kernel_matrix(64, "inv-distance", shift=0.5)
        b = rng.standard_normal(64)
        r = hodlrkit.gmres(hodlrkit.DenseOperator(a), b, hodlrkit.GmresConfig(tol=1e-13, max_iter=3))
        assert not r.converged and r.iterations == 3

    def test_zero_rhs(self):                                      # :103-105
        r = hodlrkit.gmres(lambda v: v, np.zeros(5), hodlrkit.GmresConfig())
        assert r.converged and np.array_equal(r.x, np.zeros(5))


def test_gmres_config_validation():                               # test_krylov.py:108-112
    with pytest.raises(ValueError):
        hodlrkit.GmresConfig(tol=0.0)
    with pytest.raises(ValueError):
        hodlrkit.GmresConfig(max_iter=0)


# =================================================================== test_lowrank.py
def _chain_block(a, split):
    n = a.shape[0]
    pat = hodlrkit.SparsePattern.from_edges(n, np.arange(n - 1), np.arange(1, n))
    return hodlrkit.BlockAccessor(a, pattern=pat).block(np.arange(split), np.arange(split, n))


def _smooth(n=64, kind="inv-distance"):
    """test_lowrank.py:23-32: off-diagonal block of a 2n-point chain kernel."""
    k = hodlrkit.kernel_matrix(2 * n, kind)
    return _chain_block(k, n)


def _rel_err(block, f):
    a = block.materialize()
    return np.linalg.norm(a - f.evaluate()) / max(np.linalg.norm(a), 1e-300)


@gpu
@pytest.mark.usefixtures("need_gpu")
class TestLowRank:
    def test_svd_zero(self):                                      # test_lowrank.py:40-43
        f = hodlrkit.compress_svd(hodlrkit.BlockAccessor(np.zeros((6, 9))), hodlrkit.CompressionConfig(tol=1e-8))
        assert f.rank == 0 and f.shape == (6, 9)

    def test_svd_rank_three(self, rng):                           # :46-51
        a = low_rank(rng, 20, 14, 3)
        f = hodlrkit.compress_svd(hodlrkit.BlockAccessor(a), hodlrkit.CompressionConfig(tol=1e-12))
        assert f.rank == 3
        assert np.linalg.norm(a - f.evaluate()) <= 1e-11 * np.linalg.svd(a, compute_uv=False)[0]

    def test_svd_flat_spectrum(self):                             # :54-56
        assert hodlrkit.compress_svd(hodlrkit.BlockAccessor(np.eye(8)), hodlrkit.CompressionConfig(tol=0.5)).rank == 8

    def test_aca_rank_one(self, rng):                             # :59-63
        a = np.outer(rng.standard_normal(30), rng.standard_normal(22))
        f = hodlrkit.compress_aca(hodlrkit.BlockAccessor(a), hodlrkit.CompressionConfig(scheme="aca", tol=1e-8))
        assert f.rank == 1 and np.linalg.norm(a - f.evaluate()) <= 1e-13 * np.linalg.norm(a)

    def test_aca_zero(self):                                      # :66-68
        assert hodlrkit.compress_aca(hodlrkit.BlockAccessor(np.zeros((7, 7))),
                                     hodlrkit.CompressionConfig(scheme="aca", tol=1e-6)).rank == 0

    def test_aca_smooth(self):                                    # :71-75
        blk = _smooth(64)
        f = hodlrkit.compress_aca(blk, hodlrkit.CompressionConfig(scheme="aca", tol=1e-6))
        assert f.rank < 64 and _rel_err(blk, f) <= 1e-5

    def test_aca_rank_recovery(self, rng):                        # :78-85
        for _ in range(20):
            r = int(rng.integers(1, 9))
            m, n = int(rng.integers(r + 1, 90)), int(rng.integers(r + 1, 90))
            a = low_rank(rng, m, n, r)
            f = hodlrkit.compress_aca(hodlrkit.BlockAccessor(a), hodlrkit.CompressionConfig(scheme="aca", tol=1e-12))
            assert f.rank <= r + 1 and np.linalg.norm(a - f.evaluate()) <= 1e-10 * np.linalg.norm(a)

    def test_aca_max_rank(self, rng):                             # :88-91
        f = hodlrkit.compress_aca(hodlrkit.BlockAccessor(rng.standard_normal((40, 40))),
                                  hodlrkit.CompressionConfig(scheme="aca", tol=1e-12, max_rank=5))
        assert f.rank == 5

    def test_bdlr_disconnected(self):                             # :102-106
        pat = hodlrkit.SparsePattern.from_edges(4, [0, 2], [1, 3])
        blk = hodlrkit.BlockAccessor(np.zeros((4, 4)), pattern=pat).block([0, 1], [2, 3])
        assert hodlrkit.compress_bdlr(blk, hodlrkit.CompressionConfig(scheme="bdlr", tol=1e-3, depth=2)).rank == 0

    def test_bdlr_full_selection(self, rng):                      # :109-115
        blk = _chain_block(rng.standard_normal((12, 24)), 12)
        f = hodlrkit.compress_bdlr(blk, hodlrkit.CompressionConfig(scheme="bdlr", tol=1e-14, depth=40))
        assert _rel_err(blk, f) <= 1e-12

    def test_bdlr_chain_front(self):                              # :118-124
        prob = front_of((40, 21), 1, 10)
        blk = prob.accessor().block(np.arange(20), np.arange(20, 40))
        f = hodlrkit.compress_bdlr(blk, hodlrkit.CompressionConfig(scheme="bdlr", tol=1e-1, depth=1))
        assert _rel_err(blk, f) <= 0.3

    def test_bdlr_degenerate(self):                               # :127-135
        a = np.zeros((10, 10))
        a[:, -1] = 1.0
        with pytest.raises(hodlrkit.DegenerateSkeletonError):
            hodlrkit.compress_bdlr(_chain_block(a, 5), hodlrkit.CompressionConfig(scheme="bdlr", tol=1e-2, depth=0))

    def test_pseudo_skeleton_exact(self, rng):                    # :138-146, :149-157
        for _ in range(20):
            r = int(rng.integers(1, 9))
            m, n = int(rng.integers(r + 2, 100)), int(rng.integers(r + 2, 100))
            a = low_rank(rng, m, n, r)
            while True:
                rows = rng.choice(m, size=r, replace=False)
                cols = rng.choice(n, size=r, replace=False)
                sv = np.linalg.svd(a[np.ix_(rows, cols)], compute_uv=False)
                if sv[-1] >= 1e-4 * sv[0]:
                    break
            f = hodlrkit.pseudo_skeleton(hodlrkit.BlockAccessor(a), rows, cols, tol=1e-12)
            assert np.linalg.norm(a - f.evaluate()) <= 1e-10 * np.linalg.norm(a)

    def test_schemes_share_contract(self, rng):                   # :160-169
        for blk in (_smooth(32), _chain_block(rng.standard_normal((24, 24)), 12)):
            for scheme in ("svd", "aca", "bdlr"):
                f = hodlrkit.compress(blk, hodlrkit.CompressionConfig(scheme=scheme, tol=1e-4, depth=3,
                                                                      max_rank=10))
                assert f.rank <= 10 and np.isfinite(_rel_err(blk, f))

    def test_eckart_young(self):                                  # :172-182
        blk = _smooth(48)
        a = blk.materialize()
        sigma = np.linalg.svd(a, compute_uv=False)
        tail = np.sqrt(np.concatenate([np.cumsum(sigma[::-1] ** 2)[::-1], [0.0]]))
        for scheme in ("aca", "bdlr"):
            f = hodlrkit.compress(blk, hodlrkit.CompressionConfig(scheme=scheme, tol=1e-5, depth=5))
            assert np.linalg.norm(a - f.evaluate()) >= tail[min(f.rank, sigma.size)] - 1e-12

    def test_bdlr_depth_monotone(self):                           # :185-193
        blk = _smooth(32)
        errs = []
        for depth in (1, 2, 3, 4):
            cfg = hodlrkit.CompressionConfig(scheme="bdlr", tol=1e-13, depth=depth)
            f = hodlrkit.compress_bdlr(blk, cfg)
            rows, cols = hodlrkit.held_out_samples(blk, cfg)
            errs.append(hodlrkit.monitor_error(blk, f, rows, cols))
        assert all(b <= a + 1e-12 for a, b in zip(errs, errs[1:]))

    def test_monitor_exact_factor(self, rng):                     # :196-200
        a = low_rank(rng, 16, 12, 2)
        f = hodlrkit.truncate_svd(hodlrkit.svd(a), 1e-13)
        assert hodlrkit.monitor_error(hodlrkit.BlockAccessor(a), f, np.arange(4), np.arange(4)) <= 1e-13

    def test_monitor_known_two_sigma(self, rng):                  # :210-220
        q1 = np.linalg.qr(rng.standard_normal((18, 18)))[0][:, :2]
        q2 = np.linalg.qr(rng.standard_normal((15, 15)))[0][:, :2]
        a = q1 @ np.diag([1.0, 0.1]) @ q2.T
        f = hodlrkit.truncate_svd(hodlrkit.svd(a), 0.5)
        assert f.rank == 1
        full = hodlrkit.monitor_error(hodlrkit.BlockAccessor(a), f, np.arange(18), np.arange(15))
        assert full == pytest.approx(0.1 / np.sqrt(1.01), rel=1e-10)
        assert 0.0 <= hodlrkit.monitor_error(hodlrkit.BlockAccessor(a), f, np.arange(4), np.arange(3)) <= 1.0

    def test_held_out_next_layer(self):                           # :231-238
        prob = front_of((40, 21), 1, 10)
        blk = prob.accessor().block(np.arange(20), np.arange(20, 40))
        cfg = hodlrkit.CompressionConfig(scheme="bdlr", tol=1e-2, depth=1, monitor_samples=4)
        rows, cols = hodlrkit.held_out_samples(blk, cfg)
        d = hodlrkit.distance_index(blk.graph_view, "row")
        assert np.all(d[rows] > 1) and rows.size == 4 and cols.size == 4


def test_monitor_rank_zero_and_underflow(rng, caplog):            # test_lowrank.py:203-207, :223-228
    a = rng.standard_normal((10, 10))
    err = hodlrkit.monitor_error(hodlrkit.BlockAccessor(a), hodlrkit.LowRankFactor.zero(10, 10),
                                 np.arange(3), np.arange(3))
    assert err == pytest.approx(1.0)
    f = hodlrkit.LowRankFactor(np.ones((6, 1)), np.ones((6, 1)))
    with caplog.at_level("WARNING", logger="hodlrkit"):
        err = hodlrkit.monitor_error(hodlrkit.BlockAccessor(np.zeros((6, 6))), f, np.arange(2), np.arange(2))
    assert np.isfinite(err) and err > 0
    assert any("underflow" in r.message for r in caplog.records)


# =================================================================== test_dense.py
@gpu
@pytest.mark.usefixtures("need_gpu")
class TestDense:
    def test_lu_partial_small(self):                              # test_dense.py:14-23
        assert np.allclose(hodlrkit.lu_partial(np.eye(3)).solve(np.array([1.0, 2.0, 3.0])), [1, 2, 3])
        x = hodlrkit.lu_partial(np.array([[0.0, 1.0], [1.0, 0.0]])).solve(np.array([1.0, 2.0]))
        assert np.allclose(x, [2.0, 1.0])

    def test_lu_partial_kernel_residual(self, rng):               # :26-30
        a = hodlrkit.kernel_matrix(64, "inv-distance") + 10.0 * np.eye(64)
        b = rng.standard_normal((64, 3))
        assert np.linalg.norm(a @ hodlrkit.lu_partial(a).solve(b) - b) <= 1e-12 * np.linalg.norm(b)

    def test_lu_partial_reconstruction_and_round_trip(self, rng):  # :33-51
        for n in (5, 17, 60, 128, 256):
            a = rng.standard_normal((n, n)) + n * np.eye(n)
            f = hodlrkit.lu_partial(a)
            low, up = np.tril(f.lu, -1) + np.eye(n), np.triu(f.lu)
            assert np.linalg.norm(a[f.row_perm] - low @ up) <= 1e-13 * np.linalg.norm(a)
            x = rng.standard_normal((n, 2))
            assert np.linalg.norm(f.solve(a @ x) - x) <= 1e-10 * np.linalg.norm(x)

    def test_lu_partial_errors(self):                             # :54-64
        with pytest.raises(hodlrkit.SingularMatrixError):
            hodlrkit.lu_partial(np.zeros((3, 3)))
        a = np.eye(2)
        a[0, 1] = np.nan
        with pytest.raises(ValueError):
            hodlrkit.lu_partial(a)

    def test_lu_full_known_answers(self):                         # :67-89, :108-114
        assert hodlrkit.lu_full(np.array([[1.0, 2.0], [3.0, 4.0]])).pivot_magnitudes[0] == 4.0
        z = hodlrkit.lu_full(np.zeros((3, 3)))
        assert z.pivot_magnitudes.size == 0 and z.numerical_rank(1e-12) == 0 and z.numerical_rank(0.5) == 0
        assert hodlrkit.lu_full(np.outer([1.0, 2.0, 3.0], [1.0, 1.0])).numerical_rank(1e-12) == 1
        assert np.all(np.diff(hodlrkit.lu_full(np.diag([8.0, 4.0, 2.0, 1.0])).pivot_magnitudes) <= 0)
        assert np.all(np.diff(hodlrkit.lu_full(np.outer([3.0, 1.0], [2.0, 1.0])).pivot_magnitudes) <= 1e-12)

    def test_lu_full_reconstruction_and_growth(self, rng):        # :92-105
        for m, n in ((8, 8), (40, 25), (256, 256)):
            a = rng.standard_normal((m, n))
            assert np.linalg.norm(hodlrkit.lu_full(a).reconstruct() - a) <= 1e-12 * np.linalg.norm(a)
        for _ in range(25):
            p = hodlrkit.lu_full(rng.standard_normal((30, 30))).pivot_magnitudes
            assert np.all(p[1:] <= 2.0 * p[:-1] * (1 + 1e-12))

    def test_svd(self, rng):                                      # :117-145
        assert np.allclose(hodlrkit.svd(np.diag([3.0, 2.0, 1.0])).singular_values, [3, 2, 1])
        z = hodlrkit.svd(np.zeros((2, 5)))
        assert z.singular_values.shape == (2,) and np.allclose(z.singular_values, 0.0)
        q1 = np.linalg.qr(rng.standard_normal((6, 6)))[0][:, :2]
        q2 = np.linalg.qr(rng.standard_normal((7, 7)))[0][:, :2]
        s = hodlrkit.svd(q1 @ np.diag([1.0, 1e-4]) @ q2.T).singular_values
        assert abs(s[0] - 1.0) <= 1e-12 and abs(s[1] - 1e-4) <= 1e-12
        a = rng.standard_normal((20, 12))
        r = hodlrkit.svd(a)
        assert np.linalg.norm(r.u @ np.diag(r.singular_values) @ r.v.T - a) <= 1e-12 * np.linalg.norm(a)
        assert np.all(np.diff(r.singular_values) <= 0)
        assert np.abs(r.u.T @ r.u - np.eye(12)).max() <= 1e-12
        assert np.abs(r.v.T @ r.v - np.eye(12)).max() <= 1e-12

    @pytest.mark.parametrize("sigma,tol,rank", [([1.0, 1e-3, 1e-9], 1e-6, 2), ([5.0], 1e-1, 1)])
    def test_truncate_from_spectrum(self, sigma, tol, rank):      # :148-155
        a = np.zeros((4, 3))
        a[:len(sigma), :len(sigma)] = np.diag(sigma)
        assert hodlrkit.truncate_svd(hodlrkit.svd(a), tol).rank == rank

    def test_truncate_rank_and_bound(self, rng):                  # :158-172
        a = sum(np.outer(rng.standard_normal(32), rng.standard_normal(32)) for _ in range(4))
        f = hodlrkit.truncate_svd(hodlrkit.svd(a), 1e-10)
        assert f.rank == 4 and np.linalg.norm(a - f.evaluate()) <= 1e-10 * np.linalg.norm(a)
        a = rng.standard_normal((24, 18))
        s = hodlrkit.svd(a)
        for tol in (1e-1, 1e-3):
            gap = np.linalg.norm(a - hodlrkit.truncate_svd(s, tol).evaluate(), ord=2)
            assert gap <= tol * s.singular_values[0] * (1 + 1e-12)


# =================================================================== test_graph.py (host integer code)
def _path(n):
    return hodlrkit.SparsePattern.from_edges(n, np.arange(n - 1), np.arange(1, n))


def _grid5():
    """test_graph.py:20-33: 5x5 grid, vertex id = 5*column + row."""
    r, c = [], []
    for col in range(5):
        for row in range(5):
            v = 5 * col + row
            if row < 4:
                r.append(v), c.append(v + 1)
            if col < 4:
                r.append(v), c.append(v + 5)
    return hodlrkit.SparsePattern.from_edges(25, r, c)


def _random_view(rng, n, p_edge=0.05):                           # test_graph.py:143-149
    mask = rng.random((n, n)) < p_edge
    rows, cols = np.nonzero(np.triu(mask, 1))
    pat = hodlrkit.SparsePattern.from_edges(n, rows, cols)
    perm = rng.permutation(n)
    return pat, BlockGraphView(pat, perm[:n // 2], perm[n // 2:])


def _floyd_warshall_distance(pat, own, other):                   # test_graph.py:152-174
    own = np.asarray(own)
    k = own.size
    where = {int(v): i for i, v in enumerate(own)}
    oth = {int(v) for v in other}
    d = np.full((k, k), np.inf)
    np.fill_diagonal(d, 0.0)
    bnd = []
    for i, v in enumerate(own):
        nb = [int(u) for u in pat.neighbors(int(v))]
        for u in nb:
            if u in where:
                d[i, where[u]] = 1.0
        if any(u in oth for u in nb):
            bnd.append(i)
    for t in range(k):
        d = np.minimum(d, d[:, [t]] + d[[t], :])
    return d[:, bnd].min(axis=1) if bnd else np.full(k, np.inf)


class TestGraph:
    def test_pattern_symmetric_sorted(self):                      # test_graph.py:36-43
        p = hodlrkit.SparsePattern.from_edges(4, [0, 2, 0], [1, 1, 1])
        for v in range(4):
            nb = p.neighbors(v)
            assert np.all(np.diff(nb) > 0) and all(v in p.neighbors(int(u)) for u in nb)
        assert list(p.neighbors(1)) == [0, 2]

    def test_self_loops_dropped(self):                            # :46-49
        p = hodlrkit.SparsePattern.from_edges(3, [0, 1], [0, 2], values=[5.0, -1.0])
        assert p.degree(0) == 0 and p.diagonal[0] == 5.0

    def test_boundaries(self):                                    # :52-72
        v = BlockGraphView(_path(4), [0, 1], [2, 3])
        assert list(hodlrkit.boundary_vertices(v, "row")) == [1]
        assert list(hodlrkit.boundary_vertices(v, "col")) == [2]
        v = BlockGraphView(hodlrkit.SparsePattern.from_edges(4, [0, 2], [1, 3]), [0, 1], [2, 3])
        assert hodlrkit.boundary_vertices(v, "row").size == hodlrkit.boundary_vertices(v, "col").size == 0
        v = BlockGraphView(_grid5(), np.arange(10), np.arange(10, 25))
        assert list(hodlrkit.boundary_vertices(v, "row")) == [5, 6, 7, 8, 9]
        assert list(hodlrkit.boundary_vertices(v, "col")) == [10, 11, 12, 13, 14]

    def test_distances(self):                                     # :75-94
        assert list(hodlrkit.distance_index(BlockGraphView(_path(5), [0, 1, 2], [3, 4]), "row")) == [2, 1, 0]
        v = BlockGraphView(hodlrkit.SparsePattern.from_edges(4, [0, 2], [1, 3]), [0, 1], [2, 3])
        assert np.isinf(hodlrkit.distance_index(v, "row")).all()
        d = hodlrkit.distance_index(BlockGraphView(_grid5(), np.arange(10), np.arange(10, 25)), "row")
        assert np.all(d[:5] == 1.0) and np.all(d[5:] == 0.0)

    def test_selection(self):                                     # :97-121
        v = BlockGraphView(_path(5), [0, 1, 2], [3, 4])
        r, c = hodlrkit.select_by_depth(v, 0)
        assert list(r) == [2] and list(c) == [0]
        r, c = hodlrkit.select_by_depth(v, 10)
        assert list(r) == [2, 1, 0] and list(c) == [0, 1]
        r, _ = hodlrkit.select_by_depth(BlockGraphView(_grid5(), np.arange(10), np.arange(10, 25)), 1)
        assert list(r) == [5, 6, 7, 8, 9, 0, 1, 2, 3, 4]
        with pytest.raises(hodlrkit.EmptySelectionError):
            hodlrkit.select_by_depth(BlockGraphView(hodlrkit.SparsePattern.from_edges(4, [0, 2], [1, 3]),
                                                    [0, 1], [2, 3]), 3)

    def test_selection_monotone_and_deterministic(self, rng):     # :124-140
        _, view = _random_view(rng, 60)
        prev = set()
        for depth in range(5):
            try:
                r, _ = hodlrkit.select_by_depth(view, depth)
            except hodlrkit.EmptySelectionError:
                continue
            assert prev <= set(int(i) for i in r)
            prev = set(int(i) for i in r)
        _, view = _random_view(rng, 80)
        a, b = hodlrkit.select_by_depth(view, 2), hodlrkit.select_by_depth(view, 2)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])

    def test_bfs_vs_floyd_warshall(self, rng):                    # :177-184
        for _ in range(10):
            n = int(rng.integers(10, 120))
            pat, view = _random_view(rng, n, p_edge=3.0 / n)
            for side in ("row", "col"):
                want = _floyd_warshall_distance(pat, view.side(side), view.other(side))
                assert np.array_equal(hodlrkit.distance_index(view, side), want)

    def test_distance_lipschitz(self, rng):                       # :187-197
        pat, view = _random_view(rng, 100, p_edge=0.04)
        d = hodlrkit.distance_index(view, "row")
        where = {int(v): i for i, v in enumerate(view.row_verts)}
        for v in view.row_verts:
            for u in pat.neighbors(int(v)):
                if int(u) in where:
                    a, b = d[where[int(v)]], d[where[int(u)]]
                    if np.isfinite(a) and np.isfinite(b):
                        assert abs(a - b) <= 1.0

    def test_view_rejects_overlap(self):                          # :200-202
        with pytest.raises(ValueError):
            BlockGraphView(_path(4), [0, 1], [1, 2])
