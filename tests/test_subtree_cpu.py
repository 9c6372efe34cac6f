"""HODLR-subtree sharding (BASELINE config 4's multi-GPU path)
on the CPU: the orchestration of subtree.ShardedHodlr -- ownership, external
extensions, the per-level all-reduces of the coupling terms and the
distributed solve -- run (i) over gloo with world size 2 and (ii) as emulated
ranks in one process, with a dense CPU stand-in for the per-rank device
primitives (exact local subtree inverse; top-level blocks compressed by the
oracle's ACA).  The GPU path swaps in GpuBackend (tests/test_gpu_parity.py).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hodlr_oracle as O
from paper_1403_5337_b200 import subtree as ST
from paper_1403_5337_b200.frontgen import cell_conductivity, layered_grid_front
from paper_1403_5337_b200.lowrank import CompressionConfig


class DenseCpuBackend:
    """Test stand-in for GpuBackend: exact dense subtree inverse, oracle ACA."""

    def __init__(self, front, lo, hi, leaf):
        self.front = front
        self.lo, self.hi = lo, hi

    def compress(self, r0, r1, c0, c1, cfg):
        U, V = O.aca(self.front[r0:r1, c0:c1].numpy(), cfg.tol)
        return torch.from_numpy(np.ascontiguousarray(U.T)), torch.from_numpy(np.ascontiguousarray(V.T))

    def build(self, cfg):
        self.Kinv = torch.linalg.inv(self.front[self.lo:self.hi, self.lo:self.hi])

    def factor_ext(self, Z):
        return (self.Kinv @ Z.T).T.contiguous()

    def solve_local_(self, x):                  # x: (s, n_loc)
        x[:] = (self.Kinv @ x.T).T
        return x

    def gemm(self, C, A, B, trans_a=False, alpha=1.0, beta=0.0):
        Am = A.T if not trans_a else A       # math view of op(A): A is cm (shape cols x rows)
        res = alpha * (Am @ B.T) + (beta * C.T if beta else 0.0)
        C[...] = res.T
        return C

    def inverse(self, S):
        return torch.linalg.inv(S.T).T.contiguous()

    def rows_matvec(self, X):                   # X: (s, n) -> (s, rows)
        return (self.front[self.lo:self.hi] @ X.T).T


def _front():
    dims = (12, 12, 12)
    return torch.from_numpy(layered_grid_front(dims, "z", 6, conductivity=cell_conductivity(dims, 4)))


CFG = CompressionConfig(scheme="aca", tol=1e-12)
LEAF = 16


def _run(comm, front, b):
    sh = ST.ShardedHodlr(front, LEAF, comm, backend_factory=DenseCpuBackend)
    sh.factorize(CFG)
    return sh.solve(b), sh.apply(b)


def _run_batch(comm, front, B):
    """s = 3 right-hand sides through one sharded sweep / GEMV (rows = rhs)."""
    sh = ST.ShardedHodlr(front, LEAF, comm, backend_factory=DenseCpuBackend)
    sh.factorize(CFG)
    return sh.solve_batch(B), sh.apply_batch(B)


def _rhs3(n):
    return torch.from_numpy(np.random.default_rng(8).standard_normal((3, n)))


@pytest.mark.parametrize("G", [2, 4])
def test_emulated_ranks_match_dense_solve(G):
    front = _front()
    b = torch.from_numpy(np.random.default_rng(7).standard_normal(front.shape[0]))
    x, ax = _run(ST.EmulatedRanks(G), front, b)
    exact = torch.linalg.solve(front, b)
    # top-level blocks compressed at 1e-12, subtrees exact: the sharded HODLR inverse is exact
    assert float(torch.linalg.vector_norm(x - exact) / torch.linalg.vector_norm(exact)) < 1e-9
    assert torch.allclose(ax, front @ b, rtol=0, atol=1e-12)
    B = _rhs3(front.shape[0])
    X, AX = _run_batch(ST.EmulatedRanks(G), front, B)
    exact = torch.linalg.solve(front, B.T).T
    assert float(torch.linalg.vector_norm(X - exact) / torch.linalg.vector_norm(exact)) < 1e-9
    assert torch.allclose(AX, B @ front.T, rtol=0, atol=1e-12)


def test_emulated_rejects_shallow_trees():
    front = _front()
    with pytest.raises(ValueError):
        ST.ShardedHodlr(front, 200, ST.EmulatedRanks(4), backend_factory=DenseCpuBackend)
    with pytest.raises(ValueError):
        ST.ShardedHodlr(front, LEAF, ST.EmulatedRanks(3), backend_factory=DenseCpuBackend)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.set_num_threads(1)
        front = _front()
        b = torch.from_numpy(np.random.default_rng(7).standard_normal(front.shape[0]))
        x, ax = _run(ST.TorchDistRanks(1), front, b)
        X, AX = _run_batch(ST.TorchDistRanks(1), front, _rhs3(front.shape[0]))
        out[rank] = (x.numpy().tolist(), ax.numpy().tolist(), X.numpy().tolist(), AX.numpy().tolist())
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_matches_emulated():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    torch.set_num_threads(1)
    front = _front()
    b = torch.from_numpy(np.random.default_rng(7).standard_normal(front.shape[0]))
    x_em, ax_em = _run(ST.EmulatedRanks(2), front, b)
    X_em, AX_em = _run_batch(ST.EmulatedRanks(2), front, _rhs3(front.shape[0]))
    for r in range(world):
        assert np.array_equal(np.array(res[r][0]), x_em.numpy()), r   # same sums, same bits
        assert np.array_equal(np.array(res[r][1]), ax_em.numpy()), r
        assert np.array_equal(np.array(res[r][2]), X_em.numpy()), r
        assert np.array_equal(np.array(res[r][3]), AX_em.numpy()), r
