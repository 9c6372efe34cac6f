"""GPU front generation on this library's kernels: the
batched SPD block Gauss-Jordan inverse (hk_spd_inverse) against numpy, and
the plane-by-plane elimination through it against the cuSOLVER-backed path
and the reference's own generator recipe."""

import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_1403_5337_b200 as hk  # noqa: E402
from paper_1403_5337_b200 import _native as N  # noqa: E402
from paper_1403_5337_b200 import frontgen as fg  # noqa: E402


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("n,batch", [(1, 1), (7, 3), (64, 2), (65, 2), (200, 4), (1024, 2), (2100, 1)])
def test_spd_inverse_vs_numpy(n, batch):
    rng = np.random.default_rng(n)
    mats = []
    for _ in range(batch):
        G = rng.standard_normal((n, n))
        mats.append(G @ G.T / n + np.eye(n))
    A = np.stack(mats)
    X = torch.from_numpy(A).cuda().contiguous()
    st = (ctypes.c_int32 * batch)()
    N.check(N.lib().hk_spd_inverse(N.ptr(X), n, n, batch, n * n, st, N.stream_handle()))
    assert list(st) == [0] * batch
    Xi = X.cpu().numpy()
    for b in range(batch):
        ref = np.linalg.inv(A[b])
        assert np.abs(Xi[b] - ref).max() <= 1e-11 * np.abs(ref).max()


def test_spd_inverse_singular_block_reported():
    n = 130
    A = np.eye(n)
    A[70, 70] = 0.0                          # pivot block 1 singular
    X = torch.from_numpy(np.stack([np.eye(n), A])).cuda().contiguous()
    st = (ctypes.c_int32 * 2)()
    N.check(N.lib().hk_spd_inverse(N.ptr(X), n, n, 2, n * n, st, N.stream_handle()))
    assert list(st) == [0, 1]


@pytest.mark.parametrize("dims,plane,seed", [((12, 12, 12), 6, 3), ((32, 32, 32), 16, 0)])
def test_layered_front_hk_matches_cusolver_path(dims, plane, seed, monkeypatch):
    kc = fg.cell_conductivity(dims, seed)
    monkeypatch.setenv("HK_FRONTGEN", "torch")
    ref = fg.layered_grid_front(dims, 2, plane, conductivity=kc, device="cuda", return_torch=True)
    monkeypatch.setenv("HK_FRONTGEN", "hk")
    got = fg.layered_grid_front(dims, 2, plane, conductivity=kc, device="cuda", return_torch=True)
    assert float((got - ref).abs().max() / ref.abs().max()) <= 1e-14


def test_batched_fronts_equal_single_fronts():
    dims = (10, 10, 10)
    kcs = [fg.cell_conductivity(dims, s) for s in range(4)]
    Fb = fg.layered_grid_fronts(dims, 2, 5, kcs, device="cuda")
    for s in range(4):
        one = fg.layered_grid_front(dims, 2, 5, conductivity=kcs[s], device="cuda", return_torch=True)
        assert torch.equal(Fb[s], one)


def test_gpu_front_matches_reference_generator_recipe():
    """Constant coefficients: the plane elimination equals the reference's
    dense elimination (grid_front, src/frontgen.py:159-189) on a small grid."""
    dims = (9, 9, 9)
    ref = hk.grid_front(hk.GridSpec(dims), 2, 4).front
    got = fg.layered_grid_front(dims, 2, 4, device="cuda")
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
