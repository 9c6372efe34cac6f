"""Dense kernels of the drop-in API (reference src/dense.py) on the B200.

``lu_partial``  -> hk_lu_partial (batched partial-pivot LU kernel, lu.cu)
``lu_full``     -> hk_lu_full   (complete pivoting, numpy-identical pivot order)
``svd``         -> cuSOLVER through torch.linalg.svd (parity-only scheme;
                   SURVEY.md §2.3 K7 marks it "not performance-graded")

Results come back as the reference's frozen dataclasses holding numpy arrays.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import SingularMatrixError, SvdConvergenceError

PIVOT_UNDERFLOW = 1e-300


def as_matrix(a, name="matrix") -> np.ndarray:
    """2-D float64, finite entries only (dense.py:22-29)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got ndim={a.ndim}")
    if a.size and not np.isfinite(a).all():
        raise ValueError(f"{name} contains NaN or Inf entries")
    return a


def _row_perm_from_piv(piv: np.ndarray) -> np.ndarray:
    perm = np.arange(piv.size)
    for k, p in enumerate(piv):
        perm[k], perm[p] = perm[p], perm[k]
    return perm


@dataclass(frozen=True)
class PartialPivLU:
    """P A = L U, packed (dense.py:32-56).  ``inverse`` is the explicit A^{-1}
    the device path applies; ``solve`` uses it on the GPU."""

    lu: np.ndarray
    piv: np.ndarray
    row_perm: np.ndarray
    inverse: np.ndarray | None = None

    @property
    def n(self) -> int:
        return self.lu.shape[0]

    def solve(self, b) -> np.ndarray:
        b = np.asarray(b, dtype=np.float64)
        vector = b.ndim == 1
        if vector:
            b = b[:, None]
        if b.shape[0] != self.n:
            raise ValueError(f"rhs has {b.shape[0]} rows, expected {self.n}")
        if self.n == 0 or b.shape[1] == 0:
            x = np.zeros_like(b)
        else:
            torch = N.require_cuda()
            inv = self.inverse
            if inv is None:
                raise RuntimeError("factor was created without an inverse")
            it = torch.from_numpy(np.ascontiguousarray(inv)).cuda()
            bt = torch.from_numpy(np.ascontiguousarray(b.T)).cuda()   # column-major n x s
            y = torch.empty_like(bt)
            N.check(N.lib().hk_gemv(N.ptr(it), self.n, self.n, self.n, N.ptr(bt), self.n,
                                    b.shape[1], N.ptr(y), self.n, N.stream_handle()))
            x = y.cpu().numpy().T.copy()
        return x[:, 0] if vector else x


def lu_partial(a) -> PartialPivLU:
    """Row-pivoted LU; SingularMatrixError below 1e-300 (dense.py:59-81)."""
    a = as_matrix(a)
    m, n = a.shape
    if m != n:
        raise ValueError(f"matrix must be square, got {m}x{n}")
    if n == 0:
        z = np.zeros(0, dtype=np.intp)
        return PartialPivLU(np.zeros((0, 0)), z, z, np.zeros((0, 0)))
    torch = N.require_cuda()
    at = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    inv = torch.empty_like(at)
    piv = torch.empty(n, dtype=torch.int32, device="cuda")
    st = N.lib().hk_lu_partial(N.ptr(at), n, n, N.ptr(piv), N.ptr(inv), N.stream_handle())
    if st == 3:
        raise SingularMatrixError(f"pivot magnitude below {PIVOT_UNDERFLOW:g}")
    N.check(st)
    pv = piv.cpu().numpy().astype(np.intp)
    return PartialPivLU(at.cpu().numpy(), pv, _row_perm_from_piv(pv), inv.cpu().numpy())


def gj_inverse(a) -> np.ndarray:
    """Explicit inverse(s) by the factorization's batched Gauss-Jordan kernels
    (hk_gj_inverse): `a` is (n, n) or (batch, n, n).  Same implicit partial
    pivoting and singularity test as lu_partial (dense.py:76-77); raises
    SingularMatrixError naming the first singular matrix."""
    a = np.asarray(a, dtype=np.float64)
    single = a.ndim == 2
    a3 = a[None] if single else a
    if a3.ndim != 3 or a3.shape[1] != a3.shape[2]:
        raise ValueError(f"expected (n, n) or (batch, n, n), got {a.shape}")
    if not np.all(np.isfinite(a3)):
        raise ValueError("matrix contains NaN or Inf")
    bsz, n, _ = a3.shape
    if n == 0 or bsz == 0:
        return np.zeros_like(a)
    torch = N.require_cuda()
    at = torch.from_numpy(np.ascontiguousarray(a3)).cuda()
    out = torch.empty_like(at)
    status = np.zeros(bsz, dtype=np.int32)
    N.check(N.lib().hk_gj_inverse(N.ptr(at), n, n, bsz, n * n, N.ptr(out),
                                  status.ctypes.data, N.stream_handle()))
    if status.any():
        raise SingularMatrixError(f"matrix {int(np.argmax(status))}: pivot magnitude below "
                                  f"{PIVOT_UNDERFLOW:g}")
    inv = out.cpu().numpy().transpose(0, 2, 1)     # column-major -> row-major
    return np.ascontiguousarray(inv[0] if single else inv)


@dataclass(frozen=True)
class FullPivLU:
    """A[row_perm][:, col_perm] = L U with complete pivoting (dense.py:84-130)."""

    lu: np.ndarray
    row_perm: np.ndarray
    col_perm: np.ndarray
    pivot_magnitudes: np.ndarray

    @property
    def shape(self):
        return self.lu.shape

    def numerical_rank(self, tau: float) -> int:
        if self.pivot_magnitudes.size == 0:
            return 0
        return int(np.count_nonzero(self.pivot_magnitudes >= tau * self.pivot_magnitudes[0]))

    def lower(self, r: int) -> np.ndarray:
        l11 = np.tril(self.lu[:r, :r], -1)
        np.fill_diagonal(l11, 1.0)
        return l11

    def upper(self, r: int) -> np.ndarray:
        return np.triu(self.lu[:r, :r])

    def reconstruct(self) -> np.ndarray:
        m, n = self.lu.shape
        k = min(m, n)
        low = np.tril(self.lu[:, :k], -1)
        np.fill_diagonal(low, 1.0)
        out = np.zeros((m, n))
        out[np.ix_(self.row_perm, self.col_perm)] = low @ np.triu(self.lu[:k, :])
        return out


def lu_full(a) -> FullPivLU:
    """Complete-pivoting LU on the GPU, never erroring on rank deficiency
    (dense.py:133-166); pivots, permutations and packed factors are
    bit-identical to the reference."""
    a = as_matrix(a)
    m, n = a.shape
    if m == 0 or n == 0:
        return FullPivLU(a.copy(), np.arange(m), np.arange(n), np.zeros(0))
    torch = N.require_cuda()
    w = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    rp = torch.empty(m, dtype=torch.int64, device="cuda")
    cp = torch.empty(n, dtype=torch.int64, device="cuda")
    pv = torch.empty(min(m, n), dtype=torch.float64, device="cuda")
    cnt = N.I64(0)
    N.check(N.lib().hk_lu_full(N.ptr(w), m, n, n, N.ptr(rp), N.ptr(cp), N.ptr(pv),
                               N.C.byref(cnt), N.stream_handle()))
    return FullPivLU(w.cpu().numpy(), rp.cpu().numpy().astype(np.intp),
                     cp.cpu().numpy().astype(np.intp), pv[:cnt.value].cpu().numpy())


@dataclass(frozen=True)
class SvdResult:
    """A = u diag(s) v^T, thin (dense.py:169-175)."""

    u: np.ndarray
    singular_values: np.ndarray
    v: np.ndarray


def svd(a) -> SvdResult:
    """Thin SVD via cuSOLVER (parity-only scheme)."""
    a = as_matrix(a)
    torch = N.require_cuda()
    if a.size == 0:
        m, n = a.shape
        k = min(m, n)
        return SvdResult(np.zeros((m, k)), np.zeros(k), np.zeros((n, k)))
    try:
        u, s, vh = torch.linalg.svd(torch.from_numpy(np.ascontiguousarray(a)).cuda(),
                                    full_matrices=False)
    except RuntimeError as exc:
        raise SvdConvergenceError(str(exc)) from exc
    return SvdResult(u.cpu().numpy(), s.cpu().numpy(), vh.T.cpu().numpy())
