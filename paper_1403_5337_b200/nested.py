"""Forward/back substitution across an elimination tree: the whole grid
problem solved through its separator front (the paper's
setting, PAPER.md:488-493 -- the HODLR-compressed front inside a multifrontal
solve).

One level of nested dissection along `axis`: the planes on either side of the
separator plane form two chains that are eliminated toward it,

    D_0 = T_0,   D_k = T_k - C_k D_{k-1}^{-1} C_k       (plane Schur complements)
    S   = T_p - C_L D_L^{-1} C_L - C_R D_R^{-1} C_R     (the separator front)

where T_t is the in-plane operator and C_t = diag(c_t) the coupling between
planes t-1 and t (frontgen.PlaneOperator).  A solve of L x = b then runs

    forward   y_0 = b_0,  y_k = b_k + c_k * (D_{k-1}^{-1} y_{k-1})    per chain
    front     S x_p = b_p + c_L * (D_L^{-1} y_L) + c_R * (D_R^{-1} y_R)
              by GMRES preconditioned with the HODLR factorization of S
    backward  x_k = D_k^{-1} (y_k + c_{k+1} * x_{k+1})                 per chain

The plane inverses come from this library's block Gauss-Jordan
(hk_spd_inverse), the front from the same elimination (it is bit-for-bit the
front `frontgen.layered_grid_front` returns), the HODLR build / factor /
GMRES from the hot path, and every D^{-1} y product is this library's GEMV
(hk_gemv).  The reference has no such solver; its fronts are the separator
Schur complements this one builds.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .errors import InvalidPlaneError
from .frontgen import PlaneOperator, _torch
from .krylov import DenseOperator, GmresConfig, gmres
from .lowrank import BlockAccessor, CompressionConfig
from .hodlr import build_tree, factorize


class PlaneNestedSolver:
    """Solve the grid Laplacian of `dims` (Dirichlet boundary eliminated, cell
    conductivity `conductivity` or constant) through the separator plane
    `plane` of `axis`.  Vectors are (ext, nl) arrays: plane t along `axis`,
    nodes of a plane in row-major order of the remaining axes (the separator
    front's order)."""

    def __init__(self, dims, axis, plane, conductivity=None, leaf=64,
                 cfg: CompressionConfig | None = None, device="cuda"):
        torch = _torch()
        N.require_cuda()
        self.op = op = PlaneOperator(dims, axis, [conductivity], device=device)
        self.ext, self.nl, self.plane = op.ext, op.nl, int(plane)
        if not 0 < self.plane < self.ext - 1:
            raise InvalidPlaneError(f"plane {plane} is not strictly interior to extent {self.ext}")
        self.chains = (list(range(0, self.plane)), list(range(self.ext - 1, self.plane, -1)))
        self.dinv = {}            # plane -> D^{-1} of the chain up to it (nl x nl, on device)
        self.cin = {}             # plane -> coupling to the previous plane of its chain
        front = op.layer_matrix(self.plane)[0]
        self.csep = []
        for chain in self.chains:
            D = None
            prev = None
            for t in chain:
                T = op.layer_matrix(t)[0]
                if D is not None:
                    c = op.coupling(max(t, prev))[0]
                    self.cin[t] = c
                    T = T - c[:, None] * self.dinv[prev] * c[None, :]
                D = T
                self.dinv[t] = op.inverse(D[None])[0]
                prev = t
            c = op.coupling(max(self.plane, chain[-1]))[0]
            self.csep.append(c)
            front = front - c[:, None] * self.dinv[chain[-1]] * c[None, :]
        self.front = front.contiguous()
        self.cfg = cfg or CompressionConfig(scheme="aca", tol=1e-6)
        self.fact, self.report = factorize(BlockAccessor.from_matrix(self.front.cpu().numpy()),
                                           build_tree(self.nl, leaf), self.cfg)
        self._front_op = DenseOperator(self.front)

    def _dinv_mv(self, t, v):
        """D_t^{-1} v on the device (hk_gemv; D^{-1} is symmetric, so its
        row-major and column-major views agree)."""
        torch = _torch()
        M = self.dinv[t]
        y = torch.empty_like(v)
        n = self.nl
        N.check(N.lib().hk_gemv(N.ptr(M), n, n, n, N.ptr(v), n, 1, N.ptr(y), n, N.stream_handle()))
        return y

    def solve(self, b, gmres_cfg: GmresConfig | None = None):
        """x with L x = b (b: (ext, nl) array-like); also returns the separator
        GMRES result."""
        torch = _torch()
        B = torch.as_tensor(np.asarray(b, dtype=np.float64)).to(self.op.dev)
        if B.shape != (self.ext, self.nl):
            raise ValueError(f"rhs must have shape ({self.ext}, {self.nl})")
        y = {}
        g = B[self.plane].clone()
        for chain, cs in zip(self.chains, self.csep):
            prev = None
            for t in chain:
                y[t] = B[t].clone() if prev is None else B[t] + self.cin[t] * self._dinv_mv(prev, y[prev])
                prev = t
            g = g + cs * self._dinv_mv(chain[-1], y[chain[-1]])
        res = gmres(self._front_op, g.cpu().numpy(), gmres_cfg or GmresConfig(tol=1e-12),
                    preconditioner=self.fact)
        X = torch.empty_like(B)
        X[self.plane] = torch.from_numpy(res.x).to(self.op.dev)
        for chain, cs in zip(self.chains, self.csep):
            nxt, cn = self.plane, cs
            for t in reversed(chain):
                X[t] = self._dinv_mv(t, y[t] + cn * X[nxt])
                nxt = t
                cn = self.cin.get(t)
        return X.cpu().numpy(), res

    def apply(self, x):
        """L x for an (ext, nl) array (block tridiagonal operator)."""
        torch = _torch()
        X = torch.as_tensor(np.asarray(x, dtype=np.float64)).to(self.op.dev)
        Y = torch.empty_like(X)
        for t in range(self.ext):
            v = self.op.layer_matrix(t)[0] @ X[t]
            if t > 0:
                v = v - self.op.coupling(t)[0] * X[t - 1]
            if t + 1 < self.ext:
                v = v - self.op.coupling(t + 1)[0] * X[t + 1]
            Y[t] = v
        return Y.cpu().numpy()
