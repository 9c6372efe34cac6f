"""Front manufacture: grid operators, planar separators, dense Schur fronts.

Mirrors the input side of the reference (src/frontgen.py) with the same names
and argument meaning.  This is *not* the hot path -- it only manufactures the
dense frontal matrices the HODLR path consumes.

Where the reference eliminates the two interior sides with one dense solve
each (src/frontgen.py:159-189, O(N_interior^3)), grid fronts here are built
by plane-by-plane block elimination along the separator axis: every interior
layer couples only to its two neighbouring layers through a diagonal matrix,
so the separator Schur complement is the recursion
``D_0 = T_0;  D_t = T_t - C D_{t-1}^{-1} C``.  The dense layer solves run in
torch fp64 on whatever device is given (cuSOLVER on a B200), which makes the
32^3 / 48^3 / 96^3 fronts of BASELINE.json configs 0, 1, 3 and 4 cheap to
produce.  Constant-coefficient fronts agree with the reference's dense
elimination to ~1e-15 relative (tests/test_frontgen.py).

Variable coefficients (BASELINE configs 1 and 3, "per-cell conductivity
exp(g)"): cells of an (X+1) x (Y+1) x (Z+1) lattice surround the interior
nodes (the Dirichlet boundary nodes sit on the outer faces); the weight of a
grid edge is the mean conductivity of the four cells sharing it, and a node's
diagonal is the sum of its six incident edge weights.  With g = 0 this is the
reference's constant-coefficient operator (diagonal 6, couplings -1).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InvalidPlaneError, SingularInteriorError
from .graph import SparsePattern
from .lowrank import BlockAccessor

STENCILS = ("laplacian", "vector-laplacian")
KERNELS = ("inv-distance", "exp-decay")
AXIS_NAMES = {"x": 0, "y": 1, "z": 2}


@dataclass(frozen=True)
class GridSpec:
    """Regular grid (src/frontgen.py:28-60): extents 1 or >= 3."""

    dims: tuple
    stencil: str = "laplacian"

    def __post_init__(self):
        dims = tuple(int(d) for d in self.dims)
        object.__setattr__(self, "dims", dims)
        if len(dims) not in (2, 3):
            raise ValueError("dims must have 2 or 3 extents")
        if any(d < 1 or d == 2 for d in dims):
            raise ValueError("extents must be 1 (degenerate) or >= 3")
        if self.stencil not in STENCILS:
            raise ValueError(f"unknown stencil {self.stencil!r}")

    @property
    def dof_per_node(self) -> int:
        return 3 if self.stencil == "vector-laplacian" else 1

    @property
    def node_count(self) -> int:
        return int(np.prod(self.dims))

    @property
    def dof_count(self) -> int:
        return self.node_count * self.dof_per_node


@dataclass(frozen=True)
class FrontProblem:
    """Dense front + separator graph + ordering + seeded rhs (frontgen.py:63-81)."""

    front: np.ndarray
    graph: SparsePattern
    ordering: np.ndarray
    rhs: np.ndarray

    @property
    def n(self) -> int:
        return self.front.shape[0]

    def accessor(self) -> BlockAccessor:
        return BlockAccessor.from_matrix(self.front, pattern=self.graph)


def _strides(dims):
    s = np.ones(len(dims), dtype=np.int64)
    for a in range(len(dims) - 2, -1, -1):
        s[a] = s[a + 1] * dims[a + 1]
    return s


def _expand(nodes, dof):
    nodes = np.asarray(nodes, dtype=np.int64)
    if dof == 1:
        return nodes
    return (nodes[:, None] * dof + np.arange(dof)).ravel()


def grid_operator(spec: GridSpec) -> SparsePattern:
    """Stencil matrix with the Dirichlet boundary eliminated (frontgen.py:90-123)."""
    dims = spec.dims
    stride = _strides(dims)
    ids = np.arange(spec.node_count, dtype=np.int64).reshape(dims)
    rows, cols = [], []
    for axis, ext in enumerate(dims):
        if ext < 2:
            continue
        sl = [slice(None)] * len(dims)
        sl[axis] = slice(0, ext - 1)
        lo = ids[tuple(sl)].ravel()
        rows.append(lo)
        cols.append(lo + stride[axis])
    rows = np.concatenate(rows) if rows else np.zeros(0, np.int64)
    cols = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    dof = spec.dof_per_node
    rows, cols = _expand(rows, dof), _expand(cols, dof)
    diag = float(2 * sum(1 for d in dims if d > 1))
    ndof = spec.dof_count
    return SparsePattern.from_edges(ndof, rows, cols, np.full(rows.size, -1.0),
                                    np.full(ndof, diag))


def planar_separator(spec: GridSpec, axis, plane: int):
    """(separator, left, right) dof ids (frontgen.py:126-156)."""
    if isinstance(axis, str):
        if axis not in AXIS_NAMES:
            raise ValueError(f"axis must be one of {tuple(AXIS_NAMES)} or an integer")
        axis = AXIS_NAMES[axis]
    if not 0 <= axis < len(spec.dims):
        raise InvalidPlaneError(f"axis {axis} out of range for dims {spec.dims}")
    ext = spec.dims[axis]
    if not 0 < plane < ext - 1:
        raise InvalidPlaneError(f"plane {plane} is not strictly interior to extent {ext}")
    along = np.indices(spec.dims).reshape(len(spec.dims), -1)[axis]
    dof = spec.dof_per_node
    return (_expand(np.flatnonzero(along == plane), dof),
            _expand(np.flatnonzero(along < plane), dof),
            _expand(np.flatnonzero(along > plane), dof))


def _torch():
    import torch
    return torch


def schur_front(op: SparsePattern, sep, left, right, rhs_seed: int = 0,
                rhs_columns: int = 1, device=None) -> FrontProblem:
    """Dense separator Schur complement of a general sparse operator.

    Same contract as src/frontgen.py:159-189 (sides must not touch).  The
    interior solves run in torch fp64 on ``device``.
    """
    torch = _torch()
    sep = np.asarray(sep, dtype=np.int64)
    left = np.asarray(left, dtype=np.int64)
    right = np.asarray(right, dtype=np.int64)
    merged = np.concatenate([sep, left, right])
    if merged.size != op.n or np.unique(merged).size != merged.size:
        raise ValueError("sep, left, right must partition the vertex set")
    rmask = np.zeros(op.n, dtype=bool)
    rmask[right] = True
    for v in left:
        if rmask[op.neighbors(int(v))].any():
            raise ValueError("left and right sides are connected; the separator is invalid")
    dev = torch.device(device or "cpu")
    front = torch.from_numpy(op.submatrix_dense(sep, sep)).to(dev)
    for side in (left, right):
        if side.size == 0:
            continue
        a_si = torch.from_numpy(op.submatrix_dense(sep, side)).to(dev)
        a_ii = torch.from_numpy(op.submatrix_dense(side, side)).to(dev)
        try:
            front -= a_si @ torch.linalg.solve(a_ii, a_si.T.contiguous())
        except RuntimeError as exc:
            raise SingularInteriorError(str(exc)) from exc
    rng = np.random.default_rng(rhs_seed)
    rhs = rng.standard_normal((sep.size, rhs_columns))
    return FrontProblem(front.cpu().numpy(), op.induced(sep), sep.copy(), rhs)


# ---------------------------------------------------------------------------
# layered (plane-recursive) grid fronts
# ---------------------------------------------------------------------------

def cell_conductivity(dims, seed):
    """exp(g), g ~ N(0,1) i.i.d. on the (X+1)x(Y+1)x(Z+1) cell lattice."""
    shape = tuple(d + 1 for d in dims)
    return np.exp(np.random.default_rng(seed).standard_normal(shape))


def _edge_weights(dims, kcell):
    """Per-axis edge weights w[a] of shape dims + 1 along axis a.

    w[a][..., t, ...] is the edge between nodes t-1 and t along axis a (t = 0
    and t = ext are the edges to the eliminated boundary).  The weight is the
    mean of the 2^(d-1) cells sharing the edge.
    """
    d = len(dims)
    out = []
    for a in range(d):
        if dims[a] == 1:
            # a degenerate axis carries no couplings at all (frontgen.py:100-102)
            shape = list(dims)
            shape[a] += 1
            out.append(np.zeros(shape))
            continue
        if kcell is None:
            shape = list(dims)
            shape[a] += 1
            out.append(np.ones(shape))
            continue
        acc = None
        cnt = 0
        # cells sharing an edge along axis a: cell index along a is t (0..ext),
        # along every other axis b it is x_b or x_b + 1
        offs = [(0, 1) if b != a else (0,) for b in range(d)]
        for combo in np.ndindex(*[len(o) for o in offs]):
            sl = []
            for b in range(d):
                o = offs[b][combo[b]]
                if b == a:
                    sl.append(slice(0, dims[a] + 1))
                else:
                    sl.append(slice(o, o + dims[b]))
            part = kcell[tuple(sl)]
            acc = part.copy() if acc is None else acc + part
            cnt += 1
        out.append(acc / cnt)
    return out


def frontgen_solver() -> str:
    """Dense inverse behind the GPU plane elimination: "hk" (this library's
    block Gauss-Jordan, the default) or "torch" (cuSOLVER); HK_FRONTGEN picks."""
    import os
    return os.environ.get("HK_FRONTGEN", "hk")


def _spd_inverse_(X):
    """In place: X[b] <- X[b]^{-1} for a contiguous CUDA float64 (B, n, n) batch
    of SPD matrices (hk_spd_inverse: block Gauss-Jordan, one call per batch)."""
    import ctypes
    from . import _native as N
    B, n = X.shape[0], X.shape[1]
    st = (ctypes.c_int32 * B)()
    N.check(N.lib().hk_spd_inverse(N.ptr(X), n, n, B, n * n, st, N.stream_handle()))
    if any(st):
        raise ValueError("plane elimination: singular pivot block in a layer Schur complement")


def layered_grid_front(dims, axis, plane, conductivity=None, device=None,
                       dtype=None, return_torch=False):
    """Separator front of a scalar grid Laplacian by plane-by-plane elimination.

    ``conductivity`` is None (constant coefficients, the reference operator)
    or a cell array of shape dims+1 (see module docstring).  Returns the dense
    n x n front (numpy, or a torch tensor on ``device``) with rows ordered like
    src/frontgen.py:126-156 orders the separator.
    """
    F = layered_grid_fronts(dims, axis, plane, [conductivity], device=device, dtype=dtype)[0]
    if return_torch:
        return F
    return F.cpu().numpy()


class PlaneOperator:
    """The grid Laplacian of one or more conductivity fields, split into planes
    along `axis`: block tridiagonal with the in-plane operators T_t (nl x nl)
    on the diagonal and -diag(c_t) (the edges between planes t-1 and t) off it.
    Every field of a batch has the same stencil pattern, so the batch's plane
    operators are assembled with one scatter (leading batch axis)."""

    def __init__(self, dims, axis, conductivities, device=None, dtype=None):
        torch = _torch()
        self.dims = tuple(int(x) for x in dims)
        d = len(self.dims)
        if isinstance(axis, str):
            axis = AXIS_NAMES[axis]
        self.axis = axis
        self.ext = self.dims[axis]
        self.dev = torch.device(device or "cpu")
        self.dt = dtype or torch.float64
        # move the separator axis to the front; remaining axes keep their order
        self.perm = [axis] + [b for b in range(d) if b != axis]
        wls = []
        for kc in conductivities:
            w = _edge_weights(self.dims, kc)
            wls.append([np.transpose(w[b], self.perm) for b in range(d)])
        self.B = len(wls)
        self.layer_shape = tuple(self.dims[b] for b in self.perm[1:])
        self.nl = int(np.prod(self.layer_shape)) if self.layer_shape else 1
        self._ids = np.arange(self.nl).reshape(self.layer_shape)
        self._wlb = [np.stack([wl[b] for wl in wls]) for b in range(d)]

    def layer_matrix(self, t):
        """In-layer operators T_t of the batch (B x nl x nl)."""
        torch = _torch()
        B, nl, layer_shape, ids, wlb = self.B, self.nl, self.layer_shape, self._ids, self._wlb
        diag = np.zeros((B,) + layer_shape)
        # edges along the separator axis: t and t+1 (in w's indexing)
        wa = wlb[self.axis]
        diag += wa[:, t] + wa[:, t + 1]
        rows, cols, vals = [], [], []
        for j, b in enumerate(self.perm[1:]):
            wb = wlb[b][:, t]                     # (B, layer dims with +1 on axis j)
            n_b = layer_shape[j]
            lo = [slice(None)] * (len(layer_shape) + 1)
            hi = [slice(None)] * (len(layer_shape) + 1)
            lo[j + 1] = slice(0, n_b)
            hi[j + 1] = slice(1, n_b + 1)
            diag += wb[tuple(lo)] + wb[tuple(hi)]
            if n_b > 1:
                a_sl = [slice(None)] * len(layer_shape)
                a_sl[j] = slice(0, n_b - 1)
                inner = [slice(None)] * len(layer_shape)
                inner[j] = slice(1, n_b)
                src = ids[tuple(a_sl)].ravel()
                dst = ids[tuple(inner)].ravel()
                ww = wb[(slice(None),) + tuple(inner)].reshape(B, -1)
                rows += [src, dst]
                cols += [dst, src]
                vals += [-ww, -ww]
        T = torch.zeros((B, nl, nl), dtype=self.dt, device=self.dev)
        if rows:
            r = torch.from_numpy(np.concatenate(rows)).to(self.dev)
            c = torch.from_numpy(np.concatenate(cols)).to(self.dev)
            v = torch.from_numpy(np.concatenate(vals, axis=1)).to(device=self.dev, dtype=self.dt)
            T[:, r, c] = v
        idx = torch.arange(nl, device=self.dev)
        T[:, idx, idx] = torch.from_numpy(diag.reshape(B, nl)).to(device=self.dev, dtype=self.dt)
        return T

    def coupling(self, t):
        """Diagonals of the coupling between layers t-1 and t (edge t), B x nl."""
        torch = _torch()
        return torch.from_numpy(np.ascontiguousarray(self._wlb[self.axis][:, t]).reshape(self.B, -1)).to(
            device=self.dev, dtype=self.dt)

    def inverse(self, D):
        """D^{-1} for a (B, nl, nl) batch of SPD plane Schur complements: this
        library's block Gauss-Jordan on the GPU, torch.linalg.inv otherwise."""
        torch = _torch()
        if self.dev.type == "cuda" and self.dt == torch.float64 and frontgen_solver() == "hk":
            X = D.contiguous().clone()
            _spd_inverse_(X)
            return X
        return torch.linalg.inv(D)


def layered_grid_fronts(dims, axis, plane, conductivities, device=None, dtype=None):
    """The fronts of several conductivity fields of one grid (a batch of the
    multifrontal level of config 3), eliminated together: every plane step
    inverts the whole batch's layer Schur complements in one hk_spd_inverse
    call (block Gauss-Jordan on the DMMA GEMM) on the GPU.  Returns a
    (len(conductivities), n, n) torch tensor on ``device``."""
    torch = _torch()
    op = PlaneOperator(dims, axis, conductivities, device=device, dtype=dtype)
    ext = op.ext
    if not 0 < plane < ext - 1:
        raise InvalidPlaneError(f"plane {plane} is not strictly interior to extent {ext}")
    use_hk = op.dev.type == "cuda" and op.dt == torch.float64 and frontgen_solver() == "hk"

    def schur_term(D, c):
        """C D^{-1} C for the batch (C = diag(c)): this library's block
        Gauss-Jordan on the GPU, torch.linalg.solve (cuSOLVER / LAPACK) otherwise."""
        if use_hk:
            X = D.contiguous().clone()
            _spd_inverse_(X)
            return c[:, :, None] * X * c[:, None, :]
        return c[:, :, None] * torch.linalg.solve(D, torch.diag_embed(c))

    def eliminate(order):
        """Schur complement of the layers in ``order`` (far to near):
        D_k = T_k - C D_{k-1}^{-1} C with C the diagonal plane coupling."""
        D = None
        for k, t in enumerate(order):
            T = op.layer_matrix(t)
            if D is not None:
                T = T - schur_term(D, op.coupling(max(t, order[k - 1])))
            D = T
        return D

    front = op.layer_matrix(plane)
    left_layers = list(range(0, plane))
    right_layers = list(range(ext - 1, plane, -1))
    for layers in (left_layers, right_layers):
        if not layers:
            continue
        D = eliminate(layers)
        try:
            front = front - schur_term(D, op.coupling(max(plane, layers[-1])))
        except (RuntimeError, ValueError) as exc:
            raise SingularInteriorError(str(exc)) from exc
    return front


def grid_graph(spec: GridSpec, axis, plane) -> SparsePattern:
    """Separator subgraph relabelled to front order (frontgen.py:185)."""
    op = grid_operator(spec)
    sep, _, _ = planar_separator(spec, axis, plane)
    return op.induced(sep)


def grid_front(spec: GridSpec, axis, plane: int, rhs_seed: int = 0,
               device=None) -> FrontProblem:
    """Operator -> planar split -> Schur complement (frontgen.py:201-205).

    Scalar stencils use the layered elimination; the 3-component stencil is
    three uncoupled copies of the scalar operator, so its front is the scalar
    front with every entry expanded to a 3x3 identity block.
    """
    if isinstance(axis, str):
        if axis not in AXIS_NAMES:
            raise ValueError(f"axis must be one of {tuple(AXIS_NAMES)} or an integer")
        axis_i = AXIS_NAMES[axis]
    else:
        axis_i = axis
    sep, left, right = planar_separator(spec, axis_i, plane)
    scalar = layered_grid_front(spec.dims, axis_i, plane, device=device)
    dof = spec.dof_per_node
    front = scalar if dof == 1 else np.kron(scalar, np.eye(dof))
    graph = grid_graph(spec, axis_i, plane)
    rhs = np.random.default_rng(rhs_seed).standard_normal((sep.size, 1))
    return FrontProblem(np.ascontiguousarray(front), graph, sep.copy(), rhs)


def kernel_matrix(n: int, kind: str = "inv-distance", shift: float = 0.0) -> np.ndarray:
    """k(|i-j|) + shift*I (frontgen.py:208-218)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if kind not in KERNELS:
        raise ValueError(f"unknown kernel {kind!r}, expected one of {KERNELS}")
    dist = np.abs(np.arange(n)[:, None] - np.arange(n)[None, :]).astype(np.float64)
    a = 1.0 / (1.0 + dist) if kind == "inv-distance" else np.exp(-dist / 8.0)
    if shift:
        a = a + shift * np.eye(n)
    return a


# ---------------------------------------------------------------------------
# BASELINE config 2: unstructured-graph front (not in the reference; SURVEY.md
# §8(d) cfg 2 and Appendix A.3).  Points uniform in the unit cube, the union-
# symmetrised k-nearest-neighbour graph Laplacian L = D - W + shift*I, the slab
# S = {|x - 1/2| <= h} as the "separator" (not a true separator: a few kNN
# edges cross it, so every non-slab vertex is eliminated jointly), the front
# F = L_SS - L_SI L_II^{-1} L_IS, and S ordered by recursive coordinate
# bisection whose split sizes match build_tree's ceil(size/2).

@dataclass(frozen=True)
class KnnFront:
    """Dense slab front in RCB order, its induced kNN graph (same order), the
    slab vertex ids in that order, and generation diagnostics."""

    front: np.ndarray
    graph: SparsePattern
    ordering: np.ndarray
    info: dict

    @property
    def n(self) -> int:
        return self.front.shape[0]

    def accessor(self) -> BlockAccessor:
        return BlockAccessor.from_matrix(self.front, pattern=self.graph)


def knn_points(npoints: int, seed: int = 2) -> np.ndarray:
    """``default_rng(seed).random((npoints, 3))`` (BASELINE config 2)."""
    return np.random.default_rng(seed).random((int(npoints), 3))


def knn_graph(points: np.ndarray, k: int = 8, device=None, chunk: int = 2048) -> SparsePattern:
    """Union-symmetrised k-nearest-neighbour adjacency (no self loops).

    Exact squared distances (difference form, no |p|^2+|q|^2-2pq
    cancellation), the k smallest per point by a stable sort of
    (distance, index), so ties resolve to the lower index on any device.
    """
    torch = _torch()
    pts = np.ascontiguousarray(points, dtype=np.float64)
    npnt = pts.shape[0]
    if k < 1 or k >= npnt:
        raise ValueError("need 1 <= k < number of points")
    dev = torch.device(device or "cpu")
    if dev.type == "cpu":                  # host: a k-d tree gives the same neighbour sets
        from scipy.spatial import cKDTree
        _, nb = cKDTree(pts).query(pts, k + 1)
        nb = nb[:, 1:] if np.all(nb[:, 0] == np.arange(npnt)) else _drop_self(nb, k)
        return SparsePattern.from_edges(npnt, np.repeat(np.arange(npnt), k), nb.ravel())
    P = torch.from_numpy(pts).to(dev)
    nbr = np.empty((npnt, k), dtype=np.int64)
    for c0 in range(0, npnt, chunk):
        q = P[c0:c0 + chunk]
        d2 = ((q[:, None, 0] - P[None, :, 0]) ** 2 + (q[:, None, 1] - P[None, :, 1]) ** 2
              + (q[:, None, 2] - P[None, :, 2]) ** 2)
        rows = torch.arange(q.shape[0], device=dev)
        d2[rows, rows + c0] = float("inf")                      # no self loops
        # k + a margin of candidates, then an exact stable (distance, index) order
        cand_d, cand_i = torch.topk(d2, min(k + 8, npnt - 1), dim=1, largest=False, sorted=False)
        key_i, order = torch.sort(cand_i, dim=1)
        cand_d = torch.gather(cand_d, 1, order)
        _, o2 = torch.sort(cand_d, dim=1, stable=True)
        nbr[c0:c0 + q.shape[0]] = torch.gather(key_i, 1, o2)[:, :k].cpu().numpy()
    rows = np.repeat(np.arange(npnt), k)
    return SparsePattern.from_edges(npnt, rows, nbr.ravel())


def _drop_self(nb: np.ndarray, k: int) -> np.ndarray:
    out = np.empty((nb.shape[0], k), dtype=nb.dtype)
    for i, row in enumerate(nb):
        out[i] = row[row != i][:k]
    return out


def rcb_order(points: np.ndarray, leaf: int) -> np.ndarray:
    """Recursive coordinate bisection: split along the widest coordinate, the
    first ceil(size/2) points (stable sort by that coordinate, then index)
    going left, until a part has <= leaf points -- the split sizes of
    build_tree(n, leaf) (src/hodlr.py:76-102).  Returns positions into
    ``points``."""
    pts = np.asarray(points, dtype=np.float64)
    out = []
    stack = [np.arange(pts.shape[0])]
    while stack:
        idx = stack.pop()
        if idx.size <= leaf:
            out.append(idx)
            continue
        ext = pts[idx].max(axis=0) - pts[idx].min(axis=0)
        ax = int(np.argmax(ext))
        srt = idx[np.argsort(pts[idx, ax], kind="stable")]
        half = (idx.size + 1) // 2
        stack.append(srt[half:])
        stack.append(srt[:half])
    return np.concatenate(out) if out else np.zeros(0, dtype=np.intp)


def _laplacian_csr(graph: SparsePattern, shift: float):
    """L = D - W + shift*I as scipy CSR (unit edge weights)."""
    import scipy.sparse as sp
    n = graph.n
    deg = np.diff(graph.indptr).astype(np.float64)
    W = sp.csr_matrix((np.ones(graph.nnz), graph.indices, graph.indptr), shape=(n, n))
    return (sp.diags(deg + shift) - W).tocsr()


def _torch_csr(M, dev):
    torch = _torch()
    M = M.tocsr()
    return torch.sparse_csr_tensor(torch.from_numpy(M.indptr.astype(np.int64)),  # noqa
                                   torch.from_numpy(M.indices.astype(np.int64)),
                                   torch.from_numpy(M.data.astype(np.float64)), size=M.shape,
                                   dtype=torch.float64).to(dev)


def _cg_solve_block(L_II, L_IS, device, tol, max_iter):
    """Jacobi-preconditioned block CG (every column its own alpha/beta) for
    L_II X = L_IS on `device` in fp64 with torch sparse CSR products; the
    dense right-hand sides are formed on the device."""
    torch = _torch()
    dev = torch.device(device)
    A = _torch_csr(L_II, dev)
    dinv = torch.from_numpy(1.0 / L_II.diagonal()).to(dev)[:, None]
    Bt = _torch_csr(L_IS, dev).to_dense()
    X = torch.zeros_like(Bt)
    R = Bt.clone()
    Z = dinv * R
    Pm = Z.clone()
    rz = (R * Z).sum(0)
    bn = torch.linalg.vector_norm(Bt, dim=0).clamp_min(1e-300)
    its = 0
    for its in range(1, max_iter + 1):
        AP = A @ Pm
        pap = (Pm * AP).sum(0)
        alpha = torch.where(pap > 0, rz / torch.where(pap > 0, pap, 1.0), 0.0)
        X += alpha * Pm
        R -= alpha * AP
        rel = torch.linalg.vector_norm(R, dim=0) / bn
        if its % 10 == 0 and float(rel.max()) <= tol:
            break
        Z = dinv * R
        rz_new = (R * Z).sum(0)
        Pm = Z + torch.where(rz > 0, rz_new / torch.where(rz > 0, rz, 1.0), 0.0) * Pm
        rz = rz_new
    return X, its, float(rel.max())


def knn_front(npoints: int = 200000, k: int = 8, shift: float = 1e-3, h: float = 0.005,
              seed: int = 2, leaf: int = 64, device=None, solver: str = "auto",
              cg_tol: float = 1e-13, cg_max_iter: int = 20000) -> KnnFront:
    """BASELINE config 2 front (module note above).  ``solver``: "direct"
    (scipy SuperLU on the host; small problems), "cg" (block CG on `device`,
    the 200k-point case on a B200) or "auto" (direct below 40k interior
    vertices)."""
    import scipy.sparse.linalg as spla
    pts = knn_points(npoints, seed)
    graph = knn_graph(pts, k, device=device)
    L = _laplacian_csr(graph, shift)
    slab = np.flatnonzero(np.abs(pts[:, 0] - 0.5) <= h)
    if slab.size == 0:
        raise ValueError("empty slab")
    order = slab[rcb_order(pts[slab], leaf)]
    interior = np.setdiff1d(np.arange(npoints), order)
    L_SS = L[order][:, order].toarray()
    L_IS = L[interior][:, order].tocsc()
    L_II = L[interior][:, interior].tocsc()
    crossing = 0
    left = pts[interior, 0] < 0.5
    li = L[interior][:, interior].tocoo()
    crossing = int(np.count_nonzero(left[li.row] != left[li.col]))
    if solver == "auto":
        solver = "direct" if interior.size <= 40000 else "cg"
    info = {"npoints": int(npoints), "k": k, "shift": shift, "h": h, "n": int(order.size),
            "crossing_directed_edges": crossing, "solver": solver}
    if solver == "direct":
        X = spla.splu(L_II).solve(L_IS.toarray())
        front = L_SS - (L_IS.T @ X)
    else:
        torch = _torch()
        dev = torch.device(device or "cuda")
        Xt, its, rel = _cg_solve_block(L_II, L_IS, dev, cg_tol, cg_max_iter)
        info.update(cg_iterations=its, cg_rel_residual=rel)
        front = L_SS - (_torch_csr(L_IS.T, dev) @ Xt).cpu().numpy()
        del Xt
    return KnnFront(np.ascontiguousarray(front), graph.induced(order), order, info)
