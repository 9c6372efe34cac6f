"""HODLR-subtree sharding of one large front (BASELINE config 4).

G = 2**g ranks.  Rank r owns the level-g subtree T_r of the bisection tree
(rows [lo_r, hi_r)); the 2(G-1) blocks of the top g levels are shared.  The
reference's recursion (src/hodlr.py:217-282) splits exactly along this line:

* **Build.**  Each top-level block is compressed by one rank (round robin) and
  broadcast; every rank compresses the blocks inside its subtree locally.
* **Factor.**  _factorize_node passes every child the extension
  ``ext = [ancestors' U]`` restricted to the child's rows (hodlr.py:244-245), so
  rank r factors T_r with the external extension Z_r = the top ancestors' U on
  rows T_r (hk_factor_ext), which returns E_r = K_T^{-1} Z_r.  Then, for each
  top node p bottom-up, the coupling terms ``V_low^T d_left`` and
  ``V_up^T d_right`` (hodlr.py:269-271) -- together with the V^T-projection of
  the rest of the extension, H -- are sums over rows: every rank contributes
  its rows and one **all-reduce over the ranks under p** completes H.  The
  coupling system S is inverted redundantly in that group, and each rank
  applies ``c -= d y`` (hodlr.py:129-134) to its own rows of E.
* **Solve.**  The local levels run inside the rank's plan; each top node
  needs one all-reduce of its R x s projection ``V^T x`` (hodlr.py:298-306).
* **GMRES.**  A is row-slab partitioned (A[lo_r:hi_r] x, then an all-gather);
  the Arnoldi step runs redundantly on the replicated Krylov vectors.

Nothing else crosses ranks: per top level the collectives carry R x w
(factor) and R x s (solve) doubles.  The same orchestration runs over
``torch.distributed`` (one process per GPU, NCCL) or over G *emulated* ranks
in one process (``EmulatedRanks``): with fewer GPUs than ranks the ranks are
run one after the other on one device, and their collectives become sums over
the hosted ranks (no kernel waits on another rank).

Matrices are column-major; a column-major m x k matrix is held as a torch
tensor of shape (k, m) with unit inner stride ("cm" below).
"""

from __future__ import annotations

import math

import numpy as np

from .errors import DimensionMismatchError, SingularSchurError
from .hodlr import build_tree
from .krylov import GmresConfig, GmresResult


# ---------------------------------------------------------------- communicators
class EmulatedRanks:
    """All G ranks hosted by this process; collectives are fixed-order sums."""

    def __init__(self, world: int):
        self.world = world
        self.hosted = list(range(world))

    def allreduce(self, parts: dict, group) -> dict:
        total = None
        for r in sorted(group):
            total = parts[r].clone() if total is None else total + parts[r]
        return {r: (total if i == 0 else total.clone())
                for i, r in enumerate(r for r in sorted(group) if r in parts)}

    def allgather(self, parts: dict, sizes=None) -> list:
        return [parts[r] for r in range(self.world)]

    def broadcast(self, value, owner: int):
        return value


class TorchDistRanks:
    """One rank per process over torch.distributed (NCCL on GPUs, gloo on CPU).

    Process groups for every top-level node's rank set are created up front
    (every rank must create every group, in the same order)."""

    def __init__(self, g: int):
        import torch.distributed as dist
        self.dist = dist
        self.world = dist.get_world_size()
        if self.world != 1 << g:
            raise ValueError(f"world size {self.world} != 2**{g}")
        self.rank = dist.get_rank()
        self.hosted = [self.rank]
        self.groups = {}
        for level in range(g):
            span = self.world >> level
            for start in range(0, self.world, span):
                key = tuple(range(start, start + span))
                self.groups[key] = dist.new_group(list(key)) if span < self.world else None

    def allreduce(self, parts: dict, group) -> dict:
        t = parts[self.rank]
        key = tuple(sorted(group))
        self.dist.all_reduce(t, group=self.groups.get(key))
        return {self.rank: t}

    def allgather(self, parts: dict, sizes) -> list:
        """Gather every rank's (s, sizes[r]) block.  The sizes come from the
        tree (every rank knows them), so nothing but the data crosses ranks:
        one all_gather of blocks padded to the largest size."""
        import torch
        t = parts[self.rank]
        width = max(sizes)
        pad = t.new_zeros(t.shape[:-1] + (width,))
        pad[..., : t.shape[-1]] = t
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(outs, pad)
        return [o[..., :k] for o, k in zip(outs, sizes)]

    def broadcast(self, value, owner: int):
        """value: tuple of fp64 tensors on the owner (None elsewhere); returns it everywhere."""
        import torch
        dev = self._device()
        meta = torch.zeros(16, dtype=torch.int64, device=dev)
        if self.rank == owner:
            flat = [len(value)] + [d for v in value for d in (v.dim(), *v.shape)]
            meta[: len(flat)] = torch.tensor(flat, dtype=torch.int64)
        self.dist.broadcast(meta, src=owner)
        vals = meta.tolist()
        shapes, pos = [], 1
        for _ in range(vals[0]):
            d = vals[pos]
            shapes.append(tuple(vals[pos + 1: pos + 1 + d]))
            pos += 1 + d
        out = []
        for k, shp in enumerate(shapes):
            t = value[k].contiguous().to(dev) if self.rank == owner else \
                torch.empty(shp, dtype=torch.float64, device=dev)
            self.dist.broadcast(t, src=owner)
            out.append(t)
        return tuple(out)

    def _device(self):
        import torch
        return torch.device("cuda", torch.cuda.current_device()) \
            if self.dist.get_backend() == "nccl" else torch.device("cpu")


# ---------------------------------------------------------------- GPU local backend
class GpuBackend:
    """Per-rank device primitives: the rank's subtree plan and the C-ABI kernels."""

    def __init__(self, front, lo: int, hi: int, leaf: int):
        from . import _native as N
        from .hodlr import _Plan
        self.N = N
        self.torch = N.require_cuda()
        self.front = front                     # full n x n row-major cuda tensor (every rank)
        self.n = front.shape[0]
        self.lo, self.hi = lo, hi
        self.plan = _Plan(hi - lo, leaf, 1)

    # -- primitives used by the orchestration
    def compress(self, r0, r1, c0, c1, cfg):
        N, torch = self.N, self.torch
        m, k = r1 - r0, c1 - c0
        cap = min(m, k, cfg.max_rank or max(m, k))
        U = torch.empty((cap, m), dtype=torch.float64, device="cuda")
        V = torch.empty((cap, k), dtype=torch.float64, device="cuda")
        rank = N.I64(0)
        nr, nc = N.I64(0), N.I64(0)
        rows = np.zeros(m + cap + 1, dtype=np.int32)
        cols = np.zeros(cap + 1, dtype=np.int32)
        a = self.front[r0:, c0:]
        N.check(N.lib().hk_aca_block(N.ptr(a), m, k, self.n, cfg.tol ** 2, cap, N.ptr(U), N.ptr(V),
                                     N.C.byref(rank), N.arr_ptr(rows, N.I32), N.C.byref(nr),
                                     N.arr_ptr(cols, N.I32), N.C.byref(nc), N.stream_handle()))
        r = rank.value
        return U[:r].clone(), V[:r].clone()

    def build(self, cfg):
        N = self.N
        a = self.front[self.lo:, self.lo:]
        N.check(N.lib().hk_build_aca(self.plan.h, N.ptr(a), self.n, self.n * self.n, cfg.tol,
                                     cfg.tol ** 2, cfg.max_rank or 0, 0, N.stream_handle()))
        self.plan.fronts = self.front

    def factor_ext(self, Z):
        """Z: cm (wext, n_loc); returns E = K_T^{-1} Z as cm (wext, n_loc)."""
        N, torch = self.N, self.torch
        wext, nl = Z.shape
        Zc = Z.contiguous()
        N.check(N.lib().hk_factor_ext(self.plan.h, N.ptr(Zc) if wext else None, nl, wext,
                                      N.stream_handle()))
        E = torch.empty((wext, nl), dtype=torch.float64, device="cuda")
        if wext:
            N.check(N.lib().hk_copy_extension(self.plan.h, 0, 0, wext, N.ptr(E), nl,
                                              N.stream_handle()))
        return E

    def solve_local_(self, x):
        """x: (s, n_loc) contiguous = column-major n_loc x s; solved in place."""
        N = self.N
        s, nl = x.shape
        N.check(N.lib().hk_solve(self.plan.h, N.ptr(x), nl, s, nl * s, N.stream_handle()))
        return x

    def gemm(self, C, A, B, trans_a=False, alpha=1.0, beta=0.0):
        """C (cm n x m) = alpha op(A) B + beta C, all cm views with unit inner stride."""
        N = self.N
        if trans_a:
            k, m = A.shape[1], A.shape[0]
        else:
            k, m = A.shape[0], A.shape[1]
        n = B.shape[0]
        assert C.shape == (n, m) and B.shape[1] == k
        for t in (A, B, C):
            assert t.stride(1) == 1
        if m == 0 or n == 0:
            return C
        N.check(N.lib().hk_dgemm(1 if trans_a else 0, m, n, k, alpha, N.ptr(A), A.stride(0),
                                 N.ptr(B), B.stride(0), beta, N.ptr(C), C.stride(0),
                                 N.stream_handle()))
        return C

    def inverse(self, S):
        """S: cm (R, R); returns S^{-1} (cm).  Singular -> SingularSchurError."""
        N, torch = self.N, self.torch
        R = S.shape[0]
        a = S.t().contiguous()                 # row-major copy
        inv = torch.empty_like(a)
        perm = torch.empty(R, dtype=torch.int32, device="cuda")
        try:
            N.check(N.lib().hk_lu_partial(N.ptr(a), R, R, N.ptr(perm), N.ptr(inv),
                                          N.stream_handle()))
        except Exception as exc:              # SingularMatrixError from the kernel
            raise SingularSchurError(f"top-level coupling system singular: {exc}") from exc
        return inv.t().contiguous()            # row-major inverse -> cm

    def rows_matvec(self, X):
        """A[lo:hi, :] X for X (s, n) (row slab of the dense front); (s, rows)."""
        N, torch = self.N, self.torch
        s = X.shape[0]
        rows = self.hi - self.lo
        y = torch.empty((s, rows), dtype=torch.float64, device="cuda")
        a = self.front[self.lo:]
        N.check(N.lib().hk_gemv(N.ptr(a), self.n, rows, self.n, N.ptr(X), self.n, s,
                                N.ptr(y), rows, N.stream_handle()))
        return y


# ---------------------------------------------------------------- orchestration
class _Top:
    """A top-level node p with its two shared block factors."""

    def __init__(self, slot, node, a, b):
        self.slot, self.node, self.a, self.b = slot, node, a, b
        self.Uu = self.Vu = self.Ul = self.Vl = None   # cm tensors (rank, rows)
        self.Sinv = {}                                  # per hosted rank (redundant)

    @property
    def ru(self):
        return self.Uu.shape[0]

    @property
    def rl(self):
        return self.Ul.shape[0]


class ShardedHodlr:
    """Factor, solve and GMRES of one front sharded over G = 2**g HODLR subtrees."""

    def __init__(self, front, leaf: int, comm, backend_factory=GpuBackend):
        self.front = front
        self.n = front.shape[0]
        self.G = comm.world
        self.g = int(round(math.log2(self.G)))
        if 1 << self.g != self.G:
            raise ValueError("the number of ranks must be a power of two")
        self.comm = comm
        self.tree = build_tree(self.n, leaf)
        nodes = self.tree.nodes
        # level-g subtree roots in row order; every node above them must be internal
        frontier = [0]
        for _ in range(self.g):
            nxt = []
            for s in frontier:
                if nodes[s].is_leaf:
                    raise ValueError(f"tree too shallow for {self.G} subtrees")
                nxt += [nodes[s].left, nodes[s].right]
            frontier = nxt
        self.owned = frontier
        self.tops = []
        for s, nd in enumerate(nodes):
            if nd.level < self.g:
                self.tops.append(_Top(s, nd, nodes[nd.left], nodes[nd.right]))
        self.local = {}
        for r in comm.hosted:
            nd = nodes[self.owned[r]]
            self.local[r] = backend_factory(front, nd.lo, nd.hi, leaf)
        self.E = {}
        self._factored = False

    # rank sets and sides ------------------------------------------------------
    def ranks_under(self, nd):
        return [r for r in range(self.G) if nd.lo <= self.tree.nodes[self.owned[r]].lo < nd.hi]

    def side_of(self, top, r):
        lo = self.tree.nodes[self.owned[r]].lo
        if top.a.lo <= lo < top.a.hi:
            return 0
        if top.b.lo <= lo < top.b.hi:
            return 1
        return -1

    def _path(self, r):
        """Top ancestors of rank r's subtree, root first, with side and column offset."""
        out, w = [], 0
        for top in sorted(self.tops, key=lambda t: t.node.level):
            side = self.side_of(top, r)
            if side < 0:
                continue
            width = top.ru if side == 0 else top.rl
            out.append((top, side, w, width))
            w += width
        return out

    # factorize ----------------------------------------------------------------
    def factorize(self, cfg):
        torch = self._torch()
        hosted = self.comm.hosted
        # top-level blocks: round robin over the ranks, then shared
        jobs = []
        for top in self.tops:
            jobs.append((top, 0))
            jobs.append((top, 1))
        for j, (top, side) in enumerate(jobs):
            owner = j % self.G
            a, b = top.a, top.b
            r0, r1, c0, c1 = (a.lo, a.hi, b.lo, b.hi) if side == 0 else (b.lo, b.hi, a.lo, a.hi)
            val = None
            if owner in hosted:
                val = self.local[owner].compress(r0, r1, c0, c1, cfg)
            U, V = self.comm.broadcast(val, owner)
            if side == 0:
                top.Uu, top.Vu = U, V
            else:
                top.Ul, top.Vl = U, V
        for r in hosted:
            self.local[r].build(cfg)
        # local subtree factorization with the external extension
        for r in hosted:
            nd = self.tree.nodes[self.owned[r]]
            path = self._path(r)
            wext = sum(p[3] for p in path)
            Z = torch.empty((wext, nd.hi - nd.lo), dtype=torch.float64, device=self.front.device)
            for top, side, w, width in path:
                child = top.a if side == 0 else top.b
                U = top.Uu if side == 0 else top.Ul
                Z[w:w + width] = U[:, nd.lo - child.lo: nd.hi - child.lo]
            self.E[r] = self.local[r].factor_ext(Z)
        # top levels, deepest first: H partials -> all-reduce -> S^-1 -> c -= d y
        for level in range(self.g - 1, -1, -1):
            for top in [t for t in self.tops if t.node.level == level]:
                group = self.ranks_under(top.node)
                mine = [r for r in hosted if r in group]
                if not mine:
                    continue
                ru, rl = top.ru, top.rl
                R = ru + rl
                parts = {}
                for r in mine:
                    _, side, w, _ = next(p for p in self._path(r) if p[0] is top)
                    hcols = w + max(ru, rl)
                    H = torch.zeros((hcols, R), dtype=torch.float64, device=self.front.device)
                    nd = self.tree.nodes[self.owned[r]]
                    E = self.E[r]
                    if side == 0 and rl > 0:      # H[0:rl, 0:w+ru] = V_low^T E[:, 0:w+ru]
                        Vl = top.Vl[:, nd.lo - top.a.lo: nd.hi - top.a.lo]
                        self.local[r].gemm(H[: w + ru, 0:rl], Vl, E[: w + ru], trans_a=True)
                    if side == 1 and ru > 0:      # H[rl:R, 0:w+rl] = V_up^T E[:, 0:w+rl]
                        Vu = top.Vu[:, nd.lo - top.b.lo: nd.hi - top.b.lo]
                        self.local[r].gemm(H[: w + rl, rl:R], Vu, E[: w + rl], trans_a=True)
                    parts[r] = H
                full = self.comm.allreduce(parts, group)
                for r in mine:
                    H = full[r]
                    _, side, w, _ = next(p for p in self._path(r) if p[0] is top)
                    S = torch.eye(R, dtype=torch.float64, device=self.front.device)
                    # cm S: column j holds S[:, j]; X = H[0:rl, w:w+ru], Yc = H[rl:R, w:w+rl]
                    if ru and rl:
                        S[rl:R, 0:rl] = H[w:w + ru, 0:rl]        # X block: rows 0:rl, cols rl:R
                        S[0:rl, rl:R] = H[w:w + rl, rl:R]        # Yc block: rows rl:R, cols 0:rl
                    Sinv = self.local[r].inverse(S)
                    top.Sinv[r] = Sinv
                    if w > 0:
                        Q = torch.empty((w, R), dtype=torch.float64, device=self.front.device)
                        self.local[r].gemm(Q, Sinv, H[:w])   # Q = S^-1 H[:, 0:w]
                        E = self.E[r]
                        if side == 0 and ru > 0:          # top -= d_left y_up
                            self.local[r].gemm(E[:w], E[w:w + ru], Q[:, rl:R].contiguous(),
                                               alpha=-1.0, beta=1.0)
                        if side == 1 and rl > 0:          # bottom -= d_right y_low
                            self.local[r].gemm(E[:w], E[w:w + rl], Q[:, 0:rl].contiguous(),
                                               alpha=-1.0, beta=1.0)
        self._factored = True
        return self

    # solve ---------------------------------------------------------------------
    def _sizes(self):
        return [self.tree.nodes[self.owned[r]].size for r in range(self.G)]

    def solve(self, x):
        """HODLR solve of a full (n,) right-hand side; returns the full solution."""
        if x.shape != (self.n,):
            raise DimensionMismatchError(f"rhs has shape {tuple(x.shape)}, expected ({self.n},)")
        return self.solve_batch(x[None])[0]

    def solve_batch(self, X):
        """HODLR solve of s right-hand sides X (s, n) (row c = rhs c); (s, n).
        Per top node one all-reduce of the R x s projection V^T x."""
        if not self._factored:
            raise RuntimeError("solve requires factorize()")
        if X.dim() != 2 or X.shape[1] != self.n:
            raise DimensionMismatchError(f"rhs has shape {tuple(X.shape)}, expected (s, {self.n})")
        torch = self._torch()
        hosted = self.comm.hosted
        s = X.shape[0]
        xl = {}
        for r in hosted:
            nd = self.tree.nodes[self.owned[r]]
            xr = torch.empty((s, nd.hi - nd.lo), dtype=torch.float64, device=X.device)
            xr.copy_(X[:, nd.lo:nd.hi])           # a private copy: solved in place
            xl[r] = self.local[r].solve_local_(xr)
        for level in range(self.g - 1, -1, -1):
            for top in [t for t in self.tops if t.node.level == level]:
                group = self.ranks_under(top.node)
                mine = [r for r in hosted if r in group]
                if not mine:
                    continue
                ru, rl = top.ru, top.rl
                R = ru + rl
                parts = {}
                for r in mine:
                    _, side, w, _ = next(p for p in self._path(r) if p[0] is top)
                    nd = self.tree.nodes[self.owned[r]]
                    gp = torch.zeros((s, R), dtype=torch.float64, device=self.front.device)
                    if side == 0 and rl > 0:
                        Vl = top.Vl[:, nd.lo - top.a.lo: nd.hi - top.a.lo]
                        self.local[r].gemm(gp[:, 0:rl], Vl, xl[r], trans_a=True)
                    if side == 1 and ru > 0:
                        Vu = top.Vu[:, nd.lo - top.b.lo: nd.hi - top.b.lo]
                        self.local[r].gemm(gp[:, rl:R], Vu, xl[r], trans_a=True)
                    parts[r] = gp
                full = self.comm.allreduce(parts, group)
                for r in mine:
                    _, side, w, _ = next(p for p in self._path(r) if p[0] is top)
                    y = torch.empty((s, R), dtype=torch.float64, device=self.front.device)
                    self.local[r].gemm(y, top.Sinv[r], full[r])
                    E = self.E[r]
                    if side == 0 and ru > 0:
                        self.local[r].gemm(xl[r], E[w:w + ru], y[:, rl:R].contiguous(),
                                           alpha=-1.0, beta=1.0)
                    if side == 1 and rl > 0:
                        self.local[r].gemm(xl[r], E[w:w + rl], y[:, 0:rl].contiguous(),
                                           alpha=-1.0, beta=1.0)
        return torch.cat(self.comm.allgather(xl, self._sizes()), dim=1)

    def apply(self, x):
        """Dense product A x with row-slab ownership (src/cli.py:320-321)."""
        return self.apply_batch(x[None])[0]

    def apply_batch(self, X):
        """A X for X (s, n): each rank multiplies its row slab, one all-gather."""
        torch = self._torch()
        X = X.contiguous()
        parts = {r: self.local[r].rows_matvec(X) for r in self.comm.hosted}
        return torch.cat(self.comm.allgather(parts, self._sizes()), dim=1)

    def gmres(self, b, cfg: GmresConfig) -> GmresResult:
        """Left-preconditioned GMRES with the sharded operator and preconditioner;
        the Arnoldi step runs redundantly on the replicated Krylov vectors."""
        return self.gmres_batch(b.reshape(-1, 1), cfg)[0]

    def gmres_batch(self, B, cfg: GmresConfig) -> list:
        """GMRES for the columns of B (n x s) in lock step: per iteration one
        sharded GEMV and one sharded solve carry all s columns, so the
        collectives per iteration do not grow with s."""
        from .krylov import gmres_device_batch
        torch = self._torch()
        Bt = B.t() if isinstance(B, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(B).T))
        return gmres_device_batch(self.apply_batch, Bt.to(self.front.device), cfg, self.solve_batch)

    def _torch(self):
        import torch
        return torch
