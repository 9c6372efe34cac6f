"""HODLR tree, factorization and solve (reference src/hodlr.py) on the B200.

``factorize`` uploads the front once and runs the whole batched pipeline of
the native library (csrc/api.cpp): one launch compresses every off-diagonal
block, then a leaf pass and one upward sweep per level factor the hierarchy.
``solve`` applies the stored factorization on the device.  The factor stays
resident in HBM; the reference's test-visible attributes
(``leaf_lus[slot].lu``, ``couplings[slot].d_left`` ...) are materialised on
the host lazily, on first access.

``HodlrBatch`` is the batched device API behind BASELINE config 3: many
same-size fronts factored and solved by the same launches.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .dense import PartialPivLU, _row_perm_from_piv
from .errors import DimensionMismatchError
from .lowrank import CompressionConfig, compress_svd


@dataclass(frozen=True)
class TreeNode:
    level: int
    lo: int
    hi: int
    left: int = -1
    right: int = -1

    @property
    def size(self) -> int:
        return self.hi - self.lo

    @property
    def is_leaf(self) -> bool:
        return self.left < 0


@dataclass(frozen=True)
class HodlrTree:
    nodes: list
    leaf_threshold: int

    @property
    def n(self) -> int:
        return self.nodes[0].size

    @property
    def depth(self) -> int:
        return max(node.level for node in self.nodes)

    def internal_nodes(self):
        return [k for k, node in enumerate(self.nodes) if not node.is_leaf]

    def node_at(self, level: int, index: int) -> int:
        hits = sorted((k for k in self.internal_nodes() if self.nodes[k].level == level),
                      key=lambda k: self.nodes[k].lo)
        if index < 0 or index >= len(hits):
            raise IndexError(f"no internal node ({level}, {index})")
        return hits[index]


def build_tree(n: int, leaf_threshold: int) -> HodlrTree:
    """Balanced bisection (hodlr.py:76-102): split at ceil(size/2), leaf iff
    size <= threshold, nodes in preorder.  csrc/api.cpp builds the identical
    tree for the device (checked in tests/test_host.py)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if leaf_threshold < 1:
        raise ValueError("leaf_threshold must be >= 1")
    nodes: list = []
    todo = [(0, 0, n, -1, 0)]
    parents = {}
    while todo:
        level, lo, hi, parent, side = todo.pop()
        slot = len(nodes)
        nodes.append([level, lo, hi, -1, -1])
        if parent >= 0:
            nodes[parent][3 + side] = slot
        if hi - lo > leaf_threshold:
            mid = lo + (hi - lo + 1) // 2
            todo.append((level + 1, mid, hi, slot, 1))
            todo.append((level + 1, lo, mid, slot, 0))
    del parents
    return HodlrTree([TreeNode(*x) for x in nodes], leaf_threshold)


@dataclass(frozen=True)
class Coupling:
    """Per internal node: V factors, d blocks and the coupling LU (hodlr.py:105-134)."""

    v_upper: np.ndarray
    v_lower: np.ndarray
    d_left: np.ndarray
    d_right: np.ndarray
    schur_lu: PartialPivLU

    @property
    def rank_upper(self) -> int:
        return self.v_upper.shape[1]

    @property
    def rank_lower(self) -> int:
        return self.v_lower.shape[1]

    def correct(self, top: np.ndarray, bottom: np.ndarray):
        """Host restatement of the stored correction (used only for inspection)."""
        rhs = np.vstack([self.v_lower.T @ top, self.v_upper.T @ bottom])
        y = self.schur_lu.solve(rhs)
        y_low, y_up = y[:self.rank_lower], y[self.rank_lower:]
        return top - self.d_left @ y_up, bottom - self.d_right @ y_low


class _LazySlots:
    """List-like view that materialises per-slot host objects on demand."""

    def __init__(self, n, make):
        self._n = n
        self._make = make
        self._cache = {}

    def __len__(self):
        return self._n

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(self._n))]
        if k < 0:
            k += self._n
        if not 0 <= k < self._n:
            raise IndexError(k)
        if k not in self._cache:
            self._cache[k] = self._make(k)
        return self._cache[k]

    def __iter__(self):
        for k in range(self._n):
            yield self[k]


class _Plan:
    """Owns one native plan (tree + batch) and the device copy of its fronts."""

    def __init__(self, n, leaf, batch):
        N.require_cuda()
        h = N.P()
        N.check(N.lib().hk_plan_create(n, leaf, batch, N.C.byref(h)))
        self.h = h
        self.n, self.leaf, self.batch = n, leaf, batch
        self.fronts = None     # torch (batch, n, n) float64 on cuda
        self.nblocks = 0

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and N._LIB is not None:
            N.lib().hk_plan_destroy(h)
            self.h = None

    def ranks(self, nblocks):
        out = np.zeros(self.batch * nblocks, dtype=np.int32)
        N.check(N.lib().hk_get_ranks(self.h, N.arr_ptr(out, N.I32)))
        return out.reshape(self.batch, nblocks)

    def aca_seconds(self):
        t = N.D()
        N.check(N.lib().hk_get_aca_time(self.h, N.C.byref(t)))
        return t.value

    def timings(self):
        a, b, c = N.D(), N.D(), N.D()
        N.check(N.lib().hk_get_timings(self.h, N.C.byref(a), N.C.byref(b), N.C.byref(c)))
        return {"lowrank": a.value, "leaf_lu": b.value, "schur": c.value}


def _graph_in_front_order(front):
    """CSR (int64) of the front's graph with vertex i == front row i."""
    pattern = getattr(front, "pattern", None)
    if pattern is None:
        return None
    view = front.graph_view
    rv = np.asarray(view.row_verts, dtype=np.intp)
    cv = np.asarray(view.col_verts, dtype=np.intp) if view is not None else rv
    n = front.shape[0]
    if not np.array_equal(rv, cv):
        raise ValueError("bdlr factorization needs identical row and column vertex maps")
    if not (rv.size == pattern.n and np.array_equal(rv, np.arange(n))):
        pattern = pattern.induced(rv)
    return (np.ascontiguousarray(pattern.indptr, dtype=np.int64),
            np.ascontiguousarray(pattern.indices, dtype=np.int64))


def _front_graph_view(front):
    """front.graph_view without the row/col disjointness check of BlockGraphView
    (the whole front is not an off-diagonal block)."""
    class _V:
        pass
    v = _V()
    pattern = front.pattern
    rv = getattr(front, "_row_verts", None)
    cv = getattr(front, "_col_verts", None)
    n = front.shape[0]
    v.row_verts = np.arange(n) if rv is None else rv
    v.col_verts = np.arange(n) if cv is None else cv
    v.pattern = pattern
    return v


class HodlrFactorization:
    """Device-resident factorization with the reference's attribute surface
    (hodlr.py:137-154)."""

    def __init__(self, tree: HodlrTree, config: CompressionConfig, plan: _Plan, front_index=0,
                 ranks=None):
        self.tree = tree
        self.config = config
        self._plan = plan
        self._f = front_index
        self._ranks = ranks            # (nblocks,) for this front
        self._iidx = {s: k for k, s in enumerate(tree.internal_nodes())}
        self.leaf_lus = _LazySlots(len(tree.nodes), self._leaf_lu)
        self.couplings = _LazySlots(len(tree.nodes), self._coupling)

    @property
    def n(self) -> int:
        return self.tree.n

    @property
    def plan(self):
        return self._plan

    @property
    def front_index(self):
        return self._f

    def off_diagonal_ranks(self):
        out = []
        for s in self.tree.internal_nodes():
            k = self._iidx[s]
            out.append((self.tree.nodes[s].level + 1, int(self._ranks[2 * k]),
                        int(self._ranks[2 * k + 1])))
        return out

    def _leaf_lu(self, slot):
        node = self.tree.nodes[slot]
        if not node.is_leaf:
            return None
        b = node.size
        lu = np.zeros((b, b))
        inv = np.zeros((b, b))
        piv = np.zeros(b, dtype=np.int32)
        N.check(N.lib().hk_get_leaf_lu(self._plan.h, self._f, slot, N.arr_ptr(lu, N.D),
                                       N.arr_ptr(piv, N.I32), N.arr_ptr(inv, N.D)))
        piv = piv.astype(np.intp)
        return PartialPivLU(lu, piv, _row_perm_from_piv(piv), inv)

    def block_factor(self, block):
        m, n, cap = N.I64(), N.I64(), N.I64()
        N.check(N.lib().hk_block_shape(self._plan.h, block, N.C.byref(m), N.C.byref(n),
                                       N.C.byref(cap)))
        r = int(self._ranks[block])
        U = np.zeros(m.value * r)
        V = np.zeros(n.value * r)
        N.check(N.lib().hk_get_block_factor(self._plan.h, self._f, block, N.arr_ptr(U, N.D),
                                            N.arr_ptr(V, N.D)))
        return U.reshape(r, m.value).T.copy(), V.reshape(r, n.value).T.copy()

    def _coupling(self, slot):
        node = self.tree.nodes[slot]
        if node.is_leaf:
            return None
        k = self._iidx[slot]
        ru, rl = int(self._ranks[2 * k]), int(self._ranks[2 * k + 1])
        na = self.tree.nodes[node.left].size
        nb = self.tree.nodes[node.right].size
        _, v_up = self.block_factor(2 * k)
        _, v_low = self.block_factor(2 * k + 1)
        R = ru + rl
        dl = np.zeros((na, ru))
        dr = np.zeros((nb, rl))
        slu = np.zeros((R, R))
        sinv = np.zeros((R, R))
        sp = np.zeros(max(R, 1), dtype=np.int32)
        N.check(N.lib().hk_get_coupling(self._plan.h, self._f, slot, N.arr_ptr(dl, N.D),
                                        N.arr_ptr(dr, N.D), N.arr_ptr(slu, N.D),
                                        N.arr_ptr(sp, N.I32), N.arr_ptr(sinv, N.D)))
        piv = sp[:R].astype(np.intp)
        return Coupling(v_up, v_low, dl, dr, PartialPivLU(slu, piv, _row_perm_from_piv(piv), sinv))

    # device-side application (used by solve and the GMRES preconditioner)
    def solve_device(self, x, in_place=True):
        """Solve on a CUDA tensor shaped (n,) or (s, n) [column-major n x s]."""
        torch = N.require_cuda()
        t = x if in_place else x.clone()
        if t.dim() == 1:
            s = 1
        else:
            s = t.shape[0]
        if not t.is_contiguous():
            raise ValueError("device rhs must be contiguous")
        N.check(N.lib().hk_solve_front(self._plan.h, self._f, N.ptr(t), self.n, s,
                                       N.stream_handle()))
        del torch
        return t

    def __call__(self, r):
        """Act as the HODLR preconditioner M^{-1} r (numpy or CUDA tensor)."""
        return solve(self, r)


@dataclass
class SolveReport:
    """Per-level rank telemetry and per-phase times (hodlr.py:157-170)."""

    ranks_per_level: list = field(default_factory=list)
    timings: dict = field(default_factory=dict)
    residual: float | None = None

    def to_dict(self) -> dict:
        return {"ranks_per_level": self.ranks_per_level,
                "timings": {k: float(v) for k, v in self.timings.items()},
                "residual": self.residual}


def _ranks_summary(tree: HodlrTree, ranks_row) -> list:
    per_level: dict = {}
    for k, s in enumerate(tree.internal_nodes()):
        lvl = tree.nodes[s].level + 1
        per_level.setdefault(lvl, []).extend((int(ranks_row[2 * k]), int(ranks_row[2 * k + 1])))
    return [{"level": lvl, "max_rank": int(max(r)), "mean_rank": float(np.mean(r))}
            for lvl, r in sorted(per_level.items())]


def _upload_fronts(torch, fronts):
    if isinstance(fronts, torch.Tensor):
        t = fronts.to(device="cuda", dtype=torch.float64)
        return t.contiguous()
    return torch.from_numpy(np.ascontiguousarray(fronts, dtype=np.float64)).cuda()


def _build(plan: _Plan, tree: HodlrTree, cfg: CompressionConfig, fronts_dev, graph=None,
           trace=True):
    """Run the native build for every front of the plan."""
    n = plan.n
    st = N.stream_handle()
    ptr = N.ptr(fronts_dev)
    stride = n * n
    L = N.lib()
    nblocks = 2 * len(tree.internal_nodes())
    plan.nblocks = nblocks
    max_rank = cfg.max_rank or 0
    if cfg.scheme == "aca":
        N.check(L.hk_build_aca(plan.h, ptr, n, stride, cfg.tol, cfg.tol ** 2, max_rank,
                               1 if trace else 0, st))
    elif cfg.scheme == "bdlr":
        if graph is None:
            raise ValueError("bdlr compression requires a graph view on the block")
        ip, ix = graph
        N.check(L.hk_build_bdlr(plan.h, ptr, n, stride, cfg.tol, cfg.depth, max_rank,
                                N.arr_ptr(ip, N.I64), N.arr_ptr(ix, N.I64), st))
    else:  # svd: parity-only, per block through cuSOLVER
        torch = N.require_cuda()
        N.check(L.hk_build_external_begin(plan.h, ptr, n, stride, st))
        host = fronts_dev.cpu().numpy().reshape(plan.batch, n, n)
        from .lowrank import BlockAccessor
        for f in range(plan.batch):
            acc = BlockAccessor(host[f])
            for k, s in enumerate(tree.internal_nodes()):
                nd = tree.nodes[s]
                a, b = tree.nodes[nd.left], tree.nodes[nd.right]
                for side, (r0, r1, c0, c1) in enumerate(((a.lo, a.hi, b.lo, b.hi),
                                                          (b.lo, b.hi, a.lo, a.hi))):
                    fac = compress_svd(acc.block(np.arange(r0, r1), np.arange(c0, c1)), cfg)
                    r = fac.rank
                    if r == 0:
                        N.check(L.hk_set_block_factor(plan.h, f, 2 * k + side, 0, None, 1, None,
                                                      1, st))
                        continue
                    U = torch.from_numpy(np.ascontiguousarray(fac.u.T)).cuda()
                    V = torch.from_numpy(np.ascontiguousarray(fac.v.T)).cuda()
                    N.check(L.hk_set_block_factor(plan.h, f, 2 * k + side, r, N.ptr(U),
                                                  r1 - r0, N.ptr(V), c1 - c0, st))
    return plan.ranks(nblocks)


def factorize(front, tree: HodlrTree, cfg: CompressionConfig, threads: int = 1):
    """Factor a square front over a bisection tree (hodlr.py:183-208).

    ``threads`` is accepted for API compatibility; the device path is
    deterministic, so results are bit-identical for every value.
    """
    torch = N.require_cuda()
    m, n = front.shape
    if m != n or n != tree.n:
        raise DimensionMismatchError(f"front is {m}x{n}, tree expects {tree.n}x{tree.n}")
    A = np.ascontiguousarray(front.materialize(), dtype=np.float64)
    if A.size and not np.isfinite(A).all():
        raise ValueError("matrix contains NaN or Inf entries")
    graph = None
    if cfg.scheme == "bdlr":
        if getattr(front, "pattern", None) is None:
            raise ValueError("bdlr compression requires a graph view on the block")
        graph = _graph_in_front_order(_FrontGraph(front))
    plan = _Plan(n, tree.leaf_threshold, 1)
    dev = torch.from_numpy(A).cuda()
    plan.fronts = dev
    ranks = _build(plan, tree, cfg, dev, graph)
    N.check(N.lib().hk_factor(plan.h, N.stream_handle()))
    fact = HodlrFactorization(tree, cfg, plan, 0, ranks[0])
    report = SolveReport(ranks_per_level=_ranks_summary(tree, ranks[0]), timings=plan.timings())
    return fact, report


class _FrontGraph:
    """Adapter exposing a front accessor's pattern and vertex maps."""

    def __init__(self, front):
        self.pattern = front.pattern
        self.shape = front.shape
        self.graph_view = _front_graph_view(front)


def solve(fact: HodlrFactorization, rhs):
    """Solve against one or many right-hand sides (hodlr.py:285-306).

    numpy in -> numpy out (host copies around the device solve); a CUDA
    tensor shaped (n,) or (n, s) is solved on the device without host traffic.
    """
    torch = N.require_cuda()
    if isinstance(rhs, torch.Tensor) and rhs.is_cuda:
        if rhs.dim() not in (1, 2) or rhs.shape[0] != fact.n:
            raise DimensionMismatchError(f"rhs has shape {tuple(rhs.shape)}, expected ({fact.n}, s)")
        if rhs.dim() == 1:
            return fact.solve_device(rhs.to(torch.float64).clone())
        t = rhs.to(torch.float64).T.contiguous()      # (s, n) = column-major n x s
        fact.solve_device(t)
        return t.T.contiguous()
    b = np.asarray(rhs, dtype=np.float64)
    vector = b.ndim == 1
    if vector:
        b = b[:, None]
    if b.ndim != 2 or b.shape[0] != fact.n:
        raise DimensionMismatchError(f"rhs has shape {np.shape(rhs)}, expected ({fact.n}, s)")
    s = b.shape[1]
    if s == 0:
        x = np.zeros_like(b)
    else:
        t = torch.from_numpy(np.ascontiguousarray(b.T)).cuda()
        fact.solve_device(t)
        x = t.cpu().numpy().T.copy()
    return x[:, 0] if vector else x


def apply(front, x) -> np.ndarray:
    """Exact product with the original front on the device (hodlr.py:309-316)."""
    torch = N.require_cuda()
    a = front.materialize() if hasattr(front, "materialize") else np.asarray(front)
    a = np.ascontiguousarray(a, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    if x.shape[0] != a.shape[1]:
        raise DimensionMismatchError(f"operand has {x.shape[0]} rows, front has {a.shape[1]} columns")
    vector = x.ndim == 1
    xs = x[:, None] if vector else x
    m, n = a.shape
    s = xs.shape[1]
    if m == 0 or s == 0:
        out = np.zeros((m, s))
    else:
        at = torch.from_numpy(a).cuda()
        xt = torch.from_numpy(np.ascontiguousarray(xs.T)).cuda()
        yt = torch.empty((s, m), dtype=torch.float64, device="cuda")
        N.check(N.lib().hk_gemv(N.ptr(at), n, m, n, N.ptr(xt), n, s, N.ptr(yt), m,
                                N.stream_handle()))
        out = yt.cpu().numpy().T
    return out[:, 0].copy() if vector else out.copy()


def residual_norm(front, x, rhs) -> float:
    """||A x - b|| / ||b|| against the original front (hodlr.py:319-324)."""
    rhs = np.asarray(rhs, dtype=np.float64)
    num = np.linalg.norm(apply(front, x) - rhs)
    den = np.linalg.norm(rhs)
    return float(num / den) if den > 0 else float(num)


# ---------------------------------------------------------------- batched device API
class HodlrBatch:
    """Many same-size fronts factored by the same launches (BASELINE config 3).

    ``fronts`` is a CUDA tensor (batch, n, n) fp64 (row-major fronts).  All
    fronts share one bisection tree and one compression config.
    """

    def __init__(self, n: int, leaf_threshold: int, batch: int):
        self.tree = build_tree(n, leaf_threshold)
        self.plan = _Plan(n, leaf_threshold, batch)
        self.n, self.batch = n, batch
        self.ranks = None

    def factorize(self, fronts, cfg: CompressionConfig, graph=None, trace=False):
        torch = N.require_cuda()
        dev = _upload_fronts(torch, fronts)
        if tuple(dev.shape) != (self.batch, self.n, self.n):
            raise DimensionMismatchError(f"fronts must be ({self.batch}, {self.n}, {self.n})")
        self.plan.fronts = dev
        self.ranks = _build(self.plan, self.tree, cfg, dev, graph, trace=trace)
        N.check(N.lib().hk_factor(self.plan.h, N.stream_handle()))
        self.cfg = cfg
        return self

    def build_only(self, fronts, cfg, graph=None, trace=False):
        torch = N.require_cuda()
        dev = _upload_fronts(torch, fronts)
        self.plan.fronts = dev
        self.ranks = _build(self.plan, self.tree, cfg, dev, graph, trace=trace)
        self.cfg = cfg
        return self.ranks

    def factor_only(self):
        N.check(N.lib().hk_factor(self.plan.h, N.stream_handle()))

    def solve_(self, rhs):
        """In-place device solve of rhs shaped (batch, n) or (batch, s, n)
        (column-major n x s per front): a contiguous CUDA float64 tensor."""
        torch = N.require_cuda()
        if not isinstance(rhs, torch.Tensor) or not rhs.is_cuda or rhs.dtype != torch.float64:
            raise ValueError("rhs must be a CUDA float64 tensor")
        if not rhs.is_contiguous():
            raise ValueError("rhs must be contiguous")
        if rhs.dim() == 2 and tuple(rhs.shape) == (self.batch, self.n):
            s = 1
        elif rhs.dim() == 3 and rhs.shape[0] == self.batch and rhs.shape[2] == self.n:
            s = rhs.shape[1]
        else:
            raise DimensionMismatchError(f"rhs has shape {tuple(rhs.shape)}, expected "
                                         f"({self.batch}, {self.n}) or ({self.batch}, s, {self.n})")
        if self.ranks is None:
            raise ValueError("solve_ before factorize")
        N.check(N.lib().hk_solve(self.plan.h, N.ptr(rhs), self.n, s, self.n * s,
                                 N.stream_handle()))
        return rhs

    def run_host_stream(self, items, cfg: CompressionConfig):
        """Factor and solve a stream of host-resident batches (a multifrontal
        level streamed from host memory).

        ``items`` is a sequence of ``(fronts, rhs, out)`` CPU tensors -- pinned
        for asynchronous copies -- shaped (batch, n, n), (batch, n) and
        (batch, n).  The host->device copy of item i+1 runs on a copy stream
        while item i is built, factored and solved on the current stream (two
        device buffers), and each solution is copied back on the copy stream,
        so the PCIe transfer overlaps the compute.  Returns the per-front ranks
        of the last item.  Synchronises before returning.
        """
        torch = N.require_cuda()
        items = list(items)
        if not items:
            return self.ranks
        B, n = self.batch, self.n
        # both streams are pool streams (non-blocking): work on the legacy
        # default stream would serialise with the copies
        caller = torch.cuda.current_stream()
        comp = torch.cuda.Stream()
        copy = torch.cuda.Stream()
        comp.wait_stream(caller)
        copy.wait_stream(caller)
        dev_f = [torch.empty((B, n, n), dtype=torch.float64, device="cuda") for _ in range(2)]
        dev_r = [torch.empty((B, n), dtype=torch.float64, device="cuda") for _ in range(2)]
        loaded = [torch.cuda.Event() for _ in range(2)]
        solved = [torch.cuda.Event() for _ in range(2)]
        freed = [torch.cuda.Event() for _ in range(2)]
        used = [False, False]

        def load(i):
            slot = i % 2
            fr, rh, _ = items[i]
            if tuple(fr.shape) != (B, n, n) or tuple(rh.shape) != (B, n):
                raise DimensionMismatchError(f"item {i}: fronts must be ({B}, {n}, {n}), rhs ({B}, {n})")
            with torch.cuda.stream(copy):
                if used[slot]:
                    copy.wait_event(freed[slot])
                if fr.is_pinned() and fr.is_contiguous() and fr.dtype == torch.float64:
                    # a 4-SM copy kernel with evict-first stores: a DMA copy
                    # write-allocates in L2 and slowed the concurrent build ~2x
                    N.check(N.lib().hk_copy_h2d_streaming(N.C.c_void_p(fr.data_ptr()), N.ptr(dev_f[slot]),
                                                          fr.numel() * 8, 4,
                                                          N.C.c_void_p(copy.cuda_stream)))
                else:
                    dev_f[slot].copy_(fr, non_blocking=True)
                dev_r[slot].copy_(rh, non_blocking=True)
                loaded[slot].record(copy)
            used[slot] = True

        load(0)
        for i in range(len(items)):
            slot = i % 2
            if i + 1 < len(items):
                load(i + 1)
            with torch.cuda.stream(comp):
                comp.wait_event(loaded[slot])
                self.factorize(dev_f[slot], cfg)
                self.solve_(dev_r[slot])
                solved[slot].record(comp)
            with torch.cuda.stream(copy):
                copy.wait_event(solved[slot])
                items[i][2].copy_(dev_r[slot], non_blocking=True)
                freed[slot].record(copy)
        caller.wait_stream(copy)
        caller.wait_stream(comp)
        caller.synchronize()
        return self.ranks

    def factorization(self, f: int) -> HodlrFactorization:
        return HodlrFactorization(self.tree, self.cfg, self.plan, f, self.ranks[f])

    def report(self, f: int = 0) -> SolveReport:
        return SolveReport(ranks_per_level=_ranks_summary(self.tree, self.ranks[f]),
                           timings=self.plan.timings())

    def aca_trace(self, f: int, block: int):
        nb = len(self.tree.internal_nodes()) * 2
        assert 0 <= block < nb
        m, n, cap = N.I64(), N.I64(), N.I64()
        N.check(N.lib().hk_block_shape(self.plan.h, block, N.C.byref(m), N.C.byref(n),
                                       N.C.byref(cap)))
        rows = np.zeros(m.value + cap.value + 1, dtype=np.int32)
        cols = np.zeros(cap.value + 1, dtype=np.int32)
        nr, nc = N.I64(), N.I64()
        N.check(N.lib().hk_get_aca_trace(self.plan.h, f, block, N.arr_ptr(rows, N.I32),
                                         N.C.byref(nr), N.arr_ptr(cols, N.I32), N.C.byref(nc)))
        return rows[:nr.value].astype(np.int64), cols[:nc.value].astype(np.int64)

    def skeleton(self, f: int, block: int):
        m, n, cap = N.I64(), N.I64(), N.I64()
        N.check(N.lib().hk_block_shape(self.plan.h, block, N.C.byref(m), N.C.byref(n),
                                       N.C.byref(cap)))
        rows = np.zeros(max(cap.value, 1), dtype=np.int64)
        cols = np.zeros(max(cap.value, 1), dtype=np.int64)
        r = N.I64()
        N.check(N.lib().hk_get_skeleton(self.plan.h, f, block, N.C.byref(r),
                                        N.arr_ptr(rows, N.I64), N.arr_ptr(cols, N.I64), cap.value))
        return rows[:r.value].copy(), cols[:r.value].copy()


def factorize_traced(front, tree, cfg):
    """factorize() that also returns the per-block ACA traces / BDLR skeletons
    (parity instrumentation): (fact, report, {block: record})."""
    torch = N.require_cuda()
    A = np.ascontiguousarray(front.materialize(), dtype=np.float64)
    batch = HodlrBatch(A.shape[0], tree.leaf_threshold, 1)
    graph = None
    if cfg.scheme == "bdlr":
        graph = _graph_in_front_order(_FrontGraph(front))
    batch.factorize(torch.from_numpy(A)[None], cfg, graph=graph, trace=cfg.scheme == "aca")
    recs = {}
    for b in range(2 * len(tree.internal_nodes())):
        if cfg.scheme == "aca":
            recs[b] = batch.aca_trace(0, b)
        elif cfg.scheme == "bdlr":
            recs[b] = batch.skeleton(0, b)
    return batch.factorization(0), batch.report(0), recs
