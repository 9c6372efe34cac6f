"""CPU oracle for the HODLR hot path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this module, and only as
the checker / the timed CPU baseline.  The product package
(``paper_1403_5337_b200``) never imports it.

This is a from-scratch numpy restatement of the reference algorithm
(``hodlrkit`` 0.1.0, /root/reference/pkg/src/hodlrkit).  Every function cites
the reference lines it follows.  The elementwise arithmetic that decides
pivots (ACA residual updates, complete-pivot Schur updates) is written so that
numpy evaluates exactly the same IEEE operations in the same order as the
reference: a separate multiply followed by a separate subtract, no fused
multiply-add, first-index argmax tie-breaks.  LAPACK-backed steps (getrf,
getrs, trsm, gesdd) call the same scipy/numpy routines the reference calls.

Parity pin: ``tests/test_oracle_golden.py`` checks this module against the
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``): ACA pivot traces, ranks and U/V factors
bit-exact, BDLR skeletons bit-exact, solves and GMRES results to tolerance.
"""

from __future__ import annotations

from collections import deque

import numpy as np
import scipy.linalg as sla

PIVOT_FLOOR = 1e-300          # src/dense.py:19


# ---------------------------------------------------------------------------
# bisection tree  (src/hodlr.py:76-102)
# ---------------------------------------------------------------------------

def bisection_tree(n: int, leaf: int):
    """Preorder node list of (level, lo, hi, left_slot, right_slot).

    Split point ceil(size/2) and the leaf rule size <= leaf follow
    src/hodlr.py:88-99.
    """
    if n < 1 or leaf < 1:
        raise ValueError("n and leaf must be >= 1")
    out = []
    stack = [(0, 0, n, -1, None)]      # (level, lo, hi, parent_slot, side)
    # explicit preorder walk
    while stack:
        level, lo, hi, parent, side = stack.pop()
        slot = len(out)
        out.append([level, lo, hi, -1, -1])
        if parent >= 0:
            out[parent][3 if side == 0 else 4] = slot
        if hi - lo > leaf:
            mid = lo + (hi - lo + 1) // 2
            stack.append((level + 1, mid, hi, slot, 1))
            stack.append((level + 1, lo, mid, slot, 0))
    return [tuple(x) for x in out]


# ---------------------------------------------------------------------------
# adaptive cross approximation  (src/lowrank.py:230-286)
# ---------------------------------------------------------------------------

def aca(block: np.ndarray, tol: float, max_rank=None, trace=None):
    """Partially pivoted ACA of a dense m x n block.

    Returns (U m x r, V n x r).  ``trace`` (a list) receives ('r', i) for every
    row the reference reads and ('c', j) for every column, in order -- the
    skeleton-index record the GPU path must reproduce bit for bit.
    """
    block = np.asarray(block, dtype=np.float64)
    m, n = block.shape
    cap = min(m, n) if max_rank is None else min(m, n, max_rank)   # :198-202
    if m == 0 or n == 0 or cap == 0:
        return np.zeros((m, 0)), np.zeros((n, 0))
    ucols = np.empty((cap, m))
    vcols = np.empty((cap, n))
    rank = 0
    visited = np.zeros(m, dtype=bool)
    fro2 = 0.0
    tol2 = tol ** 2
    row = 0
    while rank < cap:
        visited[row] = True
        if trace is not None:
            trace.append(("r", row))
        resid = np.array(block[row, :], dtype=np.float64)
        for k in range(rank):                     # :254-255, k-ordered, no FMA
            resid -= ucols[k, row] * vcols[k]
        col = int(np.argmax(np.abs(resid)))       # first index on ties
        piv = resid[col]
        if piv == 0.0:                            # :258-264 restart
            free = np.flatnonzero(~visited)
            if free.size == 0:
                break
            row = int(free[0])
            continue
        vnew = resid / piv
        if trace is not None:
            trace.append(("c", col))
        unew = np.array(block[:, col], dtype=np.float64)
        for k in range(rank):                     # :267-268
            unew -= vcols[k, col] * ucols[k]
        cross = float(unew @ unew) * float(vnew @ vnew)        # :269
        est = fro2 + cross
        for k in range(rank):                     # :271-272
            est += 2.0 * float(unew @ ucols[k]) * float(vnew @ vcols[k])
        est = max(est, cross)
        if cross <= tol2 * est:                   # :274-275 discard and stop
            break
        ucols[rank] = unew
        vcols[rank] = vnew
        rank += 1
        fro2 = est
        free = np.flatnonzero(~visited)
        if free.size == 0:
            break
        row = int(free[np.argmax(np.abs(unew[free]))])       # :283
    return ucols[:rank].T.copy(), vcols[:rank].T.copy()


# ---------------------------------------------------------------------------
# complete-pivoting LU  (src/dense.py:133-166, numerical_rank :104-108)
# ---------------------------------------------------------------------------

def complete_pivot_lu(a: np.ndarray):
    """Returns (packed lu, row_perm, col_perm, pivot magnitudes)."""
    w = np.array(a, dtype=np.float64)
    m, n = w.shape
    rp = np.arange(m)
    cp = np.arange(n)
    mags = []
    for k in range(min(m, n)):
        tail = np.abs(w[k:, k:])
        flat = int(np.argmax(tail))               # row-major, first occurrence
        pr, pc = divmod(flat, n - k)
        if tail[pr, pc] == 0.0:
            break
        pr += k
        pc += k
        if pr != k:
            w[[k, pr]] = w[[pr, k]]
            rp[[k, pr]] = rp[[pr, k]]
        if pc != k:
            w[:, [k, pc]] = w[:, [pc, k]]
            cp[[k, pc]] = cp[[pc, k]]
        p = w[k, k]
        mags.append(abs(p))
        if k + 1 < m:
            w[k + 1:, k] /= p
            w[k + 1:, k + 1:] -= np.outer(w[k + 1:, k], w[k, k + 1:])
    return w, rp, cp, np.asarray(mags)


def rank_from_pivots(mags: np.ndarray, tol: float) -> int:
    if mags.size == 0:
        return 0
    return int(np.count_nonzero(mags >= tol * mags[0]))


# ---------------------------------------------------------------------------
# graph selection  (src/graph.py:55-99, 171-228)
# ---------------------------------------------------------------------------

def csr_symmetric(n, rows, cols):
    """Union-symmetrised CSR adjacency without self loops (graph.py:55-99)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    keep = rows != cols
    a = np.concatenate([rows[keep], cols[keep]])
    b = np.concatenate([cols[keep], rows[keep]])
    if a.size:
        key = np.unique(a * n + b)
        a, b = key // n, key % n
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(indptr, a + 1, 1)
    indptr = np.cumsum(indptr)
    return indptr, b.astype(np.int64)


def boundary_of(indptr, indices, own, other, nverts):
    """Sorted own-side vertices with a neighbour on the other side (:171-180)."""
    mark = np.zeros(nverts, dtype=bool)
    mark[np.asarray(other, dtype=np.int64)] = True
    hits = [int(v) for v in own if mark[indices[indptr[v]:indptr[v + 1]]].any()]
    return np.asarray(sorted(hits), dtype=np.int64)


def side_distances(indptr, indices, own, other, nverts):
    """Multi-source BFS restricted to the own side (:183-206); inf = unreached."""
    own = np.asarray(own, dtype=np.int64)
    where = np.full(nverts, -1, dtype=np.int64)
    where[own] = np.arange(own.size)
    dist = np.full(own.size, np.inf)
    q = deque()
    for v in boundary_of(indptr, indices, own, other, nverts):
        dist[where[v]] = 0.0
        q.append(int(v))
    while q:
        v = q.popleft()
        dv = dist[where[v]]
        for u in indices[indptr[v]:indptr[v + 1]]:
            k = where[u]
            if k >= 0 and dist[k] == np.inf:
                dist[k] = dv + 1.0
                q.append(int(u))
    return dist


def depth_selection(indptr, indices, row_verts, col_verts, depth, nverts):
    """Block positions within ``depth`` of the interface, ordered by (d, id).

    Returns None when either side is empty (EmptySelectionError, :226-227).
    """
    picks = []
    for own, other in ((row_verts, col_verts), (col_verts, row_verts)):
        own = np.asarray(own, dtype=np.int64)
        d = side_distances(indptr, indices, own, other, nverts)
        pos = np.flatnonzero(d <= depth)
        order = np.lexsort((own[pos], d[pos]))
        picks.append(pos[order].astype(np.int64))
    if picks[0].size == 0 or picks[1].size == 0:
        return None
    return picks[0], picks[1]


# ---------------------------------------------------------------------------
# pseudo-skeleton  (src/lowrank.py:289-350)
# ---------------------------------------------------------------------------

class DegenerateSkeleton(Exception):
    pass


def skeleton(block: np.ndarray, row_sel, col_sel, tol, max_rank=None, info=None):
    """Complete-pivot skeleton factor (U m x r, V n x r) of a dense block."""
    block = np.asarray(block, dtype=np.float64)
    m, n = block.shape
    row_sel = np.asarray(row_sel, dtype=np.int64)
    col_sel = np.asarray(col_sel, dtype=np.int64)
    rsel = block[row_sel, :]
    core = rsel[:, col_sel]
    lu, rp, cp, mags = complete_pivot_lu(core)
    r = rank_from_pivots(mags, tol)
    if max_rank is not None:
        r = min(r, max_rank)
    if info is not None:
        info.update(rank=r, row_perm=rp, col_perm=cp, pivots=mags,
                    rows=row_sel[rp[:r]], cols=col_sel[cp[:r]])
    if r == 0:
        # :322-331 probe rows against tol * max|core|
        probe = np.unique(np.linspace(0, m - 1, num=min(m, 8), dtype=np.intp))
        seen = np.abs(block[probe, :]).max() if probe.size else 0.0
        lim = tol * (np.abs(core).max() if core.size else 0.0)
        if seen > lim:
            raise DegenerateSkeleton(f"rank-0 skeleton, sampled {seen:.3e} > {lim:.3e}")
        return np.zeros((m, 0)), np.zeros((n, 0))
    upper = np.triu(lu[:r, :r])
    lower = np.tril(lu[:r, :r], -1) + np.eye(r)
    cblk = block[:, col_sel[cp[:r]]]
    ct = sla.solve_triangular(upper, cblk.T, lower=False, trans="T", check_finite=False).T
    rt = sla.solve_triangular(lower, rsel[rp[:r]], lower=True, unit_diagonal=True,
                              check_finite=False)
    return ct, rt.T.copy()


def truncated_svd(block: np.ndarray, tol, max_rank=None):
    """src/lowrank.py:205-227 (gesdd through numpy)."""
    block = np.asarray(block, dtype=np.float64)
    m, n = block.shape
    u, s, vt = np.linalg.svd(block, full_matrices=False)
    if s.size == 0 or s[0] == 0.0:
        return np.zeros((m, 0)), np.zeros((n, 0))
    small = np.flatnonzero(s <= tol * s[0])
    k = int(small[0]) if small.size else s.size
    cap = min(m, n) if max_rank is None else min(m, n, max_rank)
    k = min(k, cap)
    return u[:, :k] * s[:k], vt[:k].T.copy()


# ---------------------------------------------------------------------------
# HODLR factorization and solve  (src/hodlr.py:183-306)
# ---------------------------------------------------------------------------

class OracleFactorization:
    def __init__(self, n, nodes):
        self.n = n
        self.nodes = nodes
        self.leaf = {}        # slot -> (lu, piv)
        self.cpl = {}         # slot -> dict(v_up, v_low, d_left, d_right, lu, piv)
        self.factors = {}     # slot -> (upper (U, V), lower (U, V))
        self.traces = {}      # slot -> (upper trace, lower trace) for ACA
        self.skeletons = {}   # slot -> (upper info, lower info) for BDLR


class SingularLeaf(Exception):
    pass


class SingularSchur(Exception):
    pass


def _getrf(a):
    lu, piv = sla.lu_factor(a, check_finite=False)
    if a.shape[0] and np.min(np.abs(np.diag(lu))) < PIVOT_FLOOR:
        raise ValueError("singular")
    return lu, piv


def _getrs(f, b):
    lu, piv = f
    if lu.shape[0] == 0 or b.shape[1] == 0:
        return np.zeros_like(b)
    return sla.lu_solve((lu, piv), b, check_finite=False)


def compress_block(A, r0, r1, c0, c1, scheme, tol, depth=1, max_rank=None,
                   graph=None, record=None):
    """Compress A[r0:r1, c0:c1] with the named scheme (src/lowrank.py:353-359)."""
    blk = A[r0:r1, c0:c1]
    if scheme == "aca":
        tr = [] if record is not None else None
        u, v = aca(blk, tol, max_rank, trace=tr)
        if record is not None:
            record["trace"] = tr
        return u, v
    if scheme == "svd":
        return truncated_svd(blk, tol, max_rank)
    if scheme == "bdlr":
        indptr, indices = graph
        nverts = len(indptr) - 1
        sel = depth_selection(indptr, indices, np.arange(r0, r1), np.arange(c0, c1),
                              depth, nverts)
        m, n = blk.shape
        if sel is None:
            if record is not None:
                record["info"] = None
            return np.zeros((m, 0)), np.zeros((n, 0))
        info = {}
        cap = min(m, n) if max_rank is None else min(m, n, max_rank)
        out = skeleton(blk, sel[0], sel[1], tol, cap, info=info)
        if record is not None:
            record["info"] = info
        return out
    raise ValueError(scheme)


def factorize(A, leaf, scheme, tol, depth=1, max_rank=None, graph=None):
    """Depth-first recursion with the carried extension block (hodlr.py:217-282)."""
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    nodes = bisection_tree(n, leaf)
    fact = OracleFactorization(n, nodes)

    def visit(slot, ext):
        level, lo, hi, left, right = nodes[slot]
        if left < 0:
            try:
                f = _getrf(A[lo:hi, lo:hi])
            except ValueError:
                raise SingularLeaf(f"leaf [{lo},{hi})") from None
            fact.leaf[slot] = f
            return _getrs(f, ext)
        mid = nodes[left][2]
        recs = ({}, {})
        up = compress_block(A, lo, mid, mid, hi, scheme, tol, depth, max_rank, graph, recs[0])
        lw = compress_block(A, mid, hi, lo, mid, scheme, tol, depth, max_rank, graph, recs[1])
        fact.factors[slot] = (up, lw)
        if scheme == "aca":
            fact.traces[slot] = (recs[0]["trace"], recs[1]["trace"])
        if scheme == "bdlr":
            fact.skeletons[slot] = (recs[0]["info"], recs[1]["info"])
        na = mid - lo
        wa = visit(left, np.hstack([up[0], ext[:na]]))
        wb = visit(right, np.hstack([lw[0], ext[na:]]))
        ru, rl = up[0].shape[1], lw[0].shape[1]
        s = np.eye(ru + rl)
        s[:rl, rl:] = lw[1].T @ wa[:, :ru]
        s[rl:, :rl] = up[1].T @ wb[:, :rl]
        try:
            f = _getrf(s)
        except ValueError:
            raise SingularSchur(f"node [{lo},{hi})") from None
        fact.cpl[slot] = dict(v_up=up[1], v_low=lw[1], d_left=wa[:, :ru],
                              d_right=wb[:, :rl], lu=f[0], piv=f[1])
        return np.vstack(_correct(fact.cpl[slot], wa[:, ru:], wb[:, rl:]))

    visit(0, np.zeros((n, 0)))
    return fact


def _correct(c, top, bot):
    """Coupling.correct, src/hodlr.py:129-134."""
    rl = c["v_low"].shape[1]
    rhs = np.vstack([c["v_low"].T @ top, c["v_up"].T @ bot])
    y = _getrs((c["lu"], c["piv"]), rhs)
    return top - c["d_left"] @ y[rl:], bot - c["d_right"] @ y[:rl]


def solve(fact: OracleFactorization, rhs):
    """Bottom-up solve, src/hodlr.py:285-306."""
    b = np.asarray(rhs, dtype=np.float64)
    vec = b.ndim == 1
    if vec:
        b = b[:, None]

    def go(slot, x):
        level, lo, hi, left, right = fact.nodes[slot]
        if left < 0:
            return _getrs(fact.leaf[slot], x)
        na = fact.nodes[left][2] - lo
        t = go(left, x[:na])
        u = go(right, x[na:])
        return np.vstack(_correct(fact.cpl[slot], t, u))

    x = go(0, b)
    return x[:, 0] if vec else x


def ranks_per_level(fact: OracleFactorization):
    """src/hodlr.py:148-154, 173-180 (level = child level)."""
    per = {}
    for slot, (up, lw) in fact.factors.items():
        lvl = fact.nodes[slot][0] + 1
        per.setdefault(lvl, []).extend((up[0].shape[1], lw[0].shape[1]))
    return [{"level": k, "max_rank": int(max(v)), "mean_rank": float(np.mean(v))}
            for k, v in sorted(per.items())]


# ---------------------------------------------------------------------------
# GMRES  (src/krylov.py:69-166)
# ---------------------------------------------------------------------------

class GmresBreakdown(Exception):
    pass


def gmres(matvec, b, tol=1e-10, max_iter=1000, precond=None):
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    M = (lambda r: r) if precond is None else precond
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return dict(x=np.zeros(n), iterations=0, converged=True, history=[0.0],
                    true_residual=0.0, breakdown=False)
    r0 = M(b)
    beta = np.linalg.norm(r0)
    if beta == 0.0:
        raise GmresBreakdown("zero preconditioned rhs")
    mmax = min(max_iter, n)
    Q = np.zeros((n, mmax + 1))
    H = np.zeros((mmax + 1, mmax))
    cs = np.zeros(mmax)
    sn = np.zeros(mmax)
    g = np.zeros(mmax + 1)
    Q[:, 0] = r0 / beta
    g[0] = beta
    hist = []
    conv = brk = False
    k = 0
    for k in range(1, mmax + 1):
        j = k - 1
        w = np.array(M(matvec(Q[:, j])), dtype=np.float64)
        w_in = np.linalg.norm(w)
        for i in range(k):                        # MGS, :111-114
            H[i, j] = Q[:, i] @ w
            w -= H[i, j] * Q[:, i]
        if np.linalg.norm(w) < w_in / np.sqrt(2.0):   # :115-119
            for i in range(k):
                t = Q[:, i] @ w
                H[i, j] += t
                w -= t * Q[:, i]
        H[k, j] = np.linalg.norm(w)
        happy = H[k, j] <= 1e-14 * max(w_in, 1e-300)
        if not happy:
            Q[:, k] = w / H[k, j]
        for i in range(j):                        # Givens, :126-129
            a = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = a
        den = np.hypot(H[j, j], H[k, j])
        if den == 0.0:
            brk = True
            break
        cs[j] = H[j, j] / den
        sn[j] = H[k, j] / den
        H[j, j] = den
        H[k, j] = 0.0
        g[k] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        rel = abs(g[k]) / beta
        hist.append(float(rel))
        if rel <= tol or happy:
            conv = True
            break
    m = k if not brk else k - 1
    if m > 0:
        y = np.zeros(m)
        for i in range(m - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:m] @ y[i + 1:m]) / H[i, i]
        x = Q[:, :m] @ y
    else:
        x = np.zeros(n)
    tr = float(np.linalg.norm(b - matvec(x)) / nb)
    if brk and tr > 10.0 * tol:
        raise GmresBreakdown(f"breakdown at {k}, true residual {tr:.3e}")
    if conv and tr > 10.0 * tol:
        conv = False
    if brk:
        conv = True
    return dict(x=x, iterations=m, converged=conv, history=hist, true_residual=tr,
                breakdown=brk)


def diagonal_scaling(A):
    """src/krylov.py:44-62."""
    d = np.array(np.diag(np.asarray(A)), dtype=np.float64)
    d[d == 0.0] = 1.0
    return lambda r: r / d
