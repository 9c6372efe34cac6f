"""Left-preconditioned GMRES without restarts (reference src/krylov.py).

Fast path: ``gmres(DenseOperator(front), b, cfg, preconditioner=fact)`` (or
``HodlrPreconditioner`` / ``DiagonalPreconditioner``) runs entirely on the
device through ``hk_gmres``: fp64 GEMV operator, HODLR solve, MGS + Givens,
the whole iteration captured in one CUDA graph with a conditional WHILE node,
so the host synchronises once per solve, not once per iteration.

General path: any Python callables (as in the reference's tests,
``lambda v: a @ v``).  The Krylov basis, Hessenberg and Givens state still
live on the device and every Arnoldi column is orthogonalised by the same
CUDA kernel; only the user's callables see host arrays.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import DimensionMismatchError, GmresBreakdownError

log = logging.getLogger("hodlrkit")


@dataclass(frozen=True)
class GmresConfig:
    tol: float = 1e-10
    max_iter: int = 1000

    def __post_init__(self):
        if not 0.0 < self.tol < 1.0:
            raise ValueError("tol must lie strictly between 0 and 1")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")


@dataclass
class GmresResult:
    x: np.ndarray
    iterations: int
    converged: bool
    residual_history: list = field(default_factory=list)
    true_residual: float = np.nan
    breakdown: bool = False


class DiagonalPreconditioner:
    """r / diag(A); zero diagonal entries act as identity (krylov.py:44-62)."""

    def __init__(self, front):
        if hasattr(front, "diagonal") and not isinstance(front, np.ndarray):
            diag = front.diagonal()
        else:
            diag = np.diag(np.asarray(front))
        diag = np.asarray(diag, dtype=np.float64).copy()
        self.zero_count = int(np.count_nonzero(diag == 0.0))
        if self.zero_count:
            log.warning("diagonal preconditioner: %d zero entries replaced by 1", self.zero_count)
            diag[diag == 0.0] = 1.0
        self.diag = diag
        self.front = front

    @property
    def flagged(self) -> bool:
        return self.zero_count > 0

    def device_diag(self):
        """The (zero-replaced) diagonal as a CUDA tensor, uploaded once."""
        dev = getattr(self, "_dev", None)
        if dev is None:
            torch = N.require_cuda()
            dev = self._dev = torch.from_numpy(self.diag).cuda()
        return dev

    def __call__(self, r):
        return r / self.diag


def diagonal_preconditioner(front) -> DiagonalPreconditioner:
    return DiagonalPreconditioner(front)


class DenseOperator:
    """``v -> A v`` for a dense front kept resident on the device (cli.py:320-321)."""

    def __init__(self, front):
        torch = N.require_cuda()
        a = front.materialize() if hasattr(front, "materialize") else front
        if isinstance(a, torch.Tensor):
            self.dev = a.to(device="cuda", dtype=torch.float64).contiguous()
        else:
            self.dev = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()
        self.n = self.dev.shape[0]

    def __call__(self, v):
        torch = N.require_cuda()
        on_dev = isinstance(v, torch.Tensor)
        vt = v if on_dev else torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).cuda()
        y = torch.empty(self.n, dtype=torch.float64, device="cuda")
        N.check(N.lib().hk_gemv(N.ptr(self.dev), self.n, self.n, self.n, N.ptr(vt.contiguous()),
                                self.n, 1, N.ptr(y), self.n, N.stream_handle()))
        return y if on_dev else y.cpu().numpy()


class HodlrPreconditioner:
    """M^{-1} r = HODLR solve of a factorization (hodlr.solve)."""

    def __init__(self, fact):
        self.fact = fact

    def __call__(self, r):
        from .hodlr import solve
        return solve(self.fact, r)


def _is_fact(obj):
    from .hodlr import HodlrFactorization
    return isinstance(obj, HodlrFactorization)


def gmres(apply_op, b, cfg: GmresConfig, preconditioner=None) -> GmresResult:
    """Full-orthogonalisation GMRES on the left-preconditioned system
    (krylov.py:69-166): MGS with one re-orthogonalisation pass when the
    vector loses more than 1/sqrt(2) of its norm, Givens rotations, the
    preconditioned residual as history, and the true-residual guard."""
    b = np.asarray(b, dtype=np.float64)
    if b.ndim != 1:
        raise ValueError("rhs must be a vector")
    if isinstance(apply_op, DenseOperator):
        pre = preconditioner
        if isinstance(pre, HodlrPreconditioner):
            pre = pre.fact
        if pre is None or _is_fact(pre) or isinstance(pre, DiagonalPreconditioner):
            return _gmres_device(apply_op, b, cfg, pre)
    return _gmres_callables(apply_op, b, cfg, preconditioner)


def _device_target(op: DenseOperator, n: int, pre):
    """(plan, front, precond kind, diag pointer) of the device GMRES, with the
    reference's shape errors: a HODLR preconditioner of another order raises
    DimensionMismatchError as its solve() would (hodlr.py:291-293); an
    operator of another order raises ValueError as ``dense @ v`` does."""
    from .hodlr import _Plan
    diag = None
    if _is_fact(pre):
        if pre.n != n:
            raise DimensionMismatchError(f"rhs has {n} rows, preconditioner expects {pre.n}")
        plan, front, kind = pre.plan, pre.front_index, 1
    else:
        front, kind = 0, 0
        if isinstance(pre, DiagonalPreconditioner):
            if pre.diag.size != n:
                raise ValueError(f"diagonal preconditioner has {pre.diag.size} entries, rhs {n}")
            diag, kind = pre.device_diag(), 2
        plan = getattr(op, "_plan", None)
        if plan is None:
            plan = _Plan(op.n, max(op.n, 1), 1)
            op._plan = plan
    if op.n != n:
        raise ValueError(f"operator is {op.n}x{op.n}, rhs has {n} rows")
    return plan, front, kind, diag


def _run_device(op: DenseOperator, Bn: np.ndarray, cfg: GmresConfig, pre) -> list:
    """hk_gmres_batch on the columns of Bn (n x s): the whole Arnoldi loop runs
    on the device as one CUDA graph; the host reads the results once."""
    torch = N.require_cuda()
    n, s = Bn.shape
    plan, front, kind, diag = _device_target(op, n, pre)
    # (s, n) = column-major n x s; staged through pinned memory so the copy is
    # one async DMA on the library's stream
    bh = torch.from_numpy(np.ascontiguousarray(Bn.T)).pin_memory()
    bd = torch.empty(bh.shape, dtype=bh.dtype, device="cuda")
    bd.copy_(bh, non_blocking=True)
    xd = torch.empty_like(bd)
    its = np.zeros(s, dtype=np.int64)
    hist = np.zeros((s, cfg.max_iter))
    tres = np.zeros(s)
    flags = np.zeros(2 * s, dtype=np.int32)
    N.check(N.lib().hk_gmres_batch(plan.h, front, N.ptr(op.dev), op.dev.stride(0), n, N.ptr(bd), s,
                                   cfg.tol, cfg.max_iter, kind,
                                   N.ptr(diag) if diag is not None else None, N.ptr(xd),
                                   N.arr_ptr(its, N.I64), N.arr_ptr(hist, N.D),
                                   N.arr_ptr(tres, N.D), N.arr_ptr(flags, N.I32),
                                   N.stream_handle()))
    xh = xd.cpu().numpy()
    out = []
    for c in range(s):
        m = int(its[c])
        if not np.any(Bn[:, c]):                 # krylov.py:85-87
            out.append(GmresResult(np.zeros(n), 0, True, [0.0], 0.0))
            continue
        conv, brk = bool(flags[2 * c]), bool(flags[2 * c + 1])
        if not conv and not brk and tres[c] > 10 * cfg.tol and m and hist[c, m - 1] <= cfg.tol:
            log.warning("gmres: preconditioned residual converged but true residual %.3e exceeds "
                        "10*tol; reporting non-convergence", tres[c])
        out.append(GmresResult(xh[c].copy(), m, conv, [float(h) for h in hist[c, :m]],
                               float(tres[c]), brk))
    return out


def _gmres_device(op: DenseOperator, b, cfg, pre) -> GmresResult:
    return _run_device(op, b[:, None], cfg, pre)[0]


def _gmres_callables(apply_op, b, cfg, preconditioner) -> GmresResult:
    torch = N.require_cuda()
    n = b.size
    M = (lambda r: r) if preconditioner is None else preconditioner
    dev = "cuda"
    bd = torch.from_numpy(np.ascontiguousarray(b)).to(dev)
    norm_b = float(torch.linalg.vector_norm(bd))
    if norm_b == 0.0:
        return GmresResult(np.zeros(n), 0, True, [0.0], 0.0)

    def host(v):
        return v.cpu().numpy() if isinstance(v, torch.Tensor) else np.asarray(v, dtype=np.float64)

    r0 = torch.from_numpy(np.array(host(M(b)), dtype=np.float64)).to(dev)
    beta = float(torch.linalg.vector_norm(r0))
    if beta == 0.0:
        raise GmresBreakdownError("preconditioned rhs is exactly zero")
    mmax = min(cfg.max_iter, n)
    basis = torch.zeros((mmax + 1, n), dtype=torch.float64, device=dev)   # col-major n x (m+1)
    hess = torch.zeros((mmax, mmax + 1), dtype=torch.float64, device=dev)  # col-major (m+1) x m
    cs = torch.zeros(mmax, dtype=torch.float64, device=dev)
    sn = torch.zeros(mmax, dtype=torch.float64, device=dev)
    g = torch.zeros(mmax + 1, dtype=torch.float64, device=dev)
    basis[0] = r0 / beta
    g[0] = beta
    out = np.zeros(3)
    history = []
    converged = breakdown = False
    k = 0
    L = N.lib()
    st = N.stream_handle()
    for k in range(1, mmax + 1):
        j = k - 1
        vj = basis[j].cpu().numpy()
        w = torch.from_numpy(np.array(host(M(host(apply_op(vj)))), dtype=np.float64)).to(dev)
        N.check(L.hk_arnoldi_step(n, j, mmax, N.ptr(basis), N.ptr(hess), N.ptr(cs), N.ptr(sn),
                                  N.ptr(g), N.ptr(w), beta, N.arr_ptr(out, N.D), st))
        if out[2] != 0.0:
            breakdown = True
            break
        history.append(float(out[0]))
        if out[0] <= cfg.tol or out[1] != 0.0:
            converged = True
            break
    m = k if not breakdown else k - 1
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    if m > 0:
        N.check(L.hk_gmres_combine(n, m, mmax, N.ptr(basis), N.ptr(hess), N.ptr(g), N.ptr(x), st))
    xh = x.cpu().numpy()
    tres = float(np.linalg.norm(b - host(apply_op(xh))) / norm_b)
    if breakdown and tres > 10.0 * cfg.tol:
        raise GmresBreakdownError(
            f"Arnoldi norm underflow at iteration {k} with true residual {tres:.3e}")
    if converged and tres > 10.0 * cfg.tol:
        log.warning("gmres: preconditioned residual converged but true residual %.3e exceeds "
                    "10*tol; reporting non-convergence", tres)
        converged = False
    if breakdown:
        converged = True
    return GmresResult(xh, m, converged, history, tres, breakdown)


def gmres_device(apply_op, b, cfg: GmresConfig, preconditioner=None) -> GmresResult:
    """gmres() with callables on CUDA tensors (the sharded operator and
    preconditioner of subtree.ShardedHodlr): ``gmres_device_batch`` with one
    column."""
    torch = N.require_cuda()
    bd = b if isinstance(b, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(b))
    bd = bd.to(device="cuda", dtype=torch.float64).reshape(1, -1)
    return gmres_device_batch(lambda X: apply_op(X[0])[None],
                              bd, cfg, None if preconditioner is None else
                              (lambda X: preconditioner(X[0])[None]))[0]


def gmres_device_batch(apply_op, B, cfg: GmresConfig, preconditioner=None) -> list:
    """s GMRES systems in lock step with callables that map an (s, n) CUDA
    tensor (row c = the vector of system c) to (s, n): the sharded operator and
    preconditioner, whose collectives then carry all s columns at once.  The
    Arnoldi steps of all systems run in one launch (hk_arnoldi_step_batch) and
    the host reads their three flags once per iteration.  Same algorithm,
    flags and results per system as gmres() (krylov.py:69-166)."""
    torch = N.require_cuda()
    Bd = B.to(device="cuda", dtype=torch.float64).contiguous()
    s, n = Bd.shape
    M = (lambda X: X) if preconditioner is None else preconditioner
    norm_b = torch.linalg.vector_norm(Bd, dim=1).cpu().numpy()
    zero = norm_b == 0.0
    R0 = M(Bd).contiguous()
    beta = torch.linalg.vector_norm(R0, dim=1)
    bh = beta.cpu().numpy()
    if np.any((bh == 0.0) & ~zero):
        raise GmresBreakdownError("preconditioned rhs is exactly zero")
    mmax = min(cfg.max_iter, n)
    vs = mmax + 1
    basis = torch.zeros((s, vs, n), dtype=torch.float64, device="cuda")
    hess = torch.zeros((s, mmax, vs), dtype=torch.float64, device="cuda")
    cs = torch.zeros((s, vs), dtype=torch.float64, device="cuda")
    sn = torch.zeros((s, vs), dtype=torch.float64, device="cuda")
    g = torch.zeros((s, vs), dtype=torch.float64, device="cuda")
    safe = torch.where(beta == 0.0, torch.ones_like(beta), beta)
    basis[:, 0] = R0 / safe[:, None]
    g[:, 0] = beta
    active = ~zero
    act_d = torch.from_numpy(active.astype(np.int32)).cuda()
    out = torch.zeros((s, 3), dtype=torch.float64, device="cuda")
    hist = [[] for _ in range(s)]
    m = np.zeros(s, dtype=np.int64)
    conv = zero.copy()
    brk = np.zeros(s, dtype=bool)
    L = N.lib()
    st = N.stream_handle()
    k = 0
    for k in range(1, mmax + 1):
        if not active.any():
            break
        j = k - 1
        W = M(apply_op(basis[:, j].contiguous())).contiguous()
        N.check(L.hk_arnoldi_step_batch(n, j, mmax, N.ptr(basis), vs * n, N.ptr(hess), mmax * vs,
                                        N.ptr(cs), N.ptr(sn), N.ptr(g), N.ptr(W), N.ptr(beta),
                                        N.ptr(out), N.ptr(act_d), s, st))
        o = out.cpu().numpy()                   # the one host round trip of the iteration
        for c in np.flatnonzero(active):
            if o[c, 2] != 0.0:
                brk[c], m[c], active[c] = True, k - 1, False
                continue
            hist[c].append(float(o[c, 0]))
            m[c] = k
            if o[c, 0] <= cfg.tol or o[c, 1] != 0.0:
                conv[c], active[c] = True, False
        act_d.copy_(torch.from_numpy(active.astype(np.int32)))
    X = torch.zeros((s, n), dtype=torch.float64, device="cuda")
    for c in range(s):
        if m[c] > 0 and not zero[c]:
            N.check(L.hk_gmres_combine(n, int(m[c]), mmax, N.ptr(basis[c]), N.ptr(hess[c]),
                                       N.ptr(g[c]), N.ptr(X[c]), st))
    tres = (torch.linalg.vector_norm(Bd - apply_op(X), dim=1).cpu().numpy()
            / np.where(zero, 1.0, norm_b))
    results = []
    for c in range(s):
        if zero[c]:
            results.append(GmresResult(np.zeros(n), 0, True, [0.0], 0.0))
            continue
        tr = float(tres[c])
        if brk[c] and tr > 10.0 * cfg.tol:
            raise GmresBreakdownError(
                f"rhs {c}: Arnoldi norm underflow at iteration {m[c] + 1} with true residual {tr:.3e}")
        cv = bool(conv[c])
        if cv and tr > 10.0 * cfg.tol:
            log.warning("gmres: preconditioned residual converged but true residual %.3e exceeds "
                        "10*tol; reporting non-convergence", tr)
            cv = False
        if brk[c]:
            cv = True
        results.append(GmresResult(X[c].cpu().numpy(), int(m[c]), cv, hist[c], tr, bool(brk[c])))
    return results


def gmres_batch(apply_op, B, cfg: GmresConfig, preconditioner=None) -> list:
    """gmres() for the columns of B (n x s, s <= 16) run together on the device.

    ``apply_op`` must be a DenseOperator and ``preconditioner`` a HODLR
    factorization (or HodlrPreconditioner / DiagonalPreconditioner / None).
    Every iteration reads the dense front and the stored factor once for all
    s systems (hk_gmres_batch); each system's iterates, iteration count and
    flags equal those of gmres() on that column.
    """
    torch = N.require_cuda()
    if not isinstance(apply_op, DenseOperator):
        raise TypeError("gmres_batch needs a DenseOperator")
    Bn = B.cpu().numpy() if isinstance(B, torch.Tensor) else np.asarray(B, dtype=np.float64)
    if Bn.ndim != 2:
        raise ValueError("B must be n x s")
    if not 1 <= Bn.shape[1] <= 16:
        raise ValueError("gmres_batch takes 1..16 right-hand sides")
    pre = preconditioner
    if isinstance(pre, HodlrPreconditioner):
        pre = pre.fact
    if not (pre is None or _is_fact(pre) or isinstance(pre, DiagonalPreconditioner)):
        raise TypeError("gmres_batch takes a HODLR factorization, a DiagonalPreconditioner or None")
    return _run_device(apply_op, np.asarray(Bn, dtype=np.float64), cfg, pre)
