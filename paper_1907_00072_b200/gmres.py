"""Restarted GMRES(m), right-preconditioned by the minimum-residual polynomial,
with the Krylov basis resident on the GPU (gmres.py:98-372 of the reference).

Per inner iteration the device does the whole vector work -- d fused
polynomial passes + the wrapper SpMV (``A p(A) v_j``), and the three CGS2
phases writing the normalized v_{j+1} into the basis -- and the host receives
2k+1 reduced scalars for the Givens update and the ``implicit < tol`` branch
(gmres.py:290-313), the only host/device round trip of the iteration.  At a
cycle end: host back-substitution, device GEMV ``V y``, fused polynomial
recovery with ``x +=`` in the last pass's epilogue, and the residual SpMV with
its norm.  Control flow, history rows, counters and exceptions follow the
reference line for line.
"""

from __future__ import annotations

import gc
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .counters import CostCounters
from .device import MMAX
from .errors import (
    DimensionMismatchError,
    NumericalBreakdownError,
    ParameterError,
    SingularHessenbergError,
)
from .ortho import breakdown_test
from .polyprec import POLY_FORMS, PolyCoefficients, apply_poly, root_plan


class PolynomialWrappedOperator:
    """``v -> op(p(op) v)``: degree+1 SpMVs per call (gmres.py:98-113)."""

    kind = "polynomial-wrapped"

    def __init__(self, inner, poly: PolyCoefficients):
        self.inner = inner
        self.poly = poly
        self.dimension = inner.dimension
        self.counters = inner.counters

    def apply(self, v):
        return self.inner.apply(apply_poly(self.poly, self.inner, v, self.counters))


@dataclass(frozen=True)
class GmresConfig:
    restart_m: int = 50
    tol: float = 1e-8
    max_iters: int = 200000
    record_history: bool = True
    # "monomial" (default): the reference's running-power evaluation, bit-
    # identical.  "roots": the same polynomial as a Leja-ordered root product
    # (polyprec.RootPlan) -- same SpMV count, half the vector
    # traffic per Arnoldi pass, and accurate at degrees where the monomial
    # form's cancellation is not.  Not a reference field.
    poly_form: str = "monomial"

    def __post_init__(self):
        if self.poly_form not in POLY_FORMS:
            raise ParameterError(f"poly_form must be one of {POLY_FORMS}")
        if self.restart_m < 1:
            raise ParameterError("restart_m must be at least 1")
        if not (0.0 < self.tol < 1.0):
            raise ParameterError("tol must lie in (0, 1)")
        if self.max_iters < 1:
            raise ParameterError("max_iters must be at least 1")


@dataclass
class GmresResult:
    x: object
    converged: bool
    iterations: int
    final_relres: float
    history: list = field(default_factory=list)
    counters: CostCounters = field(default_factory=CostCounters)
    cycles: int = 0


def _givens(a, b):
    r = math.hypot(a, b)
    if r == 0.0:
        return 1.0, 0.0, 0.0
    return a / r, b / r, r


def hessenberg_lsq(H, beta: float):
    """Host Givens least squares of a (j+1) x j Hessenberg matrix
    (gmres.py:172-206); kept for API parity, not on the device path."""
    H = np.array(H, dtype=np.float64)
    if H.ndim != 2 or H.shape[0] != H.shape[1] + 1:
        raise DimensionMismatchError("H must have shape (j+1, j)")
    j = H.shape[1]
    cs, sn, g = np.zeros(j), np.zeros(j), np.zeros(j + 1)
    g[0] = beta
    for col in range(j):
        for i in range(col):
            t = cs[i] * H[i, col] + sn[i] * H[i + 1, col]
            H[i + 1, col] = -sn[i] * H[i, col] + cs[i] * H[i + 1, col]
            H[i, col] = t
        c, s, r = _givens(H[col, col], H[col + 1, col])
        cs[col], sn[col] = c, s
        H[col, col], H[col + 1, col] = r, 0.0
        g[col + 1] = -s * g[col]
        g[col] = c * g[col]
    y = np.zeros(j)
    for i in range(j - 1, -1, -1):
        if H[i, i] == 0.0:
            raise SingularHessenbergError(f"zero rotated diagonal at column {i}")
        y[i] = (g[i] - H[i, i + 1:j] @ y[i + 1:]) / H[i, i]
    return y, abs(g[j])


def _engine(op):
    eng = getattr(op, "engine", None)
    if eng is None:
        raise ParameterError("the device solver needs a DeviceMatrixOperator "
                             "(there is no CPU fallback)")
    return eng


class _Workspace:
    """Device buffers of one solve (allocated once, reused across cycles)."""

    def __init__(self, e, m):
        self.V = e.cached_blocks("basis", m + 1)
        self.z = e.cached_vecs("z")       # A p(A) v_j
        self.t = e.cached_vecs("t")       # p(A) v_j / recovery update
        self.acc = e.cached_vecs("acc")
        self.w0 = e.cached_vecs("w0")
        self.w1 = e.cached_vecs("w1")
        self.r = e.cached_vecs("r")

    def col(self, j):
        return [V[j] for V in self.V]


def solve(op, b, x0=None, right_prec: PolyCoefficients | None = None,
          config: GmresConfig | None = None) -> GmresResult:
    """Restarted GMRES over the device operator (gmres.py:213-343).
    ``b`` (and ``x0``) may be numpy arrays or torch tensors; ``x`` comes back in
    the type of ``b``.

    Python's cyclic garbage collector is paused for the duration of the solve:
    the Arnoldi loop creates only short-lived acyclic objects (freed by
    reference counting), and a full collection of a process that has imported
    torch takes tens of milliseconds -- longer than several Arnoldi steps --
    during which no kernel is queued and the GPU idles."""
    enabled = gc.isenabled()
    gc.disable()
    try:
        return _solve(op, b, x0, right_prec, config)
    finally:
        if enabled:
            gc.enable()


def _solve(op, b, x0, right_prec, config) -> GmresResult:
    if config is None:
        config = GmresConfig()
    e = _engine(op)
    counters = op.counters
    n = op.dimension
    if isinstance(b, torch.Tensor):
        blen = b.shape
    else:
        b = np.asarray(b, dtype=np.float64)
        blen = b.shape
    if blen != (n,) and not (e.comm.distributed and blen == (e.local_n,)):
        raise DimensionMismatchError("right-hand side length does not match")
    m = config.restart_m
    if m + 1 > MMAX:
        raise ParameterError(f"restart_m must be at most {MMAX - 1} on the device path")
    tol = config.tol

    poly = right_prec if right_prec else None  # reference truthiness (gmres.py:261)
    plan = root_plan(poly) if (poly is not None and config.poly_form == "roots") else None
    bs = e.ingest(b)
    W = _Workspace(e, m)
    xs = e.vecs()
    early = None
    if x0 is None:
        # |b|^2 stays on the device (slot 4) while the first cycle is queued:
        # r = b, v_0 = r/|b| and Arnoldi step 0 need no host value, so the
        # host round trip for |b| overlaps step 0 (gmres.py:241-247,277).
        e.dot(bs, bs, slot=4, fetch=False)
        e.copy(bs, W.r)
        e.normalize_dev(W.r, e.slot(4), W.col(0))
        early = _launch_step(e, W, poly, 0, plan)
        norm_b = math.sqrt(e.read_slot(4))
    else:
        norm_b = math.sqrt(e.dot(bs, bs, slot=4))
    counters.scalar_dots += 1
    if norm_b == 0.0:
        return GmresResult(e.emit(e.vecs(), b), True, 0, 0.0, [], counters, 0)

    if x0 is None:
        beta = norm_b
    else:
        xs = e.ingest(x0)
        # np.any(x0) over the GLOBAL x0 (gmres.py:248): every rank must take the
        # same branch, or the collectives of the two branches would not match
        nonzero = any(bool(torch.any(x[:s.n] != 0.0)) for s, x in zip(e.shards, xs))
        if e.comm.distributed:
            nonzero = e.comm.any(nonzero)
        if nonzero:
            e.count_ops(counters, 1)
            beta = math.sqrt(e.residual(xs, bs, W.r, slot=4))
        else:
            e.copy(bs, W.r)
            beta = math.sqrt(e.dot(bs, bs, slot=4))
        counters.scalar_dots += 1

    d = poly.degree if poly is not None else 0

    history: list = []
    total_iters = 0
    cycles = 0
    true_relres = beta / norm_b
    converged = true_relres < tol
    rho = None  # per-step residual contraction, for the look-ahead guess
    Hrot = np.empty((m + 1, m))
    cs = np.empty(m)
    sn = np.empty(m)
    g = np.empty(m + 1)

    while not converged and total_iters < config.max_iters:
        if early is not None:  # first cycle already queued above
            handle, early = early, None
        else:
            # V[:, 0] = r / beta: beta = sqrt(nsq) with nsq still in device slot 4
            e.normalize_dev(W.r, e.slot(4), W.col(0))
            handle = _launch_step(e, W, poly, 0, plan)
        g[0] = beta
        j = 0
        breakdown = False
        pending_row = None
        cur_res = true_relres  # residual the next step starts from
        while j < m and total_iters < config.max_iters:
            # one step of look-ahead: step j+1's device work (it only needs
            # v_{j+1}, already normalized on the device) is queued before the
            # host waits for step j's scalars, so the GPU never idles during
            # the host Givens update.  If step j ends the cycle, the queued
            # step is abandoned unused (no counter, no history row).
            # ... unless step j is predicted to converge: the residual
            # history's last contraction factor, applied once more, lands
            # under 2 tol -- then the look-ahead would most likely be wasted
            # (a whole step of device work), while a wrong guess only costs
            # one un-overlapped host round trip.
            if handle is None:  # the previous step skipped its look-ahead
                handle = _launch_step(e, W, poly, j, plan)
            ahead = None
            likely_done = rho is not None and cur_res * rho < 2.0 * tol
            if j + 1 < m and total_iters + 1 < config.max_iters and not likely_done:
                ahead = _launch_step(e, W, poly, j + 1, plan)
            c1, c2, nsq = e.cgs2_fetch(handle)
            handle = ahead
            if poly is not None:
                e.count_ops(counters, d + 1)
                counters.vector_updates += d + 1
            else:
                e.count_ops(counters, 1)
            coeffs = c1 + c2
            new_norm = math.sqrt(nsq) if nsq >= 0.0 else float("nan")
            counters.dots += 3
            counters.scalar_dots += 2 * (j + 1) + 1
            counters.vector_updates += 2 * (j + 1)
            if not (math.isfinite(new_norm) and np.all(np.isfinite(coeffs))):
                raise NumericalBreakdownError(total_iters + 1)
            step_breakdown = breakdown_test(coeffs, new_norm)
            if not step_breakdown:
                counters.vector_updates += 1

            hcol = np.empty(j + 2)
            hcol[:j + 1] = coeffs
            hcol[j + 1] = new_norm
            for i in range(j):
                t = cs[i] * hcol[i] + sn[i] * hcol[i + 1]
                hcol[i + 1] = -sn[i] * hcol[i] + cs[i] * hcol[i + 1]
                hcol[i] = t
            c, s_, rot = _givens(hcol[j], hcol[j + 1])
            cs[j], sn[j] = c, s_
            hcol[j] = rot
            Hrot[:j + 1, j] = hcol[:j + 1]
            g[j + 1] = -s_ * g[j]
            g[j] = c * g[j]

            total_iters += 1
            j += 1
            implicit = abs(g[j]) / norm_b
            if cur_res > 0.0:
                rho = implicit / cur_res  # last per-step contraction (kept across cycles)
            cur_res = implicit
            pending_row = (total_iters, implicit)
            if step_breakdown:
                breakdown = True
                break
            # v_{j} already normalized in place on the device by Engine.cgs2
            if implicit < tol:
                break
            if j < m and total_iters < config.max_iters and config.record_history:
                history.append((total_iters, implicit) + counters.snapshot()[:3])
                pending_row = None

        # cycle end (gmres.py:318-341)
        y, zero_col = _lib.host_backsolve(Hrot, g, j)  # native loop of gmres.py:319-325
        if zero_col >= 0:
            raise SingularHessenbergError(f"zero rotated diagonal at column {zero_col}")
        e.gemv(W.V, j, y, W.t)
        counters.vector_updates += j
        if poly is not None:
            e.count_ops(counters, d)
            counters.vector_updates += d + 1
            if plan is not None:
                e.poly_roots(plan, W.t, xs, W.acc, W.w0, W.w1, base=xs)
            else:
                e.poly(poly.y, W.t, xs, W.acc, W.w0, W.w1, base=xs)  # x = x + p(A)(V y)
        else:
            e.add(xs, W.t, xs)
        counters.vector_updates += 1
        cycles += 1

        e.count_ops(counters, 1)
        beta = math.sqrt(e.residual(xs, bs, W.r, slot=4))
        counters.scalar_dots += 1
        true_relres = beta / norm_b
        if config.record_history and pending_row is not None:
            history.append(pending_row + counters.snapshot()[:3])
        if breakdown or true_relres < tol:
            converged = True

    return GmresResult(e.emit(xs, b), converged, total_iters, true_relres, history, counters,
                       cycles)


def _launch_step(e, W, poly, j, plan=None):
    """Queue Arnoldi step j on the device: w = A p(A) v_j (d fused passes +
    the wrapper SpMV, gmres.py:112-113, 283 -- or, in root form, d+1 passes
    ending in v - pi(A) v) and its CGS2 against v_0..v_j writing v_{j+1}
    (ortho.py:53-70).  Returns the scalar handle."""
    if e.fast_steps and (plan is None or plan.resid_steps):  # one native call per step
        return e.arnoldi_step(W.V, j, poly.y if (poly is not None and plan is None) else None,
                              W, j & 1, plan)
    vj = W.col(j)
    if plan is not None:
        e.wrapped_roots(plan, vj, W.z, W.acc, W.w0, W.w1)
    elif poly is not None:
        e.poly(poly.y, vj, W.t, W.acc, W.w0, W.w1)
        e.spmv(W.t, W.z)
    else:
        e.spmv(vj, W.z)
    return e.cgs2_launch(W.V, j + 1, W.z, j & 1)


def cost_report(counters: CostCounters, deg: int, restart_m: int) -> dict:
    """Communication-proxy summary (gmres.py:350-372)."""
    dots, spmvs = counters.dots, counters.spmvs
    return {
        "global_sync_proxy_dots": dots,
        "neighbor_exchange_proxy_spmvs": spmvs,
        "scalar_dots": counters.scalar_dots,
        "vector_updates": counters.vector_updates,
        "prec_applies": counters.prec_applies,
        "spmvs_per_global_sync": (spmvs / dots) if dots else 0.0,
        "spmvs_per_iteration": deg + 1,
        "dots_per_iteration": 3,
        "ca_grouping_spmvs_per_sync": deg * restart_m,
    }
