"""GMRES minimum-residual polynomial on the device (polyprec.py:24-226 of the
reference).

Construction (``build_poly`` / ``auto_degree``): the power sequence
``[v, Av, ..., A^{d+1} v]`` is built on the GPU with d+1 exact-order SpMVs
(bit-identical to the reference's), its Gram matrix with one tall-skinny
kernel plus one all-reduce; the (d+1)x(d+1) Cholesky stays on the host with the
reference's relative pivot floor (polyprec.py:60-93).

Application (``apply_poly``): the running-power recurrence fused into the
SpMV passes (``Engine.poly``): d passes, each streaming A once and updating
the accumulator in its epilogue, bit-identical to the reference.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .counters import CostCounters
from .device import KMAX
from .errors import CholeskyFailure, DimensionMismatchError, ParameterError

DEFAULT_DEGREE_CAP = 20


@dataclass(frozen=True)
class PolyCoefficients:
    """``p(A) = y[0] + y[1] A + ... + y[d] A^d`` (polyprec.py:24-43)."""

    degree: int
    y: np.ndarray
    seed_norm: float
    seed_mode: str = "unspecified"
    # roots of the residual polynomial 1 - z p(z), when the polynomial was
    # built from them (build_poly_arnoldi); the root-product form uses them
    # directly instead of re-deriving them from y.  Not a reference field.
    roots: np.ndarray | None = None

    def __post_init__(self):
        object.__setattr__(self, "y", np.asarray(self.y, dtype=np.float64))
        if self.y.shape != (self.degree + 1,):
            raise ParameterError("coefficient vector must have length degree + 1")
        if not np.all(np.isfinite(self.y)):
            raise ParameterError("polynomial coefficients must be finite")
        if self.roots is not None:
            r = np.asarray(self.roots, dtype=np.complex128)
            if r.shape != (self.degree + 1,) or not np.all(np.isfinite(r)) or np.any(r == 0):
                raise ParameterError("roots must be degree + 1 finite nonzero values")
            object.__setattr__(self, "roots", r)


@dataclass(frozen=True)
class GramSystem:
    G: np.ndarray
    rhs: np.ndarray


def dense_cholesky(system: GramSystem) -> np.ndarray:
    """Host Cholesky solve of the Gram system.  Fails (``CholeskyFailure``,
    1-based pivot) when ``pivot <= order*eps*G[k,k]`` -- the floor of the
    reference code (polyprec.py:80-82), not SPEC.md:329's."""
    G = np.asarray(system.G, dtype=np.float64)
    rhs = np.asarray(system.rhs, dtype=np.float64)
    m = G.shape[0]
    if G.shape != (m, m) or rhs.shape != (m,):
        raise DimensionMismatchError("Gram system shapes are inconsistent")
    eps = np.finfo(np.float64).eps
    L = np.zeros((m, m))
    for k in range(m):
        pivot = G[k, k] - L[k, :k] @ L[k, :k]
        if pivot <= m * eps * G[k, k]:
            raise CholeskyFailure(k + 1)
        L[k, k] = np.sqrt(pivot)
        if k + 1 < m:
            L[k + 1:, k] = (G[k + 1:, k] - L[k + 1:, :k] @ L[k, :k]) / L[k, k]
    z = np.zeros(m)
    for k in range(m):
        z[k] = (rhs[k] - L[k, :k] @ z[:k]) / L[k, k]
    y = np.zeros(m)
    for k in range(m - 1, -1, -1):
        y[k] = (z[k] - L[k + 1:, k] @ y[k + 1:]) / L[k, k]
    return y


def _engine(op):
    eng = getattr(op, "engine", None)
    if eng is None:
        raise ParameterError("the device path needs a DeviceMatrixOperator")
    return eng


#: How the degree decision's arithmetic is evaluated (polyprec.py:60-93):
#:  "reference" (default) -- the seed norm and the Gram matrix in the summation
#:     order of the reference's BLAS calls (OpenBLAS ddot / syrk, csrc/
#:     blasorder.cu) and the reference's own Cholesky loop, so build_poly's
#:     pass/fail and auto_degree's choice are the reference's;
#:  "exact" -- a double-double Gram and a compensated Cholesky: the decision
#:     exact arithmetic takes, independent of any BLAS (opt-in).
DECISIONS = ("reference", "exact")
#: OpenBLAS thread count of the host whose ddot order the seed norm follows
#: (the build container that recorded tests/golden: 8)
BLAS_THREADS = int(os.environ.get("PG_BLAS_THREADS", "8"))


def _check_decision(decision: str):
    if decision not in DECISIONS:
        raise ParameterError(f"unknown decision arithmetic {decision!r} (expected {DECISIONS})")


def _device_power_gram(op, v0, top: int, counters: CostCounters, decision: str = "reference"):
    """Unit seed, then the ``top``+1 power columns on the device and their
    Gram matrix on the host (the leading KMAX x KMAX block when top+1 > KMAX).
    Returns (Gram, seed_norm)."""
    _check_decision(decision)
    e = _engine(op)
    if isinstance(v0, torch.Tensor):
        if v0.shape != (op.dimension,) and not (e.comm.distributed and v0.shape == (e.local_n,)):
            raise DimensionMismatchError("seed vector length does not match operator")
    else:
        v0 = np.asarray(v0, dtype=np.float64)
        if v0.shape != (op.dimension,) and not (e.comm.distributed and v0.shape == (e.local_n,)):
            raise DimensionMismatchError("seed vector length does not match operator")
    if top + 1 > KMAX and decision != "reference":
        raise ParameterError(f"exact decisions take at most {KMAX} power columns")
    vs = e.ingest(v0)
    # |v0|^2 stays in device slot 6 while the power sequence and the Gram are
    # queued: one host round trip (the Gram's) instead of two
    if decision == "reference":
        e.dot_blas(vs, vs, slot=6, nthreads=BLAS_THREADS)
    else:
        e.dot(vs, vs, slot=6, fetch=False)
    P = e.cached_blocks("powers", top + 1)
    # column 0 = v0 / |v0| (exact division, as numpy's v0 / seed_norm)
    e.normalize_dev(vs, e.slot(6), [blk[0] for blk in P])
    e.power_sequence(P, top + 1)
    e.count_ops(op.counters, top)
    # past KMAX columns only the leading KMAX x KMAX block is formed: the
    # Cholesky pivots the decision needs all lie inside it (_factor)
    kg = min(top + 1, KMAX)
    G = e.gram_blas(P, kg) if decision == "reference" else e.gram(P, kg)
    seed_norm = float(np.sqrt(e.read_slot(6)))
    if seed_norm == 0.0:
        raise ParameterError("seed vector v0 must be nonzero")
    return G, seed_norm


def _normal_equations(Gfull: np.ndarray, deg: int, counters: CostCounters) -> GramSystem:
    # AV = powers[:, 1:deg+2]  ->  G = AV^T AV, rhs = AV^T v  (polyprec.py:115-122)
    counters.dots += 2
    counters.scalar_dots += (deg + 1) * (deg + 1) + (deg + 1)
    return GramSystem(Gfull[1:deg + 2, 1:deg + 2].copy(), Gfull[1:deg + 2, 0].copy())


def _cholesky_ref(G: np.ndarray, rhs: np.ndarray, order: int) -> np.ndarray:
    """dense_cholesky (polyprec.py:60-93) of the Gram block G with the pivot
    floor of an order-``order`` system -- ``order`` = G's size, or larger when
    G is the leading block of a system wider than the kernels form: pivot k of
    the full system is pivot k of its leading block, only its floor
    ``order*eps*G[k,k]`` grows with the order.  Raises CholeskyFailure."""
    m = G.shape[0]
    eps = np.finfo(np.float64).eps
    L = np.zeros((m, m))
    for k in range(m):
        pivot = G[k, k] - L[k, :k] @ L[k, :k]
        if pivot <= order * eps * G[k, k]:
            raise CholeskyFailure(k + 1)
        L[k, k] = np.sqrt(pivot)
        if k + 1 < m:
            L[k + 1:, k] = (G[k + 1:, k] - L[k + 1:, :k] @ L[k, :k]) / L[k, k]
    if order > m:  # every available pivot passed: the rest is beyond the kernels
        raise ParameterError(f"the Gram system of order {order} factors through its leading "
                             f"{m} pivots; deciding it needs more than {KMAX} power columns")
    z = np.zeros(m)
    for k in range(m):
        z[k] = (rhs[k] - L[k, :k] @ z[:k]) / L[k, k]
    y = np.zeros(m)
    for k in range(m - 1, -1, -1):
        y[k] = (z[k] - L[k + 1:, k] @ y[k + 1:]) / L[k, k]
    return y


def _factor(system: GramSystem, decision: str, order: int | None = None):
    """(y, failed 1-based pivot or 0): the reference's Cholesky loop
    (polyprec.py:60-93) or the native compensated one.  ``order`` > the
    block's size: the leading block of a wider system (_cholesky_ref)."""
    if order is None:
        order = system.G.shape[0]
    if decision == "exact":
        return _lib.host_cholesky(system.G, system.rhs)
    try:
        return _cholesky_ref(system.G, system.rhs, order), 0
    except CholeskyFailure as exc:
        return None, exc.pivot


def build_poly(op, v0, deg: int, counters: CostCounters,
               seed_mode: str = "unspecified", decision: str = "reference") -> PolyCoefficients:
    """Degree-``deg`` minimum-residual polynomial (polyprec.py:125-147):
    deg+1 device SpMVs, 2 dots, host Cholesky.  ``decision`` selects the
    arithmetic of the pass/fail decision (``DECISIONS``)."""
    if deg < 0:
        raise ParameterError("polynomial degree must be non-negative")
    Gfull, seed_norm = _device_power_gram(op, v0, deg + 1, counters, decision)
    counters.scalar_dots += 1
    full = _normal_equations(Gfull, deg, counters)
    y, pivot = _factor(full, decision, deg + 1)
    if pivot:
        raise CholeskyFailure(pivot)
    return PolyCoefficients(deg, y, seed_norm, seed_mode)


def auto_degree(op, v0, cap: int = DEFAULT_DEGREE_CAP, counters: CostCounters | None = None,
                seed_mode: str = "unspecified", decision: str = "reference") -> PolyCoefficients:
    """Largest degree <= cap whose Gram system factors (polyprec.py:150-190):
    one shared power sequence of cap+1 SpMVs, nested Gram blocks re-factored on
    the host, degree-0 fallback."""
    if cap < 1:
        raise ParameterError("degree cap must be at least 1")
    if counters is None:
        counters = CostCounters()
    Gfull, seed_norm = _device_power_gram(op, v0, cap + 1, counters, decision)
    counters.scalar_dots += 1
    return _select_degree(_normal_equations(Gfull, cap, counters), cap, seed_norm, seed_mode,
                          decision)


def _select_degree(full: GramSystem, cap: int, seed_norm: float, seed_mode: str,
                   decision: str = "reference"):
    """auto_degree's selection (polyprec.py:171-190): the largest d <= cap
    whose order-(d+1) Gram block factors with finite y, each order factored
    on its own as the reference does, then the degree-0 rule.  "reference":
    the reference's loop over every d with its Cholesky; "exact": natively
    (pg_host_degree_select, top-down, stopping at the first success)."""
    if decision == "exact":
        d, y = _lib.host_degree_select(full.G, full.rhs, cap)
    else:
        d, y = -1, None
        for dd in range(1, min(cap, full.G.shape[0] - 1) + 1):
            yy, piv = _factor(GramSystem(full.G[:dd + 1, :dd + 1], full.rhs[:dd + 1]), decision)
            if not piv and np.all(np.isfinite(yy)):
                d, y = dd, yy
        if cap + 1 > full.G.shape[0]:
            # degrees past the formed block: a leading pivot failing at the
            # floor of the next order fails at every larger one, so all of
            # them fail (_cholesky_ref raises if none does: undecidable)
            _factor(full, decision, full.G.shape[0] + 1)
    if d >= 1:
        return PolyCoefficients(d, y, seed_norm, seed_mode)
    y0, pivot = _factor(GramSystem(full.G[:1, :1], full.rhs[:1]), decision)
    if pivot:
        y0 = np.zeros(1)  # op v0 vanished; p = 0 (polyprec.py:186-187)
    return PolyCoefficients(0, y0, seed_norm, seed_mode)


def build_poly_or_auto(op, v0, deg: int, counters: CostCounters,
                       seed_mode: str = "unspecified", decision: str = "reference"):
    """Degree policy for requested degrees beyond what the power basis can
    build: the degree-``deg`` polynomial if its Gram system
    factors, else auto-degree selection with cap ``deg``.  Returns
    (PolyCoefficients, failed_pivot | None).

    ``build_poly(deg)`` and ``auto_degree(cap=deg)`` need the same power
    sequence [v, ..., A^{deg+1} v] and the same Gram matrix, so -- as
    auto_degree itself shares one sequence across candidate degrees
    (polyprec.py:150-160) -- it is built once: deg+1 SpMVs and 2 dots in total.
    The reference has no such helper; the CPU baseline runs the same policy
    (oracle.degree_policy_shared)."""
    if deg < 1:
        return build_poly(op, v0, deg, counters, seed_mode, decision), None
    Gfull, seed_norm = _device_power_gram(op, v0, deg + 1, counters, decision)
    counters.scalar_dots += 1
    full = _normal_equations(Gfull, deg, counters)
    y, pivot = _factor(full, decision, deg + 1)
    if not pivot:
        return PolyCoefficients(deg, y, seed_norm, seed_mode), None
    return _select_degree(full, deg, seed_norm, seed_mode, decision), pivot


def build_poly_arnoldi(op, v0, deg: int, counters: CostCounters | None = None,
                       seed_mode: str = "unspecified") -> PolyCoefficients:
    """Degree-``deg`` GMRES polynomial from harmonic Ritz values (SURVEY row
    f1, "a stable construction"; PAPER.md:195-202 names the power basis's
    ill-conditioning as the degree limit).  deg+1 Arnoldi steps on the operator
    from the unit seed (device SpMV + CGS2), then on the host the harmonic
    Ritz values of the (deg+1)-step Hessenberg -- the roots of the GMRES
    residual polynomial 1 - z p(z), the same minimiser build_poly finds from
    the normal equations (polyprec.py:125-147), without forming them.  Degrees
    far past the power basis's ~13 stay well conditioned; evaluate them with
    ``form="roots"``.  Costs deg+1 SpMVs, like build_poly.  No reference
    counterpart, so it is checked against build_poly's polynomial at low
    degree and by its residual minimisation at high degree."""
    if counters is None:
        counters = CostCounters()
    if deg < 0:
        raise ParameterError("polynomial degree must be non-negative")
    e = _engine(op)
    m = deg + 1
    if m + 1 > KMAX:
        raise ParameterError(f"degree {deg} exceeds the kernel limit {KMAX - 2}")
    if isinstance(v0, torch.Tensor):
        if v0.shape != (op.dimension,) and not (e.comm.distributed and v0.shape == (e.local_n,)):
            raise DimensionMismatchError("seed vector length does not match operator")
    else:
        v0 = np.asarray(v0, dtype=np.float64)
        if v0.shape != (op.dimension,) and not (e.comm.distributed and v0.shape == (e.local_n,)):
            raise DimensionMismatchError("seed vector length does not match operator")
    vs = e.ingest(v0)
    seed_norm = float(np.sqrt(e.dot(vs, vs, slot=6)))
    counters.scalar_dots += 1
    if seed_norm == 0.0:
        raise ParameterError("seed vector v0 must be nonzero")
    V = e.cached_blocks("harmonic", m + 1)
    z = e.cached_vecs("harmonic_z")
    e.normalize_dev(vs, e.slot(6), [blk[0] for blk in V])
    H = np.zeros((m + 1, m))
    for j in range(m):
        e.count_ops(counters, 1)
        e.spmv([blk[j] for blk in V], z)
        c1, c2, nsq = e.cgs2(V, j + 1, z)
        counters.dots += 3
        counters.scalar_dots += 2 * (j + 1) + 1
        counters.vector_updates += 2 * (j + 1) + 1
        H[:j + 1, j] = c1 + c2
        H[j + 1, j] = np.sqrt(max(nsq, 0.0))
        if not np.all(np.isfinite(H[:j + 2, j])):
            raise ParameterError("non-finite Arnoldi data while building the polynomial")
        if H[j + 1, j] <= 1e-14 * np.linalg.norm(H[:j + 2, j]):  # invariant subspace
            m = j + 1
            H = H[:m + 1, :m]
            break
    Hm = H[:m, :m]
    em = np.zeros(m)
    em[-1] = 1.0
    T = Hm.copy()
    if H[m, m - 1] != 0.0:
        f = np.linalg.solve(Hm.T, em)
        T[:, m - 1] += H[m, m - 1] ** 2 * f
    theta = np.linalg.eigvals(T).astype(np.complex128)
    if np.any(theta == 0) or not np.all(np.isfinite(theta)):
        raise ParameterError("singular harmonic Ritz problem (operator singular on the seed space)")
    # conjugate pairs exact: eigenvalues of a real matrix come in exact pairs;
    # the monomial coefficients follow from the product (reporting / monomial form)
    pi = np.array([1.0 + 0j])
    for th in theta:
        pi = np.convolve(pi, np.array([1.0, -1.0 / th]))
    y = -pi.real[1:]
    return PolyCoefficients(m - 1, y, seed_norm, seed_mode, roots=theta)


POLY_FORMS = ("monomial", "roots")


@dataclass(frozen=True)
class RootPlan:
    """Root-product form of ``p``.

    With ``pi(z) = 1 - z p(z) = prod_i (1 - z/theta_i)`` (degree d+1, the
    GMRES residual polynomial, roots = harmonic Ritz values), the running sum
    ``prod <- prod - A prod/theta, y <- y + prod/theta`` keeps
    ``prod = v - A y`` and ends with ``y = p(A) v``.  A complex-conjugate pair
    is one real quadratic step (two SpMVs, ``PG_ROOT_PAIR_A`` then
    ``PG_ROOT_PAIR_B``); the last root needs no SpMV, so the plan is exactly d
    fused passes, like the monomial form.  ``steps`` holds
    ``(mode, c1, c2, c3, keep_prod)`` per pass (include/pgmres.h)."""

    degree: int
    roots: np.ndarray
    steps: tuple
    y0: float  # degree-0 fallback (no roots needed)
    # d+1 passes giving A p(A) v = v - pi(A) v (the Arnoldi step's wrapped
    # operator): every root's factor, no running sum, the last one PG_ROOT_RESID
    resid_steps: tuple = ()


def leja_order(roots: np.ndarray) -> np.ndarray:
    """Modified Leja ordering with conjugate pairs adjacent (θ with Im > 0
    first): start at the largest modulus, then repeatedly take the root that
    maximises the product of distances to those already taken (log-summed)."""
    roots = np.asarray(roots, dtype=np.complex128)
    units = [complex(r) for r in roots if r.imag >= 0]
    if sum(2 if u.imag > 0 else 1 for u in units) != len(roots):
        raise ParameterError("roots are not closed under conjugation")
    taken: list = []
    out: list = []
    while units:
        if not taken:
            i = int(np.argmax([abs(u) for u in units]))
        else:
            t = np.asarray(taken)
            score = [np.sum(np.log(np.abs(u - t) + 0.0)) for u in units]
            i = int(np.argmax(score))
        u = units.pop(i)
        members = [u, u.conjugate()] if u.imag > 0 else [u]
        taken += members
        out += members
    return np.asarray(out)


def residual_poly_roots(y: np.ndarray) -> np.ndarray:
    """Roots of ``pi(z) = 1 - sum_k y_k z^{k+1}``; conjugate pairs exact
    (companion-matrix eigenvalues of a real polynomial)."""
    y = np.asarray(y, dtype=np.float64)
    coeffs = np.concatenate([-y[::-1], [1.0]])  # highest degree first
    r = np.roots(coeffs)
    # a real polynomial's complex eigenvalues come in exact conjugate pairs;
    # snap any residual asymmetry so each pair is one real quadratic step
    cplx = r[r.imag != 0]
    pos = np.sort_complex(cplx[cplx.imag > 0])
    neg = np.sort_complex(np.conj(cplx[cplx.imag < 0]))
    if len(pos) != len(neg) or not np.allclose(pos, neg, rtol=1e-12, atol=0):
        raise ParameterError("residual polynomial roots are not conjugate-closed")
    real = _polish(y, r[r.imag == 0].real.astype(np.complex128))
    pos = _polish(y, pos)
    return np.concatenate([real.real.astype(np.complex128), pos, pos.conj()])


def _polish(y: np.ndarray, roots: np.ndarray, iters: int = 4) -> np.ndarray:
    """Newton steps on pi in extended precision (np.clongdouble).  The
    companion-matrix roots carry ~1e-10 relative error at degree 10 on cfg1,
    which the running sum turns into a ~1e-10 error in p(A)v; polished roots
    bring the root form to ~3e-14 of the extended-precision p(A)v, below the
    reference monomial's own rounding."""
    if len(roots) == 0:
        return roots
    c = np.concatenate([[1.0], -np.asarray(y, dtype=np.float64)]).astype(np.longdouble)
    z = np.asarray(roots).astype(np.clongdouble)
    for _ in range(iters):
        f = np.zeros_like(z)
        df = np.zeros_like(z)
        for ck in c[::-1]:  # Horner for pi and pi'
            df = df * z + f
            f = f * z + ck
        ok = df != 0
        z = np.where(ok, z - np.where(ok, f / np.where(ok, df, 1), 0), z)
    z = z.astype(np.complex128)
    # a step that wandered (clustered roots) keeps the companion root
    moved = np.abs(z - roots) > 1e-6 * np.abs(roots)
    return np.where(moved | ~np.isfinite(z), roots, z)


def root_plan(p: PolyCoefficients) -> RootPlan:
    """Leja-ordered pass plan of ``p`` for ``Engine.poly_roots``."""
    if p.degree == 0:
        th = 1.0 / float(p.y[0]) if p.y[0] != 0.0 else None
        rs = ((_lib.PG_ROOT_REAL | _lib.PG_ROOT_RESID, float(p.y[0]), 0.0, 0.0, True),) \
            if th is not None else ()
        return RootPlan(0, np.zeros(0, np.complex128), (), float(p.y[0]), rs)
    order = leja_order(p.roots if p.roots is not None else residual_poly_roots(p.y))
    units = []
    i = 0
    while i < len(order):
        th = order[i]
        if th.imag > 0:
            units.append(("pair", th))
            i += 2
        else:
            units.append(("real", th.real))
            i += 1
    steps = []
    for j, (kind, th) in enumerate(units):
        last = j == len(units) - 1
        nxt_fold = (not last and j + 1 == len(units) - 1 and units[j + 1][0] == "real")
        c3 = 1.0 / units[j + 1][1] if nxt_fold else 0.0
        if kind == "real":
            if last:
                break  # folded into the previous pass (c3)
            steps.append((_lib.PG_ROOT_REAL, 1.0 / th, 0.0, c3, not nxt_fold))
        else:
            m2 = th.real * th.real + th.imag * th.imag
            steps.append((_lib.PG_ROOT_PAIR_A, 1.0 / m2, 2.0 * th.real, 0.0, not last))
            if not last:
                steps.append((_lib.PG_ROOT_PAIR_B, 1.0 / m2, 0.0, c3, not nxt_fold))
    if len(steps) != p.degree:
        raise ParameterError(f"root plan has {len(steps)} passes for degree {p.degree}")
    rsteps = []
    for kind, th in units:
        if kind == "real":
            rsteps.append((_lib.PG_ROOT_REAL, 1.0 / th, 0.0, 0.0, True))
        else:
            m2 = th.real * th.real + th.imag * th.imag
            rsteps.append((_lib.PG_ROOT_PAIR_A, 1.0 / m2, 2.0 * th.real, 0.0, True))
            rsteps.append((_lib.PG_ROOT_PAIR_B, 1.0 / m2, 0.0, 0.0, True))
    mode, c1, c2, c3, _ = rsteps[-1]
    rsteps[-1] = (mode | _lib.PG_ROOT_RESID, c1, c2, c3, True)
    return RootPlan(p.degree, order, tuple(steps), float(p.y[0]), tuple(rsteps))


def apply_poly(p: PolyCoefficients, op, v, counters: CostCounters, form: str = "monomial"):
    """``p(op) v`` (polyprec.py:193-212): ``degree`` fused SpMV passes,
    ``degree + 1`` counted vector updates.  ``form="monomial"`` is bit-identical
    to the reference; ``form="roots"`` evaluates the same polynomial as its
    Leja-ordered root product (``RootPlan``), also ``degree`` passes."""
    if form not in POLY_FORMS:
        raise ParameterError(f"unknown polynomial form {form!r}")
    e = _engine(op)
    if isinstance(v, np.ndarray) or not isinstance(v, torch.Tensor):
        vv = np.asarray(v, dtype=np.float64)
        if vv.shape != (op.dimension,) and not (e.comm.distributed and vv.shape == (e.local_n,)):
            raise DimensionMismatchError("vector length does not match operator")
        v = vv
    elif v.shape != (op.dimension,) and not (e.comm.distributed and v.shape == (e.local_n,)):
        raise DimensionMismatchError("vector length does not match operator")
    vs = e.ingest(v)
    out, acc, w0, w1 = e.vecs(), e.vecs(), e.vecs(), e.vecs()
    e.count_ops(op.counters, p.degree)
    counters.vector_updates += p.degree + 1
    if form == "roots":
        e.poly_roots(root_plan(p), vs, out, acc, w0, w1)
    else:
        e.poly(p.y, vs, out, acc, w0, w1)
    return e.emit(out, v)


def lambda_p_lambda(p: PolyCoefficients, points) -> np.ndarray:
    """alpha * p(alpha) by Horner (polyprec.py:215-226; host diagnostic)."""
    pts = np.asarray(points, dtype=np.float64)
    val = np.zeros_like(pts)
    for c in p.y[::-1]:
        val = val * pts + c
    return pts * val
