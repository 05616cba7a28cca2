"""CPU oracle for the PP-GMRES hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference `polygmres` algorithm
(/root/reference/pkg/src/polygmres, v0.1.0) for exactly the functions on the
hot path.  It is the *checker*: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product package ``paper_1907_00072_b200`` never imports it and has no CPU
fallback.

Parity is pinned: ``tests/golden/make_golden.py`` imports the unchanged
reference in the build container and records golden vectors; the CPU test
``tests/test_oracle_golden.py`` checks every function here against them
(bitwise for the SpMV / polynomial / RNG arithmetic, exact for counters and
iteration counts, tight tolerances where OpenBLAS ordering is involved).

Every numerical step uses the same numpy primitive, in the same order, as the
reference call site it cites, so that on the same machine (same OpenBLAS) the
results are bit-identical to the reference.
"""

from __future__ import annotations

import math
import os
import subprocess

import numpy as np

# ---------------------------------------------------------------------------
# SplitMix64 stream  (rng.py:18-37)
# ---------------------------------------------------------------------------
_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E9B5)
_M2 = np.uint64(0x94D049BB133111EB)


def sm64_raw(seed: int, count: int) -> np.ndarray:
    """Outputs 1..count of the SplitMix64 stream at ``seed`` (rng.py:25-31)."""
    k = np.arange(1, count + 1, dtype=np.uint64)
    z = np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF) + k * _G
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def sm64_uniform(seed: int, count: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Top-53-bit doubles mapped to [lo, hi) (rng.py:34-37)."""
    top = (sm64_raw(seed, count) >> np.uint64(11)).astype(np.float64)
    return lo + (hi - lo) * (top * 2.0 ** -53)


# ---------------------------------------------------------------------------
# operation tallies  (counters.py:6-46)
# ---------------------------------------------------------------------------
class Tally:
    __slots__ = ("spmvs", "dots", "scalar_dots", "vector_updates", "prec_applies")

    def __init__(self):
        self.spmvs = self.dots = self.scalar_dots = 0
        self.vector_updates = self.prec_applies = 0

    def snap(self):
        return (self.spmvs, self.dots, self.scalar_dots, self.vector_updates,
                self.prec_applies)


# ---------------------------------------------------------------------------
# CSR product  (sparse.py:151-168)
# ---------------------------------------------------------------------------
class OracleMatrix:
    """Counting CSR operator: the oracle's ``MatrixOperator`` (gmres.py:46-60).

    ``entry_row`` mirrors the precomputed row-of-entry array (sparse.py:84-85).
    """

    def __init__(self, nrows, ncols, row_ptr, col_idx, values, tally=None):
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.entry_row = np.repeat(np.arange(self.nrows, dtype=np.int64),
                                   np.diff(self.row_ptr))
        self.tally = tally if tally is not None else Tally()
        self.dimension = self.nrows

    @classmethod
    def of(cls, csr, tally=None):
        return cls(csr.nrows, csr.ncols, csr.row_ptr, csr.col_idx, csr.values, tally)

    def matvec(self, x):
        """Uncounted ``A @ x``.  Per row a sequential sum, in stored column
        order, of separately rounded products: this is what ``bincount`` with
        weights does (sparse.py:164-168)."""
        x = np.asarray(x, dtype=np.float64)
        prod = self.values * x[self.col_idx]
        return np.bincount(self.entry_row, weights=prod, minlength=self.nrows)

    def apply(self, x):
        self.tally.spmvs += 1
        return self.matvec(x)


def matvec_rowseq(row_ptr, col_idx, values, x):
    """Pure-Python loop form of the same SpMV, for the tiny bitwise cross-check
    (``s = s + v*x`` per entry, no FMA)."""
    n = len(row_ptr) - 1
    out = np.zeros(n)
    for r in range(n):
        s = 0.0
        for q in range(row_ptr[r], row_ptr[r + 1]):
            s = s + float(values[q]) * float(x[col_idx[q]])
        out[r] = s
    return out


# ---------------------------------------------------------------------------
# polynomial application  (polyprec.py:193-212)
# ---------------------------------------------------------------------------
def poly_eval(y, op, v, tally):
    """``p(A) v = sum_k y_k A^k v`` by the running power; d counted SpMVs and
    d+1 vector updates."""
    y = np.asarray(y, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    total = y[0] * v
    tally.vector_updates += 1
    cur = v
    for yk in y[1:]:
        cur = op.apply(cur)
        total += yk * cur
        tally.vector_updates += 1
    return total


def poly_eval_extended(y, op, v):
    """``p(A) v`` by the monomial running power in x87 extended precision
    (np.longdouble, 64-bit mantissa): the accuracy yardstick for the
    root-product form (the reference evaluates only the monomial
    form, polyprec.py:193-212, whose own fp64 error grows with the cancellation
    max|y_k A^k v|/|p(A)v| -- SURVEY A.5).  Per row a sequential sum in stored
    order, like ``matvec``."""
    y = np.asarray(y, dtype=np.longdouble)
    vals = np.asarray(op.values, dtype=np.longdouble)
    rp = np.asarray(op.row_ptr, dtype=np.int64)
    nz = rp[1:] > rp[:-1]

    def mv(x):
        out = np.zeros(op.nrows, dtype=np.longdouble)
        if len(vals):
            out[nz] = np.add.reduceat(vals * x[op.col_idx], rp[:-1][nz])
        return out

    cur = np.asarray(v, dtype=np.longdouble)
    total = y[0] * cur
    for yk in y[1:]:
        cur = mv(cur)
        total = total + yk * cur
    return total.astype(np.float64)


def wrapped_apply(y, op, v, tally):
    """``A p(A) v`` (gmres.py:112-113)."""
    return op.apply(poly_eval(y, op, v, tally))


# ---------------------------------------------------------------------------
# ILU(0) left preconditioning  (ilu.py:38-114, gmres.py:63-95)
# ---------------------------------------------------------------------------
class IluPivotOracle(Exception):
    def __init__(self, row, structural=False):
        super().__init__(f"pivot failure at row {row}")
        self.row = row
        self.structural = structural


def ilu0_factor(op, diag_shift=0.0):
    """IKJ elimination restricted to the pattern of ``op`` (ilu.py:38-95),
    same operation order: ``l_ik = a_ik / u_kk`` then ``a_ij -= l_ik * u_kj``
    for j in row k's upper part that is also in row i's pattern.  Returns
    (values, diag_ptr); raises IluPivotOracle(row)."""
    n = op.nrows
    rp, ci = op.row_ptr, op.col_idx
    vals = op.values.copy()
    diag = np.full(n, -1, dtype=np.int64)
    hit = op.entry_row == ci
    diag[ci[hit]] = np.nonzero(hit)[0]
    if np.any(diag < 0):
        raise IluPivotOracle(int(np.nonzero(diag < 0)[0][0]), structural=True)
    if diag_shift != 0.0:
        vals[diag] += diag_shift
    floor = np.finfo(np.float64).eps * float(np.max(np.abs(vals[diag])))
    for i in range(n):
        where = {int(ci[p]): p for p in range(rp[i], rp[i + 1])}
        for p in range(rp[i], rp[i + 1]):
            k = int(ci[p])
            if k >= i:
                break
            ukk = vals[diag[k]]
            if abs(ukk) <= floor:
                raise IluPivotOracle(k)
            vals[p] = vals[p] / ukk
            for q in range(diag[k] + 1, rp[k + 1]):
                t = where.get(int(ci[q]))
                if t is not None:
                    vals[t] -= vals[p] * vals[q]
        if abs(vals[diag[i]]) <= floor:
            raise IluPivotOracle(i)
    return vals, diag


def ilu0_apply(op, vals, diag, v):
    """``M^{-1} v`` (ilu.py:98-114): forward sweep with unit L, backward with
    U; each row's off-diagonal sum is a numpy dot as in the reference."""
    n = op.nrows
    rp, ci = op.row_ptr, op.col_idx
    y = np.empty(n)
    for i in range(n):
        y[i] = v[i] - vals[rp[i]:diag[i]] @ y[ci[rp[i]:diag[i]]]
    z = np.empty(n)
    for i in range(n - 1, -1, -1):
        d, hi = diag[i], rp[i + 1]
        z[i] = (y[i] - vals[d + 1:hi] @ z[ci[d + 1:hi]]) / vals[d]
    return z


class OracleIluOperator:
    """``v -> M^{-1} (A v)`` with its counters (gmres.py:63-95)."""

    def __init__(self, A, vals, diag):
        self.A, self.vals, self.diag = A, vals, diag
        self.tally = A.tally
        self.dimension = A.nrows
        self.nrows = A.nrows

    def apply(self, x):
        self.tally.spmvs += 1
        self.tally.prec_applies += 1
        return ilu0_apply(self.A, self.vals, self.diag, self.A.matvec(x))

    def matvec(self, x):
        return ilu0_apply(self.A, self.vals, self.diag, self.A.matvec(x))

    def precondition(self, v):
        self.tally.prec_applies += 1
        return ilu0_apply(self.A, self.vals, self.diag, v)


# ---------------------------------------------------------------------------
# two-pass classical Gram-Schmidt  (ortho.py:14, 33-70)
# ---------------------------------------------------------------------------
BREAKDOWN_RTOL = 1e-14


def cgs2(basis, w, tally):
    """Returns (coeffs, new_norm, vector, breakdown)."""
    j = basis.shape[1]
    a1 = basis.T @ w
    r1 = w - basis @ a1
    a2 = basis.T @ r1
    r2 = r1 - basis @ a2
    h = a1 + a2
    nn = float(np.linalg.norm(r2))
    tally.dots += 3
    tally.scalar_dots += 2 * j + 1
    tally.vector_updates += 2 * j
    full = math.hypot(float(np.linalg.norm(h)), nn)
    if nn <= BREAKDOWN_RTOL * full:
        return h, nn, r2, True
    tally.vector_updates += 1
    return h, nn, r2 / nn, False


# ---------------------------------------------------------------------------
# minimum-residual polynomial construction  (polyprec.py:54-190)
# ---------------------------------------------------------------------------
class CholeskyFailureOracle(Exception):
    def __init__(self, pivot):
        super().__init__(pivot)
        self.pivot = pivot


def chol_solve(G, rhs):
    """Unblocked lower Cholesky with the relative pivot floor
    ``pivot <= order*eps*G[k,k]`` (polyprec.py:60-93; the code, not
    SPEC.md:329, is authoritative), then two triangular solves."""
    G = np.asarray(G, dtype=np.float64)
    rhs = np.asarray(rhs, dtype=np.float64)
    order = G.shape[0]
    eps = np.finfo(np.float64).eps
    L = np.zeros((order, order))
    for k in range(order):
        piv = G[k, k] - L[k, :k] @ L[k, :k]
        if piv <= order * eps * G[k, k]:
            raise CholeskyFailureOracle(k + 1)
        L[k, k] = np.sqrt(piv)
        if k + 1 < order:
            L[k + 1:, k] = (G[k + 1:, k] - L[k + 1:, :k] @ L[k, :k]) / L[k, k]
    fwd = np.zeros(order)
    for k in range(order):
        fwd[k] = (rhs[k] - L[k, :k] @ fwd[:k]) / L[k, k]
    sol = np.zeros(order)
    for k in range(order - 1, -1, -1):
        sol[k] = (fwd[k] - L[k + 1:, k] @ sol[k + 1:]) / L[k, k]
    return sol


def _seed(v0):
    v0 = np.asarray(v0, dtype=np.float64)
    nrm = float(np.linalg.norm(v0))
    if nrm == 0.0:
        raise ValueError("seed vector v0 must be nonzero")
    return v0 / nrm, nrm


def power_columns(op, v, top):
    """[v, Av, ..., A^top v] as an n x (top+1) array (polyprec.py:106-112)."""
    cols = [v]
    for _ in range(top):
        cols.append(op.apply(cols[-1]))
    return np.column_stack(cols)


def gram(powers, deg, tally):
    """G = AV^T AV, rhs = AV^T v with AV = powers[:, 1:deg+2] (polyprec.py:115-122)."""
    AV = powers[:, 1:deg + 2]
    G = AV.T @ AV
    rhs = AV.T @ powers[:, 0]
    tally.dots += 2
    tally.scalar_dots += (deg + 1) * (deg + 1) + (deg + 1)
    return G, rhs


def gram_exact(powers):
    """Correctly rounded Gram matrix of the power columns (each entry: exact
    products by Dekker splitting, exactly rounded sum by math.fsum).  Not the
    reference's arithmetic -- the reference's G carries OpenBLAS rounding whose
    order depends on the host CPU -- but the arbiter of the Cholesky-failure
    degree decision in exact arithmetic."""
    split = 134217729.0  # 2^27 + 1
    k = powers.shape[1]
    G = np.zeros((k, k))

    def halves(a):
        t = split * a
        hi = t - (t - a)
        return hi, a - hi

    for i in range(k):
        ah, al = halves(powers[:, i])
        for j in range(i, k):
            b = powers[:, j]
            bh, bl = halves(b)
            p = powers[:, i] * b
            e = ((ah * bh - p) + ah * bl + al * bh) + al * bl
            G[i, j] = G[j, i] = math.fsum(np.concatenate([p, e]))
    return G


def chol_pivot_exact(G):
    """1-based failing pivot (0 = success) of the Cholesky of G with every
    inner product exactly rounded (math.fsum) and the reference's floor
    ``pivot <= order*eps*G[k,k]`` -- the exact-arithmetic pass/fail decision
    (the plain numpy loop decides the trailing pivots by its own rounding)."""
    G = np.asarray(G, dtype=np.float64)
    o = G.shape[0]
    eps = np.finfo(np.float64).eps
    L = [[0.0] * o for _ in range(o)]
    for k in range(o):
        piv = math.fsum([float(G[k, k])] + [-L[k][t] * L[k][t] for t in range(k)])
        if piv <= o * eps * G[k, k]:
            return k + 1
        L[k][k] = math.sqrt(piv)
        for i in range(k + 1, o):
            L[i][k] = math.fsum([float(G[i, k])] + [-L[i][t] * L[k][t] for t in range(k)]) / L[k][k]
    return 0


def auto_deg_exact(Gfull, cap):
    """Exact-arithmetic auto_degree decision on a (correctly rounded) Gram."""
    G = Gfull[1:cap + 2, 1:cap + 2]
    for d in range(cap, 0, -1):
        if chol_pivot_exact(G[:d + 1, :d + 1]) == 0:
            return d
    return 0


def auto_deg_from_gram(Gfull, cap):
    """auto_degree's selection loop (polyprec.py:171-190) on a given full
    Gram of [v, Av, ..., A^{cap+1} v]."""
    G = Gfull[1:cap + 2, 1:cap + 2]
    rhs = Gfull[1:cap + 2, 0]
    best = None
    for d in range(1, cap + 1):
        try:
            yy = chol_solve(G[:d + 1, :d + 1], rhs[:d + 1])
        except CholeskyFailureOracle:
            continue
        if np.all(np.isfinite(yy)):
            best = (d, yy)
    return best


# ---------------------------------------------------------------------------
# reference-order (OpenBLAS) reductions of the degree decision -- C restatement
# in oracle/blasorder.c, built into oracle/_ref/libblasorder.so
# ---------------------------------------------------------------------------
_BLAS = None
ORACLE_DIR = os.path.dirname(os.path.abspath(__file__))
BLAS_LIB = os.path.join(ORACLE_DIR, "_ref", "libblasorder.so")


def build_blasorder(force: bool = False) -> str:
    """gcc oracle/blasorder.c -> oracle/_ref/libblasorder.so (test infrastructure)."""
    src = os.path.join(ORACLE_DIR, "blasorder.c")
    if force or not os.path.exists(BLAS_LIB) or os.path.getmtime(BLAS_LIB) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(BLAS_LIB), exist_ok=True)
        tmp = BLAS_LIB + ".tmp"
        subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-ffp-contract=off", src, "-o", tmp,
                        "-lm"], check=True)
        os.replace(tmp, BLAS_LIB)
    return BLAS_LIB


def _blas():
    global _BLAS
    if _BLAS is None:
        import ctypes
        lib = ctypes.CDLL(build_blasorder())
        lib.oracle_blas_ddot.restype = ctypes.c_double
        lib.oracle_blas_ddot.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_int]
        lib.oracle_blas_gram.restype = None
        lib.oracle_blas_gram.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_int64, ctypes.c_void_p]
        _BLAS = lib
    return _BLAS


def blas_ddot(x, y, nthreads: int = 8) -> float:
    """x.y in OpenBLAS ddot order with ``nthreads`` threads (numpy's x.dot(y)
    on the build host)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return float(_blas().oracle_blas_ddot(len(x), x.ctypes.data, y.ctypes.data, nthreads))


def blas_gram(P) -> np.ndarray:
    """P^T P in OpenBLAS syrk K-block order (numpy's A.T @ A, full tiles)."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    n, k = P.shape
    G = np.zeros((k, k))
    _blas().oracle_blas_gram(n, k, P.ctypes.data, k, G.ctypes.data)
    return G


def seed_blas(v0, nthreads: int = 8):
    """_unit_seed (polyprec.py:46-51) with the norm in OpenBLAS order."""
    v0 = np.asarray(v0, dtype=np.float64)
    nrm = float(np.sqrt(blas_ddot(v0, v0, nthreads)))
    return v0 / nrm, nrm


def gram_full_blas(op, v0, top, nthreads: int = 8):
    """Full Gram of [v, Av, ..., A^top v] in reference (OpenBLAS) order, and
    the seed norm.  Column 0 pairs give rhs = AV^T v."""
    v, nrm = seed_blas(v0, nthreads)
    return blas_gram(power_columns(op, v, top)), nrm


def degree_decision_blas(Gfull, deg):
    """(build_poly(deg) failing pivot or 0, auto_degree(cap=deg) degree) from a
    full Gram of deg+2 columns, with the reference's Cholesky loop."""
    G = Gfull[1:deg + 2, 1:deg + 2]
    rhs = Gfull[1:deg + 2, 0]
    try:
        chol_solve(G, rhs)
        piv = 0
    except CholeskyFailureOracle as exc:
        piv = exc.pivot
    best = auto_deg_from_gram(Gfull, deg)
    return piv, (best[0] if best else 0)


def min_res_poly(op, v0, deg, tally):
    """``build_poly`` (polyprec.py:125-147): returns (y, seed_norm)."""
    if deg < 0:
        raise ValueError("polynomial degree must be non-negative")
    v, nrm = _seed(v0)
    tally.scalar_dots += 1
    P = power_columns(op, v, deg + 1)
    G, rhs = gram(P, deg, tally)
    return chol_solve(G, rhs), nrm


def auto_deg(op, v0, cap, tally):
    """``auto_degree`` (polyprec.py:150-190): largest successful d <= cap,
    with the degree-0 fallback.  Returns (degree, y, seed_norm)."""
    if cap < 1:
        raise ValueError("degree cap must be at least 1")
    v, nrm = _seed(v0)
    tally.scalar_dots += 1
    P = power_columns(op, v, cap + 1)
    G, rhs = gram(P, cap, tally)
    best = None
    for d in range(1, cap + 1):
        try:
            yy = chol_solve(G[:d + 1, :d + 1], rhs[:d + 1])
        except CholeskyFailureOracle:
            continue
        if np.all(np.isfinite(yy)):
            best = (d, yy)
    if best is not None:
        return best[0], best[1], nrm
    try:
        y0 = chol_solve(G[:1, :1], rhs[:1])
    except CholeskyFailureOracle:
        y0 = np.zeros(1)
    return 0, y0, nrm


def degree_policy(op, v0, deg, tally):
    """Bench/solver policy for requested degrees the power-basis construction
    cannot build: ``build_poly(deg)``; on Cholesky failure,
    ``auto_degree(cap=deg)``.  Returns (requested, effective, y, seed_norm)."""
    try:
        y, nrm = min_res_poly(op, v0, deg, tally)
        return deg, deg, y, nrm
    except CholeskyFailureOracle:
        d, y, nrm = auto_deg(op, v0, deg, tally)
        return deg, d, y, nrm


def degree_policy_shared(op, v0, deg, tally):
    """The same policy with one shared power sequence + Gram (deg+1 SpMVs,
    2 dots), as the device's build_poly_or_auto; used by the CPU baseline so
    both arms do identical work.  Returns (requested, effective, y, seed_norm)."""
    v, nrm = _seed(v0)
    tally.scalar_dots += 1
    P = power_columns(op, v, deg + 1)
    G, rhs = gram(P, deg, tally)
    try:
        return deg, deg, chol_solve(G, rhs), nrm
    except CholeskyFailureOracle:
        Gfull = np.zeros((deg + 2, deg + 2))
        Gfull[1:, 1:] = G
        Gfull[1:, 0] = rhs
        best = auto_deg_from_gram(Gfull, deg)
        if best is None:
            try:
                return deg, 0, chol_solve(G[:1, :1], rhs[:1]), nrm
            except CholeskyFailureOracle:
                return deg, 0, np.zeros(1), nrm
        return deg, best[0], best[1], nrm


# ---------------------------------------------------------------------------
# restarted GMRES(m)  (gmres.py:165-169, 213-343)
# ---------------------------------------------------------------------------
class OracleResult:
    def __init__(self, x, converged, iterations, final_relres, history, tally, cycles):
        self.x, self.converged, self.iterations = x, converged, iterations
        self.final_relres, self.history, self.tally = final_relres, history, tally
        self.cycles = cycles


def _rot(a, b):
    r = math.hypot(a, b)
    if r == 0.0:
        return 1.0, 0.0, 0.0
    return a / r, b / r, r


def gmres(op, b, x0=None, y=None, m=50, tol=1e-8, max_iters=200000,
          record_history=True):
    """Restarted GMRES(m), right-preconditioned by the polynomial with
    coefficients ``y`` (None = unpreconditioned).  Mirrors gmres.py:213-343
    step for step, including the history-row placement quirk
     and the explicit-residual stopping test."""
    t = op.tally
    n = op.dimension
    b = np.asarray(b, dtype=np.float64)
    bnorm = float(np.linalg.norm(b))
    t.scalar_dots += 1
    if bnorm == 0.0:
        return OracleResult(np.zeros(n), True, 0, 0.0, [], t, 0)
    if x0 is None:
        x = np.zeros(n)
        r = b.copy()
        beta = bnorm
    else:
        x = np.array(x0, dtype=np.float64)
        r = b - op.apply(x) if np.any(x != 0.0) else b.copy()
        beta = float(np.linalg.norm(r))
        t.scalar_dots += 1

    if y is not None:
        def A_hat(v):
            return wrapped_apply(y, op, v, t)
    else:
        A_hat = op.apply

    hist = []
    its = 0
    cycles = 0
    relres = beta / bnorm
    done = relres < tol
    V = np.empty((n, m + 1), order="F")
    R = np.empty((m + 1, m))
    cs = np.empty(m)
    sn = np.empty(m)
    g = np.empty(m + 1)

    while not done and its < max_iters:
        V[:, 0] = r / beta
        g[0] = beta
        j = 0
        happy = False
        pending = None
        while j < m and its < max_iters:
            w = A_hat(V[:, j])
            h, nn, vec, brk = cgs2(V[:, :j + 1], w, t)
            if not (math.isfinite(nn) and np.all(np.isfinite(h))):
                raise FloatingPointError(its + 1)
            col = np.empty(j + 2)
            col[:j + 1] = h
            col[j + 1] = nn
            for i in range(j):
                tmp = cs[i] * col[i] + sn[i] * col[i + 1]
                col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1]
                col[i] = tmp
            c, s, rr = _rot(col[j], col[j + 1])
            cs[j], sn[j] = c, s
            col[j] = rr
            R[:j + 1, j] = col[:j + 1]
            g[j + 1] = -s * g[j]
            g[j] = c * g[j]
            its += 1
            j += 1
            est = abs(g[j]) / bnorm
            pending = (its, est)
            if brk:
                happy = True
                break
            V[:, j] = vec
            if est < tol:
                break
            if j < m and its < max_iters and record_history:
                hist.append((its, est) + t.snap()[:3])
                pending = None

        z = np.empty(j)
        for i in range(j - 1, -1, -1):
            if R[i, i] == 0.0:
                raise ZeroDivisionError(i)
            z[i] = (g[i] - R[i, i + 1:j] @ z[i + 1:]) / R[i, i]
        upd = V[:, :j] @ z
        t.vector_updates += j
        if y is not None:
            upd = poly_eval(y, op, upd, t)
        x = x + upd
        t.vector_updates += 1
        cycles += 1
        r = b - op.apply(x)
        beta = float(np.linalg.norm(r))
        t.scalar_dots += 1
        relres = beta / bnorm
        if record_history and pending is not None:
            hist.append(pending + t.snap()[:3])
        if happy or relres < tol:
            done = True
    return OracleResult(x, done, its, relres, hist, t, cycles)
