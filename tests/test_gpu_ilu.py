"""ILU(0) left preconditioning on the device (reference
ilu.py:38-114, IluPreconditionedOperator gmres.py:63-95).  GPU only.

Bars: factors bit-identical (host native factorisation, checked on the CPU
too); M^{-1} v within 1e-14 relative of the reference's application (its short
row dots go through OpenBLAS ddot, whose order is the library's); the
left-preconditioned polynomial solve from the reference's coefficients within
+-2 iterations, relres < tol, counters (incl. prec_applies) by the reference's
laws."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_00072_b200 as pg  # noqa: E402
from oracle import pgmres_oracle as orc  # noqa: E402
from paper_1907_00072_b200 import workloads as wl  # noqa: E402

pytestmark = pytest.mark.gpu


def _rel(u, w):
    return float(np.linalg.norm(u - w) / max(np.linalg.norm(w), 1e-300))


def _cd48(a):
    n = len(a["convdiff48_row_ptr"]) - 1
    return wl.CsrHost(n, n, a["convdiff48_row_ptr"], a["convdiff48_col_idx"],
                      a["convdiff48_values"])


def test_ilu_apply_matches_reference(golden):
    a, _ = golden
    A = wl.CsrHost(4096, 4096, a["lap64_row_ptr"], a["lap64_col_idx"], a["lap64_values"])
    F = pg.ilu0_factor(A)
    got = pg.ilu0_apply(F, a["cfg1_b"])
    assert _rel(got, a["ilu_lap64_apply"]) < 1e-14
    C = _cd48(a)
    Fc = pg.ilu0_factor(C)
    bc = orc.sm64_uniform(3, C.nrows)
    assert _rel(pg.ilu0_apply(Fc, bc), a["ilu_convdiff48_apply"]) < 1e-14
    # torch in -> torch out, repeated applications reuse the device factors
    t = torch.from_numpy(bc).cuda()
    for _ in range(3):
        out = pg.ilu0_apply(Fc, t)
        assert isinstance(out, torch.Tensor) and out.is_cuda
    assert _rel(out.cpu().numpy(), a["ilu_convdiff48_apply"]) < 1e-14
    with pytest.raises(pg.DimensionMismatchError):
        pg.ilu0_apply(Fc, np.ones(5))


def test_ilu_exact_classes():
    """No-fill patterns make M = A: identity, diagonal, tridiagonal, upper."""
    ident = wl.CsrHost(5, 5, np.arange(6), np.arange(5), np.ones(5))
    v = np.arange(5.0)
    assert np.array_equal(pg.ilu0_apply(pg.ilu0_factor(ident), v), v)
    diag = wl.CsrHost(2, 2, np.arange(3), np.arange(2), np.array([2.0, 4.0]))
    assert np.array_equal(pg.ilu0_apply(pg.ilu0_factor(diag), np.array([2.0, 4.0])),
                          np.ones(2))
    gen = np.random.default_rng(12)
    for n in (2, 5, 11, 200):
        d = 4.0 + gen.random(n)
        lo, up = -gen.random(n - 1), -gen.random(n - 1)
        rows = np.concatenate([np.arange(n), np.arange(1, n), np.arange(n - 1)])
        cols = np.concatenate([np.arange(n), np.arange(n - 1), np.arange(1, n)])
        vals = np.concatenate([d, lo, up])
        o = np.lexsort((cols, rows))
        rp = np.zeros(n + 1, np.int64)
        np.add.at(rp, rows + 1, 1)
        T = wl.CsrHost(n, n, np.cumsum(rp), cols[o], vals[o])
        op = pg.DeviceIluOperator(T, pg.ilu0_factor(T))
        for _ in range(3):
            x = gen.uniform(-1, 1, n)
            np.testing.assert_allclose(op.apply(x), x, atol=1e-12)
        assert op.counters.spmvs == 3 and op.counters.prec_applies == 3
        op.close()


def test_ilu_operator_composition_and_precondition(golden):
    a, _ = golden
    C = _cd48(a)
    F = pg.ilu0_factor(C)
    c = pg.CostCounters()
    op = pg.DeviceIluOperator(C, F, c)
    assert op.kind == "left-preconditioned"
    bc = orc.sm64_uniform(3, C.nrows)
    b_eff = op.precondition(bc)
    assert _rel(b_eff, a["ilu_convdiff48_beff"]) < 1e-14
    assert c.prec_applies == 1 and c.spmvs == 0
    x = orc.sm64_uniform(5, C.nrows)
    Ao = orc.OracleMatrix.of(C)
    vals, diag = orc.ilu0_factor(Ao)
    want = orc.ilu0_apply(Ao, vals, diag, Ao.matvec(x))
    assert _rel(op.apply(x), want) < 1e-14
    assert c.spmvs == 1 and c.prec_applies == 2
    with pytest.raises(pg.ParameterError):  # the fused root form needs plain SpMV
        pg.apply_poly(pg.PolyCoefficients(2, np.array([1.0, 0.1, 0.01]), 1.0), op, x, c,
                      form="roots")
    op.close()


@pytest.mark.parametrize("x0", [False, True])
def test_ilu_left_preconditioned_polynomial_solve(golden, x0):
    """The CLI's --ilu flow on the device: precondition b, build the
    polynomial on M^{-1}A, solve; against the reference run (golden) and the
    oracle solve from the same coefficients."""
    a, meta = golden
    C = _cd48(a)
    F = pg.ilu0_factor(C)
    c = pg.CostCounters()
    op = pg.DeviceIluOperator(C, F, c)
    b_eff = op.precondition(orc.sm64_uniform(3, C.nrows))
    poly = pg.build_poly(op, wl.splitmix_uniform(4, C.nrows), 5, c)
    rec = meta["ilu_convdiff48_solve"]
    assert c.as_dict() == rec["build_counters"]
    y = a["ilu_convdiff48_y"]
    # the power-basis normal equations amplify rounding; the coefficients agree
    # to the conditioning, the solve is what must agree
    assert np.allclose(poly.y, y, rtol=1e-4, atol=0)
    x0v = orc.sm64_uniform(9, C.nrows) * 0.1 if x0 else None
    before = c.as_dict()
    res = pg.solve(op, b_eff, x0=x0v, right_prec=pg.PolyCoefficients(5, y, 1.0),
                   config=pg.GmresConfig(20, 1e-10))
    Ao = orc.OracleMatrix.of(C, orc.Tally())
    vals, diag = orc.ilu0_factor(Ao)
    oop = orc.OracleIluOperator(Ao, vals, diag)
    ref = orc.gmres(oop, a["ilu_convdiff48_beff"], x0=x0v, y=y, m=20, tol=1e-10)
    assert res.converged and ref.converged and res.final_relres < 1e-10
    assert abs(res.iterations - ref.iterations) <= 2
    if not x0:
        assert abs(res.iterations - rec["iterations"]) <= 2
        np.testing.assert_allclose(res.x, a["ilu_convdiff48_x"], rtol=0, atol=1e-8)
    got = {k: c.as_dict()[k] - before[k] for k in before}
    if (res.iterations, res.cycles) == (ref.iterations, ref.cycles):
        assert (got["spmvs"], got["dots"], got["scalar_dots"], got["vector_updates"],
                got["prec_applies"]) == Ao.tally.snap()
    assert got["prec_applies"] == got["spmvs"]
    op.close()


def test_ilu_refuses_multi_shard():
    A = wl.laplacian2d(8)
    F = pg.ilu0_factor(A)
    e = pg.DeviceMatrixOperator(A, shards=2).engine
    with pytest.raises(pg.ParameterError):
        e.attach_ilu(F)


@pytest.mark.parametrize("n,seed", [(3000, 1), (777, 2)])
def test_ilu_irregular_pattern_sweeps(n, seed):
    """Random nonsymmetric pattern (rows of 1..40 entries, columns anywhere):
    deep, irregular dependency chains for the sync-free sweeps.  Factors are
    bit-identical to the oracle restatement; M^{-1} v within 1e-13."""
    gen = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        m = int(gen.integers(1, 40))
        c = np.unique(np.concatenate([[i], gen.integers(0, n, m)]))
        v = gen.standard_normal(len(c))
        v[c == i] = 1.5 * np.abs(v).sum() + 1.0  # dominant diagonal: no tiny pivots
        rows.append(np.full(len(c), i))
        cols.append(c)
        vals.append(v)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum([len(c) for c in cols], out=rp[1:])
    A = wl.CsrHost(n, n, rp, np.concatenate(cols), np.concatenate(vals))
    F = pg.ilu0_factor(A)
    Ao = orc.OracleMatrix.of(A)
    ov, od = orc.ilu0_factor(Ao)
    assert np.array_equal(F.values, ov) and np.array_equal(F.diag_ptr, od)
    for s in range(3):
        v = gen.uniform(-1, 1, n)
        got = pg.ilu0_apply(F, v)
        want = orc.ilu0_apply(Ao, ov, od, v)
        assert _rel(got, want) < 1e-13
