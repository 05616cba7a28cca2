"""ILU(0) on the CPU side: the oracle restatement and the
native host factorisation (pg_ilu0_factor) against the reference's own
factors / applications recorded in tests/golden (ilu.py:38-114)."""

import numpy as np
import pytest

from oracle import pgmres_oracle as orc


def _mat(a, name, n):
    return orc.OracleMatrix(n, n, a[f"{name}_row_ptr"], a[f"{name}_col_idx"], a[f"{name}_values"])


def _cd48(a):
    return _mat(a, "convdiff48", len(a["convdiff48_row_ptr"]) - 1)


def test_oracle_ilu_matches_reference_bitwise(golden):
    a, _ = golden
    A = _mat(a, "lap64", 4096)
    vals, diag = orc.ilu0_factor(A)
    assert np.array_equal(vals, a["ilu_lap64_values"])
    assert np.array_equal(diag, a["ilu_lap64_diag_ptr"])
    assert np.array_equal(orc.ilu0_apply(A, vals, diag, a["cfg1_b"]), a["ilu_lap64_apply"])
    C = _cd48(a)
    vc, dc = orc.ilu0_factor(C)
    assert np.array_equal(vc, a["ilu_convdiff48_values"])
    bc = orc.sm64_uniform(3, C.nrows)
    assert np.array_equal(orc.ilu0_apply(C, vc, dc, bc), a["ilu_convdiff48_apply"])
    vs, _ = orc.ilu0_factor(C, diag_shift=0.3)
    assert np.array_equal(vs, a["ilu_convdiff48_shift_values"])


def test_native_ilu_factor_bitwise_and_pivots(golden):
    """pg_ilu0_factor (host C++, no GPU) reproduces the reference factors bit
    for bit, and its pivot failures (row, structural message)."""
    import paper_1907_00072_b200 as pg
    from paper_1907_00072_b200 import workloads as wl
    a, meta = golden
    A = wl.CsrHost(4096, 4096, a["lap64_row_ptr"], a["lap64_col_idx"], a["lap64_values"])
    F = pg.ilu0_factor(A)
    assert np.array_equal(F.values, a["ilu_lap64_values"])
    assert np.array_equal(F.diag_ptr, a["ilu_lap64_diag_ptr"]) and F.nnz == A.nnz
    n = len(a["convdiff48_row_ptr"]) - 1
    C = wl.CsrHost(n, n, a["convdiff48_row_ptr"], a["convdiff48_col_idx"],
                   a["convdiff48_values"])
    assert np.array_equal(pg.ilu0_factor(C).values, a["ilu_convdiff48_values"])
    assert np.array_equal(pg.ilu0_factor(C, diag_shift=0.3).values,
                          a["ilu_convdiff48_shift_values"])
    zp = wl.CsrHost(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]),
                    np.array([0.0, 1.0, 1.0, 1.0]))
    with pytest.raises(pg.PivotError) as err:
        pg.ilu0_factor(zp)
    assert err.value.row == meta["ilu_zero_pivot"]["row"]
    assert str(err.value) == meta["ilu_zero_pivot"]["message"]
    md = wl.CsrHost(2, 2, np.array([0, 1, 2]), np.array([1, 0]), np.array([1.0, 1.0]))
    with pytest.raises(pg.PivotError) as err:
        pg.ilu0_factor(md)
    assert err.value.row == meta["ilu_missing_diag"]["row"]
    assert "structural" in str(err.value)
    # diag_shift rescues the zero pivot; upper-triangular input is untouched
    assert pg.ilu0_factor(zp, diag_shift=2.0).values[0] == 2.0
    ut = wl.CsrHost(3, 3, np.array([0, 2, 4, 5]), np.array([0, 2, 1, 2, 2]),
                    np.array([2.0, 0.5, 3.0, -1.0, 4.0]))
    assert np.array_equal(pg.ilu0_factor(ut).values, ut.values)
    with pytest.raises(pg.ParameterError):
        pg.ilu0_factor(wl.CsrHost(2, 3, np.array([0, 1, 2]), np.array([0, 1]), np.ones(2)))


def test_oracle_ilu_left_preconditioned_solve(golden):
    """The --ilu flow (cli.py:252-277): b_eff = M^{-1} b, then the
    left-preconditioned polynomial solve from the reference's coefficients;
    iterations and every counter equal the reference's."""
    a, meta = golden
    t = orc.Tally()
    C = _cd48(a)
    C.tally = t
    vals, diag = orc.ilu0_factor(C)
    op = orc.OracleIluOperator(C, vals, diag)
    b_eff = op.precondition(orc.sm64_uniform(3, C.nrows))
    assert np.array_equal(b_eff, a["ilu_convdiff48_beff"])
    t2 = orc.Tally()
    C.tally = op.tally = t2
    res = orc.gmres(op, b_eff, y=a["ilu_convdiff48_y"], m=20, tol=1e-10)
    rec = meta["ilu_convdiff48_solve"]
    assert res.iterations == rec["iterations"] and res.converged
    want = np.array([rec["counters"][k] - rec["build_counters"][k] for k in
                     ("spmvs", "dots", "scalar_dots", "vector_updates", "prec_applies")])
    assert tuple(want) == t2.snap()
