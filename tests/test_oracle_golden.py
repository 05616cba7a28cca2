"""Pin the CPU oracle (oracle/pgmres_oracle.py) to golden vectors recorded from
the unchanged reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import pgmres_oracle as orc
from paper_1907_00072_b200 import workloads as wl


def _lap64(G):
    a, _ = G
    return orc.OracleMatrix(4096, 4096, a["lap64_row_ptr"], a["lap64_col_idx"], a["lap64_values"])


def test_rng_bitwise(golden):
    a, _ = golden
    assert np.array_equal(orc.sm64_uniform(0, 4096), a["rng_u0"])
    assert np.array_equal(orc.sm64_uniform(1, 4096), a["rng_u1"])
    assert np.array_equal(orc.sm64_uniform(7, 1000, 2.0, 5.0), a["rng_u7_hi"])
    # the product-side input generator draws the same stream, also by slices
    assert np.array_equal(wl.splitmix_uniform(0, 4096), a["rng_u0"])
    assert np.array_equal(wl.splitmix_uniform(1, 1000, start=3000), a["rng_u1"][3000:4000])


def test_laplacian_generator_matches_reference(golden):
    a, _ = golden
    h = wl.laplacian2d(64)
    assert np.array_equal(h.row_ptr, a["lap64_row_ptr"])
    assert np.array_equal(h.col_idx, a["lap64_col_idx"])
    assert np.array_equal(h.values, a["lap64_values"])
    # row-range generation concatenates to the whole matrix
    top, bot = wl.laplacian2d(64, rows=(0, 1000)), wl.laplacian2d(64, rows=(1000, 4096))
    assert np.array_equal(np.concatenate([top.col_idx, bot.col_idx]), h.col_idx)


def test_spmv_bitwise(golden):
    a, _ = golden
    A = _lap64(golden)
    x = orc.sm64_uniform(0, 4096)
    assert np.array_equal(A.matvec(x), a["cfg1_b"])
    R = orc.OracleMatrix(1000, 1000, a["rand1k_row_ptr"], a["rand1k_col_idx"], a["rand1k_values"])
    y = R.matvec(a["rand1k_x"])
    assert np.array_equal(y, a["rand1k_y"])
    # the reference SpMV is exactly a row-sequential mul-then-add loop
    loop = orc.matvec_rowseq(R.row_ptr, R.col_idx, R.values, a["rand1k_x"])
    assert np.array_equal(loop, a["rand1k_y"])


def test_apply_poly_bitwise(golden):
    a, meta = golden
    A = _lap64(golden)
    t = orc.Tally()
    A.tally = t
    out = orc.poly_eval(a["cfg1_y10"], A, a["cfg1_b"], t)
    assert np.array_equal(out, a["cfg1_pAb"])
    out2 = orc.wrapped_apply(a["cfg1_y10"], A, a["cfg1_b"], t)
    assert np.array_equal(out2, a["cfg1_ApAb"])
    assert t.spmvs == meta["cfg1_apply_counters"]["spmvs"]
    assert t.vector_updates == meta["cfg1_apply_counters"]["vector_updates"]
    assert np.array_equal(orc.poly_eval(a["cfg1_y25_rand"], A, a["cfg1_b"], orc.Tally()),
                          a["cfg1_p25b"])
    R = orc.OracleMatrix(1000, 1000, a["rand1k_row_ptr"], a["rand1k_col_idx"], a["rand1k_values"])
    assert np.array_equal(orc.poly_eval(a["rand1k_poly_y"], R, a["rand1k_x"], orc.Tally()),
                          a["rand1k_poly_out"])


def test_build_poly(golden):
    a, meta = golden
    A = _lap64(golden)
    t = orc.Tally()
    A.tally = t
    y, nrm = orc.min_res_poly(A, orc.sm64_uniform(1, 4096), 10, t)
    np.testing.assert_allclose(y, a["cfg1_y10"], rtol=1e-9, atol=0)
    assert nrm == pytest.approx(meta["cfg1_build"]["seed_norm"], rel=1e-15)
    c = meta["cfg1_build"]["counters"]
    assert (t.spmvs, t.dots, t.scalar_dots) == (c["spmvs"], c["dots"], c["scalar_dots"])
    with pytest.raises(orc.CholeskyFailureOracle) as err:
        orc.min_res_poly(A, orc.sm64_uniform(1, 4096), 13, orc.Tally())
    assert err.value.pivot == meta["cfg1_build13"]


def test_auto_degree(golden):
    a, meta = golden
    A = _lap64(golden)
    d, y, _ = orc.auto_deg(A, orc.sm64_uniform(1, 4096), 16, orc.Tally())
    assert d == meta["auto_lap64"]["degree"]
    np.testing.assert_allclose(y, a["auto_lap64_y"], rtol=1e-8)


def test_icgs(golden):
    a, meta = golden
    t = orc.Tally()
    h, nn, v, brk = orc.cgs2(a["icgs_basis"], a["icgs_w"], t)
    np.testing.assert_allclose(h, a["icgs_coeffs"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(v, a["icgs_vector"], rtol=0, atol=1e-14)
    assert nn == pytest.approx(meta["icgs"]["new_norm"], rel=1e-14)
    assert brk is False
    c = meta["icgs"]["counters"]
    assert (t.dots, t.scalar_dots, t.vector_updates) == (c["dots"], c["scalar_dots"], c["vector_updates"])


def _check_solve(res, rec, tally, exact=True):
    assert res.converged == rec["converged"]
    assert res.iterations == rec["iterations"]
    assert res.cycles == rec["cycles"]
    c = rec["counters"]
    assert (tally.spmvs, tally.dots, tally.scalar_dots, tally.vector_updates) == \
        (c["spmvs"], c["dots"], c["scalar_dots"], c["vector_updates"])
    assert res.final_relres == pytest.approx(rec["final_relres"], rel=1e-6)
    assert len(res.history) == rec["history_len"]
    for got, want in zip(res.history, rec["history"]):
        assert tuple(got[0:1]) + tuple(got[2:]) == tuple(int(v) for v in (want[0:1] + want[2:]))
        assert got[1] == pytest.approx(want[1], rel=1e-6)


def test_cfg1_solve_and_sweep(golden):
    a, meta = golden
    b = a["cfg1_b"]
    v0 = orc.sm64_uniform(1, 4096)
    for name, deg in (("cfg1_solve", 10), ("cfg1_sweep_None", None), ("cfg1_sweep_1", 1),
                      ("cfg1_sweep_4", 4), ("cfg1_sweep_8", 8), ("cfg1_sweep_12", 12)):
        t = orc.Tally()
        A = _lap64(golden)
        A.tally = t
        y = None
        if deg is not None:
            _, _, y, _ = orc.degree_policy(A, v0, deg, t)
        res = orc.gmres(A, b, y=y, m=40, tol=1e-8)
        _check_solve(res, meta[name], t)
    np.testing.assert_allclose(res.x if False else orc.gmres(
        _lap64(golden), b, y=a["cfg1_y10"], m=40, tol=1e-8).x, a["cfg1_solve_x"], rtol=0, atol=1e-9)


def test_convdiff_multicycle_and_x0(golden):
    a, meta = golden
    n = len(a["convdiff48_row_ptr"]) - 1
    mk = lambda t: orc.OracleMatrix(n, n, a["convdiff48_row_ptr"], a["convdiff48_col_idx"],
                                    a["convdiff48_values"], t)
    bc = orc.sm64_uniform(3, n)
    v0 = orc.sm64_uniform(4, n)
    t = orc.Tally()
    A = mk(t)
    _, _, y, _ = orc.degree_policy(A, v0, 6, t)
    _check_solve(orc.gmres(A, bc, y=y, m=20, tol=1e-9), meta["convdiff48_solve"], t)
    t = orc.Tally()
    A = mk(t)
    _, _, y, _ = orc.degree_policy(A, v0, 4, t)
    _check_solve(orc.gmres(A, bc, x0=a["convdiff48_x0"], y=y, m=15, tol=1e-8),
                 meta["convdiff48_x0_solve"], t)
    t = orc.Tally()
    _check_solve(orc.gmres(mk(t), bc, m=30, tol=1e-8, max_iters=400), meta["convdiff48_noprec"], t)


@pytest.mark.parametrize("c,kw", [(2, dict(grid=16)), (4, dict(grid=12)), (5, dict(grid=48))])
def test_small_configs_degree_policy(golden, c, kw):
    """Reduced configs: this repo's generators are pinned by hash, and the oracle
    reproduces the reference's degree policy, iterations and counters."""
    import hashlib
    a, meta = golden
    cfg = wl.CONFIGS[c]
    h = wl.make_matrix(cfg, **kw)
    sha = hashlib.sha256(h.row_ptr.tobytes() + h.col_idx.tobytes() + h.values.tobytes()).digest()
    assert bytes(a[f"small{c}_sha"]) == sha
    rec = meta[f"small{c}"]
    t = orc.Tally()
    A = orc.OracleMatrix.of(h, t)
    req, eff, y, _ = orc.degree_policy(A, wl.make_v0(A.nrows), cfg["degree"], t)
    assert (req, eff) == (rec["requested_degree"], rec["effective_degree"])
    res = orc.gmres(A, wl.make_rhs(cfg, h), y=y, m=cfg["m"], tol=cfg["tol"])
    _check_solve(res, rec, t)
