"""Parity of the CUDA path (through the C-ABI) with the CPU oracle and the
reference golden vectors.  GPU only.

Bars (BASELINE.json north_star):
* SpMV and p(A)v: bit-identical (the oracle restates the reference's
  row-sequential mul-then-add order; the device kernel reproduces it), which
  is stronger than the 1e-10 relative bound;
* CGS2: coefficients / vector within 1e-13 (OpenBLAS order is opaque);
* solves: iterations within +-2 of the reference, final relres < tol,
  counters exactly equal to the reference's laws.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_00072_b200 as pg  # noqa: E402
from oracle import pgmres_oracle as orc  # noqa: E402
from paper_1907_00072_b200 import workloads as wl  # noqa: E402

pytestmark = pytest.mark.gpu


def _csr(a, name, n):
    return wl.CsrHost(n, n, a[f"{name}_row_ptr"], a[f"{name}_col_idx"], a[f"{name}_values"])


def _lap64(golden):
    return _csr(golden[0], "lap64", 4096)


def _oracle(h, t=None):
    return orc.OracleMatrix.of(h, t)


# ---------------------------------------------------------------------------
# SpMV
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("shards", [1, 2, 3])
def test_spmv_bitwise_goldens(golden, shards):
    a, _ = golden
    A = _lap64(golden)
    op = pg.DeviceMatrixOperator(A, shards=shards)
    x = orc.sm64_uniform(0, 4096)
    assert np.array_equal(op.apply(x), a["cfg1_b"])
    R = _csr(a, "rand1k", 1000)
    opr = pg.DeviceMatrixOperator(R, shards=shards)
    assert np.array_equal(opr.apply(a["rand1k_x"]), a["rand1k_y"])
    assert opr.counters.spmvs == 1


@pytest.mark.parametrize("sigma", [1, 64, 4096])
def test_spmv_sell_sorting_is_exact(sigma):
    h = wl.random_lognormal(20000, seed=7)
    op = pg.DeviceMatrixOperator(h, sigma=sigma)
    x = wl.splitmix_uniform(11, h.nrows)
    assert np.array_equal(op.apply(x), _oracle(h).matvec(x))


def test_spmv_empty_rows_and_ragged():
    gen = np.random.default_rng(3)
    n = 777
    lens = gen.integers(0, 40, n)
    lens[::7] = 0
    rows = np.repeat(np.arange(n), lens)
    cols = np.concatenate([np.sort(gen.choice(n, L, replace=False)) for L in lens])
    vals = gen.standard_normal(len(cols))
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    h = wl.CsrHost(n, n, rp, cols, vals)
    x = gen.standard_normal(n)
    x[5] = -0.0
    for shards in (1, 4):
        got = pg.DeviceMatrixOperator(h, shards=shards).apply(x)
        assert np.array_equal(got, _oracle(h).matvec(x))
        assert np.all(got[lens == 0] == 0.0)


def test_spmv_torch_in_torch_out():
    A = wl.convdiff3d_7pt(20)
    op = pg.DeviceMatrixOperator(A)
    x = torch.from_numpy(wl.splitmix_uniform(2, A.nrows)).cuda()
    y = op.apply(x)
    assert isinstance(y, torch.Tensor) and y.is_cuda
    assert np.array_equal(y.cpu().numpy(), _oracle(A).matvec(x.cpu().numpy()))


def test_dimension_and_shape_errors():
    op = pg.DeviceMatrixOperator(wl.laplacian2d(8))
    with pytest.raises(pg.DimensionMismatchError):
        op.apply(np.ones(63))
    with pytest.raises(pg.ParameterError):
        pg.DeviceMatrixOperator(wl.CsrHost(2, 3, [0, 1, 2], [0, 2], [1.0, 1.0]))


# ---------------------------------------------------------------------------
# p(A)v
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("shards", [1, 2, 4])
def test_apply_poly_bitwise_cfg1(golden, shards):
    a, meta = golden
    op = pg.DeviceMatrixOperator(_lap64(golden), shards=shards)
    c = pg.CostCounters()
    op.counters = c
    p = pg.PolyCoefficients(10, a["cfg1_y10"], 1.0)
    got = pg.apply_poly(p, op, a["cfg1_b"], c)
    assert np.array_equal(got, a["cfg1_pAb"])
    wrapped = pg.PolynomialWrappedOperator(op, p).apply(a["cfg1_b"])
    assert np.array_equal(wrapped, a["cfg1_ApAb"])
    assert c.spmvs == meta["cfg1_apply_counters"]["spmvs"]
    assert c.vector_updates == meta["cfg1_apply_counters"]["vector_updates"]
    p25 = pg.PolyCoefficients(25, a["cfg1_y25_rand"], 1.0)
    assert np.array_equal(pg.apply_poly(p25, op, a["cfg1_b"], c), a["cfg1_p25b"])


def test_apply_poly_bitwise_random_and_degree0(golden):
    a, _ = golden
    op = pg.DeviceMatrixOperator(_csr(a, "rand1k", 1000))
    p = pg.PolyCoefficients(6, a["rand1k_poly_y"], 1.0)
    assert np.array_equal(pg.apply_poly(p, op, a["rand1k_x"], pg.CostCounters()),
                          a["rand1k_poly_out"])
    c = pg.CostCounters()
    op.counters = c
    out = pg.apply_poly(pg.PolyCoefficients(0, np.array([2.5]), 1.0), op, a["rand1k_x"], c)
    assert np.array_equal(out, 2.5 * a["rand1k_x"])
    assert c.spmvs == 0 and c.vector_updates == 1


@pytest.mark.parametrize("cfg,kw,deg", [(2, dict(grid=30), 25), (4, dict(grid=16), 16),
                                        (5, dict(grid=64), 32), (3, dict(size=30000), 40)])
def test_apply_poly_bitwise_configs(cfg, kw, deg):
    h = wl.make_matrix(wl.CONFIGS[cfg], **kw)
    y = np.random.default_rng(cfg).uniform(-1, 1, deg + 1) * 0.5 ** np.arange(deg + 1)
    v = wl.splitmix_uniform(5, h.nrows)
    want = orc.poly_eval(y, _oracle(h), v, orc.Tally())
    for shards in (1, 3):
        op = pg.DeviceMatrixOperator(h, shards=shards)
        got = pg.apply_poly(pg.PolyCoefficients(deg, y, 1.0), op, v, pg.CostCounters())
        assert np.array_equal(got, want)


# ---------------------------------------------------------------------------
# CGS2
# ---------------------------------------------------------------------------
def test_icgs_matches_golden(golden):
    a, meta = golden
    c = pg.CostCounters()
    res = pg.icgs(a["icgs_basis"], a["icgs_w"], c)
    np.testing.assert_allclose(res.coeffs, a["icgs_coeffs"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(res.vector, a["icgs_vector"], rtol=0, atol=1e-13)
    assert res.new_norm == pytest.approx(meta["icgs"]["new_norm"], rel=1e-13)
    assert not res.breakdown
    mc = meta["icgs"]["counters"]
    assert (c.dots, c.scalar_dots, c.vector_updates) == (mc["dots"], mc["scalar_dots"],
                                                         mc["vector_updates"])


def test_icgs_properties_and_edges():
    gen = np.random.default_rng(42)
    for _ in range(10):
        n = int(gen.integers(5, 3000))
        j = int(gen.integers(1, min(n, 51)))
        basis = np.linalg.qr(gen.standard_normal((n, j)))[0]
        w = gen.uniform(-1, 1, n)
        res = pg.icgs(basis, w, pg.CostCounters())
        h, nn, v, brk = orc.cgs2(basis, w, orc.Tally())
        np.testing.assert_allclose(res.coeffs, h, rtol=0, atol=1e-12)
        assert res.new_norm == pytest.approx(nn, rel=1e-12)
        assert np.max(np.abs(basis.T @ res.vector)) <= 1e-12
        assert abs(np.linalg.norm(res.vector) - 1.0) <= 1e-12
    # empty basis
    res = pg.icgs(np.empty((4, 0)), np.array([3.0, 0.0, 0.0, 4.0]), pg.CostCounters())
    assert res.coeffs.shape == (0,) and res.new_norm == pytest.approx(5.0)
    # dependent vector -> happy breakdown
    e0 = np.eye(3)[:, :1]
    res = pg.icgs(e0, 2.0 * e0[:, 0], pg.CostCounters())
    assert res.breakdown and res.coeffs == pytest.approx([2.0])


# ---------------------------------------------------------------------------
# polynomial construction
# ---------------------------------------------------------------------------
def test_build_poly_cfg1(golden):
    a, meta = golden
    c = pg.CostCounters()
    op = pg.DeviceMatrixOperator(_lap64(golden), c)
    v0 = orc.sm64_uniform(1, 4096)
    p = pg.build_poly(op, v0, 10, c)
    # reference-order seed norm (OpenBLAS ddot): bitwise np.linalg.norm
    assert p.seed_norm == meta["cfg1_build"]["seed_norm"]
    mc = meta["cfg1_build"]["counters"]
    assert (c.spmvs, c.dots, c.scalar_dots) == (mc["spmvs"], mc["dots"], mc["scalar_dots"])
    # the device Gram is the oracle's OpenBLAS-order Gram bit for bit
    from paper_1907_00072_b200.polyprec import _device_power_gram
    Gd, nrm = _device_power_gram(op, v0, 11, pg.CostCounters())
    t = orc.Tally()
    A = _oracle(_lap64(golden), t)
    Go, nrm_o = orc.gram_full_blas(A, v0, 11)
    assert nrm == nrm_o and np.array_equal(Gd, Go)
    # deg-10 normal equations have cond ~1e14, so y is checked by its quality:
    # the minimum-residual value |v - A p(A) v| (polyprec.py:1-9)
    v = v0 / nrm

    def resid(y):
        return np.linalg.norm(v - orc.wrapped_apply(y, A, v, orc.Tally()))

    assert resid(p.y) <= resid(a["cfg1_y10"]) * 1.01 + 1e-12
    # every recorded pass/fail decision of the reference (golden.json):
    # build_poly(12) returns, 13 and 14 fail at pivot 14
    for d in (12, 13, 14):
        rec = meta[f"cfg1_build{d}"]
        if rec == "ok":
            q = pg.build_poly(op, v0, d, pg.CostCounters())
            assert q.degree == d and np.all(np.isfinite(q.y))
        else:
            with pytest.raises(pg.CholeskyFailure) as err:
                pg.build_poly(op, v0, d, pg.CostCounters())
            assert err.value.pivot == rec
    # opt-in exact arithmetic (double-double Gram, compensated Cholesky): the
    # decision of a correctly rounded Gram, here pivot 12 for degree 13
    P13 = orc.power_columns(A, v0 / np.linalg.norm(v0), 14)
    with pytest.raises(pg.CholeskyFailure) as err:
        pg.build_poly(op, v0, 13, pg.CostCounters(), decision="exact")
    assert err.value.pivot == orc.chol_pivot_exact(orc.gram_exact(P13)[1:, 1:])
    with pytest.raises(pg.ParameterError):
        pg.build_poly(op, v0, 3, pg.CostCounters(), decision="fp32")


def test_known_answer_diag12_and_auto():
    op = pg.DeviceMatrixOperator(wl.CsrHost(2, 2, [0, 1, 2], [0, 1], [1.0, 2.0]))
    p = pg.build_poly(op, np.array([1.0, 1.0]), 1, pg.CostCounters())
    assert p.y == pytest.approx([1.5, -0.5], abs=1e-12)
    q = pg.auto_degree(op, np.array([1.0, 1.0]), 5, pg.CostCounters())
    assert q.degree == 1
    ident = pg.DeviceMatrixOperator(wl.CsrHost(4, 4, np.arange(5), np.arange(4), np.ones(4)))
    q = pg.auto_degree(ident, np.array([1.0, 2.0, 3.0, -1.0]), 5, pg.CostCounters())
    assert q.degree == 0 and q.y == pytest.approx([1.0])
    with pytest.raises(pg.ParameterError):
        pg.build_poly(op, np.zeros(2), 1, pg.CostCounters())


def test_auto_degree_lap64(golden):
    a, meta = golden
    c = pg.CostCounters()
    op = pg.DeviceMatrixOperator(_lap64(golden), c)
    v0 = orc.sm64_uniform(1, 4096)
    p = pg.auto_degree(op, v0, 16, c)
    assert p.degree == meta["auto_lap64"]["degree"]  # the reference's choice (12)
    assert (c.spmvs, c.dots) == (meta["auto_lap64"]["counters"]["spmvs"], 2)
    # opt-in exact decision (10)
    q = pg.auto_degree(op, v0, 16, pg.CostCounters(), decision="exact")
    P = orc.power_columns(_oracle(_lap64(golden)), v0 / np.linalg.norm(v0), 17)
    assert q.degree == orc.auto_deg_exact(orc.gram_exact(P), 16)


def test_auto_degree_bidiag2_and_cli_seed(golden):
    _, meta = golden
    from paper_1907_00072_b200 import problems
    op = pg.DeviceMatrixOperator(problems.bidiag2())
    p = pg.auto_degree(op, wl.splitmix_uniform(1, 5000), 20, pg.CostCounters())
    assert p.degree == meta["auto_bidiag2"]["degree"]  # 10 (exact arithmetic: 14)
    np.testing.assert_allclose(p.y, golden[0]["auto_bidiag2_y"], rtol=1e-6)
    p = pg.auto_degree(op, wl.splitmix_uniform(4, 5000), 20, pg.CostCounters())
    assert p.degree == meta["cli_auto"]["summary"]["degree"]  # 13


# ---------------------------------------------------------------------------
# solves
# ---------------------------------------------------------------------------
def _snap(c):
    return np.array(c.snapshot()[:4])


def _solve_pair(h, b, deg, m, tol, shards=1, x0=None, max_iters=200000, v0=None):
    """Device: degree policy + solve.  Oracle: the same solve from the SAME
    polynomial coefficients (the power-basis normal equations are so
    ill-conditioned that y itself is rounding-sensitive; the solve is what
    must agree).  Returns (res, solve_counters, oracle_result, oracle_tally, poly)."""
    c = pg.CostCounters()
    op = pg.DeviceMatrixOperator(h, c, shards=shards)
    poly = None
    if deg is not None:
        poly, _ = pg.build_poly_or_auto(op, wl.make_v0(h.nrows) if v0 is None else v0, deg, c)
    before = _snap(c)
    res = pg.solve(op, b, x0=x0, right_prec=poly, config=pg.GmresConfig(m, tol, max_iters))
    t = orc.Tally()
    ref = orc.gmres(_oracle(h, t), b, x0=x0, y=None if poly is None else poly.y, m=m, tol=tol,
                    max_iters=max_iters)
    op.close()
    return res, _snap(c) - before, ref, t, poly, c


def _agree(res, solve_c, ref, t, tol, c):
    assert res.converged == ref.converged
    assert abs(res.iterations - ref.iterations) <= 2, (res.iterations, ref.iterations)
    if ref.converged:
        assert res.final_relres < tol
    if (res.iterations, res.cycles) == (ref.iterations, ref.cycles):
        assert tuple(solve_c) == t.snap()[:4]  # identical accounting
    assert res.history[-1][2:] == (c.spmvs, c.dots, c.scalar_dots)
    assert [r[0] for r in res.history] == list(range(1, len(res.history) + 1))


@pytest.mark.parametrize("name,deg", [("cfg1_solve", 10), ("cfg1_sweep_None", None),
                                      ("cfg1_sweep_1", 1), ("cfg1_sweep_4", 4),
                                      ("cfg1_sweep_8", 8), ("cfg1_sweep_12", 12)])
def test_cfg1_solves(golden, name, deg):
    a, meta = golden
    rec = meta[name]
    res, sc, ref, t, poly, c = _solve_pair(_lap64(golden), a["cfg1_b"], deg, 40, 1e-8)
    _agree(res, sc, ref, t, 1e-8, c)
    # and against the unmodified reference's own run
    assert abs(res.iterations - rec["iterations"]) <= 2
    if deg is not None:
        assert poly.degree == deg == rec["effective_degree"]
        d = deg
        assert c.spmvs == (d + 1) * res.iterations + (d + 1) + d * res.cycles + res.cycles
        assert c.dots == 3 * res.iterations + 2
    if name == "cfg1_solve":
        np.testing.assert_allclose(res.x, a["cfg1_solve_x"], rtol=0, atol=1e-6)
        tr = np.linalg.norm(a["cfg1_b"] - _oracle(_lap64(golden)).matvec(res.x))
        assert res.final_relres == pytest.approx(tr / np.linalg.norm(a["cfg1_b"]), rel=1e-6)


@pytest.mark.parametrize("shards", [1, 2])
def test_convdiff_multicycle_x0_noprec(golden, shards):
    a, meta = golden
    n = len(a["convdiff48_row_ptr"]) - 1
    C = _csr(a, "convdiff48", n)
    bc = orc.sm64_uniform(3, n)
    v0 = orc.sm64_uniform(4, n)
    res, sc, ref, t, poly, c = _solve_pair(C, bc, 6, 20, 1e-9, shards, v0=v0)
    _agree(res, sc, ref, t, 1e-9, c)
    res, sc, ref, t, poly, c = _solve_pair(C, bc, 4, 15, 1e-8, shards, x0=a["convdiff48_x0"],
                                           v0=v0)
    _agree(res, sc, ref, t, 1e-8, c)
    res, sc, ref, t, poly, c = _solve_pair(C, bc, None, 30, 1e-8, shards, max_iters=400)
    rec = meta["convdiff48_noprec"]
    assert not res.converged and res.iterations == 400 == rec["iterations"]
    assert res.final_relres == pytest.approx(rec["final_relres"], rel=1e-3)
    assert c.spmvs == rec["counters"]["spmvs"] and c.dots == rec["counters"]["dots"]


@pytest.mark.parametrize("cfg,kw", [(2, dict(grid=16)), (3, dict(size=4000)), (4, dict(grid=12)),
                                    (5, dict(grid=48))])
def test_small_configs_with_degree_policy(golden, cfg, kw):
    """Reduced configs 2-5 (config 3: the random, sigma-sorted SELL operator):
    requested degree -> build or auto-degree fallback on the device, which
    takes the reference's recorded decision; the solve agrees with the oracle
    run from the same y and with the reference's own recorded run."""
    a, meta = golden
    rec = meta[f"small{cfg}"]
    conf = wl.CONFIGS[cfg]
    h = wl.make_matrix(conf, **kw)
    b = wl.make_rhs(conf, h)
    max_iters = 300 if cfg == 3 else 200000
    res, sc, ref, t, poly, c = _solve_pair(h, b, conf["degree"], conf["m"], conf["tol"],
                                           max_iters=max_iters)
    _agree(res, sc, ref, t, conf["tol"], c)
    assert poly.degree == rec["effective_degree"]
    assert res.converged == rec["converged"]
    assert abs(res.iterations - rec["iterations"]) <= 2
    if not rec["converged"]:
        assert res.final_relres == pytest.approx(rec["final_relres"], rel=0.1)


def test_identity_zero_rhs_and_nan_breakdown():
    ident = wl.CsrHost(6, 6, np.arange(7), np.arange(6), np.ones(6))
    op = pg.DeviceMatrixOperator(ident)
    b = np.array([3.0, -1.0, 0.5, 2.0, 0.0, 9.0])
    res = pg.solve(op, b)
    assert res.converged and res.iterations == 1
    np.testing.assert_allclose(res.x, b, atol=1e-14)
    assert op.counters.spmvs == 2
    res = pg.solve(op, np.zeros(6))
    assert res.converged and res.iterations == 0 and np.array_equal(res.x, np.zeros(6))
    nanop = pg.DeviceMatrixOperator(wl.CsrHost(4, 4, np.arange(5), np.arange(4),
                                               np.full(4, np.nan)))
    with pytest.raises(pg.NumericalBreakdownError) as err:
        pg.solve(nanop, np.ones(4))
    assert err.value.iteration == 1


def test_max_iters_exhaustion_and_history_law():
    A = wl.convdiff2d_9pt(40, 0.01)
    b = wl.splitmix_uniform(0, A.nrows)
    c = pg.CostCounters()
    op = pg.DeviceMatrixOperator(A, c)
    res = pg.solve(op, b, config=pg.GmresConfig(3, 1e-14, 5))
    assert not res.converged and res.iterations == 5 and res.final_relres > 1e-14
    t = orc.Tally()
    ref = orc.gmres(_oracle(A, t), b, m=3, tol=1e-14, max_iters=5)
    assert res.final_relres == pytest.approx(ref.final_relres, rel=1e-9)
    assert [r[0] for r in res.history] == [r[0] for r in ref.history]
    assert [r[2:] for r in res.history] == [r[2:] for r in ref.history]


def test_torch_solve_keeps_vectors_on_device():
    A = wl.convdiff3d_7pt(24)
    b = torch.from_numpy(wl.splitmix_uniform(0, A.nrows)).cuda()
    c = pg.CostCounters()
    op = pg.DeviceMatrixOperator(A, c)
    poly, _ = pg.build_poly_or_auto(op, torch.from_numpy(wl.make_v0(A.nrows)).cuda(), 8, c)
    res = pg.solve(op, b, right_prec=poly, config=pg.GmresConfig(50, 1e-10))
    assert isinstance(res.x, torch.Tensor) and res.x.is_cuda and res.converged
    r = b.cpu().numpy() - _oracle(A).matvec(res.x.cpu().numpy())
    assert np.linalg.norm(r) / np.linalg.norm(b.cpu().numpy()) == pytest.approx(
        res.final_relres, rel=1e-6)


# ---------------------------------------------------------------------------
# full BASELINE sizes: size-independent properties
# ---------------------------------------------------------------------------
@pytest.mark.slow
def test_cfg2_full_size_poly_bitwise_and_shard_invariance():
    h = wl.make_matrix(wl.CONFIGS[2])  # n = 1e6, nnz = 6.94M
    y = np.random.default_rng(0).uniform(-1, 1, 14) * 0.3 ** np.arange(14)
    v = wl.splitmix_uniform(1, h.nrows)
    want = orc.poly_eval(y, _oracle(h), v, orc.Tally())
    p = pg.PolyCoefficients(13, y, 1.0)
    for shards in (1, 4):
        op = pg.DeviceMatrixOperator(h, shards=shards)
        assert np.array_equal(pg.apply_poly(p, op, v, pg.CostCounters()), want)
        op.close()


@pytest.mark.slow
def test_cfg4_full_size_spmv_bitwise():
    """8M rows / 213.8M nnz: device SpMV bit-identical to the oracle, checked
    on row blocks of 2M rows (keeps host memory bounded)."""
    conf = wl.CONFIGS[4]
    h = wl.make_matrix(conf)
    assert h.nnz == 213_847_192
    op = pg.DeviceMatrixOperator(h)
    x = wl.splitmix_uniform(9, h.nrows)
    y = op.apply(x)
    for r0 in range(0, h.nrows, 2_000_000):
        blk = wl.make_matrix(conf, rows=(r0, r0 + 2_000_000))
        want = orc.OracleMatrix(blk.nrows, blk.ncols, blk.row_ptr, blk.col_idx,
                                blk.values).matvec(x)
        assert np.array_equal(y[r0:r0 + 2_000_000], want)


@pytest.mark.parametrize("env", [{}, {"PG_SPMV_WIN_MIN_ROW": "0"}, {"PG_SPMV_WIN": "0"},
                                 {"PG_SPMV_WIN": "0", "PG_SPMV_PAIR": "0"},
                                 {"PG_SPMV_WIN": "0", "PG_SPMV_PAIR": "0", "PG_SPMV_DICT": "0"}])
def test_spmv_kernel_variants_bitwise(env, monkeypatch):
    """Every SELL kernel (windowed pair ring, pair / two-stream dictionary with
    global gathers, uncompressed) is bit-identical to the reference order, on
    a 27-point and a 7-point stencil, for all four epilogue modes, including a
    misaligned x (the windowed kernel's bulk copies need 16-byte alignment and
    fall back to the gather kernel)."""
    from paper_1907_00072_b200 import _lib
    from paper_1907_00072_b200.device import ptr
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for h in (wl.aniso27(20), wl.convdiff3d_7pt(21)):
        O = _oracle(h)
        x = wl.splitmix_uniform(4, h.nrows)
        op = pg.DeviceMatrixOperator(h)
        assert np.array_equal(op.apply(x), O.matvec(x))
        y = np.random.default_rng(1).uniform(-1, 1, 6)
        got = pg.apply_poly(pg.PolyCoefficients(5, y, 1.0), op, x, pg.CostCounters())
        assert np.array_equal(got, orc.poly_eval(y, O, x, orc.Tally()))
        e = op.engine
        b = wl.splitmix_uniform(8, h.nrows)
        rs = e.vecs()
        nsq = e.residual(e.ingest(x), e.ingest(b), rs)
        r_want = b - O.matvec(x)
        assert np.array_equal(e.to_host(rs), r_want)
        assert nsq == pytest.approx(float(r_want @ r_want), rel=1e-13)
        roots = pg.apply_poly(pg.PolyCoefficients(5, y, 1.0), op, x, pg.CostCounters(),
                              form="roots")
        ext = orc.poly_eval_extended(y, O, x)
        assert np.linalg.norm(roots - ext) / np.linalg.norm(ext) < 1e-12
        s = e.shards[0]
        buf = torch.zeros(h.nrows + 2, dtype=torch.float64, device=s.device)
        buf[1:h.nrows + 1] = torch.from_numpy(x)
        out = torch.empty(h.nrows, dtype=torch.float64, device=s.device)
        _lib.call("pg_spmv", s.mat, ptr(buf) + 8, ptr(out), None)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), O.matvec(x))
        op.close()


def test_native_step_path_is_bitwise_the_kernel_by_kernel_path(golden, monkeypatch):
    """pg_arnoldi_step / pg_poly_chain (one native call per Arnoldi step or
    polynomial chain) issue the same kernels as the per-kernel entry points:
    the whole solve, x and history, is bit-identical."""
    a, _ = golden
    out = []
    for fast in ("1", "0"):
        monkeypatch.setenv("PG_FAST_STEP", fast)
        c = pg.CostCounters()
        op = pg.DeviceMatrixOperator(_lap64(golden), c)
        assert op.engine.fast_steps == (fast == "1")
        p = pg.PolyCoefficients(10, a["cfg1_y10"], 1.0)
        res = pg.solve(op, a["cfg1_b"], right_prec=p, config=pg.GmresConfig(15, 1e-10))
        out.append((res.x, res.history, c.as_dict(), res.cycles))
        op.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1] and out[0][2] == out[1][2] and out[0][3] == out[1][3] > 1


@pytest.mark.parametrize("grid", [3, 5, 7, 9, 13])
@pytest.mark.parametrize("env", [{}, {"PG_SPMV_WIN_MIN_ROW": "0"}, {"PG_SPMV_PAT": "0"},
                                 {"PG_SPMV_PAT": "0", "PG_SPMV_WIN_MIN_ROW": "0"}])
def test_stencil_kernels_ragged_sizes(grid, env, monkeypatch):
    """Windowed / short-row pair kernels at sizes that leave partial 32-row
    slices and partial 256-row blocks (n = g^3 for the 27-point operator, g^3
    for the 7-point one, forced through the windowed kernel with
    PG_SPMV_WIN_MIN_ROW=0): SpMV, the fused pass chain and the residual stay
    bit-identical."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for h in (wl.aniso27(grid), wl.convdiff3d_7pt(max(grid, 2))):
        O = _oracle(h)
        x = wl.splitmix_uniform(grid, h.nrows)
        op = pg.DeviceMatrixOperator(h)
        assert np.array_equal(op.apply(x), O.matvec(x))
        y = np.random.default_rng(grid).uniform(-1, 1, 4)
        got = pg.apply_poly(pg.PolyCoefficients(3, y, 1.0), op, x, pg.CostCounters())
        assert np.array_equal(got, orc.poly_eval(y, O, x, orc.Tally()))
        e = op.engine
        rs = e.vecs()
        b = wl.splitmix_uniform(grid + 1, h.nrows)
        e.residual(e.ingest(x), e.ingest(b), rs)
        assert np.array_equal(e.to_host(rs), b - O.matvec(x))
        op.close()


def test_recorded_step_graphs_replay_bitwise(golden, monkeypatch):
    """Repeated solves on one operator: the first issues every step, the
    second records each step as a CUDA graph, later ones replay the graphs.
    All runs are bit-identical (x, history, counters), and graphs are used."""
    a, _ = golden
    c = pg.CostCounters()
    op = pg.DeviceMatrixOperator(_lap64(golden), c)
    p = pg.PolyCoefficients(10, a["cfg1_y10"], 1.0)
    runs = []
    for _ in range(4):
        c.__init__()
        res = pg.solve(op, a["cfg1_b"], right_prec=p, config=pg.GmresConfig(15, 1e-10))
        runs.append((res.x, res.history, c.as_dict(), res.cycles, res.iterations))
    assert len(op.engine._graphs) > 0
    for r in runs[1:]:
        assert np.array_equal(r[0], runs[0][0])
        assert r[1:] == runs[0][1:]
    op.close()


# ---------------------------------------------------------------------------
# bases wider than one tall-skinny kernel call (PG_KMAX = 64 columns)
# ---------------------------------------------------------------------------
def test_restart_100_unpreconditioned_matches_oracle(golden):
    """GMRES(100) (the paper's restart length): Arnoldi steps
    past 64 basis columns orthogonalize in 64-column tiles (pg_cgs2_wide)."""
    A = _lap64(golden)
    b = golden[0]["cfg1_b"]
    res, sc, ref, t, poly, c = _solve_pair(A, b, None, 100, 1e-8, max_iters=400)
    assert res.iterations > 64  # the wide path ran
    _agree(res, sc, ref, t, 1e-8, c)
    # the same through the kernel-by-kernel path and on 2 virtual shards
    for shards in (1, 2):
        c2 = pg.CostCounters()
        op = pg.DeviceMatrixOperator(A, c2, shards=shards)
        r2 = pg.solve(op, b, config=pg.GmresConfig(100, 1e-8, 400))
        assert r2.converged and abs(r2.iterations - ref.iterations) <= 2
        op.close()


def test_restart_100_with_polynomial_and_icgs_wide(golden):
    a, _ = golden
    A = _lap64(golden)
    res, sc, ref, t, poly, c = _solve_pair(A, a["cfg1_b"], 4, 100, 1e-12)
    _agree(res, sc, ref, t, 1e-12, c)
    g = np.random.default_rng(3)
    for j in (65, 100, 130):
        basis = np.linalg.qr(g.standard_normal((700, j)))[0]
        w = g.uniform(-1, 1, 700)
        cc = pg.CostCounters()
        got = pg.icgs(basis, w, cc)
        want = orc.cgs2(basis, w, orc.Tally())
        np.testing.assert_allclose(got.coeffs, want[0], rtol=0, atol=1e-12)
        np.testing.assert_allclose(got.vector, want[2], rtol=0, atol=1e-12)
        assert (cc.dots, cc.scalar_dots) == (3, 2 * j + 1)
    with pytest.raises(pg.ParameterError):
        pg.solve(pg.DeviceMatrixOperator(A), a["cfg1_b"], config=pg.GmresConfig(256, 1e-8))


def test_degrees_past_the_kernel_width(golden):
    """build_poly / auto_degree at degrees whose power sequence is wider than
    PG_KMAX: the decision comes from the leading pivots at the full system's
    floor (polyprec._cholesky_ref), as the reference's Cholesky would take it."""
    _, meta = golden
    A = _lap64(golden)
    v0 = orc.sm64_uniform(1, 4096)
    op = pg.DeviceMatrixOperator(A)
    Gfull, _ = orc.gram_full_blas(orc.OracleMatrix.of(A), v0, 66)
    for d in (63, 64):
        want = orc.degree_decision_blas(Gfull[:d + 2, :d + 2], d)
        before = op.counters.spmvs
        with pytest.raises(pg.CholeskyFailure) as err:
            pg.build_poly(op, v0, d, pg.CostCounters())
        assert err.value.pivot == want[0]
        assert op.counters.spmvs - before == d + 1  # the reference's power sequence length
        assert pg.auto_degree(op, v0, d, pg.CostCounters()).degree == want[1]
        p, piv = pg.build_poly_or_auto(op, v0, d, pg.CostCounters())
        assert piv == want[0] and p.degree == want[1]
    assert want[1] == meta["auto_lap64"]["degree"]
    op.close()
