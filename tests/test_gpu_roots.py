"""Root-product evaluation of p(A)v on the device (BASELINE
north_star "root-product terms, complex-conjugate root pairs in real
arithmetic, running sum").  GPU only.

Bars: the reference evaluates only the monomial form (polyprec.py:193-212), so
the root form cannot be bitwise; it is checked against
* the oracle's extended-precision p(A)v (``poly_eval_extended``) to 1e-12
  relative -- the root form is the more accurate of the two fp64 forms;
* the reference-order monomial ``poly_eval`` to the north_star's 1e-10 relative
  wherever the monomial itself is that accurate (degree <= 10 on cfg1);
* solves with ``GmresConfig(poly_form="roots")``: iterations within +-2 of the
  oracle solve from the same coefficients, final relres < tol, and the
  reference's counter laws unchanged (same SpMV count per step).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_00072_b200 as pg  # noqa: E402
from oracle import pgmres_oracle as orc  # noqa: E402
from paper_1907_00072_b200 import _lib  # noqa: E402
from paper_1907_00072_b200 import workloads as wl  # noqa: E402

pytestmark = pytest.mark.gpu


def _lap64(golden):
    a = golden[0]
    return wl.CsrHost(4096, 4096, a["lap64_row_ptr"], a["lap64_col_idx"], a["lap64_values"])


def _rel(u, w):
    return float(np.linalg.norm(u - w) / np.linalg.norm(w))


def _y_from_roots(roots):
    """Coefficients y of p with 1 - z p(z) = prod (1 - z/theta)."""
    pi = np.array([1.0 + 0j])
    for th in roots:
        pi = np.convolve(pi, np.array([1.0, -1.0 / th]))
    assert np.allclose(pi.imag, 0)
    return -pi.real[1:]


@pytest.mark.parametrize("shards", [1, 2, 4])
@pytest.mark.parametrize("key", ["cfg1_sweep_1_y", "cfg1_sweep_4_y", "cfg1_sweep_8_y",
                                 "cfg1_y10", "cfg1_sweep_12_y"])
def test_apply_poly_roots_cfg1(golden, key, shards):
    a, _ = golden
    h = _lap64(golden)
    y = a[key]
    p = pg.PolyCoefficients(len(y) - 1, y, 1.0)
    c = pg.CostCounters()
    op = pg.DeviceMatrixOperator(h, c, shards=shards)
    got = pg.apply_poly(p, op, a["cfg1_b"], c, form="roots")
    assert c.spmvs == p.degree and c.vector_updates == p.degree + 1
    ext = orc.poly_eval_extended(y, orc.OracleMatrix.of(h), a["cfg1_b"])
    mono = orc.poly_eval(y, orc.OracleMatrix.of(h), a["cfg1_b"], orc.Tally())
    assert _rel(got, ext) < 1e-12
    assert _rel(got, ext) <= _rel(mono, ext) + 1e-15
    if p.degree <= 10:
        assert _rel(got, mono) < 1e-10
    if shards == 1 and key == "cfg1_y10":  # the golden p(A)b of the reference itself
        assert _rel(got, a["cfg1_pAb"]) < 1e-10
    op.close()


@pytest.mark.parametrize("roots", [
    [1.0, 2.0, 3.0, 4.0, 5.0],                        # real roots only (c3 fold)
    [2 + 1j, 2 - 1j, 4 + 0.5j, 4 - 0.5j],             # pairs only (PAIR_A last)
    [3.0, 1 + 2j, 1 - 2j, 6.0, 2 + 1j, 2 - 1j],       # mixed
    [0.5 + 0.1j, 0.5 - 0.1j, 7.5],                    # pair then a trailing real
])
def test_root_plan_shapes(roots):
    """Every plan shape (real / pair / mixed, trailing real folded into the
    previous pass) on a 3D operator, through 1 and 3 shards, and the wrapped
    A p(A) v = v - pi(A) v pass chain."""
    h = wl.convdiff3d_7pt(20)
    y = _y_from_roots(roots)
    p = pg.PolyCoefficients(len(y) - 1, y, 1.0)
    plan = pg.root_plan(p)
    assert len(plan.steps) == p.degree and len(plan.resid_steps) == p.degree + 1
    O = orc.OracleMatrix.of(h)
    v = wl.splitmix_uniform(3, h.nrows)
    ext = orc.poly_eval_extended(y, O, v)
    for shards in (1, 3):
        op = pg.DeviceMatrixOperator(h, shards=shards)
        got = pg.apply_poly(p, op, v, pg.CostCounters(), form="roots")
        assert _rel(got, ext) < 1e-12
        e = op.engine
        vs = e.ingest(v)
        z, t, p0, p1 = e.vecs(), e.vecs(), e.vecs(), e.vecs()
        e.wrapped_roots(plan, vs, z, t, p0, p1)
        torch.cuda.synchronize()
        want = O.matvec(ext)
        assert _rel(e.to_host(z), want) < 1e-12
        op.close()


def test_degree0_and_abi_errors():
    h = wl.laplacian2d(16)
    op = pg.DeviceMatrixOperator(h)
    v = wl.splitmix_uniform(1, h.nrows)
    out = pg.apply_poly(pg.PolyCoefficients(0, np.array([2.5]), 1.0), op, v, pg.CostCounters(),
                        form="roots")
    assert np.array_equal(out, 2.5 * v)
    e = op.engine
    plan0 = pg.root_plan(pg.PolyCoefficients(0, np.array([2.5]), 1.0))
    vs = e.ingest(v)
    z = e.vecs()
    e.wrapped_roots(plan0, vs, z, e.vecs(), e.vecs(), e.vecs())
    assert _rel(e.to_host(z), 2.5 * orc.OracleMatrix.of(h).matvec(v)) < 1e-13
    s = e.shards[0]
    buf = torch.zeros(s.ld, dtype=torch.float64, device=s.device)
    with pytest.raises(pg.ParameterError):
        _lib.call("pg_root_pass", s.mat, buf.data_ptr(), None, None, buf.data_ptr(), None,
                  1.0, 0.0, 0.0, 3, None)
    with pytest.raises(pg.ParameterError):  # PAIR_B needs p
        _lib.call("pg_root_pass", s.mat, buf.data_ptr(), None, None, None, buf.data_ptr(),
                  1.0, 0.0, 0.0, _lib.PG_ROOT_PAIR_B, None)
    with pytest.raises(pg.ParameterError):  # RESID needs v and writes v_out only
        _lib.call("pg_root_pass", s.mat, buf.data_ptr(), None, None, None, buf.data_ptr(),
                  1.0, 0.0, 0.0, _lib.PG_ROOT_REAL | _lib.PG_ROOT_RESID, None)
    op.close()


def _roots_solve(h, b, poly, m, tol, shards=1, x0=None):
    c = pg.CostCounters()
    op = pg.DeviceMatrixOperator(h, c, shards=shards)
    res = pg.solve(op, b, x0=x0, right_prec=poly,
                   config=pg.GmresConfig(m, tol, poly_form="roots"))
    t = orc.Tally()
    ref = orc.gmres(orc.OracleMatrix.of(h, t), b, x0=x0, y=poly.y, m=m, tol=tol)
    op.close()
    return res, c, ref, t


@pytest.mark.parametrize("key", ["cfg1_sweep_4_y", "cfg1_y10", "cfg1_sweep_12_y"])
def test_cfg1_solve_roots(golden, key):
    a, meta = golden
    y = a[key]
    d = len(y) - 1
    poly = pg.PolyCoefficients(d, y, 1.0)
    res, c, ref, t = _roots_solve(_lap64(golden), a["cfg1_b"], poly, 40, 1e-8)
    assert res.converged and ref.converged and res.final_relres < 1e-8
    assert abs(res.iterations - ref.iterations) <= 2
    assert c.spmvs == (d + 1) * res.iterations + d * res.cycles + res.cycles
    assert c.dots == 3 * res.iterations
    if key == "cfg1_y10":
        assert abs(res.iterations - meta["cfg1_solve"]["iterations"]) <= 2


@pytest.mark.parametrize("shards", [1, 2])
def test_convdiff_roots_multicycle_x0(golden, shards):
    a, _ = golden
    n = len(a["convdiff48_row_ptr"]) - 1
    h = wl.CsrHost(n, n, a["convdiff48_row_ptr"], a["convdiff48_col_idx"],
                   a["convdiff48_values"])
    b = orc.sm64_uniform(3, n)
    c = pg.CostCounters()
    op = pg.DeviceMatrixOperator(h, c)
    poly, _ = pg.build_poly_or_auto(op, orc.sm64_uniform(4, n), 6, c)
    op.close()
    for x0, m, tol in ((None, 20, 1e-9), (a["convdiff48_x0"], 15, 1e-8)):
        res, c, ref, t = _roots_solve(h, b, poly, m, tol, shards, x0)
        assert res.converged == ref.converged and res.final_relres < tol
        assert abs(res.iterations - ref.iterations) <= 2


@pytest.mark.parametrize("cfg,kw", [(2, dict(grid=16)), (4, dict(grid=12))])
def test_small_configs_roots(cfg, kw):
    conf = wl.CONFIGS[cfg]
    h = wl.make_matrix(conf, **kw)
    b = wl.make_rhs(conf, h)
    c = pg.CostCounters()
    op = pg.DeviceMatrixOperator(h, c)
    poly, _ = pg.build_poly_or_auto(op, wl.make_v0(h.nrows), conf["degree"], c)
    op.close()
    res, c, ref, t = _roots_solve(h, b, poly, conf["m"], conf["tol"])
    assert res.converged == ref.converged
    if ref.converged:
        assert res.final_relres < conf["tol"]
    assert abs(res.iterations - ref.iterations) <= 2


def _res_norm(A, y, v):
    """|| v - A p(A) v || / ||v|| in extended precision (oracle yardstick)."""
    pv = orc.poly_eval_extended(y, A, v)
    return float(np.linalg.norm(v - A.matvec(pv)) / np.linalg.norm(v))


@pytest.mark.parametrize("deg", [4, 8, 10])
def test_arnoldi_construction_matches_power_basis(golden, deg):
    """build_poly_arnoldi (harmonic Ritz values of deg+1 Arnoldi steps) finds
    the same minimum-residual polynomial as the power-basis normal equations
    (build_poly, polyprec.py:125-147) wherever those are well conditioned:
    same residual norm, same roots, same coefficients to the conditioning."""
    h = _lap64(golden)
    v0 = orc.sm64_uniform(1, h.nrows)
    c = pg.CostCounters()
    op = pg.DeviceMatrixOperator(h, c)
    pa = pg.build_poly_arnoldi(op, v0, deg, c)
    assert pa.degree == deg and len(pa.roots) == deg + 1 and c.spmvs == deg + 1
    # the exact-arithmetic power-basis minimiser (the reference-order fp64
    # Gram's rounding moves the degree-10 roots by more than the comparison)
    pp = pg.build_poly(op, v0, deg, pg.CostCounters(), decision="exact")
    O = orc.OracleMatrix.of(h)
    v = v0 / np.linalg.norm(v0)
    ra, rp = _res_norm(O, pa.y, v), _res_norm(O, pp.y, v)
    # the harmonic-Ritz minimiser is never worse; the power basis loses a
    # little to its conditioning at the top usable degree (2e-4 at deg 10)
    assert ra <= rp * (1 + 1e-6) and rp <= ra * (1 + 1e-3)
    rr = np.sort_complex(pg.residual_poly_roots(pp.y))
    assert np.allclose(np.sort_complex(pa.roots), rr, rtol=1e-4 if deg < 10 else 1e-2)
    if deg <= 8:
        np.testing.assert_allclose(pa.y, pp.y, rtol=1e-5 * 10 ** (deg / 2))
    op.close()


def test_arnoldi_high_degree_solves():
    """Degrees the power basis cannot build (cfg2 operator: Cholesky fails
    near 13): the harmonic-Ritz polynomial of degree 25 and 40, evaluated in
    root-product form, keeps decreasing the residual polynomial's norm and
    cuts GMRES iterations; the solves converge to tol."""
    conf = wl.CONFIGS[2]
    h = wl.make_matrix(conf, grid=24)
    b = wl.make_rhs(conf, h)
    v0 = wl.make_v0(h.nrows)
    O = orc.OracleMatrix.of(h)
    v = v0 / np.linalg.norm(v0)
    its, res = [], []
    for deg in (10, 25, 40):
        c = pg.CostCounters()
        op = pg.DeviceMatrixOperator(h, c)
        p = pg.build_poly_arnoldi(op, v0, deg, c)
        assert p.degree == deg
        # || v - A p(A) v || evaluated on the device in root form
        z = pg.PolynomialWrappedOperator(op, p)
        out = pg.apply_poly(p, op, v, pg.CostCounters(), form="roots")
        res.append(float(np.linalg.norm(v - O.matvec(out))))
        r = pg.solve(op, b, right_prec=p, config=pg.GmresConfig(conf["m"], conf["tol"],
                                                                   poly_form="roots"))
        assert r.converged and r.final_relres < conf["tol"]
        tr = np.linalg.norm(b - O.matvec(r.x)) / np.linalg.norm(b)
        assert tr == pytest.approx(r.final_relres, rel=1e-3)
        its.append(r.iterations)
        op.close()
        del z
    assert res[0] > res[1] > res[2]
    assert its[0] > its[1] >= its[2]


def test_roots_solve_native_and_graph_paths_bitwise(golden, monkeypatch):
    """The root-form Arnoldi chain inside pg_arnoldi_step (and its recorded
    graphs on repeated solves) is bit-identical to the per-pass path."""
    a, _ = golden
    p = pg.PolyCoefficients(10, a["cfg1_y10"], 1.0)
    outs = []
    for fast in ("0", "1"):
        monkeypatch.setenv("PG_FAST_STEP", fast)
        c = pg.CostCounters()
        op = pg.DeviceMatrixOperator(_lap64(golden), c)
        for _ in range(3):  # 3rd run replays recorded graphs on the fast path
            c.__init__()
            r = pg.solve(op, a["cfg1_b"], right_prec=p,
                         config=pg.GmresConfig(15, 1e-10, poly_form="roots"))
            outs.append((r.x, r.history, c.as_dict()))
        if fast == "1":
            assert len(op.engine._graphs) > 0
        op.close()
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and o[1:] == outs[0][1:]
