"""The dependency-driven chain kernel (csrc/chain.cu): an
Arnoldi step's d+1 SpMV passes as one kernel whose passes overlap through
per-chunk completion flags.  Its results must be bit-identical to the
pass-by-pass kernels (PG_CHAIN=0) -- same x, history and counters -- for
every chunk size, at ragged sizes, in both polynomial forms, across
repeated launches (generations) and recorded graphs, and at full cfg2 size.
GPU only."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_00072_b200 as pg  # noqa: E402
from paper_1907_00072_b200 import workloads as wl  # noqa: E402

pytestmark = pytest.mark.gpu


def _solve(monkeypatch, h, y, chain, m=12, tol=1e-12, max_iters=40, form="monomial",
           repeats=1, env=None):
    monkeypatch.setenv("PG_CHAIN", "1" if chain else "0")  # opt-in kernel
    for k, v in (env or {}).items():
        monkeypatch.setenv(k, v)
    c = pg.CostCounters()
    # natural row order (sigma = 1): tiny operators would otherwise be
    # length-sorted, which the chain kernel does not take
    op = pg.DeviceMatrixOperator(h, c, sigma=1)
    assert op.engine.shards[0].chain_fused == chain
    b = wl.splitmix_uniform(3, h.nrows)
    p = pg.PolyCoefficients(len(y) - 1, np.asarray(y, dtype=np.float64), 1.0)
    cfg = pg.GmresConfig(m, tol, max_iters=max_iters, poly_form=form)
    runs = []
    for _ in range(repeats):
        c.__init__()
        res = pg.solve(op, b, right_prec=p, config=cfg)
        runs.append((res.x, res.history, c.as_dict(), res.iterations))
    op.close()
    return runs


def _same(a, b):
    assert np.array_equal(a[0], b[0])
    assert a[1:] == b[1:]


def _coeffs(d, seed=0):
    # a contractive polynomial so that long chains stay finite
    return np.random.default_rng(seed).uniform(-1, 1, d + 1) / (d + 1)


@pytest.mark.parametrize("body", ["pattern", "pair"])
@pytest.mark.parametrize("ts", ["1", "2", "4", "8"])
@pytest.mark.parametrize("grid", [2, 3, 5, 7, 13])
def test_chain_bitwise_ragged(monkeypatch, ts, grid, body):
    """7-point operators whose n leaves partial slices and partial chunks, with
    the row-pattern and the pair-stream row bodies."""
    if body == "pair":
        monkeypatch.setenv("PG_SPMV_PAT", "0")
    h = wl.convdiff3d_7pt(grid)
    y = _coeffs(6, grid)
    want = _solve(monkeypatch, h, y, False)
    got = _solve(monkeypatch, h, y, True, env={"PG_CHAIN_TS": ts})
    _same(got[0], want[0])


@pytest.mark.parametrize("d", [1, 2, 14, 25, 40])
def test_chain_bitwise_degrees(monkeypatch, d):
    h = wl.convdiff3d_7pt(24)
    y = _coeffs(d, d)
    want = _solve(monkeypatch, h, y, False, max_iters=15)
    got = _solve(monkeypatch, h, y, True, max_iters=15)
    _same(got[0], want[0])


def test_chain_bitwise_2d_and_laplacian(monkeypatch):
    """2-D 5- and 9-point operators (one index word per lane; longer rows)."""
    for h in (wl.laplacian2d(64), wl.laplacian2d(37)):
        y = _coeffs(10, 1)
        _same(_solve(monkeypatch, h, y, True)[0], _solve(monkeypatch, h, y, False)[0])


def test_chain_root_form_bitwise(monkeypatch):
    """Root-product passes (REAL, PAIR_A / PAIR_B, the PG_ROOT_RESID last
    pass) through the chain kernel."""
    h = wl.convdiff3d_7pt(20)
    a = pg.DeviceMatrixOperator(h)
    p, _ = pg.build_poly_or_auto(a, wl.make_v0(h.nrows), 10, pg.CostCounters())
    a.close()
    y = p.y
    want = _solve(monkeypatch, h, y, False, form="roots", max_iters=20)
    got = _solve(monkeypatch, h, y, True, form="roots", max_iters=20)
    _same(got[0], want[0])


def test_chain_generations_and_graph_replays(monkeypatch):
    """Repeated solves on one operator: the chain kernel's generation counter
    advances every launch, and from the second solve on the steps replay as
    recorded graphs; every run is bit-identical to the pass-by-pass one."""
    h = wl.convdiff3d_7pt(16)
    y = _coeffs(9, 2)
    want = _solve(monkeypatch, h, y, False, max_iters=30)[0]
    for r in _solve(monkeypatch, h, y, True, max_iters=30, repeats=4):
        _same(r, want)


def test_chain_pattern_kernel_matches_oracle(monkeypatch):
    """The row-pattern matrix format is what the chain runs on stencils: its
    SpMV and p(A)v equal the oracle's bit for bit (cfg1 and a 27-point
    operator with its long rows)."""
    from oracle import pgmres_oracle as orc
    for h in (wl.laplacian2d(64), wl.aniso27(11), wl.convdiff3d_7pt(9)):
        op = pg.DeviceMatrixOperator(h, sigma=1)
        if h.nrows == 4096:
            assert op.engine.shards[0].stats["kernel"] == 5
        O = orc.OracleMatrix.of(h)
        x = wl.splitmix_uniform(5, h.nrows)
        assert np.array_equal(op.apply(x), O.matvec(x))
        y = np.random.default_rng(4).uniform(-1, 1, 8)
        got = pg.apply_poly(pg.PolyCoefficients(7, y, 1.0), op, x, pg.CostCounters())
        assert np.array_equal(got, orc.poly_eval(y, O, x, orc.Tally()))
        op.close()


def _lap_modified_boundary(g):
    """2-D Laplacian whose boundary rows carry a different diagonal: their
    row patterns are NOT masked subsequences of the interior pattern, so the
    pattern kernels take the table walk for them (and the unrolled master
    path for the interior rows)."""
    h = wl.laplacian2d(g)
    rp, ci = np.asarray(h.row_ptr), np.asarray(h.col_idx)
    vals = np.array(h.values, dtype=np.float64)
    for r in range(h.nrows):
        if rp[r + 1] - rp[r] < 5:
            for q in range(rp[r], rp[r + 1]):
                if ci[q] == r:
                    vals[q] = 5.0
    return wl.CsrHost(h.nrows, h.ncols, rp, ci, vals)


def test_pattern_master_and_table_paths_bitwise():
    """Row-pattern kernels: interior rows through the master pattern,
    modified boundary rows through the table walk, both windowed (27-point)
    and global-gather (5/7-point): SpMV and p(A)v equal the oracle."""
    from oracle import pgmres_oracle as orc
    for h in (_lap_modified_boundary(40), _lap_modified_boundary(33), wl.aniso27(12),
              wl.convdiff3d_7pt(11)):
        op = pg.DeviceMatrixOperator(h, sigma=1)
        O = orc.OracleMatrix.of(h)
        x = wl.splitmix_uniform(9, h.nrows)
        assert np.array_equal(op.apply(x), O.matvec(x))
        y = np.random.default_rng(3).uniform(-1, 1, 6)
        got = pg.apply_poly(pg.PolyCoefficients(5, y, 1.0), op, x, pg.CostCounters())
        assert np.array_equal(got, orc.poly_eval(y, O, x, orc.Tally()))
        op.close()


@pytest.mark.parametrize("grid", [5, 17, 64, 101])
def test_offset_pattern_kernel_bitwise(grid):
    """Variable-coefficient stencils (cfg5's 9-point recirculating-wind
    operator): values do not compress, the column offsets do -- the offset-
    pattern kernel (1 B per row + f64 values; master path, masked boundary
    rows) gives the oracle's SpMV, p(A)v and residual bit for bit."""
    from oracle import pgmres_oracle as orc
    h = wl.convdiff2d_9pt(grid)
    op = pg.DeviceMatrixOperator(h, sigma=1)
    # tiny grids have <= 256 distinct values: the (value) row-pattern format
    many = len(np.unique(np.asarray(h.values))) > 256
    assert op.engine.shards[0].stats["kernel"] == (7 if many else 5)
    O = orc.OracleMatrix.of(h)
    x = wl.splitmix_uniform(7, h.nrows)
    assert np.array_equal(op.apply(x), O.matvec(x))
    y = np.random.default_rng(2).uniform(-1, 1, 5)
    got = pg.apply_poly(pg.PolyCoefficients(4, y, 1.0), op, x, pg.CostCounters())
    assert np.array_equal(got, orc.poly_eval(y, O, x, orc.Tally()))
    e = op.engine
    b = wl.splitmix_uniform(8, h.nrows)
    rs = e.vecs()
    e.residual(e.ingest(x), e.ingest(b), rs)
    assert np.array_equal(e.to_host(rs), b - O.matvec(x))
    op.close()


def test_pattern_kernels_bucketed_master_with_nonfinite_x():
    """Masters shorter than their unroll bucket (5-point rows in the 8-entry
    bucket, both pattern formats): the bucket's inert tail entries are never
    added -- a non-finite x entry in a row's own slot must not leak into
    rows that do not reference it, and finite results stay bitwise."""
    from oracle import pgmres_oracle as orc
    h = wl.laplacian2d(48)
    rp, ci = np.asarray(h.row_ptr), np.asarray(h.col_idx)
    for vals in (np.asarray(h.values, dtype=np.float64),
                 np.random.default_rng(1).uniform(-1, 1, len(ci))):
        m = wl.CsrHost(h.nrows, h.ncols, rp, ci, vals)
        op = pg.DeviceMatrixOperator(m, sigma=1)
        O = orc.OracleMatrix.of(m)
        x = wl.splitmix_uniform(4, m.nrows)
        assert np.array_equal(op.apply(x), O.matvec(x))
        x[100] = np.inf
        with np.errstate(invalid="ignore"):
            want = O.matvec(x)
        got = op.apply(x)
        assert np.array_equal(np.isnan(got), np.isnan(want))
        fin = np.isfinite(want)
        assert np.array_equal(got[fin], want[fin])
        op.close()


def test_chain_full_cfg2_size(monkeypatch):
    """n = 1e6, degree 14 (the headline's effective degree): a few Arnoldi
    steps through the chain kernel equal the pass-by-pass path bit for bit."""
    h = wl.convdiff3d_7pt(100)
    y = _coeffs(14, 14)
    want = _solve(monkeypatch, h, y, False, m=50, max_iters=4)[0]
    got = _solve(monkeypatch, h, y, True, m=50, max_iters=4, repeats=3)
    for r in got:
        _same(r, want)
