"""The plane-marching SpMV kernel (csrc/march.cu, opt-in PG_SPMV_MARCH=1) on
row-pattern stencils:
bit-identical to the oracle (hence to the reference's row-sequential sum) in
every epilogue mode, at ragged sizes (partial warps, partial plane chunks,
partial last plane), on virtual shards whose boundary planes read ghost slots,
and in a full solve.  GPU only."""

import subprocess
import sys
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_00072_b200 as pg  # noqa: E402
from oracle import pgmres_oracle as orc  # noqa: E402
from paper_1907_00072_b200 import _lib, workloads as wl  # noqa: E402
from paper_1907_00072_b200.device import ptr  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [("aniso27", 11), ("aniso27", 24), ("conv7", 9), ("conv7", 23), ("lap5", 40),
         ("conv9", 33)]


def _matrix(kind, g):
    if kind == "aniso27":
        return wl.aniso27(g)
    if kind == "conv7":
        return wl.convdiff3d_7pt(g)
    if kind == "lap5":
        return wl.laplacian2d(g)
    if kind == "rand27":
        # a constant-coefficient 27-point operator with 27 distinct values (no
        # coefficient shared between the outer plane groups)
        from paper_1907_00072_b200.workloads import CsrHost
        w = np.random.default_rng(27).uniform(-1.0, 1.0, (3, 3, 3))
        w[1, 1, 1] = 9.0
        z, y, x = np.meshgrid(np.arange(g), np.arange(g), np.arange(g), indexing="ij")
        rows, cols, vals = [], [], []
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    ok = ((z + dz >= 0) & (z + dz < g) & (y + dy >= 0) & (y + dy < g)
                          & (x + dx >= 0) & (x + dx < g))
                    r = ((z * g + y) * g + x)[ok]
                    rows.append(r)
                    cols.append(r + (dz * g + dy) * g + dx)
                    vals.append(np.full(r.size, w[dz + 1, dy + 1, dx + 1]))
        rows, cols, vals = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
        order = np.lexsort((cols, rows))
        n = g ** 3
        rp = np.zeros(n + 1, dtype=np.int64)
        np.add.at(rp, rows + 1, 1)
        return CsrHost(n, n, np.cumsum(rp), cols[order].astype(np.int64), vals[order])
    # a constant-coefficient 2-D 9-point operator (row patterns, not offset patterns)
    from paper_1907_00072_b200.workloads import CsrHost
    n = g * g
    rows, cols, vals = [], [], []
    w = {(-1, -1): -1.0, (-1, 0): -4.0, (-1, 1): -1.0, (0, -1): -4.0, (0, 0): 20.5,
         (0, 1): -4.25, (1, -1): -1.0, (1, 0): -3.75, (1, 1): -1.0}
    for y in range(g):
        for x in range(g):
            for (dy, dx), v in sorted(w.items()):
                if 0 <= y + dy < g and 0 <= x + dx < g:
                    rows.append(y * g + x)
                    cols.append((y + dy) * g + x + dx)
                    vals.append(v)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, np.array(rows) + 1, 1)
    return CsrHost(n, n, np.cumsum(rp), np.array(cols, dtype=np.int64), np.array(vals))


def _check(h, shards=1):
    O = orc.OracleMatrix.of(h)
    x = wl.splitmix_uniform(3, h.nrows)
    op = pg.DeviceMatrixOperator(h, shards=shards)
    assert np.array_equal(op.apply(x), O.matvec(x))
    y = np.random.default_rng(h.nrows).uniform(-1, 1, 7)
    got = pg.apply_poly(pg.PolyCoefficients(6, y, 1.0), op, x, pg.CostCounters())
    assert np.array_equal(got, orc.poly_eval(y, O, x, orc.Tally()))
    e = op.engine
    b = wl.splitmix_uniform(8, h.nrows)
    rs = e.vecs()
    nsq = e.residual(e.ingest(x), e.ingest(b), rs)
    r_want = b - O.matvec(x)
    assert np.array_equal(e.to_host(rs), r_want)
    assert nsq == pytest.approx(float(r_want @ r_want), rel=1e-13)
    roots = pg.apply_poly(pg.PolyCoefficients(6, y, 1.0), op, x, pg.CostCounters(), form="roots")
    ext = orc.poly_eval_extended(y, O, x)
    assert np.linalg.norm(roots - ext) / np.linalg.norm(ext) < 1e-11
    op.close()


def _run_isolated(env, code):
    """Run `code` in a fresh interpreter (the kernel choice is read once per
    process) with `env` added; assert it succeeds."""
    full = dict(os.environ, PG_SPMV_MARCH="1", PG_SPMV_PLANES="0", PYTHONPATH=ROOT)
    full.update(env)
    res = subprocess.run([sys.executable, "-c", code], env=full, capture_output=True, text=True,
                         cwd=ROOT, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
    return res.stdout


def test_march_kernel_is_selected_and_bitwise():
    code = f"""
import sys; sys.path.insert(0, 'tests'); import test_gpu_march as t
import paper_1907_00072_b200 as pg
for kind, g in {CASES!r}:
    h = t._matrix(kind, g)
    t._check(h)
    for shards in (2, 3):
        t._check(h, shards)
assert pg.DeviceMatrixOperator(t._matrix("aniso27", 24)).engine.shards[0].stats["kernel"] == 8
print("ok")
"""
    out = _run_isolated({"PG_MARCH_MIN_S": "1", "PG_MARCH_Z": "3"}, code)
    assert "ok" in out


def test_march_chunks_and_default_threshold():
    code = """
import sys; sys.path.insert(0, 'tests'); import test_gpu_march as t
from paper_1907_00072_b200 import workloads as wl
h = wl.aniso27(26)
t._check(h)
t._check(wl.convdiff3d_7pt(30), 2)
print("ok")
"""
    for z in ("1", "2", "7", "0"):
        assert "ok" in _run_isolated({"PG_MARCH_Z": z}, code)


def test_march_off_matches_march_on_in_a_solve():
    code = """
import numpy as np, os, sys
import paper_1907_00072_b200 as pg
from paper_1907_00072_b200 import workloads as wl
h = wl.aniso27(30)
op = pg.DeviceMatrixOperator(h)
poly, _ = pg.build_poly_or_auto(op, wl.make_v0(h.nrows), 10, pg.CostCounters())
res = pg.solve(op, wl.splitmix_uniform(0, h.nrows), right_prec=poly, config=pg.GmresConfig(30, 1e-9))
np.save(sys.argv[1] if len(sys.argv) > 1 else "/tmp/x.npy", res.x)
print("ok", res.iterations, op.engine.shards[0].stats["kernel"])
assert (op.engine.shards[0].stats["kernel"] == 8) == (os.environ["PG_SPMV_MARCH"] == "1")
"""
    outs = []
    for on in ("1", "0"):
        path = f"/tmp/pg_march_{on}.npy"
        out = _run_isolated({"PG_SPMV_MARCH": on}, code.replace('"/tmp/x.npy"', repr(path)))
        outs.append((out.split()[1], np.load(path)))
    assert outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][1], outs[1][1])


def test_windowed_ring_wraps_bitwise_in_every_mode():
    """The windowed TMA-ring kernel with its grid capped at 2 CTAs
    (PG_SPMV_WIN_GRID): every CTA sweeps many row blocks, so the ring's slot
    reuse, empty-barrier waits and phase flips run in SpMV, the fused
    polynomial pass, the residual and the root-product passes -- all bitwise
    (ragged last stage included)."""
    code = """
import sys; sys.path.insert(0, 'tests'); import test_gpu_march as t
import paper_1907_00072_b200 as pg
from paper_1907_00072_b200 import workloads as wl
for g in (20, 23, 31):
    h = wl.aniso27(g)
    assert pg.DeviceMatrixOperator(h).engine.shards[0].stats["kernel"] == 6
    t._check(h)
    t._check(h, 2)
print("ok")
"""
    for cap in ("1", "2", "3"):
        assert "ok" in _run_isolated({"PG_SPMV_MARCH": "0", "PG_SPMV_WIN_GRID": cap}, code)
