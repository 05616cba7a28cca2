"""The plane-ring SpMV kernel (csrc/planes.cu; default for 27-point plane
stencils, every plane stencil with PG_SPMV_PLANES=2): bit-identical to the
oracle (hence to the reference's row-sequential sum, sparse.py:151-168, and
apply_poly's recurrence, polyprec.py:205-211) in every epilogue mode, with
partial tiles, many plane chunks, one-plane chunks, a 2-stage ring that wraps
on every block, forced tile widths, virtual shards, and in a full solve.
GPU only."""

import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (kind, g): the plane stride S (g^2 for 3-D, g for 2-D) must be a multiple of 16
CASES = [("aniso27", 12), ("aniso27", 20), ("aniso27", 28), ("rand27", 12), ("rand27", 20),
         ("conv7", 20), ("conv7", 28),
         ("lap5", 48), ("conv9", 32), ("conv9", 64)]


def _nonfinite(h):
    """Non-finite x entries next to boundary rows: a row that does not store
    the entry must not see it (the kernel zeroes absent window values rather
    than multiplying them), rows that do store it get the reference's inf /
    NaN."""
    import paper_1907_00072_b200 as pg
    from oracle import pgmres_oracle as orc
    from paper_1907_00072_b200 import workloads as wl
    x = wl.splitmix_uniform(5, h.nrows)
    rng = np.random.default_rng(7)
    idx = rng.choice(h.nrows, size=max(4, h.nrows // 50), replace=False)
    x[idx[0::3]] = np.inf
    x[idx[1::3]] = -np.inf
    x[idx[2::3]] = np.nan
    op = pg.DeviceMatrixOperator(h)
    got = op.apply(x)
    want = orc.OracleMatrix.of(h).matvec(x)
    assert np.array_equal(got, want, equal_nan=True)
    fin = ~np.isnan(want)  # NaN sign bits are the hardware's (x86 default NaN is negative)
    assert np.array_equal(np.signbit(got[fin]), np.signbit(want[fin]))
    op.close()


def _run(env, code):
    full = dict(os.environ, PYTHONPATH=ROOT)
    full.update(env)
    res = subprocess.run([sys.executable, "-c", code], env=full, capture_output=True, text=True,
                         cwd=ROOT, timeout=900)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
    return res.stdout


CHECK = f"""
import sys; sys.path.insert(0, 'tests'); import test_gpu_march as t
from test_gpu_planes import _nonfinite
import paper_1907_00072_b200 as pg
for kind, g in {CASES!r}:
    h = t._matrix(kind, g)
    op = pg.DeviceMatrixOperator(h)
    k = op.engine.shards[0].stats["kernel"]
    op.close()
    assert k == 9, (kind, g, k)
    import os
    want_box = int(os.environ.get("PG_PLANE_BOX", "2"))
    op = pg.DeviceMatrixOperator(h)
    plan = op.engine.shards[0].plane_plan
    assert plan["box"] == want_box, plan
    # shared outer-group products: config 4's operator (z-symmetric but for the
    # center pair), not the operator with 27 distinct coefficients
    want_sym = int(kind == "aniso27" and os.environ.get("PG_PLANE_SYM", "1") != "0")
    assert plan["sym"] == want_sym, plan
    # adjacent row pairs (16-byte operand / result accesses): 27-point tiles
    want_vec = int(kind in ("aniso27", "rand27") and os.environ.get("PG_PLANE_VEC", "1") != "0")
    assert plan["vec"] == want_vec, plan
    op.close()
    t._check(h)
    for shards in (2, 3):
        t._check(h, shards)
    _nonfinite(h)
print("ok")
"""


@pytest.mark.parametrize("env", [
    {},
    {"PG_PLANE_Q": "64", "PG_PLANE_Z": "1"},      # 1-plane chunks, many partial tiles
    {"PG_PLANE_Q": "96", "PG_PLANE_Z": "3", "PG_PLANE_STAGES": "2"},  # ring wraps every block
    {"PG_PLANE_Q": "576", "PG_PLANE_Z": "5"},     # the widest tile (second row set)
    {"PG_PLANE_STAGES": "3"},
    {"PG_PLANE_BOX": "0"},                        # per-row pattern ids on every plane
    {"PG_PLANE_BOX": "1"},                        # ids on the end planes only
    {"PG_PLANE_SYM": "0"},                        # every product computed per row
    {"PG_PLANE_Q": "64", "PG_PLANE_Z": "2"},      # 2-plane chunks: no steady stage
    {"PG_PLANE_Q": "128", "PG_PLANE_Z": "3", "PG_PLANE_STAGES": "2"},
    {"PG_PLANE_BOX": "0", "PG_PLANE_Q": "64", "PG_PLANE_Z": "4"},
    {"PG_PLANE_VEC": "0"},                        # no adjacent-pair kernels (t, t + 288 mapping)
    {"PG_PLANE_VEC": "0", "PG_PLANE_Q": "576", "PG_PLANE_Z": "5"},
    {"PG_PLANE_Q": "160", "PG_PLANE_Z": "4", "PG_PLANE_STAGES": "3"},  # two interior planes per chunk
])
def test_plane_kernel_selected_and_bitwise(env):
    env = dict(env, PG_SPMV_PLANES="2")
    assert "ok" in _run(env, CHECK)


def test_plane_kernel_default_scope_and_off_switch():
    code = """
import sys; sys.path.insert(0, 'tests'); import test_gpu_march as t
import paper_1907_00072_b200 as pg
import os
def kern(h):
    op = pg.DeviceMatrixOperator(h); k = op.engine.shards[0].stats["kernel"]; op.close(); return k
on = os.environ.get("PG_SPMV_PLANES", "1")
k27, k7, k27odd = kern(t._matrix("aniso27", 20)), kern(t._matrix("conv7", 20)), kern(t._matrix("aniso27", 11))
assert (k27 == 9) == (on != "0"), k27
assert k7 != 9 and k27odd != 9, (k7, k27odd)   # 7-point by default, S % 16 != 0: other kernels
t._check(t._matrix("aniso27", 11))
print("ok")
"""
    for on in ("1", "0"):
        assert "ok" in _run({"PG_SPMV_PLANES": on}, code)


def test_plane_kernel_solve_matches_other_kernels():
    code = """
import numpy as np, os, sys
import paper_1907_00072_b200 as pg
from paper_1907_00072_b200 import workloads as wl
h = wl.aniso27(32)
op = pg.DeviceMatrixOperator(h)
poly, _ = pg.build_poly_or_auto(op, wl.make_v0(h.nrows), 12, pg.CostCounters())
res = pg.solve(op, wl.splitmix_uniform(0, h.nrows), right_prec=poly, config=pg.GmresConfig(30, 1e-9))
np.save(sys.argv[1] if len(sys.argv) > 1 else "/tmp/x.npy", res.x)
print("ok", res.iterations, poly.degree, op.engine.shards[0].stats["kernel"])
"""
    outs = []
    for on in ("1", "0"):
        path = f"/tmp/pg_planes_{on}.npy"
        out = _run({"PG_SPMV_PLANES": on}, code.replace('"/tmp/x.npy"', repr(path)))
        tok = out.split()
        assert (tok[3] == "9") == (on == "1"), out
        outs.append((tok[1], tok[2], np.load(path)))
    # same degree and iterations; x agrees to rounding (the residual norm's
    # block reduction order follows the kernel's row-to-thread map)
    assert outs[0][:2] == outs[1][:2]
    assert np.linalg.norm(outs[0][2] - outs[1][2]) <= 1e-12 * np.linalg.norm(outs[1][2])
