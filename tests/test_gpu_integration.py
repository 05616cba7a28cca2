"""The ctypes binding shown in INTEGRATION.md §2 is executed verbatim against
the golden vectors, so the documented integration stays correct.  GPU only."""

import os
import re
import types

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_00072_b200 as pg  # noqa: E402
from paper_1907_00072_b200 import CostCounters  # noqa: E402
from paper_1907_00072_b200.polyprec import PolyCoefficients  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub_namespace():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    code = next(b for b in blocks if "pg_matrix_create" in b)
    ns = {}
    cwd = os.getcwd()
    os.chdir(ROOT)
    try:
        exec(compile(code, "INTEGRATION.md", "exec"), ns)
    finally:
        os.chdir(cwd)
    return ns


def test_integration_stub_is_bitwise(golden):
    a, meta = golden
    ns = _stub_namespace()
    A = types.SimpleNamespace(nrows=4096, ncols=4096, row_ptr=a["lap64_row_ptr"],
                              col_idx=a["lap64_col_idx"], values=a["lap64_values"])
    c = CostCounters()
    op = ns["B200Operator"](A, c)
    x = np.asarray(a["rng_u0"], dtype=np.float64)
    assert np.array_equal(op.apply(x), a["cfg1_b"])
    p = PolyCoefficients(10, a["cfg1_y10"], 1.0)
    out = ns["apply_poly_b200"](p, op, a["cfg1_b"], c)
    assert np.array_equal(out, a["cfg1_pAb"])
    assert c.spmvs == 1 + 10


def test_numpy_vectors_staged_through_pinned_chunks():
    """Large numpy vectors (the reference's call signature) move through the
    chunked pinned staging (device.HostStage): bit-exact round trips at sizes
    around the chunk boundaries, and apply() on numpy equals apply() on a
    device tensor bit for bit."""
    from paper_1907_00072_b200 import workloads as wl
    from paper_1907_00072_b200.device import HostStage
    h = wl.laplacian2d(1733)  # n = 3,003,289: three full 8 MB chunks + a tail
    op = pg.DeviceMatrixOperator(h)
    e = op.engine
    for n_cut in (HostStage.MIN, HostStage.CHUNK, HostStage.CHUNK + 1, h.nrows):
        x = wl.splitmix_uniform(n_cut, h.nrows)
        xs = e.from_host(x)
        back = e.to_host(xs)
        assert np.array_equal(back, x)
    x = wl.splitmix_uniform(5, h.nrows)
    y_np = op.apply(x)
    y_t = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(y_np, y_t)
    op.close()
