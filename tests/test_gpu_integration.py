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
