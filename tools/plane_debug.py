"""Locate plane-ring SpMV mismatches against the oracle (debug aid): for
each stencil case, the first rows whose device SpMV differs, as (plane,
in-plane index, pattern mask).  Run with PG_SPMV_PLANES=2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402

import paper_1907_00072_b200 as pg  # noqa: E402
from oracle import pgmres_oracle as orc  # noqa: E402
from paper_1907_00072_b200 import workloads as wl  # noqa: E402
import test_gpu_march as t  # noqa: E402

for kind, g in [("aniso27", 12), ("aniso27", 20), ("aniso27", 28), ("conv7", 20), ("conv7", 28),
                ("lap5", 48), ("conv9", 32), ("conv9", 64)]:
    h = t._matrix(kind, g)
    S = g * g if kind in ("aniso27", "conv7") else g
    op = pg.DeviceMatrixOperator(h)
    k = op.engine.shards[0].stats["kernel"]
    x = wl.splitmix_uniform(3, h.nrows)
    got = op.apply(x)
    want = orc.OracleMatrix.of(h).matvec(x)
    bad = np.nonzero(got != want)[0]
    print(kind, g, "kernel", k, "mismatches", len(bad), "of", h.nrows)
    for r in bad[:12]:
        print("   row", r, "plane", r // S, "q", r % S, "len", h.row_ptr[r + 1] - h.row_ptr[r],
              "got", got[r], "want", want[r])
    op.close()
