"""Full-size reference records for the BASELINE configs (build container only).

Runs the UNMODIFIED reference (`/root/reference/pkg/src/polygmres`) on a
BASELINE config at its full size, with the degree policy the bench uses
(`build_poly(d)`, else `auto_degree(cap=d)` on `CholeskyFailure`, SURVEY §7(i);
polyprec.py:125-190) and `solve` (gmres.py:213-343), and writes
`tests/golden/cfg<N>_full_reference.json`: the effective degree, the
polynomial coefficients y, iterations, cycles, final relres, counters and the
wall times.  The GPU tests feed the recorded y to the device `solve`, so
iteration parity at full size does not depend on the degree decision.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_full_records.py 4
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_full_records.py 5:100

`N:cap` stops the reference after `cap` iterations (configs whose full solve
takes hours on the CPU: cfg5 needs > 3000 iterations) and records the whole
residual history, which the GPU test compares iteration by iteration.

The operator comes from this repo's generator (`workloads.make_matrix`), the
right-hand side and v0 from the reference RNG (rng.py:25-37) -- the same
inputs `bench.py` builds.  cfg4 takes about 1.5 h on the 8-core build host.
"""

from __future__ import annotations

import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import polygmres as pg  # noqa: E402  (the unchanged reference)

from paper_1907_00072_b200 import workloads as wl  # noqa: E402

MAX_ITERS = {3: 300}


def main(config: int, cap: int | None = None):
    cfg = wl.CONFIGS[config]
    max_iters = cap if cap else MAX_ITERS.get(config, 200000)
    t0 = time.perf_counter()
    h = wl.make_matrix(cfg)
    A = pg.CsrMatrix(h.nrows, h.ncols, h.row_ptr, h.col_idx, h.values)
    del h
    n = A.nrows
    b = wl.make_rhs(cfg, A, 0)
    v0 = wl.make_v0(n, 0)
    gen_s = time.perf_counter() - t0
    print(f"cfg{config}: n={n} nnz={A.nnz} generated in {gen_s:.1f} s", flush=True)

    counters = pg.CostCounters()
    op = pg.MatrixOperator(A, counters)
    deg = cfg["degree"]
    fail = None
    t0 = time.perf_counter()
    try:
        poly = pg.build_poly(op, v0, deg, counters)
    except pg.CholeskyFailure as exc:
        fail = exc.pivot
        poly = pg.auto_degree(op, v0, deg, counters)
    build_s = time.perf_counter() - t0
    build_counters = counters.as_dict()
    print(f"  degree {deg} -> {poly.degree} (fail pivot {fail}) in {build_s:.1f} s", flush=True)

    t0 = time.perf_counter()
    res = pg.solve(op, b, right_prec=poly,
                   config=pg.GmresConfig(cfg["m"], cfg["tol"], max_iters, True))
    solve_s = time.perf_counter() - t0
    rec = dict(
        config=f"cfg{config} full ({cfg['name']}), n={n}, nnz={A.nnz}",
        generator="paper_1907_00072_b200.workloads.make_matrix; b = make_rhs(seed 0); "
                  "v0 = make_v0(seed 0)",
        requested_degree=deg, build_fail_pivot=fail, effective_degree=poly.degree,
        seed_norm=float(poly.seed_norm), y=[float(v) for v in poly.y],
        restart_m=cfg["m"], tol=cfg["tol"], max_iters=max_iters,
        iterations=res.iterations, cycles=res.cycles, converged=bool(res.converged),
        final_relres=res.final_relres, counters=counters.as_dict(),
        build_counters=build_counters,
        history_first=[list(map(float, r)) for r in res.history[:8]],
        history_last=list(map(float, res.history[-1])) if res.history else None,
        history=[list(map(float, r)) for r in res.history] if (cap or config == 3) else None,
        gen_s=gen_s, build_s=build_s, solve_s=solve_s,
        host=f"build container ({os.cpu_count()} cores, {platform.processor() or 'x86_64'}), "
             f"numpy {np.__version__}",
    )
    out = os.path.join(HERE, f"cfg{config}_full_reference.json" if not cap
                       else f"cfg{config}_full_cap{cap}_reference.json")
    with open(out, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(f"  {res.iterations} iterations, {res.cycles} cycles, relres {res.final_relres:.3e}, "
          f"solve {solve_s:.0f} s -> {out}", flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:] or ["4"]:
        if ":" in c:
            main(int(c.split(":")[0]), int(c.split(":")[1]))
        else:
            main(int(c))
