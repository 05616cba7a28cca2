"""Generate the golden vectors that pin the oracle (and, through it, the device
path) to the UNMODIFIED reference.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It writes tests/golden/golden.npz (arrays) and tests/golden/golden.json
(scalars, counters, histories).  Nothing at test / bench time reads
/root/reference; only these committed fixtures travel.

Cases:
  rng      uniform(0, 4096), uniform(1, 4096)                     (rng.py:34-37)
  lap64    gen_laplacian2d(64) CSR                                (sparse.py:329-359)
  spmv     cfg1 b = A x_true; random 1k matrix, rows up to 200    (sparse.py:151-168)
  poly     cfg1 build_poly(deg 10) y; apply_poly(y, b); A p(A) b  (polyprec.py:125-212)
  icgs     random basis n=300 j=20                                (ortho.py:33-70)
  auto     auto_degree bidiag2 cap 20; lap64 cap 16               (polyprec.py:150-190)
  solve    cfg1 full solve; degree sweep; convdiff2d multi-cycle; x0 != 0
  ilu      ILU(0) factors / applications of lap64 and convdiff48 (+ diag shift),
           an ILU-left-preconditioned polynomial solve, pivot failures
  cli      the reference command line on five experiments (incl. --ilu, --degree
           auto, a Matrix Market file lap10.mtx, a non-converged run)
  small    reduced-size versions of configs 2-5 (this repo's generators) solved
           by the reference with the SURVEY §7(i) degree policy
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import polygmres as pg  # noqa: E402  (the unchanged reference)
from polygmres import rng as pg_rng  # noqa: E402

from paper_1907_00072_b200 import workloads as wl  # noqa: E402

arrays: dict = {}
meta: dict = {}


def ref_csr(h):
    return pg.CsrMatrix(h.nrows, h.ncols, h.row_ptr, h.col_idx, h.values)


def solve_record(name, A, b, v0, deg, m, tol, max_iters=200000, x0=None, policy=True,
                 keep_x=False):
    counters = pg.CostCounters()
    op = pg.MatrixOperator(A, counters)
    poly = None
    eff = None
    if deg is not None:
        try:
            poly = pg.build_poly(op, v0, deg, counters)
            eff = deg
        except pg.CholeskyFailure as exc:
            if not policy:
                raise
            meta[name + "_build_fail_pivot"] = exc.pivot
            poly = pg.auto_degree(op, v0, deg, counters)
            eff = poly.degree
    res = pg.solve(op, b, x0=x0, right_prec=poly,
                   config=pg.GmresConfig(m, tol, max_iters, True))
    meta[name] = dict(
        requested_degree=deg, effective_degree=eff, converged=bool(res.converged),
        iterations=res.iterations, cycles=res.cycles, final_relres=res.final_relres,
        counters=counters.as_dict(),
        history=[list(map(float, row)) for row in res.history[:60]],
        history_len=len(res.history),
        history_last=list(map(float, res.history[-1])) if res.history else None,
    )
    if poly is not None:
        arrays[name + "_y"] = poly.y
    if keep_x:
        arrays[name + "_x"] = res.x
    return res


def main():
    # --- rng -------------------------------------------------------------
    arrays["rng_u0"] = pg_rng.uniform(0, 4096)
    arrays["rng_u1"] = pg_rng.uniform(1, 4096)
    arrays["rng_u7_hi"] = pg_rng.uniform(7, 1000, 2.0, 5.0)

    # --- config 1 operator + vectors --------------------------------------
    A = pg.gen_laplacian2d(64)
    arrays["lap64_row_ptr"] = A.row_ptr
    arrays["lap64_col_idx"] = A.col_idx
    arrays["lap64_values"] = A.values
    n = A.nrows
    x_true = pg_rng.uniform(0, n)
    b = pg.spmv(A, x_true)
    arrays["cfg1_b"] = b
    v0 = pg.random_seed_vector(n, 1)

    counters = pg.CostCounters()
    op = pg.MatrixOperator(A, counters)
    poly = pg.build_poly(op, v0, 10, counters)
    arrays["cfg1_y10"] = poly.y
    meta["cfg1_build"] = dict(seed_norm=poly.seed_norm, counters=counters.as_dict())
    c2 = pg.CostCounters()
    op2 = pg.MatrixOperator(A, c2)
    arrays["cfg1_pAb"] = pg.apply_poly(poly, op2, b, c2)
    arrays["cfg1_ApAb"] = pg.PolynomialWrappedOperator(op2, poly).apply(b)
    meta["cfg1_apply_counters"] = c2.as_dict()
    for d in (12, 13, 14):
        try:
            pg.build_poly(pg.MatrixOperator(A), v0, d, pg.CostCounters())
            meta[f"cfg1_build{d}"] = "ok"
        except pg.CholeskyFailure as exc:
            meta[f"cfg1_build{d}"] = exc.pivot

    # higher-degree apply with arbitrary finite coefficients (apply_poly accepts any y)
    yy = np.random.default_rng(5).uniform(-1, 1, 26) * 0.3 ** np.arange(26)
    p26 = pg.PolyCoefficients(25, yy, 1.0)
    arrays["cfg1_y25_rand"] = yy
    arrays["cfg1_p25b"] = pg.apply_poly(p26, pg.MatrixOperator(A), b, pg.CostCounters())

    solve_record("cfg1_solve", A, b, v0, 10, 40, 1e-8, keep_x=True)
    for d in (None, 1, 4, 8, 12):
        solve_record(f"cfg1_sweep_{d}", A, b, v0, d, 40, 1e-8)

    # SPEC acceptance criterion 1: lap 201, generator rhs, deg 5, m 50
    L = pg.gen_laplacian2d(201)
    solve_record("spec1_lap201", L, pg.gen_laplacian_rhs(201),
                 pg.random_seed_vector(L.nrows, 1), 5, 50, 1e-8)

    # --- random SpMV (bitwise order check) --------------------------------
    gen = np.random.default_rng(1234)
    nr = 1000
    lens = gen.integers(0, 201, nr)
    rows = np.repeat(np.arange(nr), lens)
    cols = gen.integers(0, nr, len(rows))
    vals = gen.standard_normal(len(rows))
    R = pg.CsrMatrix.from_coo(nr, nr, rows, cols, vals)
    xr = gen.standard_normal(nr)
    arrays["rand1k_row_ptr"] = R.row_ptr
    arrays["rand1k_col_idx"] = R.col_idx
    arrays["rand1k_values"] = R.values
    arrays["rand1k_x"] = xr
    arrays["rand1k_y"] = pg.spmv(R, xr)
    yr = gen.uniform(-1, 1, 7)
    arrays["rand1k_poly_y"] = yr
    arrays["rand1k_poly_out"] = pg.apply_poly(pg.PolyCoefficients(6, yr, 1.0),
                                              pg.MatrixOperator(R), xr, pg.CostCounters())

    # --- icgs ---------------------------------------------------------------
    gen = np.random.default_rng(77)
    basis = np.linalg.qr(gen.standard_normal((300, 20)))[0]
    w = gen.uniform(-1, 1, 300)
    cc = pg.CostCounters()
    res = pg.icgs(basis, w, cc)
    arrays["icgs_basis"] = basis
    arrays["icgs_w"] = w
    arrays["icgs_coeffs"] = res.coeffs
    arrays["icgs_vector"] = res.vector
    meta["icgs"] = dict(new_norm=res.new_norm, breakdown=res.breakdown, counters=cc.as_dict())

    # --- auto_degree ------------------------------------------------------
    cc = pg.CostCounters()
    p = pg.auto_degree(pg.MatrixOperator(pg.bidiag2(), cc), pg.random_seed_vector(5000, 1), 20, cc)
    arrays["auto_bidiag2_y"] = p.y
    meta["auto_bidiag2"] = dict(degree=p.degree, counters=cc.as_dict())
    cc = pg.CostCounters()
    p = pg.auto_degree(pg.MatrixOperator(A, cc), v0, 16, cc)
    arrays["auto_lap64_y"] = p.y
    meta["auto_lap64"] = dict(degree=p.degree, counters=cc.as_dict())

    # --- nonsymmetric multi-cycle solve + x0 != 0 --------------------------
    C, _ = pg.gen_convdiff2d(48, 0.05)
    bc = pg_rng.uniform(3, C.nrows)
    arrays["convdiff48_row_ptr"] = C.row_ptr
    arrays["convdiff48_col_idx"] = C.col_idx
    arrays["convdiff48_values"] = C.values
    solve_record("convdiff48_solve", C, bc, pg.random_seed_vector(C.nrows, 4), 6, 20, 1e-9,
                 keep_x=True)
    x0 = pg_rng.uniform(9, C.nrows) * 0.1
    arrays["convdiff48_x0"] = x0
    solve_record("convdiff48_x0_solve", C, bc, pg.random_seed_vector(C.nrows, 4), 4, 15, 1e-8,
                 x0=x0)
    solve_record("convdiff48_noprec", C, bc, None, None, 30, 1e-8, max_iters=400)

    # --- ILU(0) left preconditioning (ilu.py:38-114, gmres.py:63-95) --------
    F = pg.ilu0_factor(A)  # lap64
    arrays["ilu_lap64_values"] = F.values
    arrays["ilu_lap64_diag_ptr"] = F.diag_ptr
    arrays["ilu_lap64_apply"] = pg.ilu0_apply(F, b)
    Fc = pg.ilu0_factor(C)  # convdiff48 (non-symmetric)
    arrays["ilu_convdiff48_values"] = Fc.values
    arrays["ilu_convdiff48_apply"] = pg.ilu0_apply(Fc, bc)
    Fs = pg.ilu0_factor(C, diag_shift=0.3)
    arrays["ilu_convdiff48_shift_values"] = Fs.values
    # left-preconditioned polynomial solve, the CLI's --ilu flow (cli.py:252-277)
    counters = pg.CostCounters()
    opi = pg.IluPreconditionedOperator(C, Fc, counters)
    b_eff = opi.precondition(bc)
    arrays["ilu_convdiff48_beff"] = b_eff
    polyi = pg.build_poly(opi, pg.random_seed_vector(C.nrows, 4), 5, counters)
    arrays["ilu_convdiff48_y"] = polyi.y
    before = counters.as_dict()
    resi = pg.solve(opi, b_eff, right_prec=polyi, config=pg.GmresConfig(20, 1e-10))
    arrays["ilu_convdiff48_x"] = resi.x
    meta["ilu_convdiff48_solve"] = dict(
        iterations=resi.iterations, cycles=resi.cycles, converged=resi.converged,
        final_relres=resi.final_relres, counters=counters.as_dict(), build_counters=before)
    for name, dense in (("zero_pivot", [[0.0, 1.0], [1.0, 1.0]]),
                        ("missing_diag", [[0.0, 1.0], [1.0, 0.0]])):
        rows, cols = np.nonzero(np.asarray(dense) != 0.0) if name == "missing_diag" else (
            np.array([0, 0, 1, 1]), np.array([0, 1, 0, 1]))
        vals = np.asarray(dense)[rows, cols]
        M = pg.CsrMatrix.from_coo(2, 2, rows, cols, vals)
        try:
            pg.ilu0_factor(M)
            meta[f"ilu_{name}"] = dict(row=None)
        except pg.PivotError as exc:
            meta[f"ilu_{name}"] = dict(row=exc.row, message=str(exc))

    # --- reduced-size configs 2-5 (this repo's generators, reference solver) --
    small = {
        2: dict(grid=16), 3: dict(size=4000), 4: dict(grid=12), 5: dict(grid=48),
    }
    for c, kw in small.items():
        cfg = wl.CONFIGS[c]
        h = wl.make_matrix(cfg, **kw)
        Am = ref_csr(h)
        nn = Am.nrows
        arrays[f"small{c}_sha"] = np.frombuffer(
            __import__("hashlib").sha256(
                h.row_ptr.tobytes() + h.col_idx.tobytes() + h.values.tobytes()).digest(),
            dtype=np.uint8)
        bb = wl.make_rhs(cfg, h, 0)
        vv = wl.make_v0(nn, 0)
        max_iters = 300 if c == 3 else 200000
        solve_record(f"small{c}", Am, bb, vv, cfg["degree"], cfg["m"], cfg["tol"],
                     max_iters=max_iters)

    # --- the reference command line (cli.py:242-312), run in-process -------
    import tempfile

    from polygmres import cli as pg_cli
    mtx = os.path.join(HERE, "lap10.mtx")
    pg.write_matrix_market(pg.gen_laplacian2d(10), mtx)
    cli_cases = {
        "cli_cfg1": ["--generator", "laplacian2d", "--grid-n", "64", "--rhs", "axrandom",
                     "--seed", "0", "--degree", "10", "-m", "40", "--tol", "1e-8"],
        "cli_ilu": ["--generator", "convdiff2d", "--grid-n", "48", "--epsilon", "0.05",
                    "--rhs", "generator", "--ilu", "--degree", "5", "-m", "20", "--tol",
                    "1e-9", "--format", "jsonl"],
        "cli_auto": ["--generator", "bidiag2", "--rhs", "random", "--seed", "3", "--degree",
                     "auto", "--degree-cap", "20", "-m", "30", "--tol", "1e-10"],
        "cli_mtx": ["--matrix-file", "@MTX@", "--rhs", "random", "--seed", "5", "--degree", "3",
                    "--v0", "rhs", "-m", "10", "--tol", "1e-9"],
        "cli_noprec": ["--generator", "laplacian2d", "--grid-n", "32", "--rhs", "random", "-m",
                       "30", "--max-iters", "50"],
    }
    with tempfile.TemporaryDirectory() as tmp:
        for name, argv in cli_cases.items():
            out = os.path.join(tmp, name)
            argv = [a.replace("@MTX@", mtx) for a in argv] + ["-o", out]
            code = pg_cli.main(argv)
            fmt = "jsonl" if "jsonl" in argv else "csv"
            with open(out + ".summary.json") as fh:
                summary = json.load(fh)
            with open(f"{out}.history.{fmt}") as fh:
                history = fh.read()
            summary["config"]["output"] = "<OUT>"
            if summary["config"]["matrix_file"]:
                summary["config"]["matrix_file"] = "<MTX>"
            meta[name] = dict(argv=[a if a != mtx else "<MTX>" for a in argv[:-2]], exit=code,
                              summary=summary, history=history)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays,", len(meta), "records")


if __name__ == "__main__":
    main()
