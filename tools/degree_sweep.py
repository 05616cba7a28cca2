"""BASELINE config 5: polynomial degree sweep d in {1, 4, 8, 16, 32, 64} at
GMRES(50) on the 2048^2 9-point convection-diffusion operator (one GPU):
effective degree (degree policy), iterations, global reductions (the 3 dots
per iteration + 1 per cycle end + 2 for the polynomial build = all-reduces at
P > 1), SpMVs and time per solve (CUDA events, L2 flushed before each).

  python tools/degree_sweep.py [--grid 2048] [--max-iters 3000] [--out file.json]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1907_00072_b200 as pg  # noqa: E402
from paper_1907_00072_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=2048)
    ap.add_argument("--max-iters", type=int, default=3000)
    ap.add_argument("--degrees", default="1,4,8,16,32,64")
    ap.add_argument("--out", default=None)
    # policy: the reference construction (power basis, auto-degree fallback);
    # arnoldi: harmonic Ritz values at the requested degree (capped at 62),
    # evaluated in root-product form
    ap.add_argument("--construction", default="policy", choices=["policy", "arnoldi"])
    args = ap.parse_args()
    conf = wl.CONFIGS[5]
    A = wl.make_matrix(conf, grid=args.grid)
    b = torch.from_numpy(wl.make_rhs(conf, A)).cuda()
    v0 = torch.from_numpy(wl.make_v0(A.nrows)).cuda()
    op = pg.DeviceMatrixOperator(A)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    rows = []
    for d in (int(x) for x in args.degrees.split(",")):
        for rep in range(2):  # first: warm-up (allocations, first launches)
            c = pg.CostCounters()
            op.counters = c
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if args.construction == "arnoldi":
                p, piv = pg.build_poly_arnoldi(op, v0, min(d, 62), c), None
                form = "roots"
            else:
                p, piv = pg.build_poly_or_auto(op, v0, d, c)
                form = "monomial"
            res = pg.solve(op, b, right_prec=p, config=pg.GmresConfig(
                conf["m"], conf["tol"], args.max_iters, poly_form=form))
            e1.record()
            torch.cuda.synchronize()
        rec = dict(construction=args.construction, degree_requested=d,
                   degree_effective=p.degree, failed_pivot=piv,
                   iterations=res.iterations, cycles=res.cycles, converged=res.converged,
                   final_relres=res.final_relres, spmvs=c.spmvs, dots=c.dots,
                   global_reductions=c.dots + res.cycles, time_s=e0.elapsed_time(e1) / 1e3)
        print(json.dumps(rec), flush=True)
        rows.append(rec)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(dict(config=conf["name"], n=A.nrows, nnz=A.nnz, construction=args.construction,
                           rows=rows), fh, indent=1)


if __name__ == "__main__":
    main()
