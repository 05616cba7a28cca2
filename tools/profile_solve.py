"""One warm-up solve, then one profiled solve between cudaProfilerStart/Stop
(use with `ncu --profile-from-start off`).  Prints the solve summary.

  python tools/profile_solve.py [--config 2] [--max-iters N] [--grid G]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1907_00072_b200 as pg  # noqa: E402
from paper_1907_00072_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--grid", type=int, default=None)
    ap.add_argument("--max-iters", type=int, default=200000)
    args = ap.parse_args()
    conf = wl.CONFIGS[args.config]
    A = wl.make_matrix(conf, grid=args.grid)
    n = A.nrows
    b = torch.from_numpy(wl.make_rhs(conf, A)).cuda()
    v0 = torch.from_numpy(wl.make_v0(n)).cuda()
    op = pg.DeviceMatrixOperator(A)
    cfg = pg.GmresConfig(conf["m"], conf["tol"], args.max_iters)

    def one():
        c = pg.CostCounters()
        op.counters = c
        p, _ = pg.build_poly_or_auto(op, v0, conf["degree"], c)
        return p, pg.solve(op, b, right_prec=p, config=cfg), c

    one()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    p, res, c = one()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"degree {p.degree} iterations {res.iterations} cycles {res.cycles} "
          f"relres {res.final_relres:.3e} spmvs {c.spmvs} dots {c.dots}")


if __name__ == "__main__":
    main()
