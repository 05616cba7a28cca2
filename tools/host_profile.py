"""cProfile of one warm cfg2 build + solve (host-side overhead hunt).

  python tools/host_profile.py [--config 2]
"""

import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1907_00072_b200 as pg  # noqa: E402
from paper_1907_00072_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    args = ap.parse_args()
    conf = wl.CONFIGS[args.config]
    A = wl.make_matrix(conf)
    b = torch.from_numpy(wl.make_rhs(conf, A)).cuda()
    v0 = torch.from_numpy(wl.make_v0(A.nrows)).cuda()
    op = pg.DeviceMatrixOperator(A)
    cfg = pg.GmresConfig(conf["m"], conf["tol"])

    def one():
        c = pg.CostCounters()
        op.counters = c
        t0 = time.perf_counter()
        p, _ = pg.build_poly_or_auto(op, v0, conf["degree"], c)
        t1 = time.perf_counter()
        r = pg.solve(op, b, right_prec=p, config=cfg)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1, r

    for _ in range(4):  # the second solve records the step graphs
        one()
    pr = cProfile.Profile()
    pr.enable()
    tb, ts, r = one()
    pr.disable()
    print(f"build {tb*1e3:.2f} ms  solve {ts*1e3:.2f} ms  iters {r.iterations}")
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(25)
    st.sort_stats("cumulative").print_stats(40)


if __name__ == "__main__":
    main()
