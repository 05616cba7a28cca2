"""Where the e2e time goes on cfg2: public API with pinned host inputs vs
device-resident inputs, phase by phase (host clock, synchronised).

  python tools/e2e_probe.py [--config 2] [--reps 5]
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1907_00072_b200 as pg  # noqa: E402
from paper_1907_00072_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    conf = wl.CONFIGS[args.config]
    A = wl.make_matrix(conf)
    op = pg.DeviceMatrixOperator(A)
    b_host = wl.make_rhs(conf, A)
    v0_host = wl.make_v0(A.nrows)
    b_pin = torch.from_numpy(b_host).pin_memory()
    v0_pin = torch.from_numpy(v0_host).pin_memory()
    b_dev, v0_dev = b_pin.cuda(), v0_pin.cuda()
    cfg = pg.GmresConfig(conf["m"], conf["tol"])

    def run(b, v0):
        t = [time.perf_counter()]
        c = pg.CostCounters()
        op.counters = c
        p, _ = pg.build_poly_or_auto(op, v0, conf["degree"], c)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        r = pg.solve(op, b, right_prec=p, config=cfg)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        x = r.x
        if isinstance(x, torch.Tensor) and x.is_cuda:
            x = x.cpu()
        t.append(time.perf_counter())
        return np.diff(t) * 1e3

    for name, (b, v0) in (("device", (b_dev, v0_dev)), ("pinned", (b_pin, v0_pin)),
                          ("numpy", (b_host, v0_host))):
        run(b, v0)
        rows = np.array([run(b, v0) for _ in range(args.reps)])
        med = np.median(rows, axis=0)
        print(json.dumps({"inputs": name, "build_ms": round(med[0], 3),
                          "solve_ms": round(med[1], 3), "x_to_host_ms": round(med[2], 3),
                          "total_ms": round(float(med.sum()), 3)}), flush=True)


if __name__ == "__main__":
    main()
