"""Where do slow steps come from?  Per step: GPU time of build and solve
(events), host wall time, GPU time inside the fused polynomial chains, and
whether a GC generation ran.

  python tools/step_jitter.py [--steps 40] [--nogc]
"""

import argparse
import gc
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1907_00072_b200 as pg  # noqa: E402
from paper_1907_00072_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--nogc", action="store_true")
    ap.add_argument("--config", type=int, default=2)
    args = ap.parse_args()
    conf = wl.CONFIGS[args.config]
    A = wl.make_matrix(conf)
    b = torch.from_numpy(wl.make_rhs(conf, A)).cuda()
    v0 = torch.from_numpy(wl.make_v0(A.nrows)).cuda()
    op = pg.DeviceMatrixOperator(A)
    e = op.engine
    cfg = pg.GmresConfig(conf["m"], conf["tol"])
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
    gcev = []
    gc.callbacks.append(lambda phase, info: gcev.append((phase, info.get("generation"),
                                                         time.perf_counter())))
    if args.nogc:
        gc.collect()
        gc.freeze()
        gc.disable()
    rows = []
    for i in range(args.steps + 3):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e.timer = []
        n_gc = len(gcev)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        t0 = time.perf_counter()
        evs[0].record()
        c = pg.CostCounters()
        op.counters = c
        p, _ = pg.build_poly_or_auto(op, v0, conf["degree"], c)
        evs[1].record()
        pg.solve(op, b, right_prec=p, config=cfg)
        evs[2].record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        chain = sum(a.elapsed_time(bb) for a, bb, _, _ in e.timer)
        gens = [g for ph, g, _ in gcev[n_gc:] if ph == "start"]
        if i >= 3:
            rows.append(dict(step=i - 3, build_ms=round(evs[0].elapsed_time(evs[1]), 3),
                             solve_ms=round(evs[1].elapsed_time(evs[2]), 3),
                             host_ms=round(1e3 * (t1 - t0), 3), poly_chain_ms=round(chain, 3),
                             gc=gens))
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
