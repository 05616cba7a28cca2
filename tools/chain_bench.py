"""Micro-benchmark of z = A p(A) x (pg_wrapped_apply) on the cfg2 operator:
the d passes + wrapper SpMV as one chain kernel (chain.cu) vs pass by pass
(PG_CHAIN=0), over chunk sizes / blocks per SM.  CUDA events over `reps`
back-to-back applications; one line of JSON per setting.

  python tools/chain_bench.py [--degree 14] [--reps 50] [--grid 100]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1907_00072_b200 import _lib, workloads as wl  # noqa: E402
from paper_1907_00072_b200.device import Engine, ptr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--degree", type=int, default=14)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--grid", type=int, default=100)
    ap.add_argument("--settings", default="chain=0;chain=1,ts=4;chain=1,ts=2;chain=1,ts=1;chain=1,ts=8")
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    h = wl.convdiff3d_7pt(args.grid)
    e = Engine.build(h)
    s = e.shards[0]
    x, t, z, acc, w0, w1 = (s.vec() for _ in range(6))
    x.uniform_(-1, 1)
    d = args.degree
    y = np.random.default_rng(0).uniform(-1, 1, d + 1) / (d + 1)
    st = s.stream
    ref = None
    for setting in args.settings.split(";"):
        env = dict(kv.split("=") for kv in setting.split(",") if kv)
        keys = {"chain": "PG_CHAIN", "ts": "PG_CHAIN_TS", "bps": "PG_CHAIN_BLOCKS_PER_SM",
                "dyn": "PG_CHAIN_DYNAMIC"}
        for k, var in keys.items():
            os.environ.pop(var, None)
        for k, v in env.items():
            os.environ[keys[k]] = v

        def run():
            _lib.call("pg_wrapped_apply", s.mat, y.ctypes.data, d, ptr(x), ptr(t), ptr(z),
                      ptr(acc), ptr(w0), ptr(w1), s.ws, st)

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        out = z.clone()
        if ref is None:
            ref = out
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(args.reps):
            run()
        ev1.record()
        torch.cuda.synchronize()
        us = ev0.elapsed_time(ev1) * 1e3 / args.reps
        print(json.dumps({"tag": args.tag, "setting": setting, "n": s.n, "degree": d,
                          "us_per_apply": round(us, 2), "us_per_pass": round(us / (d + 1), 2),
                          "bitwise_vs_first": bool(torch.equal(out, ref))}), flush=True)


if __name__ == "__main__":
    main()
