"""Run a few fused polynomial passes of one operator (for ncu captures).

  python tools/spmv_one.py --config 4 --grid 160 [--reps 5]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1907_00072_b200 import _lib, workloads as wl  # noqa: E402
from paper_1907_00072_b200.device import Engine, ptr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--grid", type=int, default=160)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--mode", default="poly", choices=["poly", "spmv"])
    args = ap.parse_args()
    A = wl.make_matrix(wl.CONFIGS[args.config], grid=args.grid)
    e = Engine.build(A)
    s = e.shards[0]
    x, acc, w = s.vec(), s.vec(), s.vec()
    x.uniform_(-1, 1)
    for _ in range(args.reps):
        _lib.call("pg_poly_pass", s.mat, ptr(x), ptr(acc), None, ptr(acc), ptr(w), 0.5, 0.25,
                  _lib.PG_PASS_WRITE_W, s.stream)
    torch.cuda.synchronize()
    print("ok", s.stats)


if __name__ == "__main__":
    main()
