"""Micro-benchmark of the fused polynomial pass (middle pass: acc_in, w_out)
for the TMA-ring and plain SELL kernels on a few operators.  CUDA events over
`reps` back-to-back launches; algorithmic bytes = 12 nnz + 36 n per pass.

  python tools/spmv_bench.py [--reps 50]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1907_00072_b200 import _lib, workloads as wl  # noqa: E402
from paper_1907_00072_b200.device import Engine, ptr  # noqa: E402


def time_pass(e, reps):
    s = e.shards[0]
    x, acc, w = s.vec(), s.vec(), s.vec()
    x.uniform_(-1, 1)
    acc.uniform_(-1, 1)
    st = s.stream
    for _ in range(3):
        _lib.call("pg_poly_pass", s.mat, ptr(x), ptr(acc), None, ptr(acc), ptr(w), 0.5, 0.25,
                  _lib.PG_PASS_WRITE_W, st)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(reps):
        _lib.call("pg_poly_pass", s.mat, ptr(x), ptr(acc), None, ptr(acc), ptr(w), 0.5, 0.25,
                  _lib.PG_PASS_WRITE_W, st)
    ev1.record()
    torch.cuda.synchronize()
    dt = ev0.elapsed_time(ev1) / 1e3 / reps
    nb = 12 * s.nnz + 36 * s.n
    return dt, nb / dt / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    cases = [("cfg2 7pt 100^3", wl.CONFIGS[2], dict()),
             ("cfg4 27pt 160^3", wl.CONFIGS[4], dict(grid=160)),
             ("cfg5 9pt 2048^2", wl.CONFIGS[5], dict()),
             ("cfg3 random 2e6", wl.CONFIGS[3], dict())]
    out = []
    for name, conf, kw in cases:
        A = wl.make_matrix(conf, **kw)
        for plain in (False, True):
            if plain:
                os.environ.pop("PG_SPMV_TMA", None)
            else:
                os.environ["PG_SPMV_TMA"] = "1"
            e = Engine.build(A)
            dt, gbs = time_pass(e, args.reps)
            rec = dict(case=name, kernel="plain" if plain else "tma", us=dt * 1e6, gbs=gbs,
                       nnz=A.nnz, n=A.nrows, padded=e.shards[0].stats["padded_nnz"])
            print(json.dumps(rec), flush=True)
            out.append(rec)
            e.close()
            del e
        del A
    os.environ.pop("PG_SPMV_PLAIN", None)


if __name__ == "__main__":
    main()
