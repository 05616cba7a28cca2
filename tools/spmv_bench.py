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
    # PINGPONG=1: each launch reads the previous launch's w_out, like the
    # passes of a polynomial chain (default: the same x every launch)
    pp = os.environ.get("PINGPONG", "0") == "1"
    for i in range(reps):
        a, b = (x, w) if (not pp or i % 2 == 0) else (w, x)
        _lib.call("pg_poly_pass", s.mat, ptr(a), ptr(acc), None, ptr(acc), ptr(b), 0.5, 0.25,
                  _lib.PG_PASS_WRITE_W, st)
    ev1.record()
    torch.cuda.synchronize()
    dt = ev0.elapsed_time(ev1) / 1e3 / reps
    nb = 12 * s.nnz + 36 * s.n
    return dt, nb / dt / 1e9


VARIANTS = {
    "window": {"PG_SPMV_WIN_MIN_ROW": "0"},        # windowed pair kernel (TMA ring)
    "pair": {"PG_SPMV_WIN": "0"},                  # pair dictionary, global gathers
    "dict": {"PG_SPMV_WIN": "0", "PG_SPMV_PAIR": "0"},  # two 1-byte streams
    "plain": {"PG_SPMV_WIN": "0", "PG_SPMV_PAIR": "0", "PG_SPMV_DICT": "0"},  # int32 + f64
    "default": {},
    "nopat": {"PG_SPMV_PAT": "0"},                 # pair / window kernels (no row patterns)
}
ENV_KEYS = ("PG_SPMV_WIN", "PG_SPMV_PAIR", "PG_SPMV_DICT", "PG_SPMV_WIN_MIN_ROW", "PG_SPMV_PAT")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--variants", default="window,pair,dict,plain")
    ap.add_argument("--cases", default="cfg2,cfg4,cfg5,cfg3")
    args = ap.parse_args()
    cases = {"cfg2": ("cfg2 7pt 100^3", wl.CONFIGS[2], dict()),
             "cfg4": ("cfg4 27pt 160^3", wl.CONFIGS[4], dict(grid=160)),
             "cfg5": ("cfg5 9pt 2048^2", wl.CONFIGS[5], dict()),
             "cfg3": ("cfg3 random 2e6", wl.CONFIGS[3], dict())}
    out = []
    for key in args.cases.split(","):
        name, conf, kw = cases[key]
        A = wl.make_matrix(conf, **kw)
        for var in args.variants.split(","):
            for k in ENV_KEYS:
                os.environ.pop(k, None)
            os.environ.update(VARIANTS[var])
            e = Engine.build(A)
            st = e.shards[0].stats
            dt, gbs = time_pass(e, args.reps)
            eb = st["stream_bytes"]
            stored = e.shards[0].pass_bytes(24)  # middle pass: acc in/out + w out
            rec = dict(case=name, kernel=var, us=dt * 1e6, gbs_uncompressed_equiv=gbs,
                       gbs_stored=stored / dt / 1e9,
                       nnz=A.nnz, n=A.nrows, padded=st["padded_nnz"], entry_bytes=eb,
                       kernel_kind=st["kernel"])
            print(json.dumps(rec), flush=True)
            out.append(rec)
            e.close()
            del e
        del A


if __name__ == "__main__":
    main()
