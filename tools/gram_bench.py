"""Micro-benchmark of the double-double power-basis Gram (pg_gram) at the
build's sizes: n = 1e6 / 8e6 rows, 14 / 16 / 27 columns.  CUDA events over
`reps` launches.  PG_TILE_CTAS_P3 sets the co-resident CTAs its ring is
sized for.

  python tools/gram_bench.py [--reps 10]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1907_00072_b200 import _lib  # noqa: E402
from paper_1907_00072_b200.device import _pad, ptr  # noqa: E402
from paper_1907_00072_b200.ortho import workspace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    ws = workspace(torch.cuda.current_device())
    st = torch.cuda.current_stream().cuda_stream
    for n in (1_000_000, 8_000_000):
        ld = _pad(n)
        P = torch.randn((28, ld), dtype=torch.float64, device="cuda")
        G = torch.zeros(2 * 28 * 28, dtype=torch.float64, device="cuda")
        for k in (14, 16, 27):
            def run():
                _lib.call("pg_gram", ptr(P), ld, k, n, ptr(G), ws, st)
            for _ in range(2):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / args.reps
            print(json.dumps({"n": n, "cols": k, "us": round(us, 1),
                              "ctas": os.environ.get("PG_TILE_CTAS_P3", "default"),
                              "gbs": round(8 * n * k / us / 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
