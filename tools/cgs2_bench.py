"""Micro-benchmark of the three CGS2 phases (and the recovery GEMV) at the
basis widths the solver sees.  CUDA events over `reps` launches each;
algorithmic bytes: phases 1/2: 8nk + 8n, phase 3: 8nk + 16n, GEMV 8nk + 8n.

  python tools/cgs2_bench.py [--reps 20]
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


def timed(fn, reps):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--n", default="1000000,8000000")
    ap.add_argument("--k", default="10,25,51")
    args = ap.parse_args()
    ws = workspace(torch.cuda.current_device())
    st = torch.cuda.current_stream().cuda_stream
    for n in [int(v) for v in args.n.split(",")]:
        ld = _pad(n)
        V = torch.randn((52, ld), dtype=torch.float64, device="cuda")
        z = torch.randn(ld, dtype=torch.float64, device="cuda")
        out = torch.empty(ld, dtype=torch.float64, device="cuda")
        sc = torch.zeros(200, dtype=torch.float64, device="cuda")
        c1, c2, nsq = sc[:64], sc[64:128], sc[128:129]
        for k in [int(v) for v in args.k.split(",")]:
            res = {}
            res["phase1"] = timed(lambda: _lib.call("pg_cgs2_phase1", ptr(V), ld, k, ptr(z), n,
                                                    ptr(c1), ws, st), args.reps)
            res["phase2"] = timed(lambda: _lib.call("pg_cgs2_phase2", ptr(V), ld, k, ptr(z), n,
                                                    ptr(c1), ptr(c2), ws, st), args.reps)
            res["phase3"] = timed(lambda: _lib.call("pg_cgs2_phase3", ptr(V), ld, k, ptr(z), n,
                                                    ptr(c1), ptr(c2), ptr(out), ptr(nsq), ws,
                                                    st), args.reps)
            res["gemv"] = timed(lambda: _lib.call("pg_gemv", ptr(V), ld, k, ptr(c1), n,
                                                  ptr(out), st), args.reps)
            for ph, t in res.items():
                nb = 8 * n * k + (16 if ph == "phase3" else 8) * n
                print(json.dumps(dict(n=n, k=k, kernel=ph, us=round(t * 1e6, 2),
                                      gbs=round(nb / t / 1e9, 1))), flush=True)
        del V


if __name__ == "__main__":
    main()
