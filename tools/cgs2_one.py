"""Run the three CGS2 phases a few times at one (n, k) -- for ncu captures.

  python tools/cgs2_one.py --n 1000000 --k 32 [--reps 3]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1907_00072_b200 import _lib  # noqa: E402
from paper_1907_00072_b200.device import _pad, ptr  # noqa: E402
from paper_1907_00072_b200.ortho import workspace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    n, k = args.n, args.k
    ld = _pad(n)
    ws = workspace(torch.cuda.current_device())
    st = torch.cuda.current_stream().cuda_stream
    V = torch.randn((k + 1, ld), dtype=torch.float64, device="cuda")
    z = torch.randn(ld, dtype=torch.float64, device="cuda")
    sc = torch.zeros(200, dtype=torch.float64, device="cuda")
    c1, c2, nsq = sc[:64], sc[64:128], sc[128:129]
    for _ in range(args.reps):
        _lib.call("pg_cgs2_phase1", ptr(V), ld, k, ptr(z), n, ptr(c1), ws, st)
        _lib.call("pg_cgs2_phase2", ptr(V), ld, k, ptr(z), n, ptr(c1), ptr(c2), ws, st)
        _lib.call("pg_cgs2_phase3", ptr(V), ld, k, ptr(z), n, ptr(c1), ptr(c2), ptr(V[k]),
                  ptr(nsq), ws, st)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
