"""A few z = A p(A) x applications on the cfg2 operator (for ncu captures of
the chain kernel: ncu -k regex:chain_ ... python tools/chain_one.py)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1907_00072_b200 import _lib, workloads as wl  # noqa: E402
from paper_1907_00072_b200.device import Engine, ptr  # noqa: E402

grid = int(os.environ.get("GRID", "100"))
d = int(os.environ.get("DEGREE", "14"))
e = Engine.build(wl.convdiff3d_7pt(grid))
s = e.shards[0]
x, t, z, acc, w0, w1 = (s.vec() for _ in range(6))
x.uniform_(-1, 1)
y = np.random.default_rng(0).uniform(-1, 1, d + 1) / (d + 1)
for _ in range(4):
    _lib.call("pg_wrapped_apply", s.mat, y.ctypes.data, d, ptr(x), ptr(t), ptr(z), ptr(acc),
              ptr(w0), ptr(w1), s.ws, s.stream)
torch.cuda.synchronize()
print("ok", float(z.abs().sum()))
