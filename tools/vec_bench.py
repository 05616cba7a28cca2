"""Time the normalisation kernel (pg_normalize, in place as in the solver) at
n = 8M / 1M: CUDA events over back-to-back launches; bytes = 16 n."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1907_00072_b200 import _lib  # noqa: E402
from paper_1907_00072_b200.device import ptr  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
for n in (8_000_000, 1_000_000):
    x = torch.rand(n + 64, dtype=torch.float64, device="cuda") + 1.0
    nsq = torch.ones(1, dtype=torch.float64, device="cuda")
    for _ in range(3):
        _lib.call("pg_normalize", ptr(x), ptr(nsq), n, ptr(x), st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        _lib.call("pg_normalize", ptr(x), ptr(nsq), n, ptr(x), st)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 50 / 1e3
    print(json.dumps(dict(n=n, kernel="normalize", us=round(t * 1e6, 2),
                          gbs=round(16 * n / t / 1e9, 1))))
