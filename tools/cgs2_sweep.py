"""Phase 1/2 timing across k for one env configuration (n = 1e6)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1907_00072_b200 import _lib
from paper_1907_00072_b200.device import _pad, ptr
from paper_1907_00072_b200.ortho import workspace
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ld = _pad(n); ws = workspace(0); st = torch.cuda.current_stream().cuda_stream
V = torch.randn((53, ld), dtype=torch.float64, device="cuda"); z = torch.randn(ld, dtype=torch.float64, device="cuda")
sc = torch.zeros(200, dtype=torch.float64, device="cuda"); c1, c2 = sc[:64], sc[64:128]
out = {}
for k in (16, 24, 32, 40, 51):
    res = []
    for ph in (1, 2):
        f = (lambda: _lib.call("pg_cgs2_phase1", ptr(V), ld, k, ptr(z), n, ptr(c1), ws, st)) if ph == 1 else \
            (lambda: _lib.call("pg_cgs2_phase2", ptr(V), ld, k, ptr(z), n, ptr(c1), ptr(c2), ws, st))
        for _ in range(3): f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): f()
        e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 20 / 1e3
        res.append(round(8 * n * (k + 1) / t / 1e9))
    out[k] = res
print(json.dumps(out))
