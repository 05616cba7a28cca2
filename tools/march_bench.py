"""Time the fused middle polynomial pass (acc in/out + w out) of the kernel
the current environment selects, on cfg4 (8M rows, 27-point) and cfg2 (1M
rows, 7-point): CUDA events over back-to-back launches.  Run once per
environment (the kernel choice is read once per process), e.g.
PG_SPMV_MARCH=0 python tools/march_bench.py."""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1907_00072_b200 import workloads as wl  # noqa: E402
from paper_1907_00072_b200.device import Engine  # noqa: E402
from spmv_bench import time_pass  # noqa: E402

grid = int(os.environ.get("GRID", "0"))  # 0: the BASELINE grid
for key, kw in [(c, dict(grid=grid) if grid else {}) for c in os.environ.get("CASES", "cfg4,cfg2").split(",")]:
    conf = wl.CONFIGS[int(key[-1])]
    A = wl.make_matrix(conf, **kw)
    e = Engine.build(A)
    dt, _ = time_pass(e, int(os.environ.get("REPS", "50")))
    stored = e.shards[0].pass_bytes(24)
    print(json.dumps(dict(case=key, grid=grid, plan=e.shards[0].plane_plan, env={k: v for k, v in os.environ.items() if k.startswith("PG_")},
                          us=round(dt * 1e6, 2), gbs_stored=round(stored / dt / 1e9, 1),
                          stored_mb=round(stored / 1e6, 1), kernel=e.shards[0].stats["kernel"])),
          flush=True)
    e.close()
    del A, e
    torch.cuda.empty_cache()
