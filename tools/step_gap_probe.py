"""Probe: what a step-graph boundary costs.  cfg2, one Arnoldi step at k = 25
(pg_arnoldi_step), timed back to back 50x: issued on the stream (PDL), as
one recorded step graph per step (pg_step_graph_create, as the solver does),
and as graphs holding two steps each.  Events around each batch.

  python tools/step_gap_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1907_00072_b200 as pg  # noqa: E402
from paper_1907_00072_b200 import _lib, workloads as wl  # noqa: E402
from paper_1907_00072_b200.device import PgEvent, ptr  # noqa: E402


def main():
    conf = wl.CONFIGS[2]
    A = wl.make_matrix(conf)
    op = pg.DeviceMatrixOperator(A)
    e = op.engine
    c = pg.CostCounters()
    poly, _ = pg.build_poly_or_auto(op, torch.from_numpy(wl.make_v0(A.nrows)).cuda(), 25, c)
    y = np.ascontiguousarray(poly.y)
    d = poly.degree
    s = e.shards[0]
    V = e.cached_blocks("basis", 51)[0]
    V.normal_()
    z, t, acc, w0, w1 = (e.cached_vecs(k)[0] for k in ("z", "t", "acc", "w0", "w1"))
    ring = s.ring[0]
    host = s.pinned[0]
    ev = PgEvent(s.dev_ord)
    j = 24
    st = torch.cuda.Stream()
    args = (s.mat, y.ctypes.data, d, ptr(V), s.ld, j, ptr(z), ptr(t), ptr(acc), ptr(w0),
            ptr(w1), ptr(ring), host.data_ptr(), s.ws, ev.h, None, None, 0, None, None)

    def timed(fn, reps=50):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3

    out = {}
    out["stream_us_per_step"] = timed(lambda: _lib.call("pg_arnoldi_step", *args, st.cuda_stream))
    h = _lib.C.c_void_p()
    _lib.call("pg_step_graph_create", *args, _lib.C.byref(h))
    out["graph_us_per_step"] = timed(lambda: _lib.call("pg_graph_launch", h, st.cuda_stream))
    # kernel gaps inside / between back-to-back step graphs (CUPTI)
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            _lib.call("pg_graph_launch", h, st.cuda_stream)
        torch.cuda.synchronize()
    kern = sorted((ev.time_range.start, ev.time_range.end, ev.name) for ev in prof.events()
                  if ev.device_type == torch.autograd.DeviceType.CUDA and ev.name)
    per = len(kern) // 10
    gaps = [kern[i + 1][0] - kern[i][1] for i in range(len(kern) - 1)]
    out["kernels_per_step"] = per
    out["busy_us_per_step"] = sum(b - a for a, b, _ in kern) / 10
    out["boundary_gaps_us"] = [round(gaps[i], 1) for i in range(per - 1, len(gaps), per)]
    out["inner_gaps_us_mean"] = float(np.mean([g for i, g in enumerate(gaps) if (i + 1) % per]))
    out["names_tail"] = [k[2].split("(")[0][-28:] for k in kern[per - 3:per + 2]]
    out["publish"] = os.environ.get("PG_PUBLISH", "1")
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in out.items()}))
    _lib.call("pg_graph_destroy", h)


if __name__ == "__main__":
    main()
