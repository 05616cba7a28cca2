"""Probe: does replaying one Arnoldi step (pg_arnoldi_step's kernels) as a
CUDA graph beat issuing it on the stream?  cfg2, k = 25, 50 back-to-back
steps each way (events around each batch).

  python tools/graph_probe.py
"""
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

    def step(stream):
        _lib.call("pg_arnoldi_step", s.mat, y.ctypes.data, d, ptr(V), s.ld, j, ptr(z), ptr(t),
                  ptr(acc), ptr(w0), ptr(w1), ptr(ring), host.data_ptr(), s.ws, ev.h, None, None,
                  stream)

    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(5):
            step(st.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(50):
            step(st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        print(f"stream: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us per step")
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            step(st.cuda_stream)
        torch.cuda.synchronize()
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(50):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        print(f"graph:  {e0.elapsed_time(e1) / 50 * 1e3:.1f} us per step")


if __name__ == "__main__":
    main()
