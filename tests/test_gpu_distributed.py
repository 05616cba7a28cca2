"""The one-process-per-shard path (DeviceMatrixOperator.distributed +
DistComm) end to end with the real kernels: 2 ranks share the one GPU of the
test box and talk through gloo (halo exchange and the three batched
all-reduces per Arnoldi step are host-staged, so no kernel ever waits on the
other rank).  The result must equal the in-process 2-shard run.  GPU only;
multi-GPU NCCL runs use the same code with the nccl backend (bench.py)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_00072_b200 as pg  # noqa: E402
from paper_1907_00072_b200 import workloads as wl  # noqa: E402
from paper_1907_00072_b200.device import balanced_offsets  # noqa: E402

pytestmark = pytest.mark.gpu

GRID = 24
CONF = wl.CONFIGS[2]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _x0(n):
    x0 = np.zeros(n)
    x0[-GRID * GRID:] = 0.1 * wl.splitmix_uniform(9, GRID * GRID)
    return x0


def _worker(rank, world, port, offs, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        r0, r1 = int(offs[rank]), int(offs[rank + 1])
        blk = wl.convdiff3d_7pt(GRID, rows=(r0, r1))
        c = pg.CostCounters()
        op = pg.DeviceMatrixOperator.distributed(blk, offs, c, device="cuda:0")
        n = GRID ** 3
        b = wl.splitmix_uniform(0, r1 - r0, start=r0)
        v0 = wl.splitmix_uniform(1, r1 - r0, start=r0)
        y_in = wl.splitmix_uniform(5, r1 - r0, start=r0)
        p = pg.PolyCoefficients(3, np.array([1.0, -0.25, 0.05, -0.01]), 1.0)
        pav = pg.apply_poly(p, op, y_in, pg.CostCounters())
        poly, _ = pg.build_poly_or_auto(op, v0, 8, c)
        res = pg.solve(op, b, right_prec=poly, config=pg.GmresConfig(30, 1e-10))
        # x0 nonzero on rank 1's rows only: both ranks must take the global
        # np.any(x0) branch (gmres.py:248), or the collectives would not match
        x0 = _x0(n)[r0:r1]
        c0 = pg.CostCounters()
        op.counters = c0
        rx = pg.solve(op, b, x0=x0, right_prec=poly, config=pg.GmresConfig(30, 1e-10))
        q.put((rank, pav, poly.degree, poly.y, res.iterations, res.cycles, res.final_relres,
               res.x, c.spmvs, c.dots, n, rx.iterations, rx.x, c0.spmvs, c0.dots))
    finally:
        dist.destroy_process_group()


def test_two_rank_distributed_solve_matches_in_process_shards():
    import torch.multiprocessing as mp
    A = wl.convdiff3d_7pt(GRID)
    plane = GRID * GRID
    offs = np.array([0, (GRID // 2) * plane, GRID ** 3], dtype=np.int64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, offs, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=600) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0

    # in-process reference: the same two row blocks as virtual shards
    c = pg.CostCounters()
    op = pg.DeviceMatrixOperator(A, c, shards=2, offsets=offs)
    p3 = pg.PolyCoefficients(3, np.array([1.0, -0.25, 0.05, -0.01]), 1.0)
    pav = pg.apply_poly(p3, op, wl.splitmix_uniform(5, A.nrows), pg.CostCounters())
    poly, _ = pg.build_poly_or_auto(op, wl.make_v0(A.nrows), 8, c)
    res = pg.solve(op, wl.splitmix_uniform(0, A.nrows), right_prec=poly,
                   config=pg.GmresConfig(30, 1e-10))

    # p(A)v through the halo exchange: bit-identical
    assert np.array_equal(np.concatenate([g[1] for g in got]), pav)
    for g in got:
        assert g[2] == poly.degree
        assert g[4] == res.iterations and g[5] == res.cycles
        assert g[6] < 1e-10
        assert g[8] == c.spmvs and g[9] == c.dots
    x = np.concatenate([g[7] for g in got])
    np.testing.assert_allclose(x, res.x, rtol=0, atol=1e-9 * np.abs(res.x).max())
    c0 = pg.CostCounters()
    op.counters = c0
    rx = pg.solve(op, wl.splitmix_uniform(0, A.nrows), x0=_x0(A.nrows), right_prec=poly,
                  config=pg.GmresConfig(30, 1e-10))
    for g in got:
        assert g[11] == rx.iterations and g[13] == c0.spmvs and g[14] == c0.dots
    x = np.concatenate([g[12] for g in got])
    np.testing.assert_allclose(x, rx.x, rtol=0, atol=1e-9 * np.abs(rx.x).max())
