"""The native distributed path (csrc/dist.cu: NCCL halo + rank-order
reductions issued from C between the step's kernels) on the one GPU of the
test box: a world-1 NCCL communicator exercises every NCCL call the
multi-GPU path makes (grouped send/recv, all-gather, graph capture of both)
-- the halo through a rank sending to itself.  A world-1 distributed solve is
bit-identical to the single-process solve, through the native per-step calls
and the recorded step graphs.  GPU only; each case runs in a fresh process
(one NCCL process group per process)."""

import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(code, env=None):
    full = dict(os.environ, PYTHONPATH=ROOT, MASTER_ADDR="127.0.0.1")
    full.update(env or {})
    res = subprocess.run([sys.executable, "-c", code], env=full, capture_output=True, text=True,
                         cwd=ROOT, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-4000:]
    return res.stdout


HALO = r"""
import ctypes as C, numpy as np, torch
from paper_1907_00072_b200 import _lib
from paper_1907_00072_b200.device import ptr
torch.cuda.set_device(0)
uid = C.create_string_buffer(128)
_lib.call("pg_nccl_unique_id", uid, 128)
h = C.c_void_p()
_lib.call("pg_dist_create", uid, 1, 0, 0, C.byref(h))
n, m = 5000, 777
rng = np.random.default_rng(0)
idx = rng.integers(0, n, m).astype(np.int32)
half = m // 2
# two "peers" (both rank 0): sends of half and m - half entries, received
# into two contiguous ghost ranges
peers = np.array([0, 0], np.int32)
cnt = np.array([half, m - half], np.int64)
offs = np.array([n, n + half], np.int64)
_lib.call("pg_dist_set_halo", h, 2, peers.ctypes.data, cnt.ctypes.data, idx.ctypes.data,
          2, peers.ctypes.data, offs.ctypes.data, cnt.ctypes.data)
x = torch.zeros(n + m, dtype=torch.float64, device="cuda")
x[:n] = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
st = torch.cuda.current_stream().cuda_stream
_lib.call("pg_dist_halo", h, ptr(x), st)
torch.cuda.synchronize()
xh = x.cpu().numpy()
assert np.array_equal(xh[n:], xh[:n][idx]), "halo mismatch"
buf = torch.from_numpy(rng.uniform(-1, 1, 129)).cuda()
ref = buf.clone()
_lib.call("pg_dist_allreduce", h, ptr(buf), 129, st)
torch.cuda.synchronize()
assert torch.equal(buf, ref)
_lib.call("pg_dist_destroy", h)
print("ok")
"""


def test_nccl_self_halo_and_rank_sum():
    assert "ok" in _run(HALO)


SOLVE = r"""
import os, numpy as np, torch, torch.distributed as dist
import paper_1907_00072_b200 as pg
from paper_1907_00072_b200 import workloads as wl
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d", rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
h = wl.aniso27(14)
n = h.nrows
blk = wl.aniso27(14, rows=(0, n))
offs = np.array([0, n])
b = wl.splitmix_uniform(0, n)
v0 = wl.make_v0(n)
out = {}
for kind in ("dist", "solo"):
    c = pg.CostCounters()
    op = (pg.DeviceMatrixOperator.distributed(blk, offs, c, device="cuda:0") if kind == "dist"
          else pg.DeviceMatrixOperator(h, c))
    e = op.engine
    if kind == "dist":
        assert e.comm.distributed and e.native_dist is not None and e.fast_steps
    poly, piv = pg.build_poly_or_auto(op, v0, 8, c)
    runs = []
    for rep in range(3):   # issued steps, then recorded graphs, then replays
        c2 = pg.CostCounters()
        op.counters = c2
        res = pg.solve(op, b, right_prec=poly, config=pg.GmresConfig(12, 1e-10))
        runs.append((res.x, res.history, c2.as_dict(), res.iterations))
    if kind == "dist":
        assert len(e._graphs) > 0
    out[kind] = (poly.degree, poly.y, runs)
    op.close()
d, s = out["dist"], out["solo"]
assert d[0] == s[0] and np.array_equal(d[1], s[1])
for rd, rs in zip(d[2], s[2]):
    assert np.array_equal(rd[0], rs[0]) and rd[1:] == rs[1:], "solve differs"
dist.destroy_process_group()
print("ok", d[2][0][3])
"""


def test_world1_native_distributed_solve_is_bitwise_the_single_gpu_solve():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    assert "ok" in _run(SOLVE % port)
