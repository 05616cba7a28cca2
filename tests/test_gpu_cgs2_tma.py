"""CGS2 phases 1-2 (csrc/ortho.cu tma_tile_kernel) and 3 (tma_rows_kernel)
staged by TMA tensor maps (default) against a numpy fp64 restatement of the phase arithmetic
(ortho.py:53-60: c1 = V^T z, w1 = z - V c1, c2 = V^T w1, w2 = w1 - V c2),
at ragged n (partial and single tiles, rows past n zero-filled by the TMA
unit), basis widths across the 8-column box boundaries and the chunk / tile
cross-overs, both tile heights, and against the cp.async tile kernel
(PG_CGS2_TMA=0) in a separate process.  GPU only."""

import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1907_00072_b200 import _lib  # noqa: E402
from paper_1907_00072_b200.device import _pad, ptr  # noqa: E402
from paper_1907_00072_b200.ortho import workspace  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SIZES = [1, 37, 255, 257, 1000, 4097, 70001]
WIDTHS = [6, 8, 9, 13, 16, 17, 25, 33, 40, 64]


def _phases(n, k, seed):
    """Device phases 1-3 on a random basis; returns (c1, c2, w2, nsq) and the
    host inputs."""
    gen = np.random.default_rng(seed)
    ld = _pad(n)
    Vh = gen.standard_normal((k, n))
    zh = gen.uniform(-1, 1, n)
    V = torch.zeros((k, ld), dtype=torch.float64, device="cuda")
    V[:, :n] = torch.from_numpy(Vh)
    z = torch.zeros(ld, dtype=torch.float64, device="cuda")
    z[:n] = torch.from_numpy(zh)
    sc = torch.zeros(200, dtype=torch.float64, device="cuda")
    c1, c2, nsq = sc[:64], sc[64:128], sc[128:129]
    w2 = torch.zeros(ld, dtype=torch.float64, device="cuda")
    ws = workspace(torch.cuda.current_device())
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("pg_cgs2_phase1", ptr(V), ld, k, ptr(z), n, ptr(c1), ws, st)
    _lib.call("pg_cgs2_phase2", ptr(V), ld, k, ptr(z), n, ptr(c1), ptr(c2), ws, st)
    _lib.call("pg_cgs2_phase3", ptr(V), ld, k, ptr(z), n, ptr(c1), ptr(c2), ptr(w2), ptr(nsq),
              ws, st)
    torch.cuda.synchronize()
    return (c1[:k].cpu().numpy(), c2[:k].cpu().numpy(), w2[:n].cpu().numpy(),
            float(nsq.item())), Vh.T, zh


def _check(n, k, seed):
    (c1, c2, w2, nsq), V, z = _phases(n, k, seed)
    r1 = V.T @ z
    w1 = z - V @ r1
    r2 = V.T @ w1
    r3 = w1 - V @ r2
    scale = max(1.0, np.abs(V).sum(axis=0).max() * np.abs(z).max())
    assert np.max(np.abs(c1 - r1)) <= 1e-12 * scale
    assert np.max(np.abs(c2 - r2)) <= 1e-11 * scale
    assert np.max(np.abs(w2 - r3)) <= 1e-11 * scale
    assert nsq == pytest.approx(float(r3 @ r3), rel=1e-10, abs=1e-12)


@pytest.mark.parametrize("n", SIZES)
def test_tma_phases_match_numpy(n):
    for k in WIDTHS:
        _check(n, k, 1000 * n + k)


def _isolated(env):
    code = f"""
import sys; sys.path.insert(0, 'tests')
import numpy as np
import test_gpu_cgs2_tma as t
out = []
for n in (257, 4097, 70001):
    for k in (9, 25, 40):
        t._check(n, k, 7 * n + k)
        (c1, c2, w2, nsq), V, z = t._phases(n, k, 7 * n + k)
        out.append(np.concatenate([c1, c2, w2, [nsq]]))
np.save(sys.argv[1], np.concatenate(out))
print("ok")
"""
    path = f"/tmp/pg_cgs2_{abs(hash(tuple(sorted(env.items()))))}.npy"
    full = dict(os.environ, PYTHONPATH=ROOT)
    full.update(env)
    res = subprocess.run([sys.executable, "-c", code, path], env=full, capture_output=True,
                         text=True, cwd=ROOT, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
    return np.load(path)


def test_tma_and_cpasync_tile_kernels_agree():
    """Both staging paths and both tile heights give the same phases up to
    the summation order of the partial sums."""
    ref = _isolated({"PG_CGS2_TMA": "0"})
    for env in ({"PG_CGS2_TMA": "1"}, {"PG_CGS2_TMA": "1", "PG_TILE_ROWS": "128"},
                {"PG_CGS2_TMA": "1", "PG_TILE_ROWS": "256"}):
        got = _isolated(env)
        assert got.shape == ref.shape
        assert np.max(np.abs(got - ref)) <= 1e-10 * max(1.0, np.max(np.abs(ref)))


def test_phase3_tma_rows_is_bitwise_the_row_kernel():
    """Phase 3 staged by tensor maps (tma_rows_kernel, default) computes each
    row's w1 and w2 with the row-streaming kernel's operations in its order:
    w2 is bit-identical to PG_CGS2_TMA3=0 (ragged n, k across the 8-column
    boxes); ||w2||^2 agrees to the summation order of the partial sums."""
    ref = _isolated({"PG_CGS2_TMA3": "0"})
    for env in ({"PG_CGS2_TMA3": "1"}, {"PG_CGS2_TMA3": "1", "PG_TILE_CTAS_P3": "1"}):
        got = _isolated(env)
        assert got.shape == ref.shape
        pos = 0
        for n in (257, 4097, 70001):
            for k in (9, 25, 40):
                m = 2 * k + n
                assert np.array_equal(got[pos:pos + m], ref[pos:pos + m]), (n, k)
                assert got[pos + m] == pytest.approx(ref[pos + m], rel=1e-13)
                pos += m + 1
        assert pos == ref.size
