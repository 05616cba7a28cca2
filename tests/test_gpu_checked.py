"""The checked build (libpgmres_checked.so, -DPG_CHECKS=1): every
asynchronous ring kernel verifies, after each full-barrier wait, that the
slot holds the plane / row block / tile it expects (a stale or early slot
would trap), and the plane ring checks its window copies and reads against
the stage bounds.  compute-sanitizer is closed on this GPU pool, so this is
how the TMA / mbarrier rings are checked: the bitwise parity suites run
against the checked library with tiny tiles, one-plane chunks and 2-stage
rings that wrap on every block.  GPU only."""

import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1907_00072_b200", "libpgmres_checked.so")


def _env(**kw):
    env = dict(os.environ, PG_LIB_PATH=CHECKED, PYTHONPATH=ROOT)
    env.update(kw)
    return env


def test_checked_library_is_checked():
    if not os.path.exists(CHECKED):
        pytest.fail("libpgmres_checked.so missing: run __graft_entry__.build()")
    code = ("from paper_1907_00072_b200 import _lib; l = _lib.load(); "
            "assert l.pg_build_checks() == 1; print('ok')")
    res = subprocess.run([sys.executable, "-c", code], env=_env(), capture_output=True,
                         text=True, cwd=ROOT, timeout=300)
    assert res.returncode == 0 and "ok" in res.stdout, res.stderr[-2000:]


@pytest.mark.parametrize("files,extra", [
    (["tests/test_gpu_planes.py"], {}),
    (["tests/test_gpu_cgs2_tma.py"], {}),
    (["tests/test_gpu_march.py", "tests/test_gpu_parity.py"],
     {"PG_SPMV_PLANES": "0"}),  # the windowed TMA ring on the 27-point stencils
    (["tests/test_gpu_parity.py"], {"PG_CGS2_TMA": "0"}),  # the cp.async tile ring
])
def test_parity_suites_pass_on_the_checked_build(files, extra):
    cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu and not slow",
           "-p", "no:cacheprovider", *files]
    res = subprocess.run(cmd, env=_env(**extra), capture_output=True, text=True, cwd=ROOT,
                         timeout=1800)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
    assert "PG_DCHECK failed" not in res.stdout + res.stderr
