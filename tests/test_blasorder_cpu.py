"""CPU pins of the reference-order reductions behind the degree decision
(oracle/blasorder.c; device twin csrc/blasorder.cu).

* ddot: bit-identical to numpy's x.dot(y) recorded on the build host
  (tests/golden/blas_order.npz, make_blas_golden.py).
* syrk Gram: bit-identical on the full-tile entries (every entry for k <= 11),
  within a few ulp elsewhere (the kernel's M-tail unroll, see blasorder.c).
* With both, the reference's Cholesky loop takes every degree decision the
  unmodified reference recorded (tests/golden/golden.json): build_poly
  pass/fail and failing pivot, auto_degree's choice, the policy's effective
  degree -- including the cases the exact-arithmetic decision gets wrong.
"""

import json
import os
import sys

import numpy as np
import pytest

from oracle import pgmres_oracle as orc
from paper_1907_00072_b200 import workloads as wl

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_blas_golden as mb  # noqa: E402


@pytest.fixture(scope="module")
def blas_golden():
    return np.load(os.path.join(HERE, "golden", "blas_order.npz"))


def test_ddot_order_is_numpys(blas_golden):
    for (s, n), want in zip(blas_golden["dot_cases"], blas_golden["dot_values"]):
        x, y = mb.dot_inputs(int(s), int(n))
        assert orc.blas_ddot(x, y, 8) == want, (s, n)


def test_syrk_gram_order(blas_golden):
    for s, n, k in blas_golden["gram_cases"]:
        G = blas_golden[f"gram_{s}"]
        E = orc.blas_gram(mb.gram_input(int(s), int(n), int(k)))
        assert np.array_equal(E, E.T)
        if k <= 11:
            assert np.array_equal(E, G), (n, k)
        else:
            assert np.mean(E == G) > 0.4
            assert np.max(np.abs(E - G) / np.abs(G)) < 1e-12


def _op(h):
    return orc.OracleMatrix.of(h, orc.Tally())


def _decide(h, v0, deg):
    Gfull, _ = orc.gram_full_blas(_op(h), v0, deg + 1)
    return orc.degree_decision_blas(Gfull, deg)


def test_cfg1_build_and_auto_decisions(golden):
    _, meta = golden
    A = wl.laplacian2d(64)
    v0 = wl.make_v0(A.nrows, 0)
    Gfull, nrm = orc.gram_full_blas(_op(A), v0, 17)
    assert nrm == meta["cfg1_build"]["seed_norm"]  # np.linalg.norm, bitwise
    for d in (12, 13, 14):
        piv, _ = orc.degree_decision_blas(Gfull[:d + 2, :d + 2], d)
        rec = meta[f"cfg1_build{d}"]
        assert piv == (0 if rec == "ok" else rec), d
    assert orc.degree_decision_blas(Gfull[:18, :18], 16)[1] == meta["auto_lap64"]["degree"]


def test_bidiag2_auto_decisions(golden):
    _, meta = golden
    B = wl.CsrHost(*_bidiag2())
    # auto_degree(bidiag2, random_seed_vector(5000, 1), cap 20)
    assert _decide(B, wl.splitmix_uniform(1, 5000), 20)[1] == meta["auto_bidiag2"]["degree"]
    # the reference CLI's --degree auto --degree-cap 20 --seed 3 (v0 seed 4)
    assert _decide(B, wl.splitmix_uniform(4, 5000), 20)[1] == meta["cli_auto"]["summary"]["degree"]


def _bidiag2():
    from paper_1907_00072_b200 import problems
    m = problems.bidiag2()
    return m.nrows, m.ncols, m.row_ptr, m.col_idx, m.values


@pytest.mark.parametrize("c, kw", [(2, dict(grid=16)), (3, dict(size=4000)), (4, dict(grid=12)),
                                   (5, dict(grid=48))])
def test_small_config_policy_decisions(golden, c, kw):
    _, meta = golden
    cfg = wl.CONFIGS[c]
    h = wl.make_matrix(cfg, **kw)
    piv, auto = _decide(h, wl.make_v0(h.nrows, 0), cfg["degree"])
    rec = meta[f"small{c}"]
    eff = cfg["degree"] if piv == 0 else auto
    assert eff == rec["effective_degree"]
    assert (piv or None) == meta.get(f"small{c}_build_fail_pivot")


@pytest.mark.parametrize("c", [2])
def test_full_size_policy_decision(c):
    with open(os.path.join(HERE, "golden", f"cfg{c}_full_reference.json")) as fh:
        rec = json.load(fh)
    cfg = wl.CONFIGS[c]
    h = wl.make_matrix(cfg)
    piv, auto = _decide(h, wl.make_v0(h.nrows, 0), cfg["degree"])
    assert piv == rec["build_fail_pivot"]
    assert auto == rec["effective_degree"]
