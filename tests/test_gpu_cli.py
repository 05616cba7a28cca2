"""The device experiment runner against the reference command line (SURVEY
§8 row f3; cli.py:242-300): five recorded reference runs (tests/golden) are
repeated through ``paper_1907_00072_b200.cli.main``.  Same exit code, same
summary schema and configuration echo, iterations within +-2, same degree,
counters by the reference's laws, history rows in the same format.  GPU only."""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1907_00072_b200 import cli  # noqa: E402

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _num(v):
    # the reference writes relres with repr(), i.e. "np.float64(...)" under
    # numpy 2 (cli.py:224); the device runner keeps that layout
    return float(v[len("np.float64("):-1]) if v.startswith("np.float64(") else float(v)


def _history_rows(text, fmt):
    if fmt == "csv":
        lines = text.strip().split("\n")
        assert lines[0] == "iter,relres,spmvs,dots,scalar_dots"
        return [tuple(_num(v) for v in ln.split(",")) for ln in lines[1:]]
    return [tuple(float(json.loads(ln)[k]) for k in ("iter", "relres", "spmvs", "dots",
                                                      "scalar_dots"))
            for ln in text.strip().split("\n")]


@pytest.mark.parametrize("name", ["cli_cfg1", "cli_ilu", "cli_auto", "cli_mtx", "cli_noprec"])
def test_cli_matches_reference_run(golden, tmp_path, name):
    _, meta = golden
    rec = meta[name]
    argv = [a.replace("<MTX>", os.path.join(GOLDEN, "lap10.mtx")) for a in rec["argv"]]
    out = str(tmp_path / "run")
    code = cli.main(argv + ["-o", out])
    assert code == rec["exit"]
    fmt = "jsonl" if "jsonl" in argv else "csv"
    with open(out + ".summary.json") as fh:
        got = json.load(fh)
    want = rec["summary"]
    assert set(got) == set(want)
    assert set(got["config"]) == set(want["config"])
    for k, v in want["config"].items():
        if k not in ("output", "matrix_file"):
            assert got["config"][k] == v, k
    for k in ("converged", "history_residual_kind", "preconditioned_system", "v0_mode"):
        assert got[k] == want[k], k
    # the degree (also --degree auto): the device takes the reference's own
    # decision (reference-order Gram and seed norm)
    assert got["degree"] == want["degree"]
    assert abs(got["iterations"] - want["iterations"]) <= 2
    if want["converged"]:
        assert got["final_relres"] < got["config"]["tol"]
    else:
        assert got["final_relres"] == pytest.approx(want["final_relres"], rel=1e-6)
    if want["coefficients"] is not None:
        assert got["seed_norm"] == pytest.approx(want["seed_norm"], rel=1e-12)
        assert len(got["coefficients"]) == len(want["coefficients"])
    if (got["iterations"], got["cycles"]) == (want["iterations"], want["cycles"]):
        assert got["counters"] == want["counters"]
        assert got["cost_report"] == want["cost_report"]
    with open(f"{out}.history.{fmt}") as fh:
        rows = _history_rows(fh.read(), fmt)
    ref_rows = _history_rows(rec["history"], fmt)
    assert rows and ("np.float64(" in rec["history"]) == ("np.float64(" in open(
        f"{out}.history.{fmt}").read())
    n = min(len(rows), len(ref_rows))
    assert [r[0] for r in rows[:n]] == [r[0] for r in ref_rows[:n]]
    assert [r[2:] for r in rows[:n]] == [r[2:] for r in ref_rows[:n]]
    rel = np.array([r[1] for r in rows[:n]])
    ref_rel = np.array([r[1] for r in ref_rows[:n]])
    assert np.all(np.abs(np.log10(rel) - np.log10(ref_rel)) < 0.5)
