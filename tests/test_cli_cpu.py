"""Experiment runner on the CPU side: configuration
handling, validation and problem assembly mirror the reference CLI
(cli.py:49-216); the reference's own problems and runs are in tests/golden."""

import json
import os

import numpy as np
import pytest

from paper_1907_00072_b200 import cli, problems, workloads as wl
from paper_1907_00072_b200.errors import ConfigError, MatrixFormatError, ParameterError

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_defaults_and_degree_spellings():
    cfg = cli.parse_config(["--matrix-file", "a.mtx"])
    assert (cfg.degree, cfg.degree_auto, cfg.rhs_mode, cfg.restart_m, cfg.fmt) == \
        (None, False, "axrandom", 50, "csv")
    cfg = cli.parse_config(["--generator", "bidiag1", "--degree", "auto", "--degree-cap", "9"])
    assert cfg.degree is None and cfg.degree_auto and cfg.degree_cap == 9
    assert cli.parse_config(["--generator", "bidiag1", "--degree", "7"]).degree == 7
    with pytest.raises(ConfigError):
        cli.parse_config(["--generator", "bidiag1", "--degree", "seven"])


@pytest.mark.parametrize("argv", [
    [],                                                         # no matrix source
    ["--generator", "bidiag1", "--matrix-file", "a.mtx"],       # two sources
    ["--generator", "bidiag1", "--rhs", "generator"],           # bidiag has no rhs
    ["--generator", "bidiag1", "--rhs", "file"],                # file without path
    ["--generator", "bidiag1", "--tol", "1.5"],
    ["--generator", "bidiag1", "-m", "0"],
    ["--generator", "bidiag1", "--max-iters", "0"],
    ["--generator", "bidiag1", "--degree", "-1"],
    ["--generator", "bidiag1", "--degree-cap", "0"],
])
def test_validation_rejects(argv):
    with pytest.raises(ConfigError):
        cli.parse_config(argv)


def test_config_file_merge(tmp_path):
    path = tmp_path / "c.json"
    path.write_text(json.dumps({"generator": "laplacian2d", "grid_n": 9, "tol": 1e-6,
                                "degree": "auto"}))
    cfg = cli.parse_config(["--config", str(path), "--tol", "1e-9"])
    assert cfg.grid_n == 9 and cfg.tol == 1e-9 and cfg.degree_auto
    path.write_text(json.dumps({"generator": "laplacian2d", "bogus": 1}))
    with pytest.raises(ConfigError):
        cli.parse_config(["--config", str(path)])
    path.write_text("[1, 2]")
    with pytest.raises(ConfigError):
        cli.parse_config(["--config", str(path)])
    with pytest.raises(ConfigError):
        cli.parse_config(["--config", str(tmp_path / "missing.json")])


def test_problems_match_reference(golden):
    a, _ = golden
    C, rhs = problems.gen_convdiff2d(48, 0.05)
    assert np.array_equal(C.row_ptr, a["convdiff48_row_ptr"])
    assert np.array_equal(C.col_idx, a["convdiff48_col_idx"])
    assert np.array_equal(C.values, a["convdiff48_values"])
    assert rhs.shape == (C.nrows,) and np.all(rhs[(np.arange(C.nrows) % 48) != 47] == 0.0)
    M = problems.read_matrix_market(os.path.join(GOLDEN, "lap10.mtx"))
    L = wl.laplacian2d(10)
    assert np.array_equal(M.row_ptr, L.row_ptr) and np.array_equal(M.col_idx, L.col_idx)
    assert np.array_equal(M.values, L.values)
    B = problems.bidiag2()
    assert B.nnz == 9999 and B.values[0] == 0.1 and B.values[1] == 0.2
    with pytest.raises(ParameterError):
        problems.gen_convdiff2d(1, 0.1)


@pytest.mark.parametrize("text,err", [
    (b"", problems.MatrixMarketParseError),
    (b"%%MatrixMarket matrix array real general\n2 2\n", problems.UnsupportedFormatError),
    (b"%%MatrixMarket matrix coordinate complex general\n", problems.UnsupportedFormatError),
    (b"%%MatrixMarket matrix coordinate real general\n2 2\n", problems.MatrixMarketParseError),
    (b"%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
     problems.MatrixMarketParseError),
    (b"%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
     problems.MatrixMarketParseError),
])
def test_matrix_market_errors(text, err):
    with pytest.raises(err):
        problems.read_matrix_market(text)
    assert issubclass(err, MatrixFormatError)


def test_error_exit_codes(tmp_path, capsys):
    bad = tmp_path / "bad.mtx"
    bad.write_text("not a matrix market file\n")
    assert cli.main(["--matrix-file", str(bad), "-o", str(tmp_path / "x")]) == 1
    assert "polygmres: error:" in capsys.readouterr().err
    assert cli.main(["--matrix-file", str(tmp_path / "missing.mtx")]) == 1
    assert cli.main(["--generator", "bidiag1", "--tol", "2"]) == 1
