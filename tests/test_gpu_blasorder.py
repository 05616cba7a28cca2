"""Reference-order reductions on the device (csrc/blasorder.cu) against their
CPU restatement (oracle/blasorder.c), and the degree decisions they drive
against the reference's recorded ones.  GPU only."""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_00072_b200 as pg  # noqa: E402
from oracle import pgmres_oracle as orc  # noqa: E402
from paper_1907_00072_b200 import _lib, workloads as wl  # noqa: E402
from paper_1907_00072_b200.device import F64, ptr  # noqa: E402

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _dev_dot(x, y, nthreads):
    xd = torch.from_numpy(x).cuda()
    yd = torch.from_numpy(y).cuda()
    out = torch.zeros(1, dtype=F64, device="cuda")
    _lib.call("pg_dot_blas", ptr(xd), ptr(yd), len(x), nthreads, ptr(out),
              torch.cuda.current_stream().cuda_stream)
    return float(out.item())


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 31, 32, 47, 48, 377, 4096, 9999, 10000, 10001,
                               12345, 100003, 1000000])
def test_dot_blas_bitwise(n):
    g = np.random.default_rng(n)
    x = g.uniform(-1, 1, n) * 1e3
    y = g.uniform(-1, 1, n)
    for nt in (1, 8, 12):
        assert _dev_dot(x, y, nt) == (orc.blas_ddot(x, y, nt) if n else 0.0), (n, nt)
    assert _dev_dot(x, x, 8) == (orc.blas_ddot(x, x, 8) if n else 0.0)


def _dev_gram(P, cuts):
    """pg_gram_blas over row blocks [cuts[i], cuts[i+1]) chained by state."""
    n, k = P.shape
    st = torch.cuda.current_stream().cuda_stream
    npairs = k * (k + 1) // 2
    state = None
    for a, b in zip(cuts[:-1], cuts[1:]):
        blk = torch.from_numpy(np.ascontiguousarray(P[a:b].T)).cuda()  # column-major block
        need = _lib.C.c_int64(0)
        _lib.call("pg_gram_blas_scratch", b - a, a, n, k, _lib.C.byref(need))
        scratch = torch.empty(max(need.value, 1), dtype=F64, device="cuda")
        out = torch.empty(2 * npairs, dtype=F64, device="cuda")
        _lib.call("pg_gram_blas", ptr(blk), max(b - a, 1), k, b - a, a, n,
                  ptr(state) if state is not None else None, ptr(out), ptr(scratch), st)
        state = out
    packed = state[npairs:].cpu().numpy()
    G = np.zeros((k, k))
    iu = np.triu_indices(k)
    G[iu] = packed
    G.T[iu] = packed
    return G


@pytest.mark.parametrize("n,k", [(1, 1), (100, 3), (384, 7), (767, 9), (768, 17), (1151, 13),
                                 (5000, 23), (40000, 28), (3001, 64)])
def test_gram_blas_bitwise_and_partition_free(n, k):
    g = np.random.default_rng(n + k)
    P = g.uniform(-1, 1, (n, k)) * 10.0 ** g.uniform(-3, 3, k)
    want = orc.blas_gram(P)
    assert np.array_equal(_dev_gram(P, [0, n]), want)
    # shards cutting through K-blocks (chains handed over in the state)
    for cuts in ([0, n // 2, n], [0, 1, n // 3 + 5, n - 1, n] if n > 10 else [0, n]):
        cuts = sorted(set(cuts))
        assert np.array_equal(_dev_gram(P, cuts), want), cuts


def test_engine_decisions_shard_invariant(golden):
    """The reference-order decision is the same on 1, 2 and 3 virtual shards."""
    _, meta = golden
    A = wl.laplacian2d(64)
    v0 = orc.sm64_uniform(1, 4096)
    degs = []
    for shards in (1, 2, 3):
        op = pg.DeviceMatrixOperator(A, shards=shards)
        p = pg.auto_degree(op, v0, 16, pg.CostCounters())
        degs.append(p.degree)
        from paper_1907_00072_b200.polyprec import _device_power_gram
        G, nrm = _device_power_gram(op, v0, 17, pg.CostCounters())
        Go, nrm_o = orc.gram_full_blas(orc.OracleMatrix.of(A), v0, 17)
        assert nrm == nrm_o and np.array_equal(G, Go)
        op.close()
    assert degs == [meta["auto_lap64"]["degree"]] * 3


def _full_record(c):
    path = os.path.join(GOLDEN, f"cfg{c}_full_reference.json")
    if not os.path.exists(path):
        pytest.skip(f"no full-size reference record for cfg{c}")
    with open(path) as fh:
        return json.load(fh)


@pytest.mark.slow
@pytest.mark.parametrize("c", [2, 4])
def test_full_size_decision_and_solve_parity(c):
    """BASELINE size: the device degree policy takes the reference's decision
    (tests/golden/cfg<c>_full_reference.json, the unmodified reference run in
    the build container), and the device solve from the reference's own
    coefficients y converges within +-2 iterations of the reference's."""
    rec = _full_record(c)
    cfg = wl.CONFIGS[c]
    h = wl.make_matrix(cfg)
    b = wl.make_rhs(cfg, h)
    v0 = wl.make_v0(h.nrows)
    cnt = pg.CostCounters()
    op = pg.DeviceMatrixOperator(h, cnt)
    poly, piv = pg.build_poly_or_auto(op, v0, cfg["degree"], cnt)
    assert piv == rec["build_fail_pivot"]
    assert poly.degree == rec["effective_degree"]
    assert poly.seed_norm == rec["seed_norm"]
    ref_poly = pg.PolyCoefficients(rec["effective_degree"], np.array(rec["y"]), rec["seed_norm"])
    bc = rec["build_counters"]
    base = (bc["spmvs"], bc["dots"], bc["scalar_dots"])
    for p in (ref_poly, poly):
        op.counters = pg.CostCounters()
        res = pg.solve(op, b, right_prec=p, config=pg.GmresConfig(rec["restart_m"], rec["tol"],
                                                                   rec["max_iters"]))
        assert res.converged == rec["converged"]
        assert abs(res.iterations - rec["iterations"]) <= 2, (res.iterations, rec["iterations"])
        assert res.final_relres < rec["tol"]
        if p is ref_poly:
            # the recorded head of the reference's history (its build counted
            # into the same counters): iteration numbers and counters equal,
            # implicit relative residuals to 1e-6
            for got, ref in zip(res.history, rec["history_first"]):
                assert int(got[0]) == int(ref[0])
                assert tuple(int(v) for v in got[2:]) == tuple(int(v) - o
                                                               for v, o in zip(ref[2:], base))
                assert got[1] == pytest.approx(ref[1], rel=1e-6)
    op.close()


def _capped_record(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"no reference record {name}")
    with open(path) as fh:
        return json.load(fh)


@pytest.mark.slow
@pytest.mark.parametrize("c,name", [(5, "cfg5_full_cap100_reference.json"),
                                    (3, "cfg3_full_reference.json")])
def test_full_size_residual_history_parity(c, name):
    """BASELINE size, configs whose full reference solve takes hours on the
    CPU (cfg5: > 3000 iterations) or does not converge inside the bench's cap
    (cfg3: 300 iterations): the unmodified reference was stopped at the
    recorded cap (tests/golden/make_full_records.py) and its whole residual
    history kept.  The device takes the reference's degree decision, and from
    the reference's own coefficients reproduces the history row by row: the
    same iteration numbers and counters, the implicit relative residuals
    (gmres.py:306,314-316) to 1e-8 inside the first cycle and 1e-6 over the
    history (cfg3, which stagnates: 5e-3 after nine restarts), the same
    explicit residual at the cap."""
    rec = _capped_record(name)
    cfg = wl.CONFIGS[c]
    h = wl.make_matrix(cfg)
    b = wl.make_rhs(cfg, h)
    v0 = wl.make_v0(h.nrows)
    cnt = pg.CostCounters()
    op = pg.DeviceMatrixOperator(h, cnt)
    poly, piv = pg.build_poly_or_auto(op, v0, cfg["degree"], cnt)
    assert piv == rec["build_fail_pivot"]
    assert poly.degree == rec["effective_degree"]
    assert poly.seed_norm == rec["seed_norm"]
    ref_poly = pg.PolyCoefficients(rec["effective_degree"], np.array(rec["y"]), rec["seed_norm"])
    cnt = pg.CostCounters()
    op.counters = cnt
    res = pg.solve(op, b, right_prec=ref_poly,
                   config=pg.GmresConfig(rec["restart_m"], rec["tol"], rec["max_iters"]))
    assert res.converged == rec["converged"]
    assert res.iterations == rec["iterations"] and res.cycles == rec["cycles"]
    want = rec["history"]
    assert len(res.history) == len(want)
    worst = first = 0.0
    # (the reference run counted its polynomial build into the same counters)
    bc = rec["build_counters"]
    base = (bc["spmvs"], bc["dots"], bc["scalar_dots"])
    for got, ref in zip(res.history, want):
        assert int(got[0]) == int(ref[0])
        assert tuple(int(v) for v in got[2:]) == tuple(int(v) - o for v, o in zip(ref[2:], base))
        dev = abs(got[1] - ref[1]) / abs(ref[1])
        worst = max(worst, dev)
        if int(got[0]) <= rec["restart_m"]:
            first = max(first, dev)
    # cfg3 stagnates (relres 0.39 after 300 iterations) under a degree-23
    # power-basis polynomial: the first cycle agrees to 3e-10, then every
    # restart's recovery x += p(A)(V y) amplifies the 1e-13 differences of
    # the bases -- 1e-6 after one restart, 1e-3 after nine
    assert first < 1e-8, first
    tol = 5e-3 if c == 3 else 1e-6
    assert worst < tol, worst
    assert res.final_relres == pytest.approx(rec["final_relres"], rel=tol)
    op.close()
