"""CPU-only tests of the boundary and the host logic: the C-ABI library loads
and exports every symbol include/pgmres.h declares (no compute calls), the
host-built SELL-C-sigma layout reproduces the reference row order, the
row-block partition / halo plan reconstructs the global SpMV, the
torch.distributed halo exchange + all-reduce work across 2 gloo ranks, and the
host-side solver pieces mirror the reference."""

import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch

from oracle import pgmres_oracle as orc
from paper_1907_00072_b200 import _lib, workloads as wl
from paper_1907_00072_b200 import device as dv


# ---------------------------------------------------------------------------
# the C-ABI library
# ---------------------------------------------------------------------------
def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = _lib.header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing
    assert set(_lib._SIGNATURES) == set(syms)  # every declared entry point is bound
    assert lib.pg_version() == 1


def test_error_codes_and_last_error():
    lib = _lib.load()
    rp = np.array([0, 1, 2], dtype=np.int64)
    nsl, pad = C.c_int64(), C.c_int64()
    assert lib.pg_sell_size(2, rp.ctypes.data, 1, C.byref(nsl), C.byref(pad)) == 0
    bad = np.array([1, 1, 2], dtype=np.int64)  # row_ptr[0] != 0
    assert lib.pg_sell_size(2, bad.ctypes.data, 1, None, None) == _lib.PG_ERR_PARAMETER
    assert "row_ptr[0]" in _lib.last_error()
    with pytest.raises(_lib.errors.ParameterError):
        _lib.call("pg_sell_size", 2, bad.ctypes.data, 1, None, None)


def _sell_host(h, sigma):
    lib = _lib.load()
    nsl, pad = C.c_int64(), C.c_int64()
    _lib.call("pg_sell_size", h.nrows, h.row_ptr.ctypes.data, sigma, C.byref(nsl), C.byref(pad))
    ns, p = nsl.value, pad.value
    sp = np.zeros(ns + 1, np.int64)
    sw = np.zeros(ns, np.int32)
    rl = np.zeros(ns * 32, np.int32)
    pm = np.zeros(ns * 32, np.int32)
    col = np.zeros(max(p, 1), np.int32)
    val = np.zeros(max(p, 1), np.float64)
    cols = np.ascontiguousarray(h.col_idx, np.int64)
    vals = np.ascontiguousarray(h.values, np.float64)
    _lib.call("pg_sell_fill", h.nrows, h.ncols, h.row_ptr.ctypes.data, cols.ctypes.data,
              vals.ctypes.data, sigma, sp.ctypes.data, sw.ctypes.data, rl.ctypes.data,
              pm.ctypes.data, col.ctypes.data, val.ctypes.data)
    assert lib is not None
    return sp, sw, rl, pm, col, val


def _sell_spmv(sell, nrows, x):
    """Row-sequential SpMV over the SELL layout, in numpy (column j of all
    lanes at once, so each lane's sum runs in stored order)."""
    sp, sw, rl, pm, col, val = sell
    y = np.zeros(nrows)
    for s in range(len(sw)):
        lanes = np.arange(32)
        acc = np.zeros(32)
        for j in range(sw[s]):
            pos = sp[s] + j * 32 + lanes
            live = j < rl[s * 32 + lanes]
            acc = np.where(live, acc + val[pos] * x[col[pos]], acc)
        rows = pm[s * 32 + lanes]
        ok = rows >= 0
        y[rows[ok]] = acc[ok]
    return y


@pytest.mark.parametrize("sigma", [1, 64])
def test_sell_layout_reproduces_reference_order(golden, sigma):
    a, _ = golden
    R = wl.CsrHost(1000, 1000, a["rand1k_row_ptr"], a["rand1k_col_idx"], a["rand1k_values"])
    sell = _sell_host(R, sigma)
    assert np.array_equal(_sell_spmv(sell, 1000, a["rand1k_x"]), a["rand1k_y"])
    L = wl.CsrHost(4096, 4096, a["lap64_row_ptr"], a["lap64_col_idx"], a["lap64_values"])
    x = orc.sm64_uniform(0, 4096)
    assert np.array_equal(_sell_spmv(_sell_host(L, sigma), 4096, x), a["cfg1_b"])
    if sigma > 1:  # sorting makes slices uniform: padding shrinks
        assert _sell_host(R, sigma)[0][-1] <= _sell_host(R, 1)[0][-1]


def test_sell_rejects_bad_columns():
    # column 5 of a 2 x 2 matrix: the C-ABI reports ParameterError, as CsrMatrix
    # does (sparse.py:78-79)
    with pytest.raises(_lib.errors.ParameterError):
        _sell_host(wl.CsrHost(2, 2, [0, 1, 2], [0, 5], [1.0, 1.0]), 1)


# ---------------------------------------------------------------------------
# row-block partition and halo plan (host logic of device.Engine)
# ---------------------------------------------------------------------------
def _emulate_sharded_spmv(h, parts, x):
    offs = dv.balanced_offsets(h.row_ptr, parts)
    y = np.zeros(h.nrows)
    for p in range(parts):
        r0, r1 = int(offs[p]), int(offs[p + 1])
        q0, q1 = int(h.row_ptr[r0]), int(h.row_ptr[r1])
        cols = h.col_idx[q0:q1]
        ghosts = dv.ghost_columns(cols, r0, r1)
        recv = dv.plan_recv(ghosts, offs, r1 - r0)
        local_cols = dv.localize_columns(cols, r0, r1, ghosts)
        xe = np.zeros(r1 - r0 + len(ghosts))
        xe[:r1 - r0] = x[r0:r1]
        for q, (off, cnt) in recv.items():
            assert offs[q] <= ghosts[off - (r1 - r0)] < offs[q + 1]  # owned by q
            xe[off:off + cnt] = x[ghosts[off - (r1 - r0): off - (r1 - r0) + cnt]]
        blk = orc.OracleMatrix(r1 - r0, len(xe), h.row_ptr[r0:r1 + 1] - q0, local_cols,
                               h.values[q0:q1])
        y[r0:r1] = blk.matvec(xe)
    return y, offs


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_partition_halo_plan_reconstructs_spmv(parts):
    for h in (wl.convdiff3d_7pt(12), wl.random_lognormal(3000, seed=4), wl.aniso27(8)):
        x = wl.splitmix_uniform(3, h.nrows)
        y, offs = _emulate_sharded_spmv(h, parts, x)
        assert np.array_equal(y, orc.OracleMatrix.of(h).matvec(x))  # bitwise: order kept
        assert offs[0] == 0 and offs[-1] == h.nrows and np.all(np.diff(offs) >= 0)


def test_row_range_generators_concatenate():
    for make in (lambda rows=None: wl.convdiff3d_7pt(10, rows=rows),
                 lambda rows=None: wl.aniso27(7, rows=rows),
                 lambda rows=None: wl.convdiff2d_9pt(33, rows=rows),
                 lambda rows=None: wl.random_lognormal(70000, seed=3, rows=rows)):
        full = make()
        cut = full.nrows // 3
        a, b = make(rows=(0, cut)), make(rows=(cut, full.nrows))
        assert b.row_offset == cut
        assert np.array_equal(np.concatenate([a.col_idx, b.col_idx]), full.col_idx)
        assert np.array_equal(np.concatenate([a.values, b.values]), full.values)
    assert wl.aniso27(200, rows=(0, 0)).nrows == 0
    g = 20
    assert wl.aniso27(g).nnz == (3 * g - 2) ** 3


def test_choose_sigma():
    assert dv.choose_sigma(wl.convdiff3d_7pt(16).row_ptr) == 1
    assert dv.choose_sigma(wl.random_lognormal(20000, seed=1).row_ptr) > 1


# ---------------------------------------------------------------------------
# distributed halo exchange + all-reduce over 2 gloo ranks
# ---------------------------------------------------------------------------
class _CpuShard:
    """Test double of device.Shard for the gloo ranks: same plan / send-list
    fields, numpy SpMV on the local block instead of a CUDA kernel."""

    def __init__(self, h_block, offs, rank):
        self.r0, self.r1 = int(offs[rank]), int(offs[rank + 1])
        self.n = self.r1 - self.r0
        ghosts = dv.ghost_columns(h_block.col_idx, self.r0, self.r1)
        self.plan = dv.HaloPlan(ghosts, dv.plan_recv(ghosts, offs, self.n))
        self.n_ext = self.n + len(ghosts)
        self.local = orc.OracleMatrix(self.n, self.n_ext, h_block.row_ptr,
                                      dv.localize_columns(h_block.col_idx, self.r0, self.r1,
                                                          ghosts), h_block.values)

    def set_send(self, q, idx):
        self.plan.send[q] = torch.from_numpy(np.asarray(idx, dtype=np.int64))

    def packed_send(self, x, q):
        return x.index_select(0, self.plan.send[q]).contiguous()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, cfg_name, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h = wl.convdiff3d_7pt(10) if cfg_name == "7pt" else wl.random_lognormal(4000, seed=9)
        offs = dv.balanced_offsets(h.row_ptr, world)
        r0, r1 = int(offs[rank]), int(offs[rank + 1])
        blk = wl.convdiff3d_7pt(10, rows=(r0, r1)) if cfg_name == "7pt" else \
            wl.random_lognormal(4000, seed=9, rows=(r0, r1))
        s = _CpuShard(blk, offs, rank)
        comm = dv.DistComm([s])
        dv.exchange_send_lists([s], comm)
        x = wl.splitmix_uniform(5, h.nrows)
        xe = torch.zeros(s.n_ext, dtype=torch.float64)
        xe[:s.n] = torch.from_numpy(x[r0:r1])
        comm.halo([xe])
        y_local = s.local.matvec(xe.numpy())
        want = orc.OracleMatrix.of(h).matvec(x)[r0:r1]
        ok_spmv = bool(np.array_equal(y_local, want))
        part = torch.tensor([float(np.dot(y_local, y_local)), float(rank + 1)],
                            dtype=torch.float64)
        comm.allreduce([part])
        full = orc.OracleMatrix.of(h).matvec(x)
        ok_red = abs(part[0].item() - float(np.dot(full, full))) <= 1e-9 * float(np.dot(full, full))
        ok_red = ok_red and part[1].item() == world * (world + 1) / 2
        q.put((rank, ok_spmv, ok_red))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg_name", ["7pt", "random"])
def test_gloo_world2_halo_and_allreduce(cfg_name):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, cfg_name, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    got = sorted(q.get(timeout=5) for _ in range(2))
    assert got == [(0, True, True), (1, True, True)]


# ---------------------------------------------------------------------------
# host-side solver pieces
# ---------------------------------------------------------------------------
def test_host_pieces_mirror_reference():
    import paper_1907_00072_b200 as pg
    y, res = pg.hessenberg_lsq(np.array([[2.0], [0.0]]), 4.0)
    assert y == pytest.approx([2.0]) and res == pytest.approx(0.0, abs=1e-15)
    y, res = pg.hessenberg_lsq(np.array([[1.0], [1.0]]), 1.0)
    assert y == pytest.approx([0.5]) and res == pytest.approx(1 / np.sqrt(2.0))
    assert pg.dense_cholesky(pg.GramSystem(np.array([[5.0, 9.0], [9.0, 17.0]]),
                                           np.array([3.0, 5.0]))) == pytest.approx([1.5, -0.5])
    with pytest.raises(pg.CholeskyFailure) as err:
        pg.dense_cholesky(pg.GramSystem(np.ones((2, 2)), np.ones(2)))
    assert err.value.pivot == 2
    for bad in (dict(restart_m=0), dict(tol=1.5), dict(tol=0.0), dict(max_iters=0)):
        with pytest.raises(pg.ParameterError):
            pg.GmresConfig(**bad)
    with pytest.raises(pg.ParameterError):
        pg.PolyCoefficients(1, np.array([1.0]), 1.0)
    with pytest.raises(pg.ParameterError):
        pg.PolyCoefficients(0, np.array([np.nan]), 1.0)
    rep = pg.cost_report(pg.CostCounters(spmvs=5, dots=3), 4, 50)
    assert rep["spmvs_per_iteration"] == 5 and rep["ca_grouping_spmvs_per_sync"] == 200
    p = pg.PolyCoefficients(1, np.array([1.5, -0.5]), 1.0)
    assert pg.lambda_p_lambda(p, [1.0, 2.0]) == pytest.approx([1.0, 1.0])


def test_native_host_routines(golden):
    """pg_host_cholesky_solve / _degree_select / _backsolve (compensated
    inner products): known answers, and the exact-arithmetic pass/fail
    decision on the cfg1 power-basis Gram."""
    y, piv = _lib.host_cholesky(np.array([[5.0, 9.0], [9.0, 17.0]]), np.array([3.0, 5.0]))
    assert piv == 0 and y == pytest.approx([1.5, -0.5], abs=1e-12)
    assert _lib.host_cholesky(np.ones((2, 2)), np.ones(2))[1] == 2
    y, piv = _lib.host_cholesky(np.array([[4.0]]), np.array([2.0]))
    assert y == pytest.approx([0.5])
    a, _ = golden
    A = orc.OracleMatrix(4096, 4096, a["lap64_row_ptr"], a["lap64_col_idx"], a["lap64_values"])
    v0 = orc.sm64_uniform(1, 4096)
    P = orc.power_columns(A, v0 / np.linalg.norm(v0), 17)
    G = orc.gram_exact(P)
    Gs, r = np.ascontiguousarray(G[1:, 1:]), np.ascontiguousarray(G[1:, 0])
    for o in (6, 11, 12, 14):
        assert _lib.host_cholesky(Gs[:o, :o], r[:o])[1] == orc.chol_pivot_exact(Gs[:o, :o])
    d, y = _lib.host_degree_select(Gs, r, 16)
    assert d == orc.auto_deg_exact(G, 16)
    # well inside the passing range the native y agrees with the numpy loop
    y6, _ = _lib.host_cholesky(Gs[:6, :6], r[:6])
    np.testing.assert_allclose(y6, orc.chol_solve(Gs[:6, :6], r[:6]), rtol=1e-9)
    R = np.triu(np.arange(1.0, 31.0).reshape(6, 5) % 7 + 1.0)
    g = np.linspace(1, 2, 6)
    yb, zc = _lib.host_backsolve(R, g, 5)
    assert zc == -1 and np.allclose(R[:5, :5] @ yb, g[:5])
    R[2, 2] = 0.0
    assert _lib.host_backsolve(R, g, 5)[1] == 2


def test_device_path_refuses_without_gpu():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1907_00072_b200 as pg
    with pytest.raises(pg.DeviceError):
        pg.DeviceMatrixOperator(wl.laplacian2d(4))


def _simulate_root_plan(plan, A, v):
    """numpy stand-in for the pg_root_pass epilogues (include/pgmres.h) driven
    by the product's host RootPlan -- checks the plan logic without a GPU."""
    prod, t, y = v.copy(), None, np.zeros_like(v)
    for mode, c1, c2, c3, keep in plan.steps:
        if mode == _lib.PG_ROOT_REAL:
            ax = A.matvec(prod)
            pn = prod - c1 * ax
            y = y + c1 * prod + c3 * pn
            prod = pn
        elif mode == _lib.PG_ROOT_PAIR_A:
            t = c2 * prod - A.matvec(prod)
            y = y + c1 * t
        else:
            prod = prod - c1 * A.matvec(t)
            y = y + c3 * prod
    return y


@pytest.mark.parametrize("key", ["cfg1_sweep_1_y", "cfg1_sweep_4_y", "cfg1_sweep_8_y", "cfg1_y10",
                                 "cfg1_sweep_12_y"])
def test_root_plan_matches_monomial(golden, key):
    """Root-product plan: d passes, conjugate pairs adjacent;
    the running sum is within 1e-12 of the extended-precision p(A)v, and
    within the north_star's 1e-10 of the reference's fp64 monomial wherever
    the monomial itself is that accurate (deg <= 10; at deg 12 the monomial
    is 2.9e-10 off the extended value while the root form is 1.7e-13)."""
    import paper_1907_00072_b200 as pg
    a, _ = golden
    A = orc.OracleMatrix(4096, 4096, a["lap64_row_ptr"], a["lap64_col_idx"], a["lap64_values"])
    y = a[key]
    p = pg.PolyCoefficients(len(y) - 1, y, 1.0)
    plan = pg.root_plan(p)
    assert len(plan.steps) == p.degree
    r = plan.roots
    for i in range(len(r)):  # each complex root is followed by its conjugate
        if r[i].imag > 0:
            assert r[i + 1] == np.conj(r[i])
    pi = np.polynomial.polynomial.polyval(r, np.concatenate([[1.0], -y]))
    assert np.max(np.abs(pi)) < 1e-8
    b = a["cfg1_b"]
    ref = orc.poly_eval(y, A, b, orc.Tally())
    ext = orc.poly_eval_extended(y, A, b)
    got = _simulate_root_plan(plan, A, b)
    rel = lambda u, w: np.linalg.norm(u - w) / np.linalg.norm(w)
    assert rel(got, ext) < 1e-12
    assert rel(got, ext) <= rel(ref, ext) + 1e-15
    if p.degree <= 10:
        assert rel(got, ref) < 1e-10


def test_leja_order_pairs_and_start():
    import paper_1907_00072_b200 as pg
    r = np.array([1.0, 3 + 1j, 3 - 1j, -0.5, 10.0])
    o = pg.leja_order(r.astype(complex))
    assert o[0] == 10.0 and sorted(o, key=lambda z: (z.real, z.imag)) == \
        sorted(r.astype(complex), key=lambda z: (z.real, z.imag))
    i = list(o).index(3 + 1j)
    assert o[i + 1] == 3 - 1j
    with pytest.raises(pg.ParameterError):
        pg.leja_order(np.array([1 + 1j, 2.0]))
    p0 = pg.root_plan(pg.PolyCoefficients(0, np.array([2.0]), 1.0))
    assert p0.steps == () and p0.y0 == 2.0
    with pytest.raises(pg.ParameterError):
        pg.apply_poly(p0, None, np.zeros(1), pg.CostCounters(), form="chebyshev")


# ---------------------------------------------------------------------------
# row-pattern planning (the grouping behind the row-pattern and offset-pattern
# matrix formats; host-only entry point, no GPU)
# ---------------------------------------------------------------------------
def _row_patterns(h, with_values=True):
    rp = np.ascontiguousarray(h.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(h.col_idx, dtype=np.int64)
    va = np.ascontiguousarray(h.values, dtype=np.float64)
    ids = np.zeros(h.nrows, dtype=np.uint8)
    masks = np.zeros(256, dtype=np.uint32)
    npat, master, mlen = C.c_int(0), C.c_int(0), C.c_int(0)
    _lib.call("pg_row_patterns", h.nrows, rp.ctypes.data, ci.ctypes.data, va.ctypes.data,
              int(with_values), ids.ctypes.data, C.byref(npat), C.byref(master), C.byref(mlen),
              masks.ctypes.data)
    return npat.value, master.value, mlen.value, ids, masks[:max(npat.value, 0)]


def _expected_mask(h, row, master_row):
    """Bits of the master row's (offset, value) entries a row uses, in order
    (bit 31 when it is not an ordered subsequence)."""
    def seq(r):
        a, b = int(h.row_ptr[r]), int(h.row_ptr[r + 1])
        return [(int(h.col_idx[q]) - r, float(h.values[q])) for q in range(a, b)]
    ms, bits, q = seq(master_row), 0, 0
    for e in seq(row):
        while q < len(ms) and ms[q] != e:
            q += 1
        if q == len(ms):
            return 1 << 31
        bits |= 1 << q
        q += 1
    return bits


def test_row_patterns_laplacian_boundary_rows_are_master_subsequences():
    """2-D 5-point Laplacian: 9 row patterns (4 corners, 4 edges, interior);
    the interior row is the master and every boundary row is an ordered
    subsequence of it (Dirichlet rows drop neighbours) -- the property the
    unrolled master path of the pattern kernels relies on."""
    g = 8
    h = wl.laplacian2d(g)
    npat, master, mlen, ids, masks = _row_patterns(h)
    assert npat == 9 and mlen == 5
    interior = g + 1  # (1, 1)
    assert ids[interior] == master
    for r in range(h.nrows):
        assert masks[ids[r]] == _expected_mask(h, r, interior)
    assert masks[ids[0]] == 0b11100  # corner (0, 0): offsets 0, +1, +g
    assert all(m >> 31 == 0 for m in masks)


def test_row_patterns_values_and_offsets():
    """A boundary diagonal that differs from the interior one breaks the
    (offset, value) subsequence but not the offset-only one (the offset-pattern
    format, for variable-coefficient stencils)."""
    h = wl.laplacian2d(8)
    vals = np.array(h.values, dtype=np.float64)
    rp, ci = np.asarray(h.row_ptr), np.asarray(h.col_idx)
    for r in range(h.nrows):
        if rp[r + 1] - rp[r] < 5:
            vals[rp[r]:rp[r + 1]][ci[rp[r]:rp[r + 1]] == r] = 5.0
    m = wl.CsrHost(h.nrows, h.ncols, rp, ci, vals)
    npat, master, mlen, ids, masks = _row_patterns(m)
    assert npat == 9 and mlen == 5
    assert sum(1 for x in masks if x >> 31) == 8  # every boundary pattern
    npat_o, _, mlen_o, _, masks_o = _row_patterns(m, with_values=False)
    assert npat_o == 9 and mlen_o == 5 and all(x >> 31 == 0 for x in masks_o)


def test_row_patterns_stencils_and_random():
    """3-D 7- and 27-point stencils: 27 patterns (low / interior / high per
    dimension), masters of 7 and 27 entries; a random sparse matrix has more
    than 256 distinct rows (no plan)."""
    for h, ml in ((wl.convdiff3d_7pt(6), 7), (wl.aniso27(6), 27)):
        npat, _, mlen, _, masks = _row_patterns(h)
        assert (npat, mlen) == (27, ml)
        assert all(x >> 31 == 0 for x in masks)
    r = wl.random_lognormal(2000, seed=3)
    assert _row_patterns(r)[0] == -1
    assert _row_patterns(r, with_values=False)[0] == -1
