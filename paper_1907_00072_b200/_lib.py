"""ctypes binding of libpgmres.so (include/pgmres.h).

The library is loaded on first use and a missing or unloadable library is a
hard error: there is no CPU fallback anywhere in this package.
"""

from __future__ import annotations

import ctypes as C
import os
import re

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpgmres.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "pgmres.h")

PG_OK = 0
PG_ERR_DIMENSION = -1
PG_ERR_PARAMETER = -2
PG_ERR_CUDA = -3
PG_ERR_ALLOC = -4
PG_SLICE = 32
PG_KMAX = 64
PG_MMAX = 256
PG_PASS_FIRST = 1
PG_PASS_WRITE_W = 2
PG_ROOT_REAL = 0
PG_ROOT_PAIR_A = 1
PG_ROOT_PAIR_B = 2
PG_ROOT_RESID = 4

_i64 = C.c_int64
_i32 = C.c_int
_p = C.c_void_p
_d = C.c_double
_pi64 = C.POINTER(C.c_int64)

_SIGNATURES = {
    "pg_version": ([], C.c_int),
    "pg_build_checks": ([], C.c_int),
    "pg_last_error": ([C.c_char_p, C.c_size_t], C.c_int),
    "pg_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "pg_set_device": ([_i32], C.c_int),
    "pg_sell_size": ([_i64, _p, _i32, _pi64, _pi64], C.c_int),
    "pg_sell_fill": ([_i64, _i64, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p], C.c_int),
    "pg_matrix_create": ([_i32, _i64, _i64, _p, _p, _p, _i32, C.POINTER(_p)], C.c_int),
    "pg_matrix_destroy": ([_p], C.c_int),
    "pg_matrix_stats": ([_p, _pi64], C.c_int),
    "pg_plane_plan": ([_p, _pi64], C.c_int),
    "pg_workspace_create": ([_i32, C.POINTER(_p)], C.c_int),
    "pg_workspace_destroy": ([_p], C.c_int),
    "pg_spmv": ([_p, _p, _p, _p], C.c_int),
    "pg_poly_pass": ([_p, _p, _p, _p, _p, _p, _d, _d, _i32, _p], C.c_int),
    "pg_residual": ([_p, _p, _p, _p, _p, _p, _p], C.c_int),
    "pg_root_pass": ([_p, _p, _p, _p, _p, _p, _d, _d, _d, _i32, _p], C.c_int),
    "pg_cgs2_phase1": ([_p, _i64, _i32, _p, _i64, _p, _p, _p], C.c_int),
    "pg_cgs2_phase2": ([_p, _i64, _i32, _p, _i64, _p, _p, _p, _p], C.c_int),
    "pg_cgs2_phase3": ([_p, _i64, _i32, _p, _i64, _p, _p, _p, _p, _p, _p], C.c_int),
    "pg_normalize": ([_p, _p, _i64, _p, _p], C.c_int),
    "pg_gram": ([_p, _i64, _i32, _i64, _p, _p, _p], C.c_int),
    "pg_gemv": ([_p, _i64, _i32, _p, _i64, _p, _p], C.c_int),
    "pg_gemv_acc": ([_p, _i64, _i32, _p, _i64, _p, _d, _p, _p], C.c_int),
    "pg_cgs2_wide": ([_p, _i64, _i32, _p, _i64, _p, _p, _p, _p, _p, _p, _p], C.c_int),
    "pg_dot_blas": ([_p, _p, _i64, _i32, _p, _p], C.c_int),
    "pg_gram_blas_scratch": ([_i64, _i64, _i64, _i32, _pi64], C.c_int),
    "pg_gram_blas": ([_p, _i64, _i32, _i64, _i64, _i64, _p, _p, _p, _p], C.c_int),
    "pg_dot": ([_p, _p, _i64, _p, _p, _p], C.c_int),
    "pg_scale_add": ([_p, _d, _p, _i64, _p, _p], C.c_int),
    "pg_gather": ([_p, _p, _i64, _p, _p], C.c_int),
    "pg_host_cholesky_solve": ([_i32, _p, _i32, _p, _p, C.POINTER(C.c_int)], C.c_int),
    "pg_host_degree_select": ([_i32, _p, _i32, _p, _p, C.POINTER(C.c_int)], C.c_int),
    "pg_host_backsolve": ([_i32, _p, _i32, _p, _p, C.POINTER(C.c_int)], C.c_int),
    "pg_event_create": ([_i32, C.POINTER(_p)], C.c_int),
    "pg_event_destroy": ([_p], C.c_int),
    "pg_event_record": ([_p, _p], C.c_int),
    "pg_event_wait": ([_p], C.c_int),
    "pg_event_elapsed": ([_p, _p, C.POINTER(C.c_float)], C.c_int),
    "pg_chain_fused": ([_p, C.POINTER(_i32)], C.c_int),
    "pg_row_patterns": ([_i64, _p, _p, _p, _i32, _p, C.POINTER(_i32), C.POINTER(_i32),
                         C.POINTER(_i32), _p], C.c_int),
    "pg_power_sequence": ([_p, _p, _i64, _i32, _p], C.c_int),
    "pg_wrapped_apply": ([_p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p], C.c_int),
    "pg_poly_chain": ([_p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p], C.c_int),
    "pg_arnoldi_step": ([_p, _p, _i32, _p, _i64, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p,
                         _p, _i32, _p, _p, _p], C.c_int),
    "pg_step_graph_create": ([_p, _p, _i32, _p, _i64, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p,
                              _p, _p, _i32, _p, _p, C.POINTER(_p)], C.c_int),
    "pg_graph_launch": ([_p, _p], C.c_int),
    "pg_graph_destroy": ([_p], C.c_int),
    "pg_nccl_unique_id": ([_p, C.c_size_t], C.c_int),
    "pg_dist_create": ([_p, _i32, _i32, _i32, C.POINTER(_p)], C.c_int),
    "pg_dist_set_halo": ([_p, _i32, _p, _p, _p, _i32, _p, _p, _p], C.c_int),
    "pg_dist_destroy": ([_p], C.c_int),
    "pg_dist_halo": ([_p, _p, _p], C.c_int),
    "pg_dist_allreduce": ([_p, _p, _i32, _p], C.c_int),
    "pg_arnoldi_step_dist": ([_p, _p, _i32, _p, _i64, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p,
                              _p, _p, _i32, _p, _p, _p, _p], C.c_int),
    "pg_step_graph_create_dist": ([_p, _p, _i32, _p, _i64, _i32, _p, _p, _p, _p, _p, _p, _p, _p,
                                   _p, _p, _p, _i32, _p, _p, _p, C.POINTER(_p)], C.c_int),
    "pg_poly_chain_dist": ([_p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p], C.c_int),
    "pg_power_sequence_dist": ([_p, _p, _i64, _i32, _p, _p], C.c_int),
    "pg_ilu0_factor": ([_i64, _p, _p, _p, _d, _p, _p, _pi64, C.POINTER(C.c_int)], C.c_int),
    "pg_ilu_create": ([_i32, _i64, _p, _p, _p, _p, C.POINTER(_p)], C.c_int),
    "pg_ilu_destroy": ([_p], C.c_int),
    "pg_ilu_apply": ([_p, _p, _p, _p, _p], C.c_int),
}

_lib = None


def header_symbols(path: str = HEADER_PATH):
    """Names of every PG_API entry point declared in include/pgmres.h."""
    text = open(path).read()
    return sorted(set(re.findall(r"PG_API\s+[\w\s\*]+?\b(pg_\w+)\s*\(", text)))


def load():
    """Load (once) and return the library; raises if it is missing."""
    global _lib, LIB_PATH
    if _lib is not None:
        return _lib
    # PG_LIB_PATH: load an alternative build (kernel-variant A/B experiments)
    LIB_PATH = os.environ.get("PG_LIB_PATH", LIB_PATH)
    if not os.path.exists(LIB_PATH):
        raise errors.DeviceError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (the device path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def last_error() -> str:
    buf = C.create_string_buffer(1024)
    load().pg_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(code: int, what: str = ""):
    if code == PG_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if code == PG_ERR_DIMENSION:
        raise errors.DimensionMismatchError(msg)
    if code == PG_ERR_PARAMETER:
        raise errors.ParameterError(msg)
    raise errors.DeviceError(msg)


#: entry points that launch exactly one libpgmres kernel per call
LAUNCHING = frozenset({
    "pg_spmv", "pg_poly_pass", "pg_root_pass", "pg_residual", "pg_cgs2_phase1", "pg_cgs2_phase2",
    "pg_cgs2_phase3", "pg_normalize", "pg_gram", "pg_gemv", "pg_dot", "pg_scale_add",
    "pg_gather", "pg_ilu_apply", "pg_dot_blas", "pg_gemv_acc",
})
#: per-entry-point launch tally (bench.py reports it as gpu_launches)
LAUNCH_COUNT: dict = {}


def launches() -> int:
    return sum(LAUNCH_COUNT.values())


def add_launches(name: str, n: int):
    """Tally kernels launched inside one multi-kernel entry point
    (pg_arnoldi_step, pg_poly_chain)."""
    LAUNCH_COUNT[name] = LAUNCH_COUNT.get(name, 0) + int(n)


_FN: dict = {}


def host_cholesky(G, rhs):
    """(y, failed_pivot) of the order-len(rhs) Gram system (native)."""
    import numpy as np
    G = np.ascontiguousarray(G, dtype=np.float64)
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    o = len(rhs)
    y = np.zeros(o)
    piv = C.c_int(0)
    call("pg_host_cholesky_solve", o, G.ctypes.data, G.shape[1], rhs.ctypes.data, y.ctypes.data,
         C.byref(piv))
    return y, piv.value


def host_degree_select(G, rhs, cap):
    """(degree, y) chosen like auto_degree from the cap+1 blocks; degree -1 if none."""
    import numpy as np
    G = np.ascontiguousarray(G, dtype=np.float64)
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    y = np.zeros(cap + 1)
    d = C.c_int(-1)
    call("pg_host_degree_select", cap, G.ctypes.data, G.shape[1], rhs.ctypes.data,
         y.ctypes.data, C.byref(d))
    return d.value, (y[:d.value + 1].copy() if d.value >= 0 else None)


def host_backsolve(R, g, j):
    """y = R[:j,:j]^{-1} g[:j]; returns (y, zero_col) (zero_col = -1 if none)."""
    import numpy as np
    R = np.ascontiguousarray(R, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    y = np.zeros(max(j, 1))
    zc = C.c_int(-1)
    call("pg_host_backsolve", j, R.ctypes.data, R.shape[1], g.ctypes.data, y.ctypes.data,
         C.byref(zc))
    return y[:j], zc.value


def call(name: str, *args):
    fn = _FN.get(name)
    if fn is None:
        fn = _FN[name] = getattr(load(), name)
    code = fn(*args)
    if code:
        check(code, name)
    if name in LAUNCHING:
        LAUNCH_COUNT[name] = LAUNCH_COUNT.get(name, 0) + 1
