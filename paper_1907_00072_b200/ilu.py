"""ILU(0) left preconditioning on the device (reference
ilu.py:1-114 and IluPreconditionedOperator, gmres.py:63-95).

``ilu0_factor`` runs the reference's IKJ elimination restricted to the
pattern natively on the host (``pg_ilu0_factor``: same operation order, so
the factors are bit-identical); ``ilu0_apply`` and the operator's
applications run the two triangular solves on the GPU as sync-free sweeps
(``pg_ilu_apply``, csrc/ilu.cu).  The sweeps sum each row in stored column
order; the reference's short dot products go through OpenBLAS ``ddot``,
whose order is the library's, so applications agree to rounding (tests bound
the difference), not bitwise.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import DimensionMismatchError, ParameterError, PivotError


@dataclass(frozen=True)
class Ilu0Factors:
    """Combined L\\U on the matrix's pattern (ilu.py:19-35): entries left of
    the diagonal are L (unit diagonal implied), the rest U; ``diag_ptr[i]``
    locates U's diagonal in row i."""

    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    diag_ptr: np.ndarray

    @property
    def nnz(self):
        return len(self.values)


def ilu0_factor(matrix, diag_shift: float = 0.0) -> Ilu0Factors:
    """ILU(0) of a square matrix whose pattern holds every diagonal entry
    (ilu.py:38-95).  A missing diagonal or a pivot at or below
    ``eps * max|diag|`` raises :class:`PivotError` with the 0-based row."""
    if int(matrix.nrows) != int(matrix.ncols):
        raise ParameterError("ILU(0) requires a square matrix")
    n = int(matrix.nrows)
    rp = np.ascontiguousarray(matrix.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(matrix.col_idx, dtype=np.int64)
    va = np.ascontiguousarray(matrix.values, dtype=np.float64)
    out = np.empty_like(va)
    dp = np.empty(n, dtype=np.int64)
    row = C.c_int64(-1)
    kind = C.c_int(0)
    _lib.call("pg_ilu0_factor", n, rp.ctypes.data, ci.ctypes.data, va.ctypes.data,
              float(diag_shift), out.ctypes.data, dp.ctypes.data, C.byref(row), C.byref(kind))
    if kind.value == 1:
        raise PivotError(row.value, f"row {row.value} has no structural diagonal entry")
    if kind.value == 2:
        raise PivotError(row.value)
    return Ilu0Factors(n, rp, ci, out, dp)


_DEVICE_FACTORS: dict = {}


def _device_engine(factors: Ilu0Factors):
    """A single-shard engine holding these factors (cached per factors
    object) for stand-alone ``ilu0_apply`` calls."""
    key = id(factors)
    hit = _DEVICE_FACTORS.get(key)
    if hit is not None and hit[0] is factors:
        return hit[1]
    from .device import Engine
    from .workloads import CsrHost

    n = factors.n
    ident = CsrHost(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64),
                    np.ones(n))
    e = Engine.build(ident)
    e.attach_ilu(factors)
    _DEVICE_FACTORS[key] = (factors, e)
    return e


def ilu0_apply(factors: Ilu0Factors, v):
    """``M^{-1} v``: forward sweep with unit L, backward sweep with U
    (ilu.py:98-114), on the GPU.  numpy in -> numpy out, CUDA tensor in ->
    tensor out."""
    if isinstance(v, torch.Tensor):
        shape = tuple(v.shape)
    else:
        v = np.asarray(v, dtype=np.float64)
        shape = v.shape
    if shape != (factors.n,):
        raise DimensionMismatchError("vector length does not match the factors")
    e = _device_engine(factors)
    vs = e.ingest(v)
    outs = e.vecs()
    e.precondition(vs, outs)
    return e.emit(outs, v)
