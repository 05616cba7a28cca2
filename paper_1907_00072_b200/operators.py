"""Device counting operators -- the drop-in boundary for the reference's
operator protocol (gmres.py:46-113): ``.dimension``, ``.counters``, ``.kind``,
``.apply(v)``.

``DeviceMatrixOperator`` replaces ``MatrixOperator(matrix, counters)``
(gmres.py:46-60).  It accepts the reference ``CsrMatrix`` (or this package's
``CsrHost``) and keeps a SELL-C-sigma copy on the GPU(s).  ``apply`` takes and
returns the caller's vector type: numpy in -> numpy out (one H2D/D2H copy, for
code written against the reference), torch CUDA tensor in -> tensor out.
The solver itself never round-trips through the host.
"""

from __future__ import annotations

import numpy as np

from .counters import CostCounters
from .device import Engine
from .errors import ParameterError


class DeviceMatrixOperator:
    """Counting wrapper over a square sparse matrix on the GPU: apply = A @ v.

    ``shards`` > 1 splits the rows into that many *virtual* row-block shards
    (halo copies and fixed-order reductions in-process); ``device`` may be a
    list to place shards on several GPUs of this process.  For one process
    per GPU use :meth:`distributed`."""

    kind = "plain-matrix"

    def __init__(self, matrix, counters: CostCounters | None = None, *, device=None,
                 shards: int = 1, sigma: int | None = None, offsets=None):
        if int(matrix.nrows) != int(matrix.ncols):
            raise ParameterError("operator matrix must be square")
        if getattr(matrix, "row_offset", 0):
            raise ParameterError("a row block needs DeviceMatrixOperator.distributed")
        self.matrix = matrix
        self.dimension = int(matrix.nrows)
        self.counters = counters if counters is not None else CostCounters()
        self.engine = Engine.build(matrix, device=device, parts=shards, sigma=sigma,
                                   offsets=offsets)

    @classmethod
    def distributed(cls, block, offsets, counters: CostCounters | None = None, *, device,
                    group=None, sigma: int | None = None):
        """This rank's row block of an N x N matrix (``block.row_offset`` =
        ``offsets[rank]``, global column indices); one GPU per process."""
        self = cls.__new__(cls)
        self.matrix = block
        self.dimension = int(np.asarray(offsets)[-1])
        self.counters = counters if counters is not None else CostCounters()
        self.engine = Engine.build_distributed(block, offsets, device, group, sigma)
        return self

    def apply(self, v):
        self.counters.spmvs += 1
        e = self.engine
        xs = e.ingest(v)
        ys = e.vecs()
        e.spmv(xs, ys)
        return e.emit(ys, v)

    def close(self):
        self.engine.close()

    @property
    def stats(self):
        return [s.stats for s in self.engine.shards]


class DeviceIluOperator:
    """Left-preconditioned operator ``v -> M^{-1} (A v)`` with ILU(0) factors
    (IluPreconditionedOperator, gmres.py:63-95): one SpMV plus one
    preconditioner application per call, the triangular sweeps tallied in
    ``prec_applies``.  Single GPU (the reference ILU is serial)."""

    kind = "left-preconditioned"

    def __init__(self, matrix, factors, counters: CostCounters | None = None, *, device=None):
        if int(matrix.nrows) != int(matrix.ncols):
            raise ParameterError("operator matrix must be square")
        if int(factors.n) != int(matrix.nrows):
            from .errors import DimensionMismatchError
            raise DimensionMismatchError("factors do not match the matrix")
        self.matrix = matrix
        self.factors = factors
        self.dimension = int(matrix.nrows)
        self.counters = counters if counters is not None else CostCounters()
        self.engine = Engine.build(matrix, device=device)
        self.engine.attach_ilu(factors)

    def apply(self, v):
        self.counters.spmvs += 1
        self.counters.prec_applies += 1
        e = self.engine
        xs = e.ingest(v)
        ys = e.vecs()
        e.spmv(xs, ys)
        return e.emit(ys, v)

    def precondition(self, v):
        """``M^{-1} v`` for preparing the right-hand side (gmres.py:92-95)."""
        self.counters.prec_applies += 1
        e = self.engine
        xs = e.ingest(v)
        ys = e.vecs()
        e.precondition(xs, ys)
        return e.emit(ys, v)

    def close(self):
        self.engine.close()
