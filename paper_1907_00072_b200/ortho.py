"""Two-pass classical Gram-Schmidt on the device (ortho.py:14-70 of the
reference).

The solver calls ``Engine.cgs2`` directly on its device-resident basis; this
module provides the reference-shaped standalone entry point
``icgs(basis, w, counters) -> OrthoResult`` for callers (and parity tests) that
hand over arrays.  Same accounting (dots += 3, scalar_dots += 2j+1,
vector_updates += 2j (+1)), same breakdown rule
(``new_norm <= 1e-14 * hypot(|coeffs|, new_norm)``, ortho.py:64-68).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .counters import CostCounters
from .device import KMAX, MMAX, F64, _pad, ptr, require_cuda
from .errors import DimensionMismatchError

BREAKDOWN_RTOL = 1e-14


@dataclass
class OrthoResult:
    coeffs: np.ndarray
    new_norm: float
    vector: object
    breakdown: bool


_WS: dict = {}


def workspace(dev_ord: int):
    """Per-device reduction workspace for standalone calls."""
    ws = _WS.get(dev_ord)
    if ws is None:
        h = _lib.C.c_void_p()
        _lib.call("pg_workspace_create", dev_ord, _lib.C.byref(h))
        ws = _WS[dev_ord] = h
    return ws


def breakdown_test(coeffs: np.ndarray, new_norm: float) -> bool:
    w_norm = math.hypot(float(np.linalg.norm(coeffs)), new_norm)
    return new_norm <= BREAKDOWN_RTOL * w_norm


def icgs(basis, w, counters: CostCounters) -> OrthoResult:
    """Orthogonalize ``w`` against the orthonormal columns of ``basis`` (n x j)
    with the three device phases; returns the reference ``OrthoResult``
    (``vector`` in the caller's array type)."""
    require_cuda()
    as_torch = isinstance(w, torch.Tensor)
    B = basis if isinstance(basis, torch.Tensor) else torch.from_numpy(np.asarray(basis, dtype=np.float64))
    W = w if as_torch else torch.from_numpy(np.asarray(w, dtype=np.float64))
    if B.dim() != 2:
        raise DimensionMismatchError("basis must be a 2-d array of columns")
    n, j = B.shape
    if tuple(W.shape) != (n,):
        raise DimensionMismatchError("w length does not match the basis")
    if j > MMAX - 1:
        raise DimensionMismatchError(f"basis wider than {MMAX - 1} columns")
    dev = W.device if (as_torch and W.is_cuda) else torch.device("cuda", torch.cuda.current_device())
    dev_ord = dev.index if dev.index is not None else torch.cuda.current_device()
    ld = _pad(n)
    V = torch.zeros((j + 1, ld), dtype=F64, device=dev)
    if j:
        V[:j, :n].copy_(B.to(dev, F64).T)
    z = torch.zeros(ld, dtype=F64, device=dev)
    z[:n].copy_(W.to(dev, F64))
    scal = torch.zeros(2 * j + 1, dtype=F64, device=dev)
    c1, c2, nsq = scal[:j], scal[j:2 * j], scal[2 * j:]
    ws = workspace(dev_ord)
    st = torch.cuda.current_stream(dev).cuda_stream
    _lib.call("pg_set_device", dev_ord)
    if j > KMAX:  # wider than one tile: the four-pass tiled form
        w1 = torch.zeros(ld, dtype=F64, device=dev)
        _lib.call("pg_cgs2_wide", ptr(V), ld, j, ptr(z), n, ptr(c1), ptr(c2), ptr(nsq), ptr(w1),
                  ptr(V[j]), ws, st)
    else:
        if j:
            _lib.call("pg_cgs2_phase1", ptr(V), ld, j, ptr(z), n, ptr(c1), ws, st)
            _lib.call("pg_cgs2_phase2", ptr(V), ld, j, ptr(z), n, ptr(c1), ptr(c2), ws, st)
        _lib.call("pg_cgs2_phase3", ptr(V), ld, j, ptr(z), n, ptr(c1), ptr(c2), ptr(V[j]),
                  ptr(nsq), ws, st)
    host = scal.cpu().numpy()
    coeffs = host[:j] + host[j:2 * j]
    new_norm = float(np.sqrt(host[2 * j]))
    counters.dots += 3
    counters.scalar_dots += 2 * j + 1
    counters.vector_updates += 2 * j
    brk = breakdown_test(coeffs, new_norm)
    if not brk:
        counters.vector_updates += 1
        _lib.call("pg_normalize", ptr(V[j]), ptr(nsq), n, ptr(V[j]), st)
    vec = V[j, :n]
    vec = vec.clone() if as_torch else vec.cpu().numpy()
    return OrthoResult(coeffs, new_norm, vec, brk)
