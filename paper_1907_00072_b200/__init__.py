"""B200-native hot path of polynomial-preconditioned restarted GMRES(m)
(Loe, Thornquist & Boman, arxiv 1907.00072), a drop-in for the reference
``polygmres`` solver API on the path it accelerates:

* ``DeviceMatrixOperator``   <- ``MatrixOperator``      (gmres.py:46-60)
* ``PolynomialWrappedOperator``                         (gmres.py:98-113)
* ``apply_poly`` / ``build_poly`` / ``auto_degree``     (polyprec.py:125-212)
* ``icgs`` / ``OrthoResult``                            (ortho.py:17-70)
* ``solve`` / ``GmresConfig`` / ``GmresResult``         (gmres.py:120-343)
* ``CostCounters`` and the exception types              (counters.py, errors.py)

Every vector operation runs in hand-written sm_100a kernels of libpgmres.so
(include/pgmres.h) called through ctypes; there is no CPU fallback.
"""

from .counters import CostCounters
from .errors import (
    CholeskyFailure,
    ConfigError,
    DeviceError,
    DimensionMismatchError,
    MatrixFormatError,
    NumericalBreakdownError,
    ParameterError,
    PivotError,
    SingularHessenbergError,
)
from .workloads import CsrHost

__version__ = "0.1.0"

_LAZY = {
    "DeviceMatrixOperator": "operators",
    "PolynomialWrappedOperator": "gmres",
    "GmresConfig": "gmres",
    "GmresResult": "gmres",
    "solve": "gmres",
    "hessenberg_lsq": "gmres",
    "cost_report": "gmres",
    "PolyCoefficients": "polyprec",
    "GramSystem": "polyprec",
    "apply_poly": "polyprec",
    "build_poly": "polyprec",
    "auto_degree": "polyprec",
    "build_poly_or_auto": "polyprec",
    "build_poly_arnoldi": "polyprec",
    "dense_cholesky": "polyprec",
    "lambda_p_lambda": "polyprec",
    "RootPlan": "polyprec",
    "root_plan": "polyprec",
    "leja_order": "polyprec",
    "residual_poly_roots": "polyprec",
    "icgs": "ortho",
    "DeviceIluOperator": "operators",
    "Ilu0Factors": "ilu",
    "ilu0_factor": "ilu",
    "ilu0_apply": "ilu",
    "OrthoResult": "ortho",
}


def __getattr__(name):
    # torch-dependent modules load on first use so that `workloads` / errors can
    # be imported by tooling without initialising CUDA.
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = sorted(list(_LAZY) + [
    "CostCounters", "CsrHost", "CholeskyFailure", "DeviceError", "DimensionMismatchError",
    "NumericalBreakdownError", "ParameterError", "SingularHessenbergError", "PivotError",
    "ConfigError", "MatrixFormatError",
])
