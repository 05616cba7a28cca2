"""Exception types of the device path.  Same names, bases and payloads as the
reference (errors.py:4-70) so callers catch the same things; the C-ABI status
codes of include/pgmres.h map onto them in ``_lib.check``."""


class DimensionMismatchError(ValueError):
    """Operand shapes are incompatible with the operator or vector (errors.py:4)."""


class ParameterError(ValueError):
    """An argument value is outside the accepted range (errors.py:8)."""


class CholeskyFailure(Exception):
    """Gram-matrix Cholesky hit a non-positive pivot; ``pivot`` is 1-based
    (errors.py:32-42).  The auto-degree stop signal."""

    def __init__(self, pivot):
        super().__init__(f"Cholesky pivot {pivot} is not positive")
        self.pivot = pivot


class NumericalBreakdownError(RuntimeError):
    """Non-finite Krylov data at an inner iteration (errors.py:55-62)."""

    def __init__(self, iteration):
        super().__init__(f"non-finite Krylov data at inner iteration {iteration}")
        self.iteration = iteration


class SingularHessenbergError(RuntimeError):
    """The rotated Hessenberg matrix has a zero diagonal entry (errors.py:65)."""


class DeviceError(RuntimeError):
    """A CUDA / library failure reported by libpgmres (no reference analogue:
    the reference has no device).  Never silently replaced by a CPU path."""


class PivotError(ValueError):
    """An ILU pivot is zero, below the floor, or structurally missing; ``row``
    is the 0-based row at which factorisation stopped (errors.py:44-52)."""

    def __init__(self, row, message=None):
        super().__init__(message or f"zero or near-zero pivot in row {row}")
        self.row = row


class ConfigError(ValueError):
    """Experiment configuration is malformed or inconsistent (errors.py:69)."""


class MatrixFormatError(ValueError):
    """A matrix file cannot be used (errors.py:12)."""
