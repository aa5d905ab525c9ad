"""Exception types of the reference API (same names, same bases).

imaging.py:19-28, objective.py:40-41, solvers.py:37-42, extrapolation.py:41-54.
"""

from __future__ import annotations


class InvalidSize(ValueError):
    """PSF sizes that are not odd positive integers (imaging.py:19-20)."""


class KernelTooLarge(ValueError):
    """A PSF that does not fit inside the image (imaging.py:23-24)."""


class ShapeMismatch(ValueError):
    """Array shapes that do not match an operator's contract (imaging.py:27-28)."""


class CgNoConvergence(ArithmeticError):
    """Inner CG solve left a residual above the abort threshold (objective.py:40-41)."""


class NonFiniteIterate(ArithmeticError):
    """An iterate (or its cost) became NaN/Inf; carries the trace (solvers.py:37-42)."""

    def __init__(self, message: str, trace=None):
        super().__init__(message)
        self.trace = trace


class ZeroFirstColumn(ArithmeticError):
    """First difference column is numerically zero (extrapolation.py:41-42)."""


class DegenerateSum(ArithmeticError):
    """The normalizing coefficient sum vanished (extrapolation.py:45-46)."""


class RankDeficient(ArithmeticError):
    """Difference matrix rank below the requested order (extrapolation.py:49-50)."""


class NoConvergence(ArithmeticError):
    """The small SVD failed to converge (extrapolation.py:53-54)."""


class NativeFailure(RuntimeError):
    """CUDA / unsupported-configuration failure inside libredve_b200."""


def from_code(code: int, msg: str) -> Exception:
    from . import _native as n

    if code == n.E_VALUE:
        return ValueError(msg)
    if code == n.E_SHAPE:
        return ShapeMismatch(msg)
    if code == n.E_KERNEL:
        return KernelTooLarge(msg)
    if code == n.E_NONFINITE:
        return NonFiniteIterate(msg)
    if code == n.E_CG:
        return CgNoConvergence(msg)
    return NativeFailure(f"[redve_b200 code {code}] {msg}")
