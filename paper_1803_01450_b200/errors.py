"""Exception types of the reference (errors.py:4-37 under
/root/reference/pkg/src/mlamr), re-declared so the drop-in shims raise the
same names.  The C-ABI status bits map onto them in :func:`raise_status`."""


class MlamrError(Exception):
    """Base class for all package errors."""


class NotRefinedError(MlamrError):
    """A coarse cell has no finer patch covering it."""


class GeometryError(MlamrError):
    """Patch geometry is inconsistent (box outside available data footprint)."""


class TimeSyncError(MlamrError):
    """Levels are not at the same simulation time when they must be."""


class CflViolationError(MlamrError):
    """Observed wave speed times dt/dx exceeded 1."""


class NumericalAbortError(MlamrError):
    """Non-finite state detected; the run cannot continue."""


def raise_status(status: int, where: str = "") -> None:
    """Map the device status word (include/mlamr_b200.h) to an exception."""
    from ._native import ST_CFL, ST_GEOMETRY, ST_NONFINITE
    if status == 0:
        return
    if status & ST_CFL:
        raise CflViolationError(f"Courant number > 1 {where}")
    if status & ST_GEOMETRY:
        raise GeometryError(f"coarse data footprint incomplete {where}")
    if status & ST_NONFINITE:
        raise NumericalAbortError(f"non-finite state {where}")
    raise MlamrError(f"device status {status:#x} {where}")
