"""Exception types of the reference (errors.py:4-37 under
/root/reference/pkg/src/mlamr).

When the reference package ``mlamr`` is importable -- the drop-in case of
INTEGRATION.md, where these shims are patched into the reference -- the
classes ARE ``mlamr.errors``' classes, so the reference's own handlers
(``run_simulation``'s abort dump, driver.py:394-401; the CLI's exit codes,
cli.py:126-134) catch what the GPU path raises.  Without it they are
declared here with the same names, bases and constructor signatures.  The
C-ABI status bits map onto them in :func:`raise_status`.
"""

try:  # the reference's own classes (identity, not look-alikes)
    from mlamr.errors import (  # type: ignore[import-not-found]
        CflViolationError,
        ConfigError,
        FrameFormatError,
        GeometryError,
        MlamrError,
        NotRefinedError,
        NumericalAbortError,
        TimeSyncError,
    )
    FROM_REFERENCE = True
except ImportError:
    FROM_REFERENCE = False

    class MlamrError(Exception):
        """Base class for all package errors."""

    class ConfigError(MlamrError):
        """Invalid or unknown configuration input; carries the offending key path."""

        def __init__(self, key: str, message: str):
            self.key = key
            super().__init__(f"{key}: {message}")

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

    class FrameFormatError(MlamrError):
        """Frame file is malformed or has an unsupported format version."""


__all__ = ["MlamrError", "ConfigError", "NotRefinedError", "GeometryError", "TimeSyncError",
           "CflViolationError", "NumericalAbortError", "FrameFormatError", "raise_status",
           "FROM_REFERENCE"]


def raise_status(status: int, where: str = "") -> None:
    """Map the device status word (include/mlamr_b200.h) to an exception."""
    from ._native import ST_BATHY, ST_CFL, ST_GEOMETRY, ST_NONFINITE
    if status == 0:
        return
    if status & ST_BATHY:
        # check_bathymetry_consistency raises a plain AssertionError (coarsen.py:95-100)
        raise AssertionError(f"bathymetry ladder does not telescope {where}")
    if status & ST_CFL:
        raise CflViolationError(f"Courant number > 1 {where}")
    if status & ST_GEOMETRY:
        raise GeometryError(f"coarse data footprint incomplete {where}")
    if status & ST_NONFINITE:
        raise NumericalAbortError(f"non-finite state {where}")
    raise MlamrError(f"device status {status:#x} {where}")
