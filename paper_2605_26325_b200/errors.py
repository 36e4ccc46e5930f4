"""Exception types of the drop-in (pkg/src/dare/errors.py:1-33).

When the reference package `dare` is importable, its classes are re-exported
so that callers catching `dare.errors.InvalidArgumentError` keep working
after switching to this package.  Otherwise an identical hierarchy is defined.
"""
from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from dare.errors import (  # type: ignore
        DareError,
        InvalidArgumentError,
        OutOfBoundsError,
        ProtocolError,
        SweepFormatError,
        SynchronizationError,
        UndefinedMetricError,
        VolumeFormatError,
    )
except Exception:  # the reference is not installed: stand-alone hierarchy

    class DareError(Exception):
        """Root of every error this package raises."""

    class InvalidArgumentError(DareError, ValueError):
        """A documented precondition on an argument does not hold."""

    class OutOfBoundsError(DareError, ValueError):
        """A sample or index lies outside the volume grid."""

    class SynchronizationError(DareError, RuntimeError):
        """The image and pose streams do not overlap in time."""

    class SweepFormatError(DareError, ValueError):
        """A sweep recording on disk is malformed."""

    class VolumeFormatError(DareError, ValueError):
        """A volume file is malformed or has the wrong magic/version."""

    class UndefinedMetricError(DareError, ValueError):
        """A similarity metric is undefined for its inputs."""

    class ProtocolError(DareError, ValueError):
        """A wire message cannot be decoded."""


__all__ = [
    "DareError", "InvalidArgumentError", "OutOfBoundsError", "SynchronizationError",
    "SweepFormatError", "VolumeFormatError", "UndefinedMetricError", "ProtocolError",
]
