"""Exception classes raised by the backend.

The backend must raise the same classes as the reference simulator
(`/root/reference/pkg/src/qasm2cudaq/errors.py:84-101`; `ArityMismatch` at
`errors.py:44` for `bind`).  When the reference package is importable the names
below *are* the reference's classes, so `except qasm2cudaq.errors.DegenerateNorm`
in caller code keeps working after the switch.  Otherwise an identical hierarchy
is defined here.
"""

from __future__ import annotations

try:  # drop-in: share exception identity with the reference package
    from qasm2cudaq.errors import (  # type: ignore
        ArityMismatch,
        BadPauliString,
        DegenerateNorm,
        DimensionMismatch,
        DynamicCircuit,
        Qasm2CudaqError,
        SimError,
    )
except Exception:  # pragma: no cover - exercised on hosts without the frontend

    class Qasm2CudaqError(Exception):
        """Root of the hierarchy (errors.py:6-7)."""

    class SemaErrorBase(Qasm2CudaqError):
        def __init__(self, message: str, span: tuple = (0, 0)):
            super().__init__(f"semantic error at {span[0]}:{span[1]}: {message}")
            self.message = message
            self.span = span

    class ArityMismatch(SemaErrorBase):
        pass

    class SimError(Qasm2CudaqError):
        pass

    class DynamicCircuit(SimError):
        pass

    class DegenerateNorm(SimError):
        pass

    class BadPauliString(SimError):
        pass

    class DimensionMismatch(SimError):
        pass


class BackendError(SimError):
    """CUDA / NCCL / allocation failure inside the B200 backend (no reference
    equivalent; derives from SimError so reference callers still catch it)."""


class NativeLibraryMissing(BackendError):
    """The sm_100a shared library is absent or failed to load.  There is no CPU
    fallback: every entry point raises this instead."""


__all__ = [
    "Qasm2CudaqError",
    "ArityMismatch",
    "SimError",
    "DynamicCircuit",
    "DegenerateNorm",
    "BadPauliString",
    "DimensionMismatch",
    "BackendError",
    "NativeLibraryMissing",
]
