"""Error taxonomy mirrored from the reference (pkg/src/qlrt/errors.py:23-63).

The GPU entry points raise these exact classes (and ``ValueError`` for plain
argument misuse) with the reference's message texts, so callers that catch
``qlrt`` errors keep working.
"""


class QlrtError(Exception):
    """Base class for structured toolkit errors."""


class CorruptDataError(QlrtError):
    """Quantized data violates its own invariants."""


class ContainerError(QlrtError):
    """Container read/write failure (container format is out of scope here)."""


class TrainingDivergedError(QlrtError):
    """Training produced a non-finite loss or gradient norm."""


__all__ = ["QlrtError", "CorruptDataError", "ContainerError", "TrainingDivergedError"]
