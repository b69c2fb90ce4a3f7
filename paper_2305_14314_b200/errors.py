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
    """Container read/write failure (pkg/docs/FORMAT.md failure taxonomy)."""


class BadMagicError(ContainerError):
    """The first four bytes are not ``QLRT``."""


class UnsupportedVersionError(ContainerError):
    """The version field is not 1."""


class TruncatedFileError(ContainerError):
    """A section is cut short, or bytes trail the checksum."""


class ChecksumMismatchError(ContainerError):
    """The stored crc32 differs from the recomputed one."""


class TrainingDivergedError(QlrtError):
    """Training produced a non-finite loss or gradient norm."""


__all__ = ["QlrtError", "CorruptDataError", "ContainerError", "BadMagicError", "UnsupportedVersionError",
           "TruncatedFileError", "ChecksumMismatchError", "TrainingDivergedError"]
