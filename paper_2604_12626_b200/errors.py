"""Exception types. Same names and bases as the reference (splatnav/errors.py:4-41), so callers
that catch the reference's errors keep working after switching to this package."""


class SplatNavError(Exception):
    """Base class for all package errors."""


class ValidationError(SplatNavError, ValueError):
    """Input data violates a container invariant (non-finite values, bad weights...)."""


class ConsistencyError(SplatNavError, ValueError):
    """Cross-array mismatch inside a bundle (frame counts, joint counts...)."""


class ContractViolation(SplatNavError, ValueError):
    """An operation was called outside its documented precondition."""


class NativeError(SplatNavError, RuntimeError):
    """The CUDA extension reported an error (message comes from sn_last_error())."""


class PlyParseError(SplatNavError, ValueError):
    """Malformed PLY header or payload; message names the offending part."""


class UnsupportedLayoutError(SplatNavError, ValueError):
    """PLY field layout does not match any supported SH degree."""


class SchemaError(SplatNavError, ValueError):
    """Config or manifest JSON is missing required keys or has wrong types."""
