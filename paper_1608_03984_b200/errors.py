"""Exception conventions of the reference, kept so callers can catch the same types.

Mirrors /root/reference/pkg/src/fdroof/errors.py:4-9: every error derives from
`FdroofError`; bad parameters raise `ValidationError`, which is also a
`ValueError`.  The C-ABI wrapper maps return code -1 to `ValidationError` and
-2 (CUDA failure) to `DeviceError`.
"""


class FdroofError(Exception):
    """Base class for all errors raised by this package."""


class ValidationError(FdroofError, ValueError):
    """Invalid parameter values or mismatched wavefield/config shapes."""


class DeviceError(FdroofError, RuntimeError):
    """The CUDA library reported a launch or runtime failure."""


class ExtensionMissingError(FdroofError, ImportError):
    """The compiled sm_100a library is absent; there is no CPU fallback."""
