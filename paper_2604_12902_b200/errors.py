"""Error classes of the host surface (same hierarchy as raspvisor/errors.py:6-32
for the classes the batch path raises)."""


class RaspError(Exception):
    """Root of every error this package raises on purpose."""


class CapacityError(RaspError):
    """A program, input vector or batch exceeds the declared resources."""


class NativeError(RaspError):
    """The CUDA extension is missing, failed to load, or returned an error code.

    There is no CPU fallback: the batch path fails loudly instead."""
