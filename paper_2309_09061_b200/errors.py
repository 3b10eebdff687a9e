"""Error types of the drop-in surface (reference: h2mul/errors.py:4-13).

The C-ABI returns status codes that map onto these: 1 -> InvalidInputError,
2 -> StructureError, 3 -> CudaError (a RuntimeError for CUDA failures).
"""


class InvalidInputError(ValueError):
    """An argument violates a documented precondition (h2mul/errors.py:4-5)."""


class StructureError(RuntimeError):
    """An internal structural invariant is violated (h2mul/errors.py:8-13)."""


class CudaError(RuntimeError):
    """A CUDA launch or allocation failed inside the native library."""
