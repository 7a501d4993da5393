"""Error types raised at the drop-in boundary (reference `errors.py:1-6`).

The C ABI returns status codes; `_abi.py` maps them: 1 -> ValueError,
2 -> ConsistencyError, 3 -> RuntimeError (CUDA failure), 4 -> NotImplementedError.

When the reference package (`lodforge`) is importable, its exception classes ARE these
classes, so code written against the reference (`except lodforge.errors.ConsistencyError`)
catches what the drop-in raises.  Without it, look-alike classes with the same names and
bases are defined here.
"""
try:  # pragma: no cover - depends on the caller's environment
    from lodforge.errors import ConsistencyError, FormatError  # type: ignore  # noqa: F401
    REFERENCE_CLASSES = True
except Exception:  # lodforge absent (e.g. on the GPU box)
    REFERENCE_CLASSES = False

    class FormatError(Exception):
        """Malformed or unsupported input file."""

    class ConsistencyError(Exception):
        """Internal invariant violated, or the 20-bit random-sampling index limit exceeded."""
