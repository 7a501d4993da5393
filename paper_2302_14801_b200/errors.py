"""Error types raised at the drop-in boundary (reference `errors.py:1-6`).

The C ABI returns status codes; `_abi.py` maps them: 1 -> ValueError,
2 -> ConsistencyError, 3 -> RuntimeError (CUDA failure), 4 -> NotImplementedError.
"""


class FormatError(Exception):
    """Malformed or unsupported input file."""


class ConsistencyError(Exception):
    """Internal invariant violated, or the 20-bit random-sampling index limit exceeded."""
