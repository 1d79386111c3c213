"""Exception types of the reference (errors.py:1-14), restated so the mirror
raises the same classes without importing derivedpq."""


class FormatError(ValueError):
    """Malformed or corrupted container/vector file."""


class InvariantError(RuntimeError):
    """A fitted model violates a structural invariant."""
