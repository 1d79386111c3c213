"""B200-native derived two-pass PQ search (arXiv 1905.06900).

Drop-in GPU twins of the reference `derivedpq` search API:

    from paper_1905_06900_b200 import FlatIndex, IVFIndex

Both keep the reference's constructor, fit (delegated to the reference
quantizer / trainer), search signature, argument checks, exceptions and
result conventions; every search runs in libdpq.so on the GPU (no CPU
fallback: a missing library or device raises).
"""

from .errors import FormatError, InvariantError  # noqa: F401
from .flat import ArrayQuantizer, FlatIndex  # noqa: F401
from .ivf import IVFIndex  # noqa: F401

__all__ = ["FlatIndex", "IVFIndex", "ArrayQuantizer", "FormatError", "InvariantError"]
