"""B200-native (sm_100a) SsNAL-EN hot path: C-ABI library + thin ctypes binding.

The compute lives in libssnal_en.so (csrc/*.cu); this package only marshals
arguments.  There is no CPU fallback: importing the binding fails loudly if the
library is missing.
"""
from .ssnal_en import Problem, Stats, load_library, SsnalError  # noqa: F401

__all__ = ["Problem", "Stats", "load_library", "SsnalError"]
