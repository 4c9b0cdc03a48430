"""B200-native LeMix placement step (arXiv 2507.21276).

The product is liblemix.so (C ABI in include/lemix.h, CUDA kernels in csrc/);
`lemix` is the thin ctypes binding.  Nothing in this package imports the
CPU oracle (oracle/), which is test infrastructure only.
"""
from . import lemix  # noqa: F401

__all__ = ["lemix"]
