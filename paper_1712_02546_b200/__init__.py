"""B200-native kernel-partitioned convolutional-layer training (arXiv 1712.02546).

The product path: libconvpart.so (CUDA kernels for sm_100a + NCCL, C ABI in
include/convpart.h) and its thin ctypes binding.  Importing this package requires the
built library; there is no CPU fallback.
"""
from . import convpart  # noqa: F401
from .convpart import *  # noqa: F401,F403

__all__ = ["convpart", "net"]
