"""B200-native lensless RF volumetric renderer (arxiv 2605.29097): the data-parallel hot path.

The compute path is librfr.so (csrc/, sm_100a CUDA kernels behind the C ABI in include/librfr.h);
`rfr` is its thin ctypes binding.  See DESIGN.md.
"""
from . import rfr  # noqa: F401

__all__ = ["rfr"]
