"""B200-native BBC1 activation codec (BloomBee hot path, arXiv 2604.21072).

The compute path is the sm_100a library ``libbbcodec.so`` behind the C ABI in
include/bbcodec.h; this package mirrors the reference's codec API on top of it.
"""
from . import codec  # noqa: F401
from ._lib import LIB_PATH, kernel_launches, load  # noqa: F401

__all__ = ["codec", "load", "kernel_launches", "LIB_PATH"]
