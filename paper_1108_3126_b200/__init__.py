"""B200-native lockstep regular-expression matcher (arXiv 1108.3126, §8).

The product is librxg.so: host C++ front end + sm_100a CUDA kernels behind
the C ABI in include/rxg.h. ``rx`` mirrors the reference's rx:: API on top.
"""
from . import rx  # noqa: F401
from ._lib import LIB_PATH, lib  # noqa: F401

__all__ = ["rx", "lib", "LIB_PATH"]
