"""B200-native vocabulary-parallel layers (arXiv 2411.05288).

Product path: sm_100a kernels + C ABI in lib/libvpipe_b200.so
(include/vpipe_b200.h), driven from C++ (include/vpipe/vocab_math.hpp) or
from Python (paper_2411_05288_b200.vocab_math).  No CPU fallback.
"""
from ._lib import LIB_PATH, load  # noqa: F401

__all__ = ["LIB_PATH", "load"]
