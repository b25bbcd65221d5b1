"""B200-native (sm_100a) hot path of the Realistic Sparse Fourier Transform (arXiv 1610.01050).

The product is librsft.so (C ABI: include/rsft.h); `rsft` is its thin ctypes binding.
"""
from .rsft import Plan, RsftError, bitmap_to_bool, lib  # noqa: F401
