"""B200-native (sm_100a) DISC per-frame mapping hot path (arXiv 2603.03935).

The product is libdisc.so (C ABI: include/disc.h); `disc` is its thin ctypes binding.
"""
from .disc import DiscMap, DiscError, default_config, lib, LIB_PATH  # noqa: F401
