"""B200-native RO-MAP multi-object NeRF training path (arXiv 2304.05735).

The product is libromap.so (paper_2304_05735_b200/csrc, sm_100a CUDA behind the
C ABI in include/romap.h); ``romap`` is its thin ctypes binding.
"""
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libromap.so")
