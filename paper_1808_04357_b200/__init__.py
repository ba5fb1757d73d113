"""B200-native RedSync Residual Gradient Compression (arXiv 1808.04357) hot path.

``librgc.so`` (csrc/, C ABI in include/rgc.h) holds every kernel; ``rgc`` is the
thin ctypes binding.  Build with ``python -m paper_1808_04357_b200.build``.
"""
from .rgc import *  # noqa: F401,F403
from .rgc import RGC, LayerSpec, lib  # noqa: F401
