"""B200-native KIOPS hot path (arXiv 1804.05126): C ABI in include/kiops.h, sm_100a
kernels in csrc/, thin ctypes binding in kiops.py."""
from .kiops import Kiops, KiopsEpirk, KiopsError, default_options, lib  # noqa: F401
