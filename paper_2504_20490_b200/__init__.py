"""hshard-b200: B200-native HSPMD resharding executor (Hetu v2, arXiv 2504.20490).

The product is libhshard_b200.so (host planner + sm_100a kernels + C ABI);
this package is the thin Python mirror of the reference hshard API over it.
"""
from . import hshard  # noqa: F401
from ._lib import LIB, LIB_PATH, HshardError  # noqa: F401
