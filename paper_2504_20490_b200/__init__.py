"""hshard-b200: B200-native HSPMD resharding executor (Hetu v2, arXiv 2504.20490).

The product is libhshard_b200.so (host planner + sm_100a kernels + C ABI);
this package is the thin Python mirror of the reference hshard API over it.
Importing the package itself loads no native code (so `bench.py --impl
reference` can use the workload tables without mapping the product library);
the first use of `hshard`, `LIB` or any binding module loads
lib/libhshard_b200.so and fails loudly if it is missing.
"""
import importlib

_LAZY = {"LIB": "_lib", "LIB_PATH": "_lib", "HshardError": "_lib"}


def __getattr__(name):
    if name in _LAZY:
        return getattr(importlib.import_module(f"{__name__}.{_LAZY[name]}"), name)
    if name in ("hshard", "executor", "graph", "strategy", "formats", "accounting", "cli"):
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
