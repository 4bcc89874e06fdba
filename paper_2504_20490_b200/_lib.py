"""ctypes loader for libhshard_b200.so (the C ABI in include/hshard_c.h).

The library is built in-tree (paper_2504_20490_b200/lib) by
``__graft_entry__.build()``.  There is no fallback: importing the package
without the built library raises immediately.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_int, c_int64, c_size_t, c_uint32, c_ulonglong, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libhshard_b200.so")
if os.environ.get("HS_LIB_VARIANT"):  # exploration builds only (tools/stage_sweep.sh)
    LIB_PATH = os.path.join(_HERE, "lib", "variants", os.environ["HS_LIB_VARIANT"], "libhshard_b200.so")

ERRC_NAMES = [
    "OverlappingSubgroups", "CardinalityMismatch", "BadSplitDim", "IndivisibleSplit",
    "BadRatios", "DeviceNotInAnnotation", "NotRefinable", "InexactDivision", "MissingSymbol",
    "NonPositive", "CycleDetected", "DgUnionMismatch", "UnderivableSharding", "PartialUnderBsr",
    "UnsupportedHdimTransition", "NoOwner", "UnknownDevice", "ConflictingStageOrder",
    "SymbolBindingError", "ShapeMismatch", "DeadlockDetected", "ReplicaDivergence",
    "MissingShard", "UnsupportedOp", "UndeducedStrategy", "ParseError", "UnexecutableStep",
    "CudaError", "CommError",
]


class HshardError(RuntimeError):
    """Mirror of hshard::Error (reference common.hpp:74-84): carries the Errc name."""

    def __init__(self, code: str, message: str):
        super().__init__(message)
        self.code = code


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P = POINTER
    sig = {
        "hs_last_error": (c_char_p, []),
        "hs_errc_name": (c_char_p, [c_int]),
        "hs_free": (None, [c_void_p]),
        "hs_version": (c_int, []),
        "hs_classify": (c_int, [c_char_p, c_char_p, P(c_int64), c_int, c_int, c_char_p, P(c_void_p)]),
        "hs_plan_switch": (c_int, [c_int, P(c_int), P(c_char_p), P(c_char_p), P(c_int64), P(c_int),
                                   c_int, c_char_p, P(c_void_p)]),
        "hs_plan_dump": (c_int, [c_void_p, P(c_void_p)]),
        "hs_plan_destroy": (None, [c_void_p]),
        "hs_build_table": (c_int, [c_char_p, c_char_p, P(c_int64), c_int, c_int, c_int, P(c_void_p)]),
        "hs_make_plan": (c_int, [c_char_p, c_char_p, P(c_int64), c_int, c_int, c_char_p, c_int,
                                 P(c_void_p)]),
        "hs_placement": (c_int, [c_char_p, P(c_int64), c_int, c_int, P(c_int64), P(c_int64), P(c_int)]),
        "hs_convert_hsize": (c_int, [c_char_p, c_int, P(c_void_p)]),
        "hs_annotations_equal": (c_int, [c_char_p, c_char_p, P(c_int)]),
        "hs_validate": (c_int, [c_char_p, P(c_int64), c_int, P(c_void_p)]),
        "hs_align_shard_specs": (c_int, [c_char_p, c_char_p, P(c_void_p)]),
        # strategy source
        "hs_graph_deduce": (c_int, [c_char_p, P(c_void_p)]),
        "hs_graph_diff": (c_int, [c_char_p, c_int, c_int, c_char_p, P(c_void_p)]),
        "hs_graph_specialize": (c_int, [c_char_p, c_int, c_char_p, P(c_void_p)]),
        # executor
        "hs_ctx_create": (c_int, [c_int, c_int, c_int, c_size_t, P(c_void_p)]),
        "hs_ctx_destroy": (None, [c_void_p]),
        "hs_ctx_arena": (c_int, [c_void_p, P(c_void_p), P(c_size_t)]),
        "hs_ctx_ipc_handle": (c_int, [c_void_p, c_char_p]),
        "hs_ctx_open_peers": (c_int, [c_void_p, c_char_p]),
        "hs_ctx_alloc": (c_int, [c_void_p, c_size_t, P(c_size_t)]),
        "hs_nccl_unique_id": (c_int, [c_char_p]),
        "hs_ctx_nccl_init": (c_int, [c_void_p, c_char_p]),
        "hs_ctx_reset_alloc": (c_int, [c_void_p, c_size_t]),
        "hs_prog_compile": (c_int, [c_void_p, c_void_p, P(c_int), c_int, P(c_size_t), P(c_size_t),
                                    c_int, P(c_void_p)]),
        "hs_prog_destroy": (None, [c_void_p]),
        "hs_prog_run": (c_int, [c_void_p, c_void_p]),
        "hs_prog_run_host": (c_int, [c_void_p, P(c_void_p), P(c_void_p)]),
        "hs_prog_run_host_async": (c_int, [c_void_p, P(c_void_p), P(c_void_p), c_void_p, c_void_p, c_void_p]),
        "hs_prog_stats": (c_int, [c_void_p, P(c_void_p)]),
        "hs_prog_profile": (c_int, [c_void_p, c_int]),
        "hs_prog_phase_ms": (c_int, [c_void_p, P(ctypes.c_double), c_int, P(c_int)]),
        "hs_analyze": (c_int, [c_void_p, c_int, c_int, P(c_int), c_int, c_int, P(c_void_p), P(c_void_p)]),
        "hs_fill_shard": (c_int, [c_void_p, c_char_p, P(c_int64), c_int, c_int, c_int, c_size_t,
                                  c_uint32, c_int, c_int, c_void_p]),
        "hs_verify_shard": (c_int, [c_void_p, c_char_p, P(c_int64), c_int, c_int, c_int, c_size_t,
                                    c_uint32, c_int, P(c_ulonglong), c_void_p]),
        "hs_ctx_read": (c_int, [c_void_p, c_size_t, c_void_p, c_size_t]),
        "hs_ctx_write": (c_int, [c_void_p, c_size_t, c_void_p, c_size_t]),
        "hs_ctx_sync": (c_int, [c_void_p]),
        "hs_ctx_barrier": (c_int, [c_void_p, c_void_p]),
        "hs_ctx_clear_error": (c_int, [c_void_p]),
        "hs_volume_report": (c_int, [c_void_p, c_int, P(c_int), P(c_int), P(c_void_p)]),
        "hs_prog_compile_ptrs": (c_int, [c_void_p, c_void_p, P(c_int), c_int, P(c_void_p), P(c_void_p), c_int,
                                         P(c_void_p)]),
        "hs_ipc_export": (c_int, [c_void_p, c_void_p, c_char_p]),
        "hs_ipc_import": (c_int, [c_void_p, c_char_p, P(c_void_p)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue  # reported by exported_symbols(); tests assert completeness
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()


def check(rc: int) -> None:
    if rc != 0:
        code = ERRC_NAMES[rc - 1] if 0 < rc <= len(ERRC_NAMES) else f"Errc{rc - 1}"
        raise HshardError(code, LIB.hs_last_error().decode(errors="replace"))


def take_string(ptr: c_void_p) -> str:
    """Copy a malloc'd C string returned through char** and free it."""
    s = ctypes.cast(ptr, c_char_p).value.decode()
    LIB.hs_free(ptr)
    return s


def i64_array(values) -> ctypes.Array:
    values = list(values)
    return (c_int64 * max(1, len(values)))(*values)
