"""Python mirror of the reference hshard planner API over the C ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/hshard: annotation.hpp, bsr.hpp, resolve.hpp)
so tests read like the reference's own API usage.  Annotations are passed in
the reference's HetAnnotation::str() text form; helpers below build it.
Every call goes through libhshard_b200.so; errors raise HshardError carrying
the reference Errc name.
"""
from __future__ import annotations

import ctypes
import json
from ctypes import c_char_p, c_int, c_int64, c_void_p
from fractions import Fraction
from typing import Dict, List, Optional, Sequence, Tuple

from ._lib import LIB, HshardError, check, i64_array, take_string

__all__ = [
    "HshardError", "DTYPES", "anno", "single", "Plan", "classify", "plan_switch", "build_table",
    "make_plan", "make_plan_naive", "placement", "convert_hsize", "annotations_equal",
    "validate", "align_shard_specs", "parse_annotation",
]

# Pure-text helpers (no native code): annotation strings, dtype tables.
from .annotext import (DTYPE_BYTES, DTYPES, anno, kDuplicate, kPartial,  # noqa: F401
                       parse_annotation, single)


def _shape(shape):
    shape = [int(x) for x in shape]
    return i64_array(shape), len(shape)


class Plan:
    """Owning handle to a CommPlan (classify) or a fused switch plan (plan_switch)."""

    def __init__(self, handle: c_void_p, kind: str, meta: Optional[dict] = None):
        self._h = handle
        self.kind = kind
        self.meta = meta or {}
        self._dump: Optional[str] = None

    @property
    def handle(self) -> c_void_p:
        return self._h

    def dump(self) -> str:
        if self._dump is None:
            out = c_void_p()
            check(LIB.hs_plan_dump(self._h, ctypes.byref(out)))
            self._dump = take_string(out)
        return self._dump

    def json(self) -> dict:
        return json.loads(self.dump())

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and LIB is not None:  # module globals may already be gone at exit
            LIB.hs_plan_destroy(h)


def classify(src: str, dst: str, shape, dtype: str = "f64", bandwidth: str = "u") -> Plan:
    """hshard::classify (reference resolve.hpp:95-97).  Default dtype F64 as in the reference."""
    arr, n = _shape(shape)
    h = c_void_p()
    check(LIB.hs_classify(src.encode(), dst.encode(), arr, n, DTYPES[dtype], bandwidth.encode(),
                          ctypes.byref(h)))
    return Plan(h, "comm", {"src": src, "dst": dst, "shape": list(shape), "dtype": dtype})


def plan_switch(entries: Sequence[Tuple[int, str, str, Sequence[int]]], dtype: str = "f32",
                bandwidth: str = "u") -> Plan:
    """SPEC.md:419-427 plan_switch: build_table per (tensor_id, src, dst, shape), then fuse."""
    n = len(entries)
    ids = (c_int * max(1, n))(*[e[0] for e in entries])
    srcs = (c_char_p * max(1, n))(*[e[1].encode() for e in entries])
    dsts = (c_char_p * max(1, n))(*[e[2].encode() for e in entries])
    flat = [int(x) for e in entries for x in e[3]]
    shapes = i64_array(flat)
    nd = (c_int * max(1, n))(*[len(e[3]) for e in entries])
    h = c_void_p()
    check(LIB.hs_plan_switch(n, ids, srcs, dsts, shapes, nd, DTYPES[dtype], bandwidth.encode(),
                             ctypes.byref(h)))
    return Plan(h, "switch", {"entries": [(e[0], e[1], e[2], list(e[3])) for e in entries],
                              "dtype": dtype})


def build_table(src: str, dst: str, shape, tensor_id: int = 0, elem_bytes: int = 4) -> dict:
    arr, n = _shape(shape)
    out = c_void_p()
    check(LIB.hs_build_table(src.encode(), dst.encode(), arr, n, tensor_id, elem_bytes,
                             ctypes.byref(out)))
    return json.loads(take_string(out))


def _make(src, dst, shape, elem_bytes, bandwidth, naive) -> dict:
    arr, n = _shape(shape)
    out = c_void_p()
    check(LIB.hs_make_plan(src.encode(), dst.encode(), arr, n, elem_bytes, bandwidth.encode(),
                           naive, ctypes.byref(out)))
    return json.loads(take_string(out))


def make_plan(src: str, dst: str, shape, elem_bytes: int = 4, bandwidth: str = "u") -> dict:
    return _make(src, dst, shape, elem_bytes, bandwidth, 0)


def make_plan_naive(src: str, dst: str, shape, elem_bytes: int = 4) -> dict:
    return _make(src, dst, shape, elem_bytes, "u", 1)


def placement(a: str, shape, device: int) -> dict:
    """hshard::placement -> {"bounds": [[lo,hi],...], "partial": (i,n), "replica": (i,n)}."""
    arr, n = _shape(shape)
    lo = (c_int64 * max(1, n))()
    hi = (c_int64 * max(1, n))()
    ordv = (c_int * 4)()
    check(LIB.hs_placement(a.encode(), arr, n, device, lo, hi, ordv))
    return {"bounds": [[lo[i], hi[i]] for i in range(n)], "partial": (ordv[0], ordv[1]),
            "replica": (ordv[2], ordv[3])}


def convert_hsize(a: str, target: int) -> str:
    out = c_void_p()
    check(LIB.hs_convert_hsize(a.encode(), target, ctypes.byref(out)))
    return take_string(out)


def annotations_equal(a: str, b: str) -> bool:
    eq = c_int()
    check(LIB.hs_annotations_equal(a.encode(), b.encode(), ctypes.byref(eq)))
    return bool(eq.value)


def validate(a: str, shape) -> List[str]:
    arr, n = _shape(shape)
    out = c_void_p()
    check(LIB.hs_validate(a.encode(), arr, n, ctypes.byref(out)))
    return json.loads(take_string(out))


def align_shard_specs(a, b):
    out = c_void_p()
    check(LIB.hs_align_shard_specs(_ds_str(a).encode(), _ds_str(b).encode(), ctypes.byref(out)))
    return json.loads(take_string(out))


def volume_report(plan: "Plan", node_of: Dict[int, int]) -> Dict[int, List[int]]:
    """Reference volume_report (bsr.hpp:107-108, bsr.cpp:244-261) through the C ABI:
    {device: [intra-node bytes, inter-node bytes]} over the plan's transfers."""
    devs = sorted(node_of)
    n = len(devs)
    d = (c_int * max(1, n))(*devs)
    nd = (c_int * max(1, n))(*[node_of[x] for x in devs])
    out = c_void_p()
    check(LIB.hs_volume_report(plan.handle, n, d, nd, ctypes.byref(out)))
    return {int(k): v for k, v in json.loads(take_string(out)).items()}
