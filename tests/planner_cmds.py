"""Replays ref_tool line-protocol commands (oracle/ref_tool.cpp) through the
PRODUCT planner (libhshard_b200.so C ABI) and renders the same canonical text,
so golden outputs recorded from the reference compare byte-for-byte."""
from __future__ import annotations

import ctypes
import json
from ctypes import c_int, c_void_p

from paper_2504_20490_b200 import hshard as H
from paper_2504_20490_b200._lib import LIB, HshardError, check, i64_array, take_string

ELEM_DTYPE = {2: "bf16", 4: "f32", 8: "f64"}


def _shape(s):
    v = [int(x) for x in s.split(",") if x.strip()]
    return i64_array(v), len(v), v


def _region_str(p):
    s = "x".join(f"[{lo},{hi})" for lo, hi in p["bounds"])
    if p["partial"][1] > 1:
        s += f" partial {p['partial'][0]}/{p['partial'][1]}"
    if p["replica"][1] > 1:
        s += f" replica {p['replica'][0]}/{p['replica'][1]}"
    return s


def _raw(fn, *args):
    out = c_void_p()
    check(fn(*args, ctypes.byref(out)))
    return take_string(out)


def run(lines):
    try:
        return _run(lines)
    except HshardError as e:
        return json.dumps({"error": e.code}, separators=(",", ":"))


def _run(lines):
    f = lines[0].split("|")
    c = f[0]
    if c == "C":
        _, dt, shp, bw, src, dst = f
        return H.classify(src, dst, [int(x) for x in shp.split(",")], dt, bw).dump()
    if c == "T":
        _, eb, shp, tid, src, dst = f
        arr, n, _ = _shape(shp)
        return _raw(LIB.hs_build_table, src.encode(), dst.encode(), arr, n, int(tid), int(eb))
    if c == "M":
        _, bw, naive, eb, shp, src, dst = f
        arr, n, _ = _shape(shp)
        return _raw(LIB.hs_make_plan, src.encode(), dst.encode(), arr, n, int(eb), bw.encode(),
                    int(naive))
    if c == "F":
        _, bw, n = f
        entries, ebs = [], set()
        for ln in lines[1:1 + int(n)]:
            g = ln.split("|")
            ebs.add(int(g[1]))
            entries.append((int(g[0]), g[3], g[4], [int(x) for x in g[2].split(",")]))
        assert len(ebs) <= 1
        dt = ELEM_DTYPE[ebs.pop()] if ebs else "f32"
        return H.plan_switch(entries, dt, bw).dump()
    if c == "P":
        _, shp, a = f
        shape = [int(x) for x in shp.split(",")]
        devs = sorted(d for g in H.parse_annotation(a)["groups"] for d in g)
        return "{" + ",".join(f"\"{d}\":" + json.dumps(_region_str(H.placement(a, shape, d)))
                              for d in devs) + "}"
    if c == "H":
        return json.dumps(H.convert_hsize(f[1], int(f[2])))
    if c == "Q":
        return "true" if H.annotations_equal(f[1], f[2]) else "false"
    if c == "A":
        return _raw(LIB.hs_align_shard_specs, f[1].encode(), f[2].encode())
    if c == "V":
        arr, n, _ = _shape(f[1])
        return _raw(LIB.hs_validate, f[2].encode(), arr, n)
    raise ValueError(c)
