"""Byte accounting of a resharding plan under the NCCL bus-bytes convention
(SURVEY §8(d) item 2).  Host logic only; no GPU work.

Per virtual device v, the bytes v would put on the wire if every virtual
device were its own GPU and every step ran as the NCCL-convention collective:

* AllReduce over P devices, input N bytes:        2 (P-1)/P * N
* ReduceScatter (input N) / AllGather (output N):   (P-1)/P * N
* SendRecv pair (s -> r, s != r):                   the box s sends
* Bsr transfer:                                     its bytes, charged to the sender
* Split-collectives, per slice: every contributor piece crosses once to
  every receiver other than the contributor itself.

Step semantics follow resolve.hpp:24-78 (StepKind / SliceCollective) and
bsr.hpp:60-87 (Transfer); the split rule follows SURVEY §8(d).
"""
from __future__ import annotations

import math
from collections import defaultdict

from . import hshard as H


def _box_bytes(box, elem):
    return math.prod(hi - lo for lo, hi in box) * elem


def _plan_bus(pj: dict, elem: int, bus: dict, tensor_slot: int = 0):
    shape = pj["shape"]
    src, tgt = pj["src"], pj["mid"] or pj["dst"]
    for st in pj["bottom"]:
        kind = st["kind"]
        for g in st["groups"]:
            p = len(g)
            for v in g:
                if kind == "AllReduce":
                    bus[v] += 2 * (p - 1) * _box_bytes(H.placement(src, shape, v)["bounds"], elem) // p
                elif kind == "ReduceScatter":
                    bus[v] += (p - 1) * _box_bytes(H.placement(src, shape, v)["bounds"], elem) // p
                elif kind == "AllGather":
                    bus[v] += (p - 1) * _box_bytes(H.placement(tgt, shape, v)["bounds"], elem) // p
        for s, r in st["pairs"]:
            if s != r:
                bus[s] += _box_bytes(H.placement(src, shape, s)["bounds"], elem)
        if st["bsr"]:
            for x in st["bsr"]["xfer"]:
                bus[x[2]] += x[4]
    for st in pj["top"]:
        for sl in st["slices"]:
            b = _box_bytes(sl["reg"], elem)
            for c in sl["c"]:
                bus[c] += b * sum(1 for r in sl["r"] if r != c)
        if st["bsr"]:
            for x in st["bsr"]["xfer"]:
                bus[x[2]] += x[4]


def bus_bytes(plan) -> dict:
    """{virtual device: NCCL-convention bus bytes} of a classify or switch plan."""
    pj = plan.json()
    bus = defaultdict(int)
    if "xfer" in pj:  # fused Bsr switch plan: transfers charged to senders
        for x in pj["xfer"]:
            bus[x[2]] += x[4]
        return dict(bus)
    _plan_bus(pj, H.DTYPE_BYTES[pj["dtype"]], bus)
    return dict(bus)
