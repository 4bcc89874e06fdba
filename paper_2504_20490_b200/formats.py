"""Wire / on-disk formats of the SPEC's CLI.

* Annotation JSON, canonical key order:
  {"dg_union": [[0,1],[2,3]], "ds_union": [{"-1": 2}, {"0": 2}], "hdim": 0, "hsize": 2,
   "hsplit_ratios": ["3/4", "1/4"]}
  ds_union entries are ordered {key: count} maps (key -1 Duplicate, -2 Partial,
  d >= 0 Split(d)); converted to / from the annotation text the C ABI speaks.
* Graph JSON "v1": {"version": "v1", "strategies": N, "nodes": [
  {"id", "kind", "inputs": [tensor ids], "name", "shape": ["B", "64"], "dtype",
   "func", "axis", "target", "once", "annotations": {"<strategy>": annotation JSON}}]}
  nodes in creation order; node i produces tensor i.
* Tensor binary: b"HSTB", little-endian u32 header length,
  the header JSON {"shape": [...], "dtype": "bf16", "version": "v1"}, then the
  dense row-major little-endian payload.
* Plan JSON: the canonical planner dump (identical to the reference's, see
  tests/test_plan_parity.py) wrapped as {"version": "v1", "kind", "plan": ...}.
"""
from __future__ import annotations

import json
import struct
from fractions import Fraction
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import hshard as H
from .graph import Graph

VERSION = "v1"
NP_DTYPES = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64, "bf16": np.uint16}


# ---------------------------------------------------------------- annotations
def anno_to_json(text: str) -> dict:
    p = H.parse_annotation(text)
    for spec in p["specs"]:
        keys = [k for k, _ in spec]
        if len(set(keys)) != len(keys):  # a {key: count} map cannot hold a repeated key
            raise H.HshardError("ParseError", f"{text}: a DS with a repeated key has no annotation-JSON form")
    return {"dg_union": p["groups"],
            "ds_union": [{str(k): c for k, c in spec} for spec in p["specs"]],
            "hdim": p["hdim"], "hsize": p["hsize"],
            "hsplit_ratios": [f"{r.numerator}/{r.denominator}" for r in p["ratios"]]}


def anno_from_json(obj) -> str:
    """Annotation JSON (dict or JSON text) or already the text form -> text form."""
    if isinstance(obj, str):
        s = obj.strip()
        if not s.startswith("{"):
            return s
        obj = json.loads(s)
    groups = [list(map(int, g)) for g in obj["dg_union"]]
    specs = [[(int(k), int(c)) for k, c in ds.items()] for ds in obj["ds_union"]]
    if len(groups) != len(specs):
        raise H.HshardError("ParseError", "dg_union and ds_union lengths differ")
    hsize = int(obj.get("hsize", len(groups)))
    if hsize != len(groups):
        raise H.HshardError("ParseError", f"hsize {hsize} but {len(groups)} device groups")
    ratios = [Fraction(r) for r in obj.get("hsplit_ratios", [])]
    return H.anno(groups, specs, int(obj.get("hdim", -1)), ratios or None)


# ---------------------------------------------------------------- graphs
def graph_from_json(obj) -> Graph:
    if isinstance(obj, str):
        obj = json.loads(obj)
    if obj.get("version") != VERSION:
        raise H.HshardError("ParseError", f"graph JSON version {obj.get('version')!r}, expected {VERSION!r}")
    g = Graph(int(obj.get("strategies", 1)))
    for i, n in enumerate(obj["nodes"]):
        if int(n.get("id", i)) != i:
            raise H.HshardError("ParseError", f"node {n.get('id')} out of creation order (expected {i})")
        kind, ins = n["kind"], n.get("inputs", [])
        if kind in ("Placeholder", "Parameter"):
            fn = g.placeholder if kind == "Placeholder" else g.parameter
            fn(n["name"], [str(d) for d in n["shape"]], n.get("dtype", "f64"))
        elif kind == "Elementwise":
            g.elementwise(n.get("func", "identity"), ins[0])
        elif kind == "Dot":
            g.dot(ins[0], ins[1])
        elif kind == "Sum":
            g.sum(ins[0], int(n["axis"]))
        elif kind == "Reshape":
            g.reshape(ins[0], [str(d) for d in n["target"]])
        elif kind == "CommOp":
            g.comm(ins[0], n.get("once"))
        else:
            raise H.HshardError("ParseError", f"unknown node kind {kind!r}")
        for s, a in n.get("annotations", {}).items():
            g.annotate(i, int(s), anno_from_json(a))
    return g


def graph_to_json(g: Graph) -> dict:
    nodes = []
    for n in g.nodes:
        rec = {k: v for k, v in n.items() if k != "annotations"}
        rec["annotations"] = {s: anno_to_json(a) for s, a in n["annotations"].items()}
        nodes.append(rec)
    return {"version": VERSION, "strategies": g.strategies, "nodes": nodes}


def deduced_graph_json(g: Graph) -> dict:
    """The `deduce` subcommand's output: every tensor with its annotation per strategy."""
    d = g.deduce()
    tensors = []
    for t in d["tensors"]:
        per = {}
        for s, st in enumerate(d["strategies"]):
            if st["ok"]:
                per[str(s)] = anno_to_json(st["slots"][t["id"]])
        tensors.append({**t, "annotations": per})
    return {"version": VERSION, "tensors": tensors, "topo": d["topo"], "symbols": d["symbols"],
            "strategies": [{"ok": bool(s["ok"]), **({} if s["ok"] else {"error": s["error"]})}
                           for s in d["strategies"]]}


# ---------------------------------------------------------------- tensors
MAGIC = b"HSTB"


def write_tensor(path: str, array: np.ndarray, dtype: str) -> None:
    if array.dtype != NP_DTYPES[dtype]:
        raise ValueError(f"array dtype {array.dtype} does not store {dtype}")
    head = json.dumps({"shape": list(array.shape), "dtype": dtype, "version": VERSION}).encode()
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<I", len(head)) + head)
        f.write(np.ascontiguousarray(array).astype(array.dtype.newbyteorder("<"), copy=False).tobytes())


def read_tensor(path: str):
    """-> (array, dtype name)."""
    with open(path, "rb") as f:
        if f.read(4) != MAGIC:
            raise H.HshardError("ParseError", f"{path}: not an hshard tensor file")
        (n,) = struct.unpack("<I", f.read(4))
        head = json.loads(f.read(n))
        dt = head["dtype"]
        a = np.frombuffer(f.read(), dtype=np.dtype(NP_DTYPES[dt]).newbyteorder("<"))
    shape = tuple(head["shape"])
    if a.size != int(np.prod(shape)):
        raise H.HshardError("ShapeMismatch", f"{path}: payload has {a.size} elements, header says {shape}")
    return a.reshape(shape).astype(NP_DTYPES[dt]), dt


# ---------------------------------------------------------------- reports
def volume_report(xfer: Sequence, devices_per_node: int = 8, node_of: Optional[Dict[int, int]] = None
                  ) -> Dict[int, List[int]]:
    """The reference volume_report (bsr.hpp:107-108, bsr.cpp:244-261) over a plan JSON's
    transfers: {device: [intra-node bytes, inter-node bytes]} with every device of
    `node_of` present (zeros included), UnknownDevice for a transfer end outside it.
    Without node_of, the devices the transfers touch on nodes of `devices_per_node`."""
    if node_of is None:
        devs = {int(x[i]) for x in xfer for i in (2, 3)}
        node_of = {d: d // devices_per_node for d in devs}
    out: Dict[int, List[int]] = {d: [0, 0] for d in node_of}
    for x in xfer:
        s, r, b = int(x[2]), int(x[3]), int(x[4])
        for d, role in ((s, "sender"), (r, "receiver")):
            if d not in node_of:
                raise H.HshardError("UnknownDevice", f"{role} {d} not in cluster")
        out[s][0 if node_of[s] == node_of[r] else 1] += b
    return dict(sorted(out.items()))


def table(rows: Sequence[Sequence], head: Sequence[str]) -> str:
    cols = [list(map(str, head))] + [[str(c) for c in r] for r in rows]
    w = [max(len(r[i]) for r in cols) for i in range(len(head))]
    line = lambda r: "  ".join(c.rjust(w[i]) for i, c in enumerate(r))
    return "\n".join([line(cols[0]), "  ".join("-" * x for x in w)] + [line(r) for r in cols[1:]])
