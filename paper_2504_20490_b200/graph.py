"""Strategy source for graph switches: an annotated computation graph
(reference graph.hpp:105-141), sharding deduction (deduction.hpp:19-31) and
diff_strategies(graph, a, b), through the C ABI
(hs_graph_deduce / hs_graph_diff).

    g = Graph(strategies=2)
    x = g.placeholder("x", ["B", 4096], "f32")
    w = g.parameter("w", [4096, 4096], "f32")
    y = g.dot(x, w)
    g.annotate(x, 0, H.single([0, 1], {-1: 2})); g.annotate(w, 0, H.single([0, 1], {1: 2}))
    ...
    g.deduce()                       # every tensor's annotation per strategy
    entries = g.diff(0, 1)           # changed Parameters -> plan_switch entries

The graph travels as the line form hshard::parse_graph reads
(include/hshard/graph.hpp); node ids and tensor ids coincide.
"""
from __future__ import annotations

import json
from ctypes import c_void_p
from typing import Dict, List, Optional, Sequence, Union

from . import hshard as H
from ._lib import LIB, check, take_string

Dim = Union[int, str]


class Graph:
    def __init__(self, strategies: int = 1):
        if strategies < 1:
            raise ValueError("a graph has at least one strategy")
        self.strategies = strategies
        self._lines = [f"strategies {strategies}"]
        self._n = 0
        self.names: Dict[str, int] = {}
        self.nodes: List[dict] = []  # graph JSON v1 node records (formats.graph_to_json)

    # ---- builders (each returns the new node / tensor id)
    def _add(self, stmt: str, **node) -> int:
        self._lines.append(stmt)
        self.nodes.append({"id": self._n, **node, "annotations": {}})
        self._n += 1
        return self._n - 1

    @staticmethod
    def _dims(shape: Sequence[Dim]) -> str:
        return " ".join(str(d) for d in shape)

    def placeholder(self, name: str, shape: Sequence[Dim], dtype: str = "f64") -> int:
        self.names[name] = self._n
        return self._add(f"placeholder {name} {dtype} {self._dims(shape)}", kind="Placeholder", name=name,
                         shape=[str(d) for d in shape], dtype=dtype)

    def parameter(self, name: str, shape: Sequence[Dim], dtype: str = "f64") -> int:
        self.names[name] = self._n
        return self._add(f"parameter {name} {dtype} {self._dims(shape)}", kind="Parameter", name=name,
                         shape=[str(d) for d in shape], dtype=dtype)

    def elementwise(self, func: str, x: int) -> int:
        return self._add(f"elementwise {func} {x}", kind="Elementwise", inputs=[x], func=func)

    def dot(self, x: int, w: int) -> int:
        return self._add(f"dot {x} {w}", kind="Dot", inputs=[x, w])

    def sum(self, x: int, axis: int) -> int:
        return self._add(f"sum {x} {axis}", kind="Sum", inputs=[x], axis=axis)

    def reshape(self, x: int, shape: Sequence[Dim]) -> int:
        return self._add(f"reshape {x} {self._dims(shape)}", kind="Reshape", inputs=[x],
                         target=[str(d) for d in shape])

    def comm(self, x: int, once: Optional[bool] = None) -> int:
        return self._add(f"comm {x} {'auto' if once is None else int(bool(once))}", kind="CommOp", inputs=[x],
                         once=once)

    def annotate(self, node: int, strategy: int, anno: str) -> None:
        if not 0 <= strategy < self.strategies:
            raise ValueError(f"strategy {strategy} out of range")
        self._lines.append(f"annotate {node} {strategy} {anno}")
        self.nodes[node]["annotations"][str(strategy)] = anno

    # ---- queries
    def text(self) -> str:
        return "\n".join(self._lines)

    def deduce(self) -> dict:
        """{"tensors", "topo", "symbols", "strategies": [{"ok", "slots"} | {"ok": 0, "error"}]}."""
        out = c_void_p()
        check(LIB.hs_graph_deduce(self.text().encode(), out))
        return json.loads(take_string(out))

    def diff(self, a: int, b: int, bindings: Optional[Dict[str, int]] = None) -> List[dict]:
        """Parameters whose annotation differs between strategies a and b:
        [{"tensor", "name", "src", "dst", "shape"}] (UndeducedStrategy / deduction errors raise)."""
        out = c_void_p()
        bind = ",".join(f"{k}={v}" for k, v in (bindings or {}).items())
        check(LIB.hs_graph_diff(self.text().encode(), a, b, bind.encode(), out))
        return json.loads(take_string(out))

    def specialize(self, strategy: int, bindings: Optional[Dict[str, int]] = None) -> dict:
        """Executable graphs per device, node phases and pipelines of one strategy
        (reference specialize.hpp): {"phases", "exec_graphs", "pipelines" | "pipelines_error"}."""
        out = c_void_p()
        bind = ",".join(f"{k}={v}" for k, v in (bindings or {}).items())
        check(LIB.hs_graph_specialize(self.text().encode(), strategy, bind.encode(), out))
        return json.loads(take_string(out))

    def switch_plan(self, a: int, b: int, dtype: str = "bf16", bindings: Optional[Dict[str, int]] = None,
                    bandwidth: str = "u") -> H.Plan:
        """plan_switch over diff(a, b): the fused Bsr plan that moves the weights."""
        entries = [(e["tensor"], e["src"], e["dst"], tuple(e["shape"])) for e in self.diff(a, b, bindings)]
        return H.plan_switch(entries, dtype, bandwidth)
