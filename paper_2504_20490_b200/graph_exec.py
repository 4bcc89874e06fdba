"""Executable-graph integration on the GPU: the CommOps of
a specialized graph run through compiled programs, with their regions
re-derived for every micro-batch binding.

The reference resolves each CommOp into a CommPlan at the reference binding
(specialize.cpp:57-122, `instantiate`) and notes that "kinds and groups do not
depend on shapes; regions are re-derived per micro-batch"
(specialize.hpp:35-38).  `CommOpExecutor` is that execution step:

    ex = CommOpExecutor(ctx, graph, strategy, dtype, n_virtual, reference_bindings)
    ex.comm_ops                      # the CommOp nodes of the ExecGraphs (with the
                                     # reference-binding plan instantiate() produced)
    prog, lay, info = ex.program(node, {"B": 3})   # classify at the bound shape
    lay.fill_src(seed); prog.run()   # the micro-batch's collective on the GPU

Plans and programs are cached per (node, binding); a schedule's micro-batches
of equal size reuse one program.  Only the CommOps execute here -- the
compute nodes around them are outside the resharding path.
"""
from __future__ import annotations

import re
from typing import Dict, List, Optional, Tuple

from . import hshard as H
from .executor import Context, Program, ShardLayout
from .graph import Graph


def bind_shape(sym_shape: str, bindings: Dict[str, int]) -> List[int]:
    """'[B,64]' with {'B': 3} -> [3, 64]; products / quotients of a symbol ('B/2',
    '2*B') as graph.hpp's SymDim forms them."""
    dims = [d.strip() for d in sym_shape.strip()[1:-1].split(",") if d.strip()]
    out = []
    for d in dims:
        if re.fullmatch(r"-?\d+", d):
            out.append(int(d))
            continue
        m = re.fullmatch(r"(?:(\d+)\*)?([A-Za-z_]\w*)(?:/(\d+))?", d)
        if not m or m.group(2) not in bindings:
            raise H.HshardError("SymbolBindingError", f"cannot bind {d} with {bindings}")
        v = bindings[m.group(2)] * int(m.group(1) or 1)
        div = int(m.group(3) or 1)
        if v % div:
            raise H.HshardError("InexactDivision", f"{d} with {bindings}")
        out.append(v // div)
    return out


class CommOpExecutor:
    def __init__(self, ctx: Context, graph: Graph, strategy: int, dtype: str, n_virtual: int,
                 reference_bindings: Dict[str, int], flags: int = 0):
        self.ctx, self.graph, self.strategy, self.dtype = ctx, graph, strategy, dtype
        self.n_virtual, self.flags = n_virtual, flags
        self.spec = graph.specialize(strategy, reference_bindings)
        ded = graph.deduce()
        if not ded["strategies"][strategy].get("ok"):
            raise H.HshardError(ded["strategies"][strategy].get("error", "UnderivableSharding"),
                                "strategy does not deduce")
        slots = ded["strategies"][strategy]["slots"]
        tensors = {t["id"]: t for t in ded["tensors"]}
        # CommOp node -> (input annotation, output annotation, symbolic shape, reference plan)
        self.comm_ops: Dict[int, dict] = {}
        for eg in self.spec["exec_graphs"]:
            for n in eg["nodes"]:
                if not n["comm"] or n["node"] in self.comm_ops:
                    continue
                node = n["node"]
                src_tensor = graph.nodes[node]["inputs"][0]
                self.comm_ops[node] = {"src": slots[src_tensor], "dst": slots[node],
                                       "shape": tensors[node]["shape"], "phase": n["phase"],
                                       "reference_plan": n["plan"],
                                       "devices": sorted(e["device"] for e in self.spec["exec_graphs"]
                                                         if any(x["node"] == node for x in e["nodes"]))}
        self._plans: Dict[Tuple[int, tuple], H.Plan] = {}
        self._progs: Dict[Tuple[int, tuple], Tuple[Program, ShardLayout]] = {}

    def plan(self, node: int, bindings: Dict[str, int]) -> Tuple[H.Plan, bool]:
        """The CommOp's plan re-derived at `bindings` (classify over the bound shape)."""
        key = (node, tuple(sorted(bindings.items())))
        p = self._plans.get(key)
        if p is not None:
            return p, True
        op = self.comm_ops[node]
        p = H.classify(op["src"], op["dst"], bind_shape(op["shape"], bindings), self.dtype)
        self._plans[key] = p
        return p, False

    def program(self, node: int, bindings: Dict[str, int]):
        """(program, shard layout, {"plan_cached", "program_cached"}) for one micro-batch."""
        key = (node, tuple(sorted(bindings.items())))
        hit = key in self._progs
        plan, plan_hit = self.plan(node, bindings)
        if not hit:
            lay = ShardLayout(self.ctx, plan, self.n_virtual)
            self._progs[key] = (Program(self.ctx, plan, lay, self.flags), lay)
        prog, lay = self._progs[key]
        return prog, lay, {"plan_cached": plan_hit, "program_cached": hit}

    def close(self):
        for prog, lay in self._progs.values():
            prog.close()
        self._progs.clear()
