"""Parallel strategies as annotated model graphs: the strategy source for graph
switches (reference graph.hpp:105-141, deduction.hpp:29-31,
SPEC.md:413-418).

A Llama-shaped block graph is built once with one annotation slot per named
strategy; leaves (the one-hot token batch and every weight) and CommOps (the
all-reduces after row-parallel matmuls, and the hand-off to the next layer's
devices -- a pipeline send at stage edges) are annotated, everything else is
deduced, and specialize / construct_pipelines recover each strategy's stages.  diff_strategies
between two slots yields exactly the parameter moves plan_switch executes --
the same (src, dst) pairs workloads.config4 / config5 spell out by hand.

    g, names = llama_graph(32, 4096, 11008, 32000, {"A": tp_pp(2, 4, 32), "B": tp_pp(4, 2, 32)})
    plan = g.switch_plan(names["A"], names["B"], "bf16")
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Dict, Sequence, Tuple

from .graph import Graph
from .hshard import anno, single
from . import workloads as W

# stage key: a layer index, or "embed" / "head"
Layout = Callable[[int, object, str], str]


@dataclass
class Strategy:
    """params(split_key, layer, role) -> annotation of a weight;
    acts(split_key, layer, role) -> annotation of an activation entering /
    produced in that layer (split_key -1 = replicated, 1 = column split)."""
    params: Layout
    acts: Layout


def tp_pp(tp: int, pp: int, layers: int) -> Strategy:
    """TPtp x PPpp on tp*pp devices, layer l on stage l*pp//layers (as workloads.tp_pp)."""
    def acts(key, layer, role):
        s = 0 if role == "embed" else pp - 1 if role == "head" else layer * pp // layers
        return single(list(range(s * tp, (s + 1) * tp)), f"{{{key}:{tp}}}")
    return Strategy(W.tp_pp(tp, pp, layers), acts)


def dp_tp(groups: Sequence[Sequence[int]]) -> Strategy:
    """len(groups) data-parallel replicas (batch split across subgroups), TP inside each."""
    def acts(key, layer, role):
        return anno(groups, [f"{{{key}:{len(g)}}}" for g in groups], 0 if len(groups) > 1 else -1)
    return Strategy(W.dp_tp(groups), acts)


def llama_graph(layers: int, hidden: int, ffn: int, vocab: int, strategies: Dict[str, Strategy],
                dtype: str = "bf16", batch="B") -> Tuple[Graph, Dict[str, int]]:
    """Returns (graph, {strategy name: slot}); parameter names follow workloads.llama_params."""
    names = {n: i for i, n in enumerate(strategies)}
    g = Graph(len(strategies))
    todo = []  # (node, layout kind, split key, layer, role)

    def param(name, shape, key, layer, role):
        t = g.parameter(name, shape, dtype)
        todo.append((t, "params", key, layer, role))
        return t

    def comm(x, layer, role, key=-1):
        t = g.comm(x)
        todo.append((t, "acts", key, layer, role))
        return t

    tokens = g.placeholder("tokens", [batch, vocab], dtype)       # one-hot rows
    todo.append((tokens, "acts", 1, None, "embed"))                # vocab split like embed rows
    embed = param("embed", [vocab, hidden], 0, None, "embed")
    h = comm(g.dot(tokens, embed), 0, "layer")                     # partial sums -> all-reduce
    for l in range(layers):
        param(f"l{l}.attn_norm", [hidden], -1, l, "layer")
        wq = param(f"l{l}.wq", [hidden, hidden], 1, l, "layer")
        wk = param(f"l{l}.wk", [hidden, hidden], 1, l, "layer")
        wv = param(f"l{l}.wv", [hidden, hidden], 1, l, "layer")
        wo = param(f"l{l}.wo", [hidden, hidden], 0, l, "layer")
        q = g.dot(h, wq)
        g.dot(h, wk)
        g.dot(h, wv)
        h = comm(g.dot(q, wo), l, "layer")                         # row-parallel -> all-reduce
        param(f"l{l}.ffn_norm", [hidden], -1, l, "layer")
        gate = param(f"l{l}.gate", [hidden, ffn], 1, l, "layer")
        up = param(f"l{l}.up", [hidden, ffn], 1, l, "layer")
        down = param(f"l{l}.down", [ffn, hidden], 0, l, "layer")
        a = g.elementwise("gelu", g.dot(h, gate))
        g.dot(h, up)
        h = comm(g.dot(a, down), l, "layer")  # row-parallel -> all-reduce on this layer's devices
        # hand-off to the next layer's devices: a pipeline send at stage edges, identity elsewhere
        h = comm(h, l + 1, "layer") if l + 1 < layers else comm(h, None, "head")
    param("final_norm", [hidden], -1, None, "head")
    head = param("lm_head", [hidden, vocab], 1, None, "head")
    g.dot(h, head)
    for n, s in strategies.items():
        for t, kind, key, layer, role in todo:
            g.annotate(t, names[n], getattr(s, kind)(key, layer, role))
    return g, names
