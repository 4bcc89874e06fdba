"""The BASELINE.json workloads as concrete annotation pairs.

Every config is a list of (tensor_id, src, dst, shape) "transitions" plus a
dtype.  Single-tensor configs (1-3) are planned with classify(); the graph
switches (4, 5) with plan_switch() over every parameter whose annotation
changes.  Virtual device ids are 0..n_virtual-1; on G GPUs virtual device v
lives on GPU v // (n_virtual // G) (block mapping).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

from .annotext import anno, single

Transition = Tuple[int, str, str, Tuple[int, ...]]


@dataclass
class Workload:
    name: str
    kind: str                     # "classify" | "switch"
    dtype: str
    n_virtual: int
    transitions: List[Transition]
    note: str = ""
    meta: Dict = field(default_factory=dict)


D4 = [[0, 1], [2, 3]]
G8 = [list(range(4)), list(range(4, 8))]


def config1(variant: str = "A") -> Workload:
    """4096^2 fp32, Split(0) 3:1 over two subgroups -> Duplicate, 4 virtual devices."""
    src = anno(D4, ["{-1:2}", "{-1:2}"], 0, ["3/4", "1/4"])
    if variant == "A":    # keep the DG union: SplitAllGather (2 slices)
        dst = anno(D4, ["{-1:2}", "{-1:2}"], -1)
    elif variant == "B":  # hsize 1 Duplicate: global Bsr
        dst = single([0, 1, 2, 3], "{-1:4}")
    elif variant == "C":  # bottom split inside subgroups -> Duplicate over all
        src = anno(D4, ["{0:2}", "{0:2}"], 0, ["3/4", "1/4"])
        dst = single([0, 1, 2, 3], "{-1:4}")
    elif variant == "D":  # AllGather per subgroup then SplitAllGather
        src = anno(D4, ["{0:2}", "{0:2}"], 0, ["3/4", "1/4"])
        dst = anno(D4, ["{-1:2}", "{-1:2}"], -1)
    else:
        raise ValueError(variant)
    return Workload(f"cfg1{variant}", "classify", "f32", 4, [(0, src, dst, (4096, 4096))])


def config2(variant: str = "e") -> Workload:
    """Partial -> Split(1) hierarchical RS, 8192^2 bf16, DS union {TP4, TP2+TP2}."""
    shape = (8192, 8192)
    if variant == "e":
        src = anno(G8, ["{-2:4}", "{-1:2,-2:2}"], -2)
        dst = anno(G8, ["{1:4}", "{-1:2,1:2}"], 1)
    elif variant == "a":
        src = anno(G8, ["{-2:4}", "{-2:4}"], -2)
        dst = anno(G8, ["{1:4}", "{1:4}"], 1)
    elif variant == "b":
        g3 = [[0, 1, 2, 3], [4, 5], [6, 7]]
        src = anno(g3, ["{-2:4}", "{-2:2}", "{-2:2}"], -2)
        dst = anno(g3, ["{1:4}", "{1:2}", "{1:2}"], 1, ["1/2", "1/4", "1/4"])
    elif variant == "d":
        src = single(list(range(8)), "{-2:8}")
        dst = single(list(range(8)), "{1:8}")
    else:
        raise ValueError(variant)
    return Workload(f"cfg2{variant}", "classify", "bf16", 8, [(0, src, dst, shape)])


def config3(variant: str = "b") -> Workload:
    """DP gradient sync, 1 GiB bf16, heterogeneous 5:3 sub-meshes."""
    if variant == "b":    # Partial -> Split(0) with 5:3 top-tier ratios
        shape = (8192, 65536)
        src = anno(G8, ["{-2:4}", "{-2:4}"], -2)
        dst = anno(G8, ["{0:4}", "{0:4}"], 0, ["5/8", "3/8"])
    elif variant == "a":  # Partial -> Duplicate
        shape = (8192, 65536)
        src = anno(G8, ["{-2:4}", "{-2:4}"], -2)
        dst = anno(G8, ["{-1:4}", "{-1:4}"], -1)
    elif variant == "c":  # 5 + 3 devices, Partial -> Duplicate
        shape = (15360, 34952)
        g = [[0, 1, 2, 3, 4], [5, 6, 7]]
        src = anno(g, ["{-2:5}", "{-2:3}"], -2)
        dst = anno(g, ["{-1:5}", "{-1:3}"], -1)
    else:
        raise ValueError(variant)
    return Workload(f"cfg3{variant}", "classify", "bf16", 8, [(0, src, dst, shape)])


# ---------------------------------------------------------------- graph switches
def llama_params(layers: int, hidden: int, ffn: int, vocab: int):
    """(name, shape, split key or -1 for Duplicate, layer or None, role) per parameter.
    Roles: 'embed' (first stage), 'head' (last stage), 'layer'."""
    ps = [("embed", (vocab, hidden), 0, None, "embed")]
    for l in range(layers):
        ps += [
            (f"l{l}.wq", (hidden, hidden), 1, l, "layer"),
            (f"l{l}.wk", (hidden, hidden), 1, l, "layer"),
            (f"l{l}.wv", (hidden, hidden), 1, l, "layer"),
            (f"l{l}.wo", (hidden, hidden), 0, l, "layer"),
            (f"l{l}.gate", (hidden, ffn), 1, l, "layer"),
            (f"l{l}.up", (hidden, ffn), 1, l, "layer"),
            (f"l{l}.down", (ffn, hidden), 0, l, "layer"),
            (f"l{l}.attn_norm", (hidden,), -1, l, "layer"),
            (f"l{l}.ffn_norm", (hidden,), -1, l, "layer"),
        ]
    ps += [("final_norm", (hidden,), -1, None, "head"),
           ("lm_head", (hidden, vocab), 1, None, "head")]
    return ps


def tp_pp(tp: int, pp: int, layers: int):
    """Strategy: TPtp x PPpp on tp*pp devices; layer l on stage l*pp//layers."""
    def layout(split_key: int, layer, role: str) -> str:
        if role == "embed":
            s = 0
        elif role == "head":
            s = pp - 1
        else:
            s = layer * pp // layers
        devs = list(range(s * tp, (s + 1) * tp))
        return single(devs, f"{{{split_key}:{tp}}}")
    return layout


def dp_tp(groups: Sequence[Sequence[int]]):
    """Strategy: hsize = len(groups) replicas (hdim -1), TP inside each subgroup."""
    def layout(split_key: int, layer, role: str) -> str:
        return anno(groups, [f"{{{split_key}:{len(g)}}}" for g in groups], -1)
    return layout


def switch_workload(name: str, params, a, b, n_virtual: int, dtype: str = "bf16") -> Workload:
    trans = []
    for tid, (pname, shape, key, layer, role) in enumerate(params):
        sa, sb = a(key, layer, role), b(key, layer, role)
        trans.append((tid, sa, sb, tuple(shape)))
    return Workload(name, "switch", dtype, n_virtual, trans,
                    meta={"params": len(params)})


def config4() -> Workload:
    """Llama-2-7B shaped params, TP2xPP4 -> TP4xPP2 on 8 virtual devices."""
    ps = llama_params(32, 4096, 11008, 32000)
    return switch_workload("cfg4", ps, tp_pp(2, 4, 32), tp_pp(4, 2, 32), 8)


def config4_reverse() -> Workload:
    """The switch back, TP4xPP2 -> TP2xPP4 (with config4, a two-step strategy cycle)."""
    ps = llama_params(32, 4096, 11008, 32000)
    return switch_workload("cfg4_rev", ps, tp_pp(4, 2, 32), tp_pp(2, 4, 32), 8)


LLAMA13B = dict(layers=40, hidden=5120, ffn=13824, vocab=32000)


def config5_strategies():
    L = LLAMA13B["layers"]
    return {
        "S1": tp_pp(8, 1, L),                                   # TP8
        "S2": dp_tp([[0, 1, 2, 3], [4, 5, 6, 7]]),              # DP2 x TP4
        "S3": dp_tp([[0, 1, 2, 3], [4, 5], [6, 7]]),            # TP4 | TP2 | TP2 (CP-style)
        "S4": tp_pp(4, 2, L),                                   # TP4 x PP2
    }


def config5(step: str = "S1S2") -> Workload:
    """Llama-13B shaped params, one step of the S1->S2->S3->S4->S1 cycle."""
    ps = llama_params(**LLAMA13B)
    st = config5_strategies()
    a, b = step[:2], step[2:]
    return switch_workload(f"cfg5_{step}", ps, st[a], st[b], 8)


CONFIG5_CYCLE = ["S1S2", "S2S3", "S3S4", "S4S1"]


def resident_bytes(w: Workload) -> int:
    """Bytes of every source plus every destination shard of the workload."""
    from .hshard import DTYPE_BYTES, parse_annotation, placement
    total = 0
    for tid, src, dst, shape in w.transitions:
        for anno in (src, dst):
            for g in parse_annotation(anno)["groups"]:
                for d in g:
                    n = 1
                    for lo, hi in placement(anno, shape, d)["bounds"]:
                        n *= hi - lo
                    total += n * DTYPE_BYTES[w.dtype]
    return total


def all_workloads() -> List[Workload]:
    ws = [config1(v) for v in "ABCD"] + [config2(v) for v in "eabd"] + \
         [config3(v) for v in "bac"] + [config4()] + [config5(s) for s in CONFIG5_CYCLE]
    return ws


def link_probes() -> List[Workload]:
    """Not BASELINE configs: 1 GiB SendRecv between two virtual devices, one
    direction (p2p_uni: device 1 -> 0) or both (p2p_bi), to measure the NVLink
    transport in isolation at N = 2."""
    shape = (16384, 32768)
    uni = Workload("p2p_uni", "classify", "bf16", 2,
                   [(0, single([1], "{}"), single([0], "{}"), shape)])
    bi = Workload("p2p_bi", "classify", "bf16", 2,
                  [(0, single([0, 1], "{0:2}"), single([1, 0], "{0:2}"), shape)])
    return [uni, bi]


def by_name(name: str) -> Workload:
    for w in all_workloads() + link_probes():
        if w.name == name:
            return w
    raise KeyError(name)
