"""Strategy source parity: CompGraph + deduce_graph + diff_strategies.

* tests/golden/graphs.jsonl holds the REFERENCE's deduction (ref_tool G: the
  reference CompGraph and deduce_graph compiled from /root/reference) of 308
  graphs (tests/golden/graph_cases.py); ours must match every slot string,
  the topological order and every error code.  With the reference build
  present, fresh random graphs and a Llama-shaped model graph are also
  compared live.
* The model graphs of paper_2504_20490_b200/strategy.py reproduce the
  hand-built switch workloads: diff_strategies(TP2xPP4, TP4xPP2) == cfg4's 291
  parameter moves; each step of the Llama-13B S1..S4 cycle == cfg5's 363.
"""
import json
import os
import subprocess
import sys

import pytest

from paper_2504_20490_b200 import hshard as H
from paper_2504_20490_b200 import workloads as W
from paper_2504_20490_b200.graph import Graph
from paper_2504_20490_b200.strategy import dp_tp, llama_graph, tp_pp
from paper_2504_20490_b200._lib import ERRC_NAMES, LIB, take_string

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from graph_cases import random_graph  # noqa: E402

REF_TOOL = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "ref_tool")
GOLDEN = os.path.join(HERE, "golden", "graphs.jsonl")


def ours(text):
    from ctypes import c_void_p
    out = c_void_p()
    rc = LIB.hs_graph_deduce(text.encode(), out)
    if rc:
        return {"error": ERRC_NAMES[rc - 1]}
    return json.loads(take_string(out))


def same(ref, mine):
    if "error" in ref or "error" in mine:
        return ref.get("error") == mine.get("error")
    key = lambda s: (s["ok"], s.get("error"), s.get("slots"))
    return ref["topo"] == mine["topo"] and [key(s) for s in ref["strategies"]] == \
        [key(s) for s in mine["strategies"]]


def reference(texts):
    inp = "".join("G|" + t.replace("\n", "&") + "\n" for t in texts)
    out = subprocess.run([REF_TOOL], input=inp, capture_output=True, text=True, timeout=600, check=True)
    return [json.loads(l) for l in out.stdout.strip().splitlines()]


def test_golden_graph_deduction():
    cases = [json.loads(l) for l in open(GOLDEN)]
    assert len(cases) >= 300
    bad = [c["graph"] for c in cases if not same(c["out"], ours(c["graph"]))]
    assert not bad, f"{len(bad)} mismatches, first:\n{bad[0]}"
    # the fixtures exercise success and every deduction error path
    kinds = {s.get("error", "ok") for c in cases if "strategies" in c["out"] for s in c["out"]["strategies"]}
    assert {"ok", "UnderivableSharding", "DgUnionMismatch", "BadSplitDim", "UndeducedStrategy"} <= kinds


@pytest.mark.skipif(not os.path.exists(REF_TOOL), reason="reference build (oracle/_ref) absent")
def test_live_random_graphs():
    texts = [random_graph(50000 + i) for i in range(120)]
    refs = reference(texts)
    bad = [t for t, r in zip(texts, refs) if not same(r, ours(t))]
    assert not bad, f"{len(bad)} mismatches, first:\n{bad[0]}"


@pytest.mark.skipif(not os.path.exists(REF_TOOL), reason="reference build (oracle/_ref) absent")
def test_live_llama_graph():
    st = {"S1": tp_pp(8, 1, 4), "S2": dp_tp([[0, 1, 2, 3], [4, 5, 6, 7]]),
          "S3": dp_tp([[0, 1, 2, 3], [4, 5], [6, 7]]), "S4": tp_pp(4, 2, 4)}
    g, _ = llama_graph(4, 64, 128, 256, st, dtype="f32")
    ref = reference([g.text()])[0]
    mine = ours(g.text())
    assert all(s["ok"] for s in mine["strategies"])
    assert same(ref, mine)


def _check_moves(diff, workload, params):
    byname = {p[0]: t for p, t in zip(params, workload.transitions)}
    got = {e["name"] for e in diff}
    for e in diff:
        _, s, d, shape = byname[e["name"]]
        assert H.annotations_equal(s, e["src"]) and H.annotations_equal(d, e["dst"]), e["name"]
        assert list(shape) == e["shape"]
    for name, (_, s, d, _) in byname.items():
        assert name in got or H.annotations_equal(s, d), name


def test_graph_reproduces_config4():
    g, n = llama_graph(32, 4096, 11008, 32000, {"A": tp_pp(2, 4, 32), "B": tp_pp(4, 2, 32)})
    diff = g.diff(n["A"], n["B"], {"B": 8})
    assert len(diff) == 291
    _check_moves(diff, W.config4(), W.llama_params(32, 4096, 11008, 32000))


def test_graph_reproduces_config5_cycle():
    st = W.config5_strategies()
    L = W.LLAMA13B["layers"]
    g, n = llama_graph(L, 5120, 13824, 32000, {"S1": tp_pp(8, 1, L), "S2": dp_tp([[0, 1, 2, 3], [4, 5, 6, 7]]),
                                                 "S3": dp_tp([[0, 1, 2, 3], [4, 5], [6, 7]]), "S4": tp_pp(4, 2, L)})
    assert set(n) == set(st)
    for step in W.CONFIG5_CYCLE:
        _check_moves(g.diff(n[step[:2]], n[step[2:]]), W.config5(step), W.llama_params(**W.LLAMA13B))


def test_diff_properties():
    g, n = llama_graph(4, 64, 128, 256, {"A": tp_pp(2, 2, 4), "B": tp_pp(4, 1, 4), "C": tp_pp(2, 2, 4)})
    ab, ba = g.diff(n["A"], n["B"]), g.diff(n["B"], n["A"])
    assert {e["name"]: (e["src"], e["dst"]) for e in ab} == {e["name"]: (e["dst"], e["src"]) for e in ba}
    assert g.diff(n["A"], n["C"]) == [] and g.diff(n["A"], n["A"]) == []
    kinds = {t["id"]: t["kind"] for t in g.deduce()["tensors"]}
    assert all(kinds[e["tensor"]] == "Parameter" for e in ab)
    # a strategy that does not deduce cannot be diffed
    bad = Graph(2)
    x = bad.placeholder("x", [8, 8], "f32")
    w = bad.parameter("w", [8, 8], "f32")
    bad.dot(x, w)
    bad.annotate(x, 0, "hsize=1 hdim=-1 [(0,1){-1:2}]")
    bad.annotate(w, 0, "hsize=1 hdim=-1 [(0,1){1:2}]")
    bad.annotate(x, 1, "hsize=1 hdim=-1 [(0,1){-1:2}]")
    with pytest.raises(H.HshardError) as ei:
        bad.diff(0, 1)
    assert ei.value.code == "UndeducedStrategy"


def test_switch_plan_from_graph_conserves_bytes():
    g, n = llama_graph(32, 4096, 11008, 32000, {"A": tp_pp(2, 4, 32), "B": tp_pp(4, 2, 32)})
    p = g.switch_plan(n["A"], n["B"], "bf16").json()
    moved = sum(x[4] for x in p["xfer"])
    cells = lambda box: __import__("math").prod(hi - lo for lo, hi in box)
    local = sum(cells(c[2]) * 2 for c in p["local"])
    dst = 0
    for e in g.diff(n["A"], n["B"]):
        for grp in H.parse_annotation(e["dst"])["groups"]:
            for d in grp:
                dst += cells(H.placement(e["dst"], e["shape"], d)["bounds"]) * 2
    assert moved + local == dst
    assert abs(moved / 1e9 - 10.108) < 0.001  # 10.108 GB of transfers for cfg4


def test_golden_specialization():
    """instantiate_all / node_phases / construct_pipelines vs the reference's
    (ref_tool S; tests/golden/specialize.jsonl): executable graphs per device,
    the CommPlan each CommOp resolves to, phases and pipeline stages."""
    from ctypes import c_void_p
    cases = [json.loads(l) for l in open(os.path.join(HERE, "golden", "specialize.jsonl"))]
    assert len(cases) >= 150
    bad = []
    for c in cases:
        out = c_void_p()
        rc = LIB.hs_graph_specialize(c["graph"].encode(), c["strategy"], c["bindings"].encode(), out)
        mine = {"error": ERRC_NAMES[rc - 1]} if rc else json.loads(take_string(out))
        if mine != c["out"]:
            bad.append((c["strategy"], c["graph"][:200]))
    assert not bad, f"{len(bad)} mismatches, first: {bad[0]}"
    # the Llama graph recovers each strategy's pipeline structure
    pipes = [c["out"]["pipelines"] for c in cases[:5]]
    assert pipes == [[[list(range(8))]], [[[0, 1, 2, 3]], [[4, 5, 6, 7]]], [[[0, 1, 2, 3]], [[4, 5]], [[6, 7]]],
                     [[[0, 1, 2, 3], [4, 5, 6, 7]]], [[[0, 1], [2, 3], [4, 5], [6, 7]]]]
    assert any("pipelines_error" in c["out"] for c in cases)  # ConflictingStageOrder is exercised
