"""Records tests/golden/graphs.jsonl: each graph case of graph_cases.py with
the REFERENCE's deduction of it -- oracle/_ref/ref_tool command G, i.e. the
reference CompGraph builders and deduce_graph (graph.cpp, deduction.cpp
compiled from /root/reference/proj/src).  Run from the repo root after
`make -C oracle`:

    python tests/golden/make_graph_golden.py
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from graph_cases import all_cases  # noqa: E402

REF_TOOL = os.path.join(HERE, "..", "..", "oracle", "_ref", "ref_tool")


def reference(cases):
    inp = "".join("G|" + c.replace("\n", "&") + "\n" for c in cases)
    out = subprocess.run([REF_TOOL], input=inp, capture_output=True, text=True, timeout=600, check=True)
    lines = out.stdout.strip().splitlines()
    assert len(lines) == len(cases)
    return lines


def spec_cases(graph_records):
    """(graph text, strategy, bindings) for every strategy that deduces, plus a
    Llama-shaped graph under TP8 / DP2xTP4 / TP4|TP2|TP2 / TP4xPP2 / TP2xPP4."""
    sys.path.insert(0, os.path.join(HERE, "..", ".."))
    from paper_2504_20490_b200.strategy import dp_tp, llama_graph, tp_pp
    st = {"S1": tp_pp(8, 1, 4), "S2": dp_tp([[0, 1, 2, 3], [4, 5, 6, 7]]),
          "S3": dp_tp([[0, 1, 2, 3], [4, 5], [6, 7]]), "S4": tp_pp(4, 2, 4), "P": tp_pp(2, 4, 4)}
    g, _ = llama_graph(4, 64, 128, 256, st, dtype="f32")
    out = [(g.text(), s, "B=8") for s in range(len(st))]
    for text, ref in graph_records:
        for s, r in enumerate(ref.get("strategies", [])):
            if r["ok"]:
                out.append((text, s, "B=8,S=4"))
    return out


def main():
    cases = all_cases()
    refs = [json.loads(r) for r in reference(cases)]
    with open(os.path.join(HERE, "graphs.jsonl"), "w") as f:
        for c, r in zip(cases, refs):
            f.write(json.dumps({"graph": c, "out": r}, separators=(",", ":")) + "\n")
    specs = spec_cases(list(zip(cases, refs)))
    inp = "".join(f"S|{s}|{b}|" + t.replace("\n", "&") + "\n" for t, s, b in specs)
    out = subprocess.run([REF_TOOL], input=inp, capture_output=True, text=True, timeout=600, check=True)
    lines = out.stdout.strip().splitlines()
    assert len(lines) == len(specs)
    with open(os.path.join(HERE, "specialize.jsonl"), "w") as f:
        for (t, s, b), r in zip(specs, lines):
            f.write(json.dumps({"graph": t, "strategy": s, "bindings": b, "out": json.loads(r)},
                               separators=(",", ":")) + "\n")
    print(f"{len(cases)} graph cases, {len(specs)} specializations")


if __name__ == "__main__":
    main()
