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


def main():
    cases = all_cases()
    with open(os.path.join(HERE, "graphs.jsonl"), "w") as f:
        for c, r in zip(cases, reference(cases)):
            f.write(json.dumps({"graph": c, "out": json.loads(r)}, separators=(",", ":")) + "\n")
    print(f"{len(cases)} graph cases")


if __name__ == "__main__":
    main()
