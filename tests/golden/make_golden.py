#!/usr/bin/env python3
"""Generate the golden plan/data fixtures from the REFERENCE implementation.

Runs oracle/_ref/ref_tool (the reference hshard planner compiled from
/root/reference/proj/src by oracle/Makefile, plus the reference-primitive
executor) on:
  * the SPEC / SURVEY known-answer cases,
  * every BASELINE workload (paper_2504_20490_b200/workloads.py),
  * a seeded random sweep of annotation pairs (SPEC.md:533 acceptance #2 shape
    limits: <= 8 devices, shapes <= [16,16]),
and records the reference's output for each command in plans.jsonl (large
outputs as sha256 + length) and executor vectors in data.jsonl.

Only needed when the fixtures change; tests read the committed files and never
touch /root/reference.  Usage:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import subprocess
import sys
from fractions import Fraction

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from gen_cases import kat_commands, random_commands, random_exec_commands, workload_commands  # noqa: E402

REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
BIG = 64 * 1024


def run_ref(cmds):
    """cmds: list of lists of lines (one command may span several lines)."""
    text = "".join("\n".join(c) + "\n" for c in cmds)
    res = subprocess.run([REF_TOOL], input=text, capture_output=True, text=True, timeout=3600)
    if res.returncode != 0:
        raise SystemExit(f"ref_tool failed: {res.stderr[-2000:]}")
    outs = res.stdout.splitlines()
    assert len(outs) == len(cmds), (len(outs), len(cmds))
    return outs


def record(cmd, out):
    if len(out) > BIG:
        return {"cmd": cmd, "sha256": hashlib.sha256(out.encode()).hexdigest(), "len": len(out),
                "summary": summarize(out)}
    return {"cmd": cmd, "out": out}


def summarize(out):
    try:
        j = json.loads(out)
    except Exception:
        return None
    if "xfer" in j:
        return {"xfer": len(j["xfer"]), "local": len(j["local"]), "fg": len(j["fg"]),
                "bytes": sum(t[4] for t in j["xfer"])}
    return None


def main():
    if not os.path.exists(REF_TOOL):
        raise SystemExit("build the reference first: make -C oracle")
    cmds = kat_commands() + workload_commands() + random_commands(seed=20250428, n=1400)
    outs = run_ref(cmds)
    with open(os.path.join(HERE, "plans.jsonl"), "w") as f:
        for c, o in zip(cmds, outs):
            f.write(json.dumps(record(c, o)) + "\n")
    print(f"plans.jsonl: {len(cmds)} cases")

    xcmds = random_exec_commands(seed=7, n=700)
    xouts = run_ref(xcmds)
    kept = 0
    with open(os.path.join(HERE, "data.jsonl"), "w") as f:
        for c, o in zip(xcmds, xouts):
            j = json.loads(o)
            if "error" in j:
                continue
            j.pop("seconds", None)
            f.write(json.dumps({"cmd": c, "out": j}) + "\n")
            kept += 1
    print(f"data.jsonl: {kept} executed cases")


if __name__ == "__main__":
    main()
