"""hshard command line.

    python -m paper_2504_20490_b200.cli deduce      --graph g.json [--strategy S] [--out F]
    python -m paper_2504_20490_b200.cli plan-comm   --src A --dst B --shape 8192,8192 [--dtype bf16]
    python -m paper_2504_20490_b200.cli switch-plan --graph g.json --strategy A --strategy B [--bindings B=8]
    python -m paper_2504_20490_b200.cli report      --plan plan.json [--devices-per-node 8]
    python -m paper_2504_20490_b200.cli simulate    --plan plan.json --input x.bin --out DIR   (B200)
    python -m paper_2504_20490_b200.cli specialize  --graph g.json --strategy S [--bindings B=8]
    python -m paper_2504_20490_b200.cli pipelines   --graph g.json --strategy S [--bindings B=8]

Annotations (--src / --dst) are annotation JSON files, inline annotation
JSON, or the annotation text form; graphs are graph JSON v1; tensors use the
binary format of formats.py.  Every JSON output carries "version".  Exit 0 on
success, 1 with a structured error report {"version", "error": {"module",
"op", "code", "message"}} on a failure, 2 on a usage error (including an
unknown subcommand).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

from . import formats as F
from . import hshard as H

SUBCOMMANDS = ["deduce", "plan-comm", "switch-plan", "report", "simulate", "specialize", "pipelines"]


def _read_json_arg(v: str):
    """A path to a JSON file, or inline JSON / text."""
    if os.path.exists(v):
        with open(v) as f:
            return f.read()
    return v


def _bindings(items):
    out = {}
    for item in items or []:
        for kv in item.split(","):
            if kv.strip():
                k, _, v = kv.partition("=")
                if not _:
                    raise H.HshardError("ParseError", f"binding {kv!r} lacks '='")
                out[k.strip()] = int(v)
    return out


def _emit(obj, out, text=None):
    s = json.dumps(obj, separators=(",", ":"))
    if out:
        with open(out, "w") as f:
            f.write(s + "\n")
    else:
        print(s)
    if text:
        print(text, file=sys.stderr)


# ---------------------------------------------------------------- subcommands
def cmd_deduce(a):
    g = F.graph_from_json(_read_json_arg(a.graph))
    res = F.deduced_graph_json(g)
    if a.strategy:
        s = int(a.strategy[0])
        if not 0 <= s < len(res["strategies"]):
            raise H.HshardError("UndeducedStrategy", f"graph has no strategy {s}")
        if not res["strategies"][s]["ok"]:
            raise H.HshardError(res["strategies"][s]["error"], f"strategy {s} does not deduce")
        for t in res["tensors"]:
            t["annotations"] = {str(s): t["annotations"][str(s)]}
        res["strategies"] = [res["strategies"][s]]
    _emit(res, a.out)


def cmd_plan_comm(a):
    src, dst = F.anno_from_json(_read_json_arg(a.src)), F.anno_from_json(_read_json_arg(a.dst))
    shape = [int(x) for x in a.shape.split(",")]
    plan = H.classify(src, dst, shape, a.dtype, a.bandwidth)
    _emit({"version": F.VERSION, "kind": "comm", "src": F.anno_to_json(src), "dst": F.anno_to_json(dst),
           "shape": shape, "dtype": a.dtype, "plan": json.loads(plan.dump())}, a.out)


def cmd_switch_plan(a):
    if not a.strategy or len(a.strategy) != 2:
        raise H.HshardError("ParseError", "switch-plan needs exactly two --strategy")
    g = F.graph_from_json(_read_json_arg(a.graph))
    sa, sb = int(a.strategy[0]), int(a.strategy[1])
    entries = g.diff(sa, sb, _bindings(a.bindings))
    plan = H.plan_switch([(e["tensor"], e["src"], e["dst"], tuple(e["shape"])) for e in entries], a.dtype,
                         a.bandwidth)
    pj = json.loads(plan.dump())
    devs = sorted({d for e in entries for an in (e["src"], e["dst"])
                   for g in H.parse_annotation(an)["groups"] for d in g})
    vol = H.volume_report(plan, {d: d // a.devices_per_node for d in devs})  # reference bsr.cpp:244-261
    rows = [(d, f"{v[0] / 2**20:.1f}", f"{v[1] / 2**20:.1f}") for d, v in vol.items()]
    _emit({"version": F.VERSION, "kind": "switch", "strategies": [sa, sb], "dtype": a.dtype,
           "entries": [{**e, "src": F.anno_to_json(e["src"]), "dst": F.anno_to_json(e["dst"])} for e in entries],
           "plan": pj, "volume": {str(d): v for d, v in vol.items()}},
          a.out, F.table(rows, ["device", "intra-node MiB", "inter-node MiB"]))


def _plan_from_file(obj):
    if obj.get("version") != F.VERSION:
        raise H.HshardError("ParseError", "plan JSON version mismatch")
    if obj["kind"] == "comm":
        return H.classify(F.anno_from_json(obj["src"]), F.anno_from_json(obj["dst"]), obj["shape"], obj["dtype"])
    entries = [(e["tensor"], F.anno_from_json(e["src"]), F.anno_from_json(e["dst"]), tuple(e["shape"]))
               for e in obj["entries"]]
    return H.plan_switch(entries, obj["dtype"])


def cmd_report(a):
    obj = json.loads(_read_json_arg(a.plan))
    pj = obj["plan"]
    lines = []
    if obj["kind"] == "comm":
        rows = [(ph, s["kind"], s["sub"], len(s["groups"]) or len(s["pairs"]) or len(s["slices"]))
                for ph in ("bottom", "top") for s in pj[ph]]
        lines.append(F.table(rows, ["phase", "step", "subgroup", "groups/pairs/slices"]))
        xfer = [x for ph in ("bottom", "top") for s in pj[ph] if s["bsr"] for x in s["bsr"]["xfer"]]
    else:
        xfer = pj["xfer"]
        lines.append(f"{len(obj['entries'])} parameters, {len(pj['xfer'])} transfers, "
                     f"{len(pj['local'])} local copies, {len(pj['fg'])} fusion groups")
    vol = F.volume_report(xfer, a.devices_per_node)
    if vol:
        lines.append(F.table([(d, f"{v[0] / 2**20:.1f}", f"{v[1] / 2**20:.1f}") for d, v in vol.items()],
                             ["device", "intra-node MiB", "inter-node MiB"]))
    print("\n\n".join(lines))


def cmd_simulate(a):
    """Execute a plan on cuda:0 (every virtual device on one B200) from a logical input tensor."""
    import numpy as np
    from .executor import Context, Program, ShardLayout
    obj = json.loads(_read_json_arg(a.plan))
    if obj.get("kind") != "comm":
        raise H.HshardError("UnsupportedOp", "simulate takes a plan-comm plan (one tensor)")
    plan = _plan_from_file(obj)
    src, dst = F.anno_from_json(obj["src"]), F.anno_from_json(obj["dst"])
    x, dt = F.read_tensor(a.input)
    if list(x.shape) != list(obj["shape"]) or dt != obj["dtype"]:
        raise H.HshardError("ShapeMismatch", f"input {list(x.shape)} {dt} vs plan {obj['shape']} {obj['dtype']}")
    devs = sorted({d for an in (src, dst) for g in H.parse_annotation(an)["groups"] for d in g})
    cluster = json.loads(_read_json_arg(a.cluster)) if a.cluster else {}
    n_virtual = int(cluster.get("n_virtual", devs[-1] + 1))
    ctx = Context(max(1 << 30, 4 * x.nbytes * len(devs)))
    try:
        lay = ShardLayout(ctx, plan, n_virtual)
        top_partial = H.parse_annotation(src)["hdim"] == -2 and H.parse_annotation(src)["hsize"] > 1
        groups = H.parse_annotation(src)["groups"]
        for (slot, d), rec in lay.src.items():  # scatter (sim.hpp / SPEC.md:476-489)
            p = H.placement(src, obj["shape"], d)
            box = tuple(slice(lo, hi) for lo, hi in p["bounds"])
            carries = p["partial"][0] == 0 and (not top_partial or d in groups[0])
            lay.write("src", slot, d, x[box] if carries else np.zeros_like(x[box]))
        prog = Program(ctx, plan, lay)
        prog.run()
        ctx.sync()
        t0 = time.perf_counter()
        prog.run()
        ctx.sync()
        ms = (time.perf_counter() - t0) * 1e3
        os.makedirs(a.out, exist_ok=True)
        shards = {}
        for (slot, d), rec in sorted(lay.dst.items()):
            path = os.path.join(a.out, f"dst_dev{d}.bin")
            F.write_tensor(path, lay.read("dst", slot, d), dt)
            shards[str(d)] = {"file": os.path.basename(path), "bounds": H.placement(dst, obj["shape"], d)["bounds"]}
        st = prog.stats()
        report = {"version": F.VERSION, "shards": shards, "wall_ms": ms,
                  "traffic": {k: st[k] for k in ("hbm_read", "hbm_write", "nvlink_in", "nvlink_out", "dst_bytes")},
                  "kernels_per_run": st["kernels_per_run"]}
        with open(os.path.join(a.out, "traffic.json"), "w") as f:
            json.dump(report, f, indent=1)
        print(json.dumps(report, indent=1))
        prog.close()
    finally:
        ctx.close()


def _specialized(a):
    g = F.graph_from_json(_read_json_arg(a.graph))
    if not a.strategy:
        raise H.HshardError("ParseError", f"{a.cmd} needs --strategy")
    s = int(a.strategy[0])
    return s, g.specialize(s, _bindings(a.bindings))


def cmd_specialize(a):
    """One ExecGraph JSON per device: nodes with their phase and resolved CommPlans."""
    s, r = _specialized(a)
    _emit({"version": F.VERSION, "strategy": s, "phases": r["phases"],
           "exec_graphs": [{**e, "strategy": s} for e in r["exec_graphs"]]}, a.out)


def cmd_pipelines(a):
    """Pipeline structure JSON: stages of device groups per pipeline."""
    s, r = _specialized(a)
    if "pipelines_error" in r:
        raise H.HshardError(r["pipelines_error"], "the strategy's communication is not a set of pipelines")
    rows = [(p, st, ",".join(map(str, devs))) for p, pipe in enumerate(r["pipelines"]) for st, devs in enumerate(pipe)]
    _emit({"version": F.VERSION, "strategy": s, "pipelines": r["pipelines"]}, a.out,
          F.table(rows, ["pipeline", "stage", "devices"]))


COMMANDS = {"deduce": cmd_deduce, "plan-comm": cmd_plan_comm, "switch-plan": cmd_switch_plan,
            "report": cmd_report, "simulate": cmd_simulate, "specialize": cmd_specialize,
            "pipelines": cmd_pipelines}


def parser():
    ap = argparse.ArgumentParser(prog="hshard", description=__doc__.split("\n\n")[0])
    ap.add_argument("cmd", choices=SUBCOMMANDS)
    ap.add_argument("--graph")
    ap.add_argument("--strategy", action="append")
    ap.add_argument("--cluster")
    ap.add_argument("--src")
    ap.add_argument("--dst")
    ap.add_argument("--shape")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--bandwidth", default="u")
    ap.add_argument("--bindings", action="append")
    ap.add_argument("--plan")
    ap.add_argument("--input")
    ap.add_argument("--devices-per-node", type=int, default=8)
    ap.add_argument("--out")
    ap.add_argument("--seed", type=int, default=0)
    return ap


def main(argv=None) -> int:
    a = parser().parse_args(argv)  # usage errors exit 2
    need = {"deduce": ["graph"], "plan-comm": ["src", "dst", "shape"], "switch-plan": ["graph"],
            "report": ["plan"], "simulate": ["plan", "input", "out"], "specialize": ["graph", "strategy"],
            "pipelines": ["graph", "strategy"]}.get(a.cmd, [])
    missing = [f"--{n}" for n in need if getattr(a, n) is None]
    if missing:
        parser().print_usage(sys.stderr)
        print(f"hshard {a.cmd}: missing {' '.join(missing)}", file=sys.stderr)
        return 2
    try:
        COMMANDS[a.cmd](a)
        return 0
    except H.HshardError as e:
        err = {"module": a.cmd, "op": COMMANDS[a.cmd].__name__, "code": e.code, "message": str(e)}
    except (OSError, ValueError, KeyError, json.JSONDecodeError) as e:
        err = {"module": a.cmd, "op": COMMANDS[a.cmd].__name__, "code": "ParseError", "message": repr(e)}
    print(json.dumps({"version": F.VERSION, "error": err}))
    return 1


if __name__ == "__main__":
    sys.exit(main())
