"""The SPEC's command line and wire formats (SPEC.md:93, 149, 270, 343, 445, 497,
504-528): annotation / graph JSON round trips, the tensor
binary format, each subcommand's output (plan-comm plans are checked against
the reference planner's recorded dumps), the exit-code contract, and
`simulate` on the B200."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2504_20490_b200 import formats as F
from paper_2504_20490_b200 import hshard as H
from paper_2504_20490_b200 import workloads as W
from paper_2504_20490_b200.strategy import dp_tp, llama_graph, tp_pp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def cli(*args, check_rc=None):
    r = subprocess.run([sys.executable, "-m", "paper_2504_20490_b200.cli", *args], capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    if check_rc is not None:
        assert r.returncode == check_rc, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])
    return r


def test_annotation_json_round_trip():
    from graph_cases import _anno, _groups
    import random
    rng = random.Random(7)
    annos = [t[1] for w in W.all_workloads() if w.kind == "classify" for t in w.transitions]
    annos += [t[2] for w in W.all_workloads() if w.kind == "classify" for t in w.transitions]
    annos += [_anno(rng, _groups(rng), 3) for _ in range(200)]
    for a in annos:
        keys = [[k for k, _ in spec] for spec in H.parse_annotation(a)["specs"]]
        if any(len(set(k)) != len(k) for k in keys):
            with pytest.raises(H.HshardError):  # the SPEC's {key: count} maps cannot repeat a key
                F.anno_to_json(a)
            continue
        j = F.anno_to_json(a)
        assert list(j) == ["dg_union", "ds_union", "hdim", "hsize", "hsplit_ratios"]  # canonical order
        back = F.anno_from_json(json.dumps(j))
        assert H.parse_annotation(back) == H.parse_annotation(a), a
    assert F.anno_from_json("hsize=1 hdim=-1 [(0){}]") == "hsize=1 hdim=-1 [(0){}]"


def test_tensor_binary_round_trip(tmp_path):
    for dt, arr in [("f32", np.arange(24, dtype=np.float32).reshape(2, 3, 4)),
                    ("bf16", np.arange(10, dtype=np.uint16)), ("i64", np.array([[-1, 2]], dtype=np.int64))]:
        p = str(tmp_path / f"{dt}.bin")
        F.write_tensor(p, arr, dt)
        back, bdt = F.read_tensor(p)
        assert bdt == dt and back.dtype == arr.dtype and np.array_equal(back, arr)
        raw = open(p, "rb").read()
        assert raw[:4] == b"HSTB" and json.loads(raw[8:8 + int.from_bytes(raw[4:8], "little")])["dtype"] == dt
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"nope")
    with pytest.raises(H.HshardError):
        F.read_tensor(str(bad))


def test_plan_comm_matches_reference_dumps(tmp_path):
    """plan-comm's "plan" is the canonical dump the reference planner produced (tests/golden/plans.jsonl)."""
    cases = [json.loads(l) for l in open(os.path.join(ROOT, "tests", "golden", "plans.jsonl"))]
    picked = [c for c in cases if c["cmd"][0].startswith("C|") and c.get("out", "").startswith('{"src"')][:12]
    assert len(picked) == 12
    for c in picked:
        _, dt, shape, bw, src, dst = c["cmd"][0].split("|")[:6]
        out = tmp_path / "p.json"
        cli("plan-comm", "--src", json.dumps(F.anno_to_json(src)), "--dst", dst, "--shape", shape,
            "--dtype", dt, "--bandwidth", bw, "--out", str(out), check_rc=0)
        got = json.load(open(out))
        assert got["version"] == "v1" and got["kind"] == "comm"
        assert got["plan"] == json.loads(c["out"]), c["cmd"][0]


def test_plan_comm_fig6_allreduce():
    r = cli("plan-comm", "--src", "hsize=1 hdim=-1 [(0,1,2,3){-2:4}]", "--dst", "hsize=1 hdim=-1 [(0,1,2,3){-1:4}]",
            "--shape", "8,8", check_rc=0)
    p = json.loads(r.stdout)["plan"]
    assert [s["kind"] for s in p["bottom"] + p["top"]] == ["AllReduce"]


def _graph_file(tmp_path):
    st = {"A": tp_pp(2, 2, 2), "B": tp_pp(4, 1, 2), "C": dp_tp([[0, 1, 2, 3], [4, 5], [6, 7]])}
    g, n = llama_graph(2, 64, 128, 256, st, dtype="f32")
    path = tmp_path / "g.json"
    path.write_text(json.dumps(F.graph_to_json(g)))
    return g, n, str(path)


def test_deduce_and_switch_plan(tmp_path):
    g, n, path = _graph_file(tmp_path)
    r = cli("deduce", "--graph", path, check_rc=0)
    d = json.loads(r.stdout)
    assert d["version"] == "v1" and all(s["ok"] for s in d["strategies"])
    ref = g.deduce()
    for t in d["tensors"]:
        for s in range(3):
            assert H.parse_annotation(F.anno_from_json(t["annotations"][str(s)])) == \
                H.parse_annotation(ref["strategies"][s]["slots"][t["id"]])
    one = json.loads(cli("deduce", "--graph", path, "--strategy", "2", check_rc=0).stdout)
    assert all(list(t["annotations"]) == ["2"] for t in one["tensors"])

    out = tmp_path / "sw.json"
    r = cli("switch-plan", "--graph", path, "--strategy", "0", "--strategy", "2", "--dtype", "f32",
            "--devices-per-node", "4", "--out", str(out), check_rc=0)
    sw = json.load(open(out))
    assert len(sw["entries"]) == len(g.diff(0, 2))
    assert sum(sum(v) for v in sw["volume"].values()) == sum(x[4] for x in sw["plan"]["xfer"])
    assert any(v[1] > 0 for v in sw["volume"].values())  # devices 4..7 are another "node"
    assert "intra-node MiB" in r.stderr  # the human table
    rep = cli("report", "--plan", str(out), check_rc=0).stdout
    assert "fusion groups" in rep and "device" in rep


def test_exit_codes(tmp_path):
    assert cli("frobnicate").returncode == 2                  # unknown subcommand: usage error
    assert cli("plan-comm", "--src", "x").returncode == 2     # missing flags: usage error
    r = cli("plan-comm", "--src", "hsize=1 hdim=-1 [(0,1,2,3){-2:4}]", "--dst", "hsize=1 hdim=-1 [(0,1){0:2}]",
            "--shape", "8,8", check_rc=1)
    err = json.loads(r.stdout)["error"]
    assert err["code"] == "PartialUnderBsr" and err["module"] == "plan-comm"
    assert cli("specialize").returncode == 2  # needs --graph and --strategy
    bad = tmp_path / "g.json"
    bad.write_text(json.dumps({"version": "v0", "nodes": []}))
    assert json.loads(cli("deduce", "--graph", str(bad), check_rc=1).stdout)["error"]["code"] == "ParseError"


@pytest.mark.gpu
def test_simulate_on_b200(tmp_path):
    """Partial -> hierarchical Split(1): every destination shard equals the input's slice."""
    w = W.config2("e")
    _, src, dst, _ = w.transitions[0]
    shape = (64, 256)
    plan = tmp_path / "p.json"
    cli("plan-comm", "--src", src, "--dst", dst, "--shape", "64,256", "--dtype", "f32", "--out", str(plan),
        check_rc=0)
    x = (np.arange(np.prod(shape)) % 97 - 48).astype(np.float32).reshape(shape)
    F.write_tensor(str(tmp_path / "x.bin"), x, "f32")
    out = tmp_path / "out"
    r = cli("simulate", "--plan", str(plan), "--input", str(tmp_path / "x.bin"), "--out", str(out), check_rc=0)
    rep = json.loads(r.stdout)
    assert rep["traffic"]["dst_bytes"] == x.nbytes * 3 // 2  # 4 devices x 1/8 (TP4 half) + 4 x 1/4 (TP2 half, x2)
    for d, s in rep["shards"].items():
        got, _ = F.read_tensor(str(out / s["file"]))
        box = tuple(slice(lo, hi) for lo, hi in s["bounds"])
        assert np.array_equal(got, x[box]), d


def test_specialize_and_pipelines(tmp_path):
    st = {"A": tp_pp(2, 2, 2), "B": tp_pp(2, 4, 4)}
    g, n = llama_graph(4, 64, 128, 256, {"A": tp_pp(2, 2, 4), "P": tp_pp(2, 4, 4)}, dtype="f32")
    path = tmp_path / "g.json"
    path.write_text(json.dumps(F.graph_to_json(g)))
    sp = json.loads(cli("specialize", "--graph", str(path), "--strategy", "1", "--bindings", "B=8",
                        check_rc=0).stdout)
    assert [e["device"] for e in sp["exec_graphs"]] == list(range(8))
    assert all(node["plan"] is not None for e in sp["exec_graphs"] for node in e["nodes"] if node["comm"])
    r = cli("pipelines", "--graph", str(path), "--strategy", "1", "--bindings", "B=8", check_rc=0)
    assert json.loads(r.stdout)["pipelines"] == [[[0, 1], [2, 3], [4, 5], [6, 7]]]
    assert "stage" in r.stderr
