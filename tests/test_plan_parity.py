"""Plan parity: the product planner (libhshard_b200.so) vs the REFERENCE planner.

Golden outputs in tests/golden/plans.jsonl were recorded by
tests/golden/make_golden.py from oracle/_ref/ref_tool, i.e. the reference's own
classify / build_table / make_plan / fuse / placement / convert_hsize
(compiled from /root/reference/proj/src).  Every case must match
byte-for-byte, errors by Errc name.  When the reference build is present the
comparison is also re-run live on fresh random cases.
"""
import hashlib
import json
import os
import random
import subprocess

import pytest

from planner_cmds import run

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "plans.jsonl")
REF_TOOL = os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref", "ref_tool")


def _cases():
    with open(GOLDEN) as f:
        return [json.loads(l) for l in f]


CASES = _cases()


def _canon_error(s):
    if s.startswith('{"error"'):
        return json.dumps({"error": json.loads(s)["error"]}, separators=(",", ":"))
    return s


@pytest.mark.parametrize("chunk", range(8))
def test_golden_plans(chunk):
    bad = []
    for i, case in enumerate(CASES):
        if i % 8 != chunk:
            continue
        got = run(case["cmd"])
        if "out" in case:
            ok = _canon_error(got) == _canon_error(case["out"])
        else:
            ok = hashlib.sha256(got.encode()).hexdigest() == case["sha256"]
        if not ok:
            bad.append((case["cmd"][0][:200], got[:300], case.get("out", case.get("summary"))))
    assert not bad, f"{len(bad)} mismatches, first: {bad[:3]}"


def test_golden_covers_every_step_kind():
    kinds = set()
    for case in CASES:
        o = case.get("out", "")
        if case["cmd"][0].startswith("C|") and o.startswith('{"src"'):
            p = json.loads(o)
            kinds |= {s["kind"] for s in p["bottom"] + p["top"]}
    assert kinds == {"Identity", "SendRecv", "AllReduce", "ReduceScatter", "AllGather",
                     "SplitAllReduce", "SplitReduceScatter", "SplitAllGather", "Bsr"}


def test_workload_plans_match_survey_numbers():
    """cfg4 808 transfers / 356 local / 20 groups / 10,108,289,024 B and the
    cfg5 cycle counts -- recorded from the reference, recomputed by the product."""
    from paper_2504_20490_b200 import hshard as H, workloads as W
    w = W.config4()
    j = H.plan_switch([(t, s, d, sh) for t, s, d, sh in w.transitions], "bf16").json()
    assert (len(j["xfer"]), len(j["local"]), len(j["fg"])) == (808, 356, 20)
    assert sum(t[4] for t in j["xfer"]) == 10108289024
    expect = {"S1S2": (3948, 1212, 14, 45554073600), "S2S3": (1692, 2340, 8, 39046348800),
              "S3S4": (282, 1170, 6, 6507724800), "S4S1": (2298, 606, 22, 22780354560)}
    for step, (nx, nl, ng, nb) in expect.items():
        w = W.config5(step)
        j = H.plan_switch([(t, s, d, sh) for t, s, d, sh in w.transitions], "bf16").json()
        assert (len(j["xfer"]), len(j["local"]), len(j["fg"]), sum(t[4] for t in j["xfer"])) == \
            (nx, nl, ng, nb), step


def test_bf16_plans_equal_f32_plans_up_to_bytes():
    """The reference has no BF16 (common.hpp:28); a bf16 plan must be the f32 plan with every
    byte count halved (heuristic III loads scale uniformly)."""
    from paper_2504_20490_b200 import hshard as H, workloads as W
    for w in [W.config2("e"), W.config3("b"), W.config1("B"), W.config1("C")]:
        t, s, d, sh = w.transitions[0]
        a = H.classify(s, d, sh, "f32").json()
        b = H.classify(s, d, sh, "bf16").json()
        assert b["dtype"] == "bf16"
        for step in a["bottom"] + a["top"]:
            if step["bsr"]:
                for x in step["bsr"]["xfer"]:
                    x[4] //= 2
        a["dtype"] = "bf16"
        assert a == b


@pytest.mark.skipif(not os.path.exists(REF_TOOL), reason="reference build (oracle/_ref) absent")
def test_live_random_sweep_against_reference():
    from gen_cases import random_commands
    cmds = random_commands(seed=random.randrange(1 << 30), n=300)
    text = "".join("\n".join(c) + "\n" for c in cmds)
    res = subprocess.run([REF_TOOL], input=text, capture_output=True, text=True, timeout=600)
    outs = res.stdout.splitlines()
    assert len(outs) == len(cmds)
    bad = [(c, o) for c, o in zip(cmds, outs) if _canon_error(run(c)) != _canon_error(o)]
    assert not bad, bad[:3]


def test_volume_report_matches_reference():
    """volume_report (reference bsr.hpp:107-108, bsr.cpp:244-261) over fused
    switch plans: the C ABI (hs_volume_report) and the CLI's JSON form
    (formats.volume_report) against the reference's own output recorded by
    ref_tool R (tests/golden/volume.jsonl, make_volume_golden.py)."""
    import json as _json
    from paper_2504_20490_b200 import formats as F
    from paper_2504_20490_b200 import hshard as H
    path = os.path.join(os.path.dirname(__file__), "golden", "volume.jsonl")
    cases = [_json.loads(l) for l in open(path)]
    assert len(cases) >= 40
    for c in cases:
        node_of = {int(k): v for k, v in c["node_of"].items()}
        ents = [(tid, src, dst, tuple(shape)) for tid, eb, shape, src, dst in c["entries"]]
        want = c["out"]
        try:
            plan = H.plan_switch(ents, {2: "bf16", 4: "f32", 8: "f64"}[c["entries"][0][1]])
            got = H.volume_report(plan, node_of)
        except H.HshardError as e:
            assert "error" in want and e.code == want["error"], (c["name"], e)
            continue
        assert "error" not in want, c["name"]
        assert {str(k): v for k, v in got.items()} == want, c["name"]
        js = F.volume_report(_json.loads(plan.dump())["xfer"], node_of=node_of)
        assert {str(k): v for k, v in js.items()} == want, c["name"]


@pytest.mark.skipif(not os.path.exists(REF_TOOL), reason="reference build (oracle/_ref) absent")
def test_live_align_sweep_against_reference():
    """align_shard_specs (reference annotation.cpp:431-472) on random count chains, half of
    them with equal totals so the common refinement usually exists."""
    rng = random.Random(random.randrange(1 << 30))
    keys = [-2, -1, 0, 1]

    def spec(counts):
        return "{" + ",".join(f"{rng.choice(keys)}:{c}" for c in counts) + "}"

    chains = [[2, 2, 2], [4, 2], [2, 4], [8], [2, 3], [3, 2], [6], [4, 4], [2, 8], [1, 4, 1]]
    cmds = [[f"A|{spec(rng.choice(chains))}|{spec(rng.choice(chains))}"] for _ in range(2000)]
    cmds += [[f"A|{spec([rng.choice([1, 2, 3, 4]) for _ in range(rng.randint(0, 3))])}|"
              f"{spec([rng.choice([1, 2, 3, 4]) for _ in range(rng.randint(0, 3))])}"] for _ in range(2000)]
    text = "".join(c[0] + "\n" for c in cmds)
    res = subprocess.run([REF_TOOL], input=text, capture_output=True, text=True, timeout=600)
    outs = res.stdout.splitlines()
    assert len(outs) == len(cmds)
    bad = [(c, o) for c, o in zip(cmds, outs) if run(c) != o]
    assert not bad, bad[:3]
