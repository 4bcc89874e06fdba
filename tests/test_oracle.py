"""Pins the numpy oracle executor (oracle/executor.py) before it is trusted.

1. Against the REFERENCE: tests/golden/data.jsonl holds, for random plans, the
   destination shards produced by oracle/_ref/ref_tool's executor, which runs
   the reference planner's CommPlan through the reference's own per-cell
   Tensor::slice / write_slice / add_slice (tensor.cpp:84-114).  On the exact
   integer grid the oracle must reproduce every value bit-exactly.
2. SPEC acceptance #2: reassembly invariance over a random
   sweep; only the reference's align_shard_specs defect class
   may fail, and it must fail loudly with UnexecutableStep.
"""
import json
import os
import random

import numpy as np
import pytest

from gen_cases import rand_pair, zero_width
from oracle import datagen as dg
from oracle import executor as ox
from paper_2504_20490_b200 import hshard as H

DATA = os.path.join(os.path.dirname(__file__), "golden", "data.jsonl")


def _data_cases():
    with open(DATA) as f:
        return [json.loads(l) for l in f]


def test_oracle_matches_reference_primitive_executor():
    cases = _data_cases()
    assert len(cases) > 300
    for case in cases:
        _, dt, shp, bw, src, dst, seed, mode, _, _ = case["cmd"][0].split("|")
        shape = [int(x) for x in shp.split(",")]
        plan = H.classify(src, dst, shape, dt, bw).json()
        out = ox.execute_plan(plan, ox.scatter(src, shape, dt, int(seed), 0, mode), dt)
        ref = case["out"]["shards"]
        assert sorted(int(d) for d in ref) == sorted(out), case["cmd"]
        for d, v in ref.items():
            got = dg.decode(out[int(d)], dt).ravel()
            assert np.array_equal(got, np.asarray(v["v"], dtype=np.float64)), (case["cmd"], d)
        nbytes = sum(a.size for a in out.values()) * H.DTYPE_BYTES[dt]
        assert nbytes == case["out"]["dst_bytes"]


def test_datagen_pieces_sum_to_logical():
    rng = random.Random(3)
    for _ in range(200):
        src, dst, shape = rand_pair(rng)
        try:
            H.validate(src, shape)
            if H.validate(src, shape):
                continue
        except H.HshardError:
            continue
        if zero_width(src, shape):
            continue
        shards = ox.scatter(src, shape, "bf16", 11, 0, "grid")
        x = ox.reassemble(src, shards, shape, "bf16")
        lin = dg.box_linear_indices(shape, [[0, s] for s in shape])
        assert np.array_equal(x, dg.logical_grid(lin, 11, 0).astype(np.float64)), src


@pytest.mark.parametrize("dtype", ["bf16", "f32", "i64"])
def test_reassembly_invariance_sweep(dtype):
    rng = random.Random({"bf16": 1, "f32": 2, "i64": 3}[dtype])
    executed = unexecutable = 0
    kinds = set()
    while executed < 500:
        src, dst, shape = rand_pair(rng)
        if zero_width(src, shape) or zero_width(dst, shape):
            continue
        try:
            plan = H.classify(src, dst, shape, dtype).json()
        except H.HshardError:
            continue
        seed = rng.randrange(1 << 20)
        try:
            out = ox.execute_plan(plan, ox.scatter(src, shape, dtype, seed, 0, "grid"), dtype)
        except ox.OracleError as e:
            assert e.code == "UnexecutableStep"
            assert any(s["kind"] in ("AllGather", "ReduceScatter", "AllReduce")
                       for s in plan["bottom"]), plan
            unexecutable += 1
            continue
        executed += 1
        kinds |= {s["kind"] for s in plan["bottom"] + plan["top"]}
        x = ox.reassemble(dst, out, shape, dtype)
        lin = dg.box_linear_indices(shape, [[0, s] for s in shape])
        assert np.array_equal(x, dg.logical_grid(lin, seed, 0).astype(np.float64)), (src, dst)
    assert len(kinds) == 9, kinds
    assert unexecutable < 25


def test_appendix_b1_repros_rejected():
    for src, dst, shape in [
        ("hsize=1 hdim=-1 [(3,5,2,7){1:4}]", "hsize=1 hdim=-1 [(3,5,2,7){-1:2,1:2}]", [12, 4]),
        ("hsize=1 hdim=-1 [(2,5,6,4){-2:2,0:2}]", "hsize=1 hdim=-1 [(2,5,6,4){0:4}]", [16, 8]),
    ]:
        plan = H.classify(src, dst, shape, "f32").json()
        with pytest.raises(ox.OracleError) as ei:
            ox.execute_plan(plan, ox.scatter(src, shape, "f32", 1), "f32")
        assert ei.value.code == "UnexecutableStep"
