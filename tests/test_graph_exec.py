"""Executable-graph integration (reference specialize.cpp:57-122,
specialize.hpp:35-38): the CommOps of the specialized ExecGraphs, re-derived per
micro-batch binding, and executed on the GPU against the oracle."""
import numpy as np
import pytest

from oracle import executor as ox
from paper_2504_20490_b200 import hshard as H
from paper_2504_20490_b200 import strategy as S
from paper_2504_20490_b200.graph_exec import CommOpExecutor


def _graph():
    strategies = {"tp2pp2": S.tp_pp(2, 2, 2), "tp4": S.tp_pp(4, 1, 2),
                  "dp2tp2": S.dp_tp([[0, 1], [2, 3]])}
    return S.llama_graph(2, 64, 128, 64, strategies)


def _strip_regions(plan):
    """Kinds and groups of a plan (what does not depend on shapes, specialize.hpp:35-38)."""
    return [(s["kind"], s["sub"], s["groups"], s["pairs"]) for s in plan["bottom"] + plan["top"]]


@pytest.mark.parametrize("strategy", ["tp2pp2", "tp4", "dp2tp2"])
def test_comm_ops_rederived_per_binding(strategy):
    g, names = _graph()
    ex = CommOpExecutor(None, g, names[strategy], "bf16", 4, {"B": 8})
    assert ex.comm_ops
    for node, op in ex.comm_ops.items():
        # at the reference binding: byte-identical to the plan instantiate() embedded
        # (which test_graph_parity pins to the reference's specialize)
        p, hit = ex.plan(node, {"B": 8})
        assert not hit and p.json() == op["reference_plan"], node
        assert ex.plan(node, {"B": 8})[1]  # cached
        for b in (2, 4, 6):
            q, _ = ex.plan(node, {"B": b})
            assert q.json()["shape"][0] in (b, 64)
            assert _strip_regions(q.json()) == _strip_regions(op["reference_plan"]), (node, b)


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["tp2pp2", "dp2tp2"])
def test_comm_ops_execute_per_micro_batch(gpu_ctx, strategy):
    """Every CommOp of the ExecGraphs, for micro-batches of 2, 4 and 6 rows (a
    GPipe-style schedule's sizes), runs on the GPU bit-exactly vs the oracle;
    equal sizes reuse one compiled program."""
    g, names = _graph()
    mark = gpu_ctx.alloc(0)
    ex = CommOpExecutor(gpu_ctx, g, names[strategy], "bf16", 4, {"B": 8})
    try:
        for rnd in range(2):
            for b in (2, 4, 6):
                for node, op in ex.comm_ops.items():
                    prog, lay, info = ex.program(node, {"B": b})
                    assert info["program_cached"] == (rnd == 1)
                    seed = 100 * b + node
                    lay.fill_src(seed, "real")
                    prog.run()
                    gpu_ctx.sync()
                    plan = ex.plan(node, {"B": b})[0]
                    src = ox.scatter(op["src"], plan.json()["shape"], "bf16", seed, 0, "real")
                    want = ox.execute_plan(plan.json(), src, "bf16")
                    for (slot, dev) in lay.dst:
                        got = lay.read("dst", slot, dev)
                        assert np.array_equal(got, want[dev]), (strategy, node, b, dev)
    finally:
        ex.close()
        gpu_ctx.reset(mark)
