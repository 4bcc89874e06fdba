"""GPU parity: the sm_100a executor (libhshard_b200.so) vs the CPU oracle.

* random plans of every step kind, every dtype, exact-grid and real-valued
  payloads: destination shards must be BIT-IDENTICAL to oracle/executor.py
  (same fixed reduction order, fp32 accumulation for bf16/f32, one rounding
  per plan phase -- the stated tolerance for Partial reductions is therefore
  zero ulp against the oracle; against the reference's double-precision
  executor it is exact on the grid, see test_oracle.py);
* the on-GPU payload generator must equal oracle/datagen.py;
* BASELINE workloads at FULL size: configs 1-2 against the oracle; every
  reduction config (2a/2b/2d/2e, 3a/3b/3c) with real-valued, order-sensitive
  payloads against the native CPU executor (oracle/_ref/ref_tool N); configs
  3-5 also through size-independent properties (every Partial-free
  destination shard equals the logical counter-hash tensor on its box);
* the host-buffer (e2e) path and the Appendix-B1 rejection.
"""
import random

import numpy as np
import pytest

from gen_cases import rand_pair, zero_width
from oracle import datagen as dg
from oracle import executor as ox
from paper_2504_20490_b200 import hshard as H
from paper_2504_20490_b200 import workloads as W

pytestmark = pytest.mark.gpu


# default (fused, TMA, merged outputs), the plain register path, TMA bulk stores for
# copies with 16 KB items
FLAG_SETS = [0, 2 | 4 | 8, (1 << 25) | (1 << 27)]


def _gpu_case(ctx, plan, src, dst, shape, dtype, seed, mode, n_virtual=10, flag_sets=FLAG_SETS):
    from paper_2504_20490_b200.executor import Program, ShardLayout
    mark = ctx.alloc(0)
    try:
        lay = ShardLayout(ctx, plan, n_virtual)
        lay.fill_src(seed, mode)
        ref_src = ox.scatter(src, shape, dtype, seed, 0, mode)
        for (slot, dev) in lay.src:
            got = lay.read("src", 0, dev)
            assert np.array_equal(got.view(np.uint8), ref_src[dev].view(np.uint8)), ("fill", dev)
        want = ox.execute_plan(plan.json(), ref_src, dtype)
        stats = None
        for flags in flag_sets:
            lay.clear_dst()
            prog = Program(ctx, plan, lay, flags)
            prog.run()
            ctx.sync()
            for (slot, dev) in lay.dst:
                got = lay.read("dst", 0, dev)
                assert np.array_equal(got.view(np.uint8), want[dev].view(np.uint8)), \
                    (flags, src, dst, dev)
            stats = stats or prog.stats()
            prog.close()
        return stats
    finally:
        ctx.reset(mark)


@pytest.mark.parametrize("dtype", ["bf16", "f32", "f64", "i32", "i64"])
def test_random_plans_bit_exact(gpu_ctx, dtype):
    rng = random.Random({"bf16": 1, "f32": 2, "f64": 3, "i32": 4, "i64": 5}[dtype])
    kinds, done = set(), 0
    while done < 120:
        src, dst, shape = rand_pair(rng)
        if zero_width(src, shape) or zero_width(dst, shape):
            continue
        try:
            plan = H.classify(src, dst, shape, dtype)
        except H.HshardError:
            continue
        j = plan.json()
        try:
            ox.execute_plan(j, ox.scatter(src, shape, dtype, 1), dtype)
        except ox.OracleError:
            continue  # Appendix-B1 class, covered below
        mode = "real" if (done % 2 and dtype in ("bf16", "f32", "f64")) else "grid"
        _gpu_case(gpu_ctx, plan, src, dst, shape, dtype, rng.randrange(1 << 30), mode)
        kinds |= {s["kind"] for s in j["bottom"] + j["top"]}
        done += 1
    assert len(kinds) >= 8, kinds


def test_zero_width_top_tier_slices(gpu_ctx):
    """validate accepts top-tier ratio slices that floor to zero
    width (annotation.cpp:304-318); the reference's Tensor::slice then throws
    (tensor.cpp:55-57).  Here an empty box is simply no work: the devices of a
    zero-width subgroup hold empty shards and every other shard must still be
    bit-identical to the oracle."""
    rng = random.Random(33)
    done = tries = 0
    while done < 40 and tries < 20000:
        tries += 1
        src, dst, shape = rand_pair(rng)
        shape = [rng.choice([1, 2, 3, 4, 6]) if rng.random() < 0.7 else x for x in shape]
        if not (zero_width(src, shape) or zero_width(dst, shape)):
            continue
        try:
            plan = H.classify(src, dst, shape, "f32")
            ox.execute_plan(plan.json(), ox.scatter(src, shape, "f32", 1), "f32")
        except (H.HshardError, ox.OracleError):
            continue
        _gpu_case(gpu_ctx, plan, src, dst, shape, "f32", rng.randrange(1 << 30), "grid")
        done += 1
    assert done >= 20, done


def test_appendix_b1_rejected_on_compile(gpu_ctx):
    from paper_2504_20490_b200.executor import Program, ShardLayout
    src, dst = "hsize=1 hdim=-1 [(3,5,2,7){1:4}]", "hsize=1 hdim=-1 [(3,5,2,7){-1:2,1:2}]"
    plan = H.classify(src, dst, [12, 4], "f32")
    mark = gpu_ctx.alloc(0)
    lay = ShardLayout(gpu_ctx, plan, 8)
    with pytest.raises(H.HshardError) as ei:
        Program(gpu_ctx, plan, lay)
    assert ei.value.code == "UnexecutableStep"
    gpu_ctx.reset(mark)


def test_switch_random_bit_exact(gpu_ctx):
    from paper_2504_20490_b200.executor import Program, ShardLayout
    rng = random.Random(5)
    for it in range(30):
        entries = []
        while len(entries) < rng.randint(1, 5):
            s, d, shp = rand_pair(rng, partial_ok=False)
            if zero_width(s, shp) or zero_width(d, shp):
                continue
            try:
                H.build_table(s, d, shp)
            except H.HshardError:
                continue
            entries.append((len(entries) * 2 + 1, s, d, shp))
        plan = H.plan_switch(entries, "bf16")
        mark = gpu_ctx.alloc(0)
        lay = ShardLayout(gpu_ctx, plan, 10)
        lay.fill_src(it, "real")
        src = {}
        for slot, (tid, s, d, shp) in enumerate(entries):
            for dev, a in ox.scatter(s, shp, "bf16", it, tid, "real").items():
                src[(tid, dev)] = a
        want = ox.execute_switch(plan.json(), entries, src, "bf16")
        for flags in (0, 1 << 25):  # default and TMA bulk stores
            lay.clear_dst()
            prog = Program(gpu_ctx, plan, lay, flags)
            prog.run()
            gpu_ctx.sync()
            for (slot, dev) in lay.dst:
                tid = entries[slot][0]
                assert np.array_equal(lay.read("dst", slot, dev), want[(tid, dev)]), (it, flags, slot, dev)
            prog.close()
        gpu_ctx.reset(mark)


@pytest.mark.parametrize("name", ["cfg1A", "cfg1B", "cfg1C", "cfg1D", "cfg2e", "cfg2b"])
def test_workload_full_size_vs_oracle(gpu_ctx, name):
    w = W.by_name(name)
    tid, src, dst, shape = w.transitions[0]
    plan = H.classify(src, dst, shape, w.dtype)
    st = _gpu_case(gpu_ctx, plan, src, dst, shape, w.dtype, 1234, "real", w.n_virtual)
    assert st["hbm_write"] == st["dst_bytes"] or plan.json()["mid"] is not None


@pytest.mark.parametrize("name", ["cfg3b", "cfg3a", "cfg3c", "cfg2a", "cfg2d", "cfg2e", "cfg2b",
                                  "cfg2e:f32", "cfg3b:f32"])
def test_workload_full_size_real_vs_native(gpu_ctx, name, tmp_path):
    """Rounding- and order-sensitive parity at FULL size: real-valued payloads
    through the reduction configs, every destination shard byte-compared with
    the native CPU executor (oracle/_ref/ref_tool N, pinned to the numpy oracle
    in test_native_oracle.py): ascending-id fp32 sums, one rounding per plan
    phase, reproduced by the fused GPU program and by the plain register path.
    In bf16 the rounding points decide the bits; the ":f32" variants (same
    annotations, f32 storage) make the summation order decide them too."""
    import native_ref
    from paper_2504_20490_b200.executor import Program, ShardLayout
    if not native_ref.available():
        pytest.skip("oracle/_ref/ref_tool not built")
    w = W.by_name(name.split(":")[0])
    dtype = name.split(":")[1] if ":" in name else w.dtype
    tid, src, dst, shape = w.transitions[0]
    plan = H.classify(src, dst, shape, dtype)
    _, want = native_ref.run(src, dst, shape, dtype, 4321, "real", 0, str(tmp_path))
    mark = gpu_ctx.alloc(0)
    try:
        lay = ShardLayout(gpu_ctx, plan, w.n_virtual)
        lay.fill_src(4321, "real")
        for flags in (0, 2 | 4 | 8):
            lay.clear_dst()
            prog = Program(gpu_ctx, plan, lay, flags)
            prog.run()
            gpu_ctx.sync()
            for (slot, dev) in lay.dst:
                got = lay.read("dst", 0, dev).ravel()
                assert np.array_equal(got.view(np.uint8), want[dev].view(np.uint8)), (name, flags, dev)
            prog.close()
    finally:
        gpu_ctx.reset(mark)


@pytest.mark.parametrize("name", ["cfg3b", "cfg3a", "cfg3c", "cfg2a", "cfg2d"])
def test_workload_full_size_properties(gpu_ctx, name):
    from paper_2504_20490_b200.executor import Program, ShardLayout
    w = W.by_name(name)
    tid, src, dst, shape = w.transitions[0]
    plan = H.classify(src, dst, shape, w.dtype)
    mark = gpu_ctx.alloc(0)
    try:
        lay = ShardLayout(gpu_ctx, plan, w.n_virtual)
        lay.fill_src(77, "grid")
        lay.clear_dst()
        Program(gpu_ctx, plan, lay).run()
        gpu_ctx.sync()
        assert lay.verify_dst(77) == 0
    finally:
        gpu_ctx.reset(mark)


@pytest.mark.parametrize("name", ["cfg4", "cfg5_S3S4", "cfg5_S4S1", "cfg5_S1S2", "cfg5_S2S3"])
def test_switch_full_size_properties(gpu_ctx, name):
    from paper_2504_20490_b200.executor import Program, ShardLayout
    w = W.by_name(name)
    need = W.resident_bytes(w)
    if need * 1.02 > gpu_ctx.arena_bytes:
        pytest.skip("arena too small for this switch at full size")
    plan = H.plan_switch(w.transitions, w.dtype)
    mark = gpu_ctx.alloc(0)
    try:
        lay = ShardLayout(gpu_ctx, plan, w.n_virtual)
        lay.fill_src(5, "grid")
        for flags in (0, 1 << 25):  # default and TMA bulk stores
            lay.clear_dst()
            prog = Program(gpu_ctx, plan, lay, flags)
            prog.run()
            gpu_ctx.sync()
            assert lay.verify_dst(5) == 0, flags
            prog.close()
    finally:
        gpu_ctx.reset(mark)


def test_host_buffer_path(gpu_ctx):
    from paper_2504_20490_b200.executor import Program, ShardLayout
    w = W.config2("e")
    tid, src, dst, shape = w.transitions[0]
    shape = (1024, 2048)
    plan = H.classify(src, dst, shape, "bf16")
    mark = gpu_ctx.alloc(0)
    try:
        lay = ShardLayout(gpu_ctx, plan, 8)
        srcs = ox.scatter(src, shape, "bf16", 9, 0, "real")
        host_src = {(0, d): a for d, a in srcs.items()}
        host_dst = {(0, d): np.zeros(r["ext"], dtype=np.uint16) for (s, d), r in lay.dst.items()}
        Program(gpu_ctx, plan, lay).run_host(host_src, host_dst)
        want = ox.execute_plan(plan.json(), srcs, "bf16")
        for (s, d), a in host_dst.items():
            assert np.array_equal(a, want[d])
    finally:
        gpu_ctx.reset(mark)


def test_host_buffer_path_pipelined(gpu_ctx):
    """hs_prog_run_host_async: two programs over two layouts alternate on three
    streams; every step's outputs are that step's inputs resharded."""
    import torch
    from paper_2504_20490_b200.executor import Program, ShardLayout
    w = W.config2("e")
    tid, src, dst, shape = w.transitions[0]
    shape = (512, 1024)
    plan = H.classify(src, dst, shape, "bf16")
    mark = gpu_ctx.alloc(0)
    try:
        lays = [ShardLayout(gpu_ctx, plan, 8) for _ in range(2)]
        progs = [Program(gpu_ctx, plan, l) for l in lays]
        streams = [torch.cuda.Stream() for _ in range(3)]
        h2d, comp, d2h = (s.cuda_stream for s in streams)
        steps = []
        for k in range(4):
            srcs = ox.scatter(src, shape, "bf16", 20 + k, 0, "real")
            host_src = {(0, d): a for d, a in srcs.items()}
            host_dst = {(0, d): np.zeros(r["ext"], dtype=np.uint16) for (s, d), r in lays[k % 2].dst.items()}
            progs[k % 2].run_host_async(host_src, host_dst, h2d, comp, d2h)
            steps.append((srcs, host_src, host_dst))
        streams[2].synchronize()
        for srcs, _, host_dst in steps:
            want = ox.execute_plan(plan.json(), srcs, "bf16")
            for (s, d), a in host_dst.items():
                assert np.array_equal(a, want[d])
    finally:
        gpu_ctx.reset(mark)


def test_graph_derived_switch_on_gpu(gpu_ctx):
    """Strategy source -> executor: diff_strategies of a Llama-shaped graph
    (TP2xPP2 -> TP4 on 4 virtual devices), planned and executed on the B200,
    every destination shard checked against the counter-hash ground truth."""
    from paper_2504_20490_b200.executor import Program, ShardLayout
    from paper_2504_20490_b200.strategy import llama_graph, tp_pp
    g, n = llama_graph(4, 256, 512, 1024, {"A": tp_pp(2, 2, 4), "B": tp_pp(4, 1, 4)})
    plan = g.switch_plan(n["A"], n["B"], "bf16")
    assert len(plan.json()["xfer"]) > 0
    mark = gpu_ctx.alloc(0)
    try:
        lay = ShardLayout(gpu_ctx, plan, 4)
        lay.fill_src(8, "grid")
        lay.clear_dst()
        Program(gpu_ctx, plan, lay).run()
        gpu_ctx.sync()
        assert lay.verify_dst(8) == 0
    finally:
        gpu_ctx.reset(mark)


def _random_param_anno(rng, rank):
    """A random Partial-free annotation on 4 virtual devices (switches move weights)."""
    devs = [0, 1, 2, 3]
    rng.shuffle(devs)
    h = rng.choice([1, 1, 2])
    sizes = rng.choice([[4], [2], [1]]) if h == 1 else rng.choice([[2, 2], [2, 1], [1, 1]])
    groups, i = [], 0
    for s in sizes:
        groups.append(sorted(devs[i:i + s]))
        i += s
    specs = []
    for g in groups:
        n = len(g)
        ent = [] if n == 1 else [(rng.choice([-1] + list(range(rank))), n)]
        specs.append(ent)
    hdim = -1 if h == 1 else rng.choice([-1] + list(range(rank)))
    return H.anno(groups, specs, hdim)


def test_switch_round_trip_random_strategies(gpu_ctx):
    """SPEC acceptance 6: for 20 random strategy pairs over a 3-parameter model,
    apply_switch(A->B) then (B->A) restores bit-identical shards (every shard
    checked against the counter-hash ground truth after each leg)."""
    import random
    from paper_2504_20490_b200.executor import Program, ShardLayout
    from paper_2504_20490_b200.graph import Graph
    rng = random.Random(3)
    shapes = [(64, 128), (128, 64), (64,)]
    done = 0
    for trial in range(60):
        g = Graph(2)
        ps = [g.parameter(f"p{i}", list(sh), "bf16") for i, sh in enumerate(shapes)]
        for s in range(2):
            for p, sh in zip(ps, shapes):
                g.annotate(p, s, _random_param_anno(rng, len(sh)))
        try:
            ab, ba = g.switch_plan(0, 1, "bf16"), g.switch_plan(1, 0, "bf16")
        except H.HshardError:  # a random annotation that does not validate on these shapes
            continue
        if not ab.json()["xfer"] and not ab.json()["local"]:
            continue
        mark = gpu_ctx.alloc(0)
        try:
            lay_ab, lay_ba = ShardLayout(gpu_ctx, ab, 4), ShardLayout(gpu_ctx, ba, 4)
            lay_ab.fill_src(trial, "grid")
            lay_ab.clear_dst()
            Program(gpu_ctx, ab, lay_ab).run()
            gpu_ctx.sync()
            assert lay_ab.verify_dst(trial) == 0
            for key in lay_ba.src:  # B -> A starts from the moved shards
                lay_ba.write("src", key[0], key[1], lay_ab.read("dst", key[0], key[1]))
            lay_ba.clear_dst()
            Program(gpu_ctx, ba, lay_ba).run()
            gpu_ctx.sync()
            assert lay_ba.verify_dst(trial) == 0
            for key in lay_ab.src:  # bit-identical to the original A shards
                assert np.array_equal(lay_ba.read("dst", key[0], key[1]).view(np.uint8),
                                      lay_ab.read("src", key[0], key[1]).view(np.uint8))
        finally:
            gpu_ctx.reset(mark)
        done += 1
        if done == 20:
            break
    assert done == 20


def test_strategy_cycle_cached_round_trip(gpu_ctx):
    """A Llama-shaped 4-strategy cycle (cfg5's S1->S2->S3->S4->S1, shapes / 32)
    through chained layout states twice: the second cycle re-plans and
    recompiles nothing (SwitchCache hits), every state equals the logical
    tensors, and the round trip returns S1 bit-exactly."""
    from paper_2504_20490_b200.executor import StrategyCycle
    steps = []
    for x in W.CONFIG5_CYCLE:
        steps.append([(tid, s, d, tuple(max(8, v // 32) for v in shp)) for tid, s, d, shp in W.config5(x).transitions])
    mark = gpu_ctx.alloc(0)
    cyc = StrategyCycle(gpu_ctx, steps, "bf16", 8)
    try:
        assert cyc.states[-1] is cyc.states[0]
        cyc.states[0].fill(7)
        gpu_ctx.sync()
        for rnd in range(2):
            for k in range(len(steps)):
                prog, info = cyc.prepare(k)
                assert info["plan_cached"] == (rnd == 1) and info["program_cached"] == (rnd == 1)
                prog.run()
                gpu_ctx.sync()
                assert cyc.states[k + 1].verify(7) == 0, (rnd, k)
    finally:
        cyc.close()
        gpu_ctx.reset(mark)


@pytest.mark.parametrize("name", ["cfg2e", "cfg3b", "cfg1C"])
def test_caller_owned_torch_buffers(gpu_ctx, name):
    """hs_prog_compile_ptrs: the program reshards framework-allocated tensors
    (torch.empty on cuda:0, caching-allocator sub-allocations) in place -- no
    arena -- bit-exact against the oracle (shards are
    {device, gpu_ptr, box}; reference sim.hpp:77-79)."""
    import torch
    from paper_2504_20490_b200.executor import PointerLayout, Program
    w = W.by_name(name)
    tid, src, dst, shape = w.transitions[0]
    shape = [s // 16 for s in shape]
    plan = H.classify(src, dst, shape, w.dtype)
    ref_src = ox.scatter(src, shape, w.dtype, 8, 0, "real")
    want = ox.execute_plan(plan.json(), ref_src, w.dtype)
    tdt = {"bf16": torch.int16, "f32": torch.float32}[w.dtype]
    keep, sp, dp = [], {}, {}
    for dev, a in ref_src.items():
        t = torch.from_numpy(a.view(np.int16) if w.dtype == "bf16" else a).to("cuda:0")
        keep.append(t)
        sp[(0, dev)] = t.data_ptr()
    outs = {}
    for dev, a in want.items():
        t = torch.full(a.shape, 7, dtype=tdt, device="cuda:0")
        keep.append(t)
        outs[dev] = t
        dp[(0, dev)] = t.data_ptr()
    lay = PointerLayout(w.n_virtual, 1, sp, dp, [0] * w.n_virtual)
    for flags in (0, 2 | 4 | 8):
        prog = Program(gpu_ctx, plan, lay, flags)
        prog.run(torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        for dev, a in want.items():
            got = outs[dev].cpu().numpy()
            assert np.array_equal(got.view(np.uint8), a.view(np.uint8)), (name, flags, dev)
        prog.close()
