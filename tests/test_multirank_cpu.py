"""Multi-rank partitioning on CPU: the executor compiler's dry run (hs_analyze)
per rank, under a real world-size-2 gloo process group and, in-process, for
4 and 8 ranks.  Checks, for every BASELINE workload and program variant:

* every destination cell is written exactly once by the union of all ranks'
  tasks, in whichever phase finalises it (no gaps, no double writes);
* every relay / intermediate buffer a task reads was written by an earlier
  phase of some rank, and every NCCL receive slot by an earlier send of a peer;
* NVLink bytes leaving all ranks equal the bytes arriving;
* a task's outputs are on its own rank unless they are relay stores or pushed
  (multi-output) results, never source shards.
"""
import json
import os
import subprocess
import sys

import pytest

from paper_2504_20490_b200 import hshard as H
from paper_2504_20490_b200 import workloads as W
from paper_2504_20490_b200.executor import analyze

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FLAG_SETS = [0, 14, 1, 32, 128, 256, 512, 1024, 1152, 2048, 2062, 4096, 8192, 12288, 16384, 16896,
             32768, 32769, 32896, 16789504, 1073745920, 1610616832]
# last three: STATIC_LOCAL | PULL_MID | NO_STREAM; SPLIT_RELAY | NO_STREAM; the same + INTERLEAVE
HEAVY = {"cfg3a", "cfg3c"}  # thousands of streamed pieces: default and unstreamed only
NAMES = ["cfg1A", "cfg1B", "cfg1C", "cfg1D", "cfg2e", "cfg2a", "cfg2b", "cfg2d", "cfg3b", "cfg3a",
         "cfg3c", "cfg4"]


def _plan(w):
    if w.kind == "classify":
        t, s, d, sh = w.transitions[0]
        return H.classify(s, d, sh, w.dtype)
    return H.plan_switch(w.transitions, w.dtype)


def _boxes_tile(box, parts):
    """parts exactly tile box: volumes add up and no two overlap."""
    vol = lambda b: __import__("math").prod(hi - lo for lo, hi in b)
    if sum(vol(p) for p in parts) != vol(box):
        return False
    for i in range(len(parts)):
        for j in range(i + 1, len(parts)):
            if all(max(a[0], b[0]) < min(a[1], b[1]) for a, b in zip(parts[i], parts[j])):
                return False
    return all(all(bl <= lo and hi <= bh for (lo, hi), (bl, bh) in zip(p, box)) for p in parts)


def check_partition(w, plan, per_rank, world):
    """per_rank: [(stats, tasks)] for every rank."""
    stats = [s for s, _ in per_rank]
    tasks = [t for _, ts in per_rank for t in ts]
    assert sum(s["nvlink_in"] for s in stats) == sum(s["nvlink_out"] for s in stats)
    # destination coverage
    entries = ([(0, plan.meta["dst"], plan.meta["shape"])] if plan.kind == "comm"
               else [(i, d, sh) for i, (tid, s, d, sh) in enumerate(plan.meta["entries"])])
    written = {}
    for t in tasks:
        for kind, dev, rank in t["dsts"]:
            if kind == "dst":
                written.setdefault((t["tensor"], dev), []).append(t["box"])
    for slot, dst, shape in entries:
        for g in H.parse_annotation(dst)["groups"]:
            for dev in g:
                box = H.placement(dst, shape, dev)["bounds"]
                assert _boxes_tile(box, written.get((slot, dev), [])), (w.name, slot, dev)
    # relay / mid buffers are produced by an earlier phase before they are read
    produced = {}
    for t in tasks:
        for kind, dev, rank in t["dsts"]:
            if kind in ("relay", "mid"):
                produced.setdefault((kind, t["tensor"], dev, rank), []).append((t["phase"], t["box"]))
            if kind == "send":  # NCCL staging slot: one index space across ranks
                produced.setdefault(("recv", t["tensor"], dev), []).append((t["phase"], t["box"], rank))
    signallers = {}
    for t in tasks:
        for r, f in t.get("targets", []):
            signallers.setdefault((r, f), []).append(t)
    streamed = any(s.get("streamed") for s in stats)
    for t in tasks:
        if t.get("wait", -1) >= 0:
            assert len(signallers.get((t["rank"], t["wait"]), [])) == t["need"], t
        for kind, dev, rank in t["terms"]:
            if kind == "relay":
                assert rank == t["rank"], t
            if kind in ("relay", "mid") and streamed:
                # one launch: the pieces that signal this task's flag must cover what it reads
                assert t["wait"] >= 0, t
                cover = [p["box"] for p in signallers[(t["rank"], t["wait"])]
                         if any(o[0] == kind and o[1] == dev for o in p["dsts"])]
            elif kind in ("relay", "mid", "recv"):
                if kind == "recv":
                    cover = [b for ph, b, r in produced.get((kind, t["tensor"], dev), [])
                             if ph < t["phase"] and r != t["rank"]]
                else:
                    cover = [b for ph, b in produced.get((kind, t["tensor"], dev, rank), []) if ph < t["phase"]]
            if kind in ("relay", "mid", "recv"):
                inside = [[[max(lo, a), min(hi, b)] for (lo, hi), (a, b) in zip(c, t["box"])] for c in cover
                          if all(max(lo, a) < min(hi, b) for (lo, hi), (a, b) in zip(c, t["box"]))]
                assert _boxes_tile(t["box"], inside), (w.name, t)
        for kind, dev, rank in t["dsts"]:
            if rank != t["rank"]:
                assert kind in ("relay", "dst", "mid"), t


def flag_sets(name):
    return [0, 4096, 8192, 16384, 32769, 16789504, 1073745920, 1610616832] if name in HEAVY else FLAG_SETS


def _analyze_all(w, plan, world, flags):
    return [analyze(plan, world, r, w.n_virtual, flags) for r in range(world)]


def _partition_or_unsupported(w, plan, world, flags):
    """check_partition, unless the variant refuses the plan (UnsupportedOp) on every rank."""
    try:
        per_rank = _analyze_all(w, plan, world, flags)
    except H.HshardError as e:
        assert e.code == "UnsupportedOp", e
        return
    check_partition(w, plan, per_rank, world)


def test_zero_width_slices_partition():
    """top-tier ratio slices that floor to zero width compile
    (empty boxes are dropped -- they once divided by a zero extent) and still
    tile every destination shard, on 1, 2 and 5 ranks and across variants."""
    import random
    from types import SimpleNamespace
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from gen_cases import rand_pair, zero_width
    rng = random.Random(33)
    done = tries = 0
    while done < 40 and tries < 20000:
        tries += 1
        s, d, sh = rand_pair(rng)
        sh = [rng.choice([1, 2, 3, 4, 6]) if rng.random() < 0.7 else x for x in sh]
        if not (zero_width(s, sh) or zero_width(d, sh)):
            continue
        try:
            plan = H.classify(s, d, sh, "f32")
        except H.HshardError:
            continue
        w = SimpleNamespace(name=f"zero-width {s} -> {d} {sh}", n_virtual=10)
        try:
            for world in (1, 2, 5):
                for flags in (0, 14, 8192, 32768):
                    _partition_or_unsupported(w, plan, world, flags)
        except H.HshardError as e:
            assert e.code == "UnexecutableStep", e  # Appendix-B1 plans, as without zero widths
            continue
        done += 1
    assert done >= 30, done


@pytest.mark.parametrize("world", [4, 8])
def test_partitioning_in_process(world):
    for name in NAMES:
        w = W.by_name(name)
        plan = _plan(w)
        for flags in flag_sets(name):
            _partition_or_unsupported(w, plan, world, flags)


def test_partitioning_gloo_world2(tmp_path):
    """Two real processes (gloo): each compiles its own rank, results all-gathered."""
    out = tmp_path / "res"
    code = f"""
import json, os, sys
sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {os.path.join(ROOT, 'tests')!r})
import torch.distributed as dist
from paper_2504_20490_b200 import workloads as W
from paper_2504_20490_b200.executor import analyze
from test_multirank_cpu import NAMES, flag_sets, _plan, check_partition
from paper_2504_20490_b200 import hshard as H
dist.init_process_group('gloo')
rank, world = dist.get_rank(), dist.get_world_size()
ok = True
for name in NAMES:
    w = W.by_name(name); plan = _plan(w)
    for flags in flag_sets(name):
        try:
            mine = analyze(plan, world, rank, w.n_virtual, flags)
        except H.HshardError as e:
            assert e.code == "UnsupportedOp"
            mine = None
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        if rank == 0 and all(a is not None for a in allr):
            check_partition(w, plan, allr, world)
if rank == 0:
    open({str(out)!r}, 'w').write('ok')
dist.destroy_process_group()
"""
    script = tmp_path / "worker.py"
    script.write_text(code)
    res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr=127.0.0.1", "--master-port=29641", str(script)],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-4000:]
    assert out.read_text() == "ok"


def test_interleave_slots_partition():
    """HS_PROG_INTERLEAVE's launch order (kernels.cu expand_records_kernel): the
    k-th item of the NVLink class goes to slot ceil((k+1) n / na) - 1, the k-th
    local item to floor(k n / (n - na)); together a permutation of [0, n) that
    spreads the classes evenly (every prefix holds its share of each class)."""
    for n in range(1, 400):
        for na in range(1, n):
            a = [((k + 1) * n + na - 1) // na - 1 for k in range(na)]
            b = [(k * (n)) // (n - na) for k in range(n - na)]
            assert sorted(a + b) == list(range(n)), (n, na)
            # evenness: within any prefix of j slots, the NVLink-class count is within 1 of j*na/n
            is_a = [0] * n
            for x in a:
                is_a[x] = 1
            c = 0
            for j in range(n):
                c += is_a[j]
                assert abs(c - (j + 1) * na / n) <= 1.0 + 1e-9, (n, na, j)


def test_state_layouts_chain_and_transition_offsets():
    """executor.StateLayout packs one strategy's shards symmetrically (identical offsets
    on every rank by construction, within the requested base); Transition indexes them
    by the switch plan's tensor order, matched by tensor id -- a plan that lists only
    some parameters, in its own order, still finds every shard."""
    import numpy as np
    from paper_2504_20490_b200 import hshard as H
    from paper_2504_20490_b200 import workloads as W
    from paper_2504_20490_b200.executor import SIZE_MAX, StateLayout, Transition, block_map

    class Ctx:
        def __init__(self, rank, world):
            self.rank, self.world, self.arena_bytes = rank, world, 1 << 40

        def alloc(self, n):
            raise AssertionError("explicit bases only")

    w = W.config4()
    src = [(i, t, s, shp) for i, (t, s, d, shp) in enumerate(w.transitions)]
    dst = [(i, t, d, shp) for i, (t, s, d, shp) in enumerate(w.transitions)]
    for world in (1, 2, 4, 8):
        size = StateLayout.bytes_needed(src, "bf16", 8, world)
        lays = [StateLayout(Ctx(r, world), src, "bf16", 8, base=4096) for r in range(world)]
        recs = [sorted((k, v["offset"], v["rank"], v["bytes"]) for k, v in l.recs.items()) for l in lays]
        assert all(r == recs[0] for r in recs)                      # symmetric
        assert max(o + b for _, o, _, b in recs[0]) <= 4096 + size  # within the reservation
        vmap = block_map(8, world)
        assert all(rank == vmap[k[1]] for k, _, rank, _ in recs[0])
    # a plan over a reversed subset of the tensors: offsets follow tensor ids
    sub = list(reversed(w.transitions[:5]))
    plan = H.plan_switch(sub, "bf16")
    a = StateLayout(Ctx(0, 1), src, "bf16", 8, base=0)
    b = StateLayout(Ctx(0, 1), dst, "bf16", 8, base=1 << 36)
    tr = Transition(plan, a, b)
    offs = np.array(tr._offs[0])
    for slot, (tid, s, d, shp) in enumerate(sub):
        for dev in range(8):
            rec = next((v for (sl, dv), v in a.recs.items() if v["tid"] == tid and dv == dev), None)
            want = rec["offset"] if rec else SIZE_MAX
            assert offs[slot * 8 + dev] == want, (tid, dev)
