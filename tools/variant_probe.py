"""Times given program variants (HS_PROG_* flag sets) of one workload at N ranks
(torchrun), every variant verified on-device; prints one JSON line per variant
(rank 0).  Exploration tool: candidates that win here join executor.AUTOTUNE_CANDIDATES.

    torchrun --nproc-per-node N tools/variant_probe.py --workload cfg2e --flags 0,8192,...
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    from paper_2504_20490_b200 import hshard as H
    from paper_2504_20490_b200 import workloads as W
    from paper_2504_20490_b200.executor import Context, Program, ShardLayout
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2e")
    ap.add_argument("--flags", default="0")
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    free, _ = torch.cuda.mem_get_info(local)
    arena = free - (12 << 30)
    if world > 1:  # one arena size on every rank (the arena is symmetric)
        t_ = torch.tensor([float(arena)], dtype=torch.float64)
        dist.all_reduce(t_, op=dist.ReduceOp.MIN)
        arena = int(t_.item()) // (1 << 20) << 20
    ctx = Context(arena, rank=rank, world=world, gpu=local)
    w = W.by_name(a.workload)
    tid, s, d, shp = w.transitions[0]
    plan = H.classify(s, d, shp, w.dtype)
    lay = ShardLayout(ctx, plan, w.n_virtual)
    lay.fill_src(3, "grid")
    stream = torch.cuda.Stream()
    for f in [int(x) for x in a.flags.split(",")]:
        prog = Program(ctx, plan, lay, f)
        for _ in range(5):
            prog.run(stream.cuda_stream)
        stream.synchronize()
        ctx.sync()
        if world > 1:
            dist.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ev0.record()
            for _ in range(a.steps):
                prog.run(stream.cuda_stream)
            ev1.record()
        ev1.synchronize()
        ctx.sync()
        t = torch.tensor([ev0.elapsed_time(ev1) / a.steps], dtype=torch.float64)
        bad = torch.tensor([float(lay.verify_dst(3)) if not any(r["partial"][1] > 1 for r in lay.dst.values())
                            else 0.0])
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dist.all_reduce(bad, op=dist.ReduceOp.MAX)
        st = prog.stats()
        prog.profile(True)  # separate pass: per-phase durations on every rank
        for _ in range(20):
            prog.run(stream.cuda_stream)
        stream.synchronize()
        ctx.sync()
        ph, runs = prog.phase_ms()
        mine = {"rank": rank, "phase_ms": [x / max(1, runs) for x in ph], "phase_bytes": st["phase_bytes"],
                "kernels": st["phase_kernels"]}
        per = [mine]
        if world > 1:
            per = [None] * world
            dist.all_gather_object(per, mine)
        if rank == 0:
            print(json.dumps({"workload": a.workload, "n": world, "flags": f, "ms": t.item(),
                              "verified": bad.item() == 0, "streamed": st["streamed"],
                              "phases": st["phases"], "ranks": per}), flush=True)
        prog.close()
        if world > 1:
            dist.barrier()
    ctx.close()


if __name__ == "__main__":
    main()
