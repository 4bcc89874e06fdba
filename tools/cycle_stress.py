"""Stress: the cfg5 strategy cycle (executor.StrategyCycle) at N ranks, several
fresh cycles back to back, every state verified on-device after every step.
Exploration / regression tool for intermittent multi-GPU failures.

    torchrun --nproc-per-node N tools/cycle_stress.py [--rounds 3] [--cycles 2]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    from paper_2504_20490_b200 import workloads as W
    from paper_2504_20490_b200.executor import Context, StrategyCycle
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--cycles", type=int, default=2)
    ap.add_argument("--workload", default="cfg5")
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
    steps = ([W.config5(x) for x in W.CONFIG5_CYCLE] if a.workload == "cfg5"
             else [W.config4(), W.config4_reverse()])
    stream = torch.cuda.Stream()
    for rnd in range(a.rounds):
        ctx.reset(0)
        cyc = StrategyCycle(ctx, [w.transitions for w in steps], "bf16", 8)
        cyc.states[0].fill(5, "grid", stream.cuda_stream)
        stream.synchronize()
        ctx.sync()
        for c in range(a.cycles):
            for k, w in enumerate(steps):
                if world > 1:
                    dist.barrier()
                t0 = time.perf_counter()
                prog, info = cyc.prepare(k)
                prog.run(stream.cuda_stream)
                stream.synchronize()
                ctx.sync()
                bad = cyc.states[k + 1].verify(5)
                if rank == 0 or bad:
                    print(json.dumps({"rank": rank, "round": rnd, "cycle": c, "step": w.name, "bad": bad,
                                      "ms": (time.perf_counter() - t0) * 1e3}), flush=True)
        cyc.close()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
