"""Exploration: warm time of every step of the cfg4 pair and the cfg5 strategy cycle
under given program variants (StrategyCycle with fixed flags), every state verified.
Cheaper than bench.py --config (no host path).  rank 0 prints one JSON line per
(cycle, flags).

    torchrun --nproc-per-node N tools/cycle_flags_probe.py --flags 1024,570426496
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

    from paper_2504_20490_b200 import workloads as W
    from paper_2504_20490_b200.executor import Context, StrategyCycle
    ap = argparse.ArgumentParser()
    ap.add_argument("--flags", default="1024")
    ap.add_argument("--runs", type=int, default=5)
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(rank)
    if world > 1:
        dist.init_process_group("gloo")
    free, _ = torch.cuda.mem_get_info(rank)
    t_ = torch.tensor([float(free - (12 << 30))], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_, op=dist.ReduceOp.MIN)
    ctx = Context(int(t_.item()) // (1 << 20) << 20, rank=rank, world=world, gpu=rank)
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    for cname, steps in (("cfg4", [W.config4(), W.config4_reverse()]),
                         ("cfg5", [W.config5(x) for x in W.CONFIG5_CYCLE])):
        for f in [int(x) for x in a.flags.split(",")]:
            ctx.reset(0)
            cyc = StrategyCycle(ctx, [w.transitions for w in steps], "bf16", 8, f)
            cyc.states[0].fill(5, "grid", sp)
            stream.synchronize()
            ctx.sync()
            out = {}
            for k, w in enumerate(steps):
                prog, _ = cyc.prepare(k)
                for _ in range(2):
                    prog.run(sp)
                stream.synchronize()
                ctx.sync()
                if world > 1:
                    dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    e0.record()
                    for _ in range(a.runs):
                        prog.run(sp)
                    e1.record()
                e1.synchronize()
                ctx.sync()
                ms = torch.tensor([e0.elapsed_time(e1) / a.runs], dtype=torch.float64)
                bad = torch.tensor([float(cyc.states[k + 1].verify(5))], dtype=torch.float64)
                if world > 1:
                    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
                    dist.all_reduce(bad, op=dist.ReduceOp.MAX)
                out[w.name] = (round(ms.item(), 3), bad.item() == 0)
            if rank == 0:
                print(json.dumps({"cycle": cname, "n": world, "flags": f, "steps": out}), flush=True)
            cyc.close()
    ctx.close()


if __name__ == "__main__":
    main()
