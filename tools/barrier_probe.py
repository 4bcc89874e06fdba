"""Cost of the device-side cross-rank barrier (hs_ctx_barrier), alone and
between two empty-ish launches, timed with CUDA events (max over ranks).

    torchrun --nproc-per-node 2 tools/barrier_probe.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_20490_b200.executor import Context  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    ctx = Context(1 << 30, rank=rank, world=world, gpu=local)
    s = torch.cuda.Stream()
    out = {}
    for n in (1, 2, 4):
        for _ in range(20):
            for _ in range(n):
                ctx.barrier(s.cuda_stream)
        s.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record()
            for _ in range(200):
                for _ in range(n):
                    ctx.barrier(s.cuda_stream)
            b.record()
        b.synchronize()
        t = torch.tensor([a.elapsed_time(b) / 200 / n * 1e3])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[f"us_per_barrier_x{n}"] = round(float(t), 2)
    ctx.sync()
    if rank == 0:
        print(json.dumps({"world": world, **out}))


if __name__ == "__main__":
    main()
