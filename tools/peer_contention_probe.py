"""Does a pull over NVLink slow down when the peer's (or the puller's own) HBM
is saturated, and does the pull slow the local HBM work?

Rank 0 pulls 1 GiB from rank 1's HBM (p2p_uni, HS_PROG_PULL_COPIES) while
both GPUs are otherwise idle ("idle"), while rank 1 runs back-to-back 2 GiB
device copies on a side stream ("peer_busy"), and while rank 0 itself runs
them ("self_busy"; the copies' own rate is reported too).  CUDA events;
DESIGN.md §9.

    torchrun --nproc-per-node 2 tools/peer_contention_probe.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_20490_b200 import hshard as H  # noqa: E402
from paper_2504_20490_b200 import workloads as W  # noqa: E402
from paper_2504_20490_b200.executor import (HS_PROG_PULL_COPIES, Context, Program,  # noqa: E402
                                            ShardLayout)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    ctx = Context(8 << 30, rank=rank, world=world, gpu=local)
    w = W.by_name("p2p_uni")
    tid, s, d, shape = w.transitions[0]
    plan = H.classify(s, d, shape, w.dtype)
    lay = ShardLayout(ctx, plan, w.n_virtual)
    lay.fill_src(1, "grid")
    ctx.sync()
    prog = Program(ctx, plan, lay, HS_PROG_PULL_COPIES)
    stream = torch.cuda.Stream()
    side = torch.cuda.Stream()
    a = torch.empty(1 << 30, dtype=torch.int16, device="cuda")  # 2 GiB
    b = torch.empty_like(a)
    out = {}
    copy_ms = {}
    for busy in ("idle", "peer_busy", "self_busy", "idle", "peer_busy", "self_busy"):
        for _ in range(3):
            prog.run(stream.cuda_stream)
        stream.synchronize()
        ctx.sync()
        dist.barrier()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if (busy == "peer_busy" and rank == 1) or (busy == "self_busy" and rank == 0):
            with torch.cuda.stream(side):
                c0.record()
                for _ in range(40):  # ~27 ms of HBM-bound copies, longer than the timed pulls
                    b.copy_(a)
                c1.record()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record()
            for _ in range(8):
                prog.run(stream.cuda_stream)
            e1.record()
        e1.synchronize()
        side.synchronize()
        ctx.sync()
        t = torch.tensor([e0.elapsed_time(e1) / 8])
        dist.broadcast(t, 0)
        out.setdefault(busy, []).append(round(float(t), 4))
        if busy == "self_busy" and rank == 0:
            copy_ms.setdefault("self_busy_copy_GBps", []).append(round(40 * 2 * a.numel() * 2 / (c0.elapsed_time(c1) * 1e-3) / 1e9, 1))
        dist.barrier()
    if rank == 0:
        gib = 1 << 30
        # an uncontended 2 GiB copy for comparison
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(side):
            c0.record()
            for _ in range(20):
                b.copy_(a)
            c1.record()
        c1.synchronize()
        copy_ms["alone_copy_GBps"] = round(20 * 2 * a.numel() * 2 / (c0.elapsed_time(c1) * 1e-3) / 1e9, 1)
        print(json.dumps({"pull_1GiB_ms": out,
                          "pull_GBps": {k: round(gib / (min(v) * 1e-3) / 1e9, 1) for k, v in out.items()},
                          "local_copy": copy_ms}))


if __name__ == "__main__":
    main()
