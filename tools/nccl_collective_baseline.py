"""NCCL collective baseline for the reduction configs.

    torchrun --nproc-per-node N tools/nccl_collective_baseline.py [--configs cfg2d,cfg3a,cfg3b]

What the plans compute, lowered onto NCCL's own collectives the standard way:
virtual devices sharing a GPU are pre-reduced locally (torch, fp32 accumulate,
one rounding), then one collective per step runs among the GPUs over
torch.distributed's NCCL communicators (sub-communicators where the group
spans a subset), then each local device's destination box is copied out:

* cfg2d  {-2:8} -> {1:8}, ReduceScatter{0..7}: local sum, columns packed rank
  by rank, ncclReduceScatter, unpacked into the 8192 x 1024 column shards.
* cfg3a  AR{0..3}, AR{4..7} + SplitAllReduce c{0,4}: every device ends with
  the sum of all 8 partials -> local sum + ncclAllReduce over all GPUs (the
  flat all-reduce SURVEY §8(d) quotes as the 1.75 GiB alternative) + copies.
* cfg3b  RS x2 + SplitReduceScatter, rows 5:3: device d ends with rows R_d of
  the full sum -> local sum + one ncclReduce per GPU onto the GPU owning those
  rows (rows are uneven, 5:3, so ncclReduceScatter's equal counts do not fit).

Tolerance: NCCL's reduction order differs from the oracle's ascending-id,
round-once-per-phase order, so real-valued results would differ by rounding
(bf16 <= 1 ulp per phase).  This baseline runs on the exact integer grid, where
every order gives the same sums, and checks its destination shards bit-exactly
against the logical sums.  Prints one JSON line per config (rank 0): device
ms per step (CUDA events, max over ranks) and GB/s destination-resident.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def partial(dev, shape, seed=7):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed * 1000 + dev)
    return torch.randint(-8, 8, shape, generator=g, device="cuda", dtype=torch.int32).to(torch.bfloat16)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg2d,cfg3a,cfg3b")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--hierarchical", action="store_true",
                    help="cfg3a lowered literally on NCCL sub-communicators (N=4): AllReduce within each "
                         "subgroup's GPUs, then between the subgroups' GPU pairs (i, i + N/2)")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    V = 8
    per = V // world
    mine = list(range(rank * per, (rank + 1) * per))
    sub_groups = pair_groups = None
    if a.hierarchical:
        half = world // 2
        # every rank creates every group (torch.distributed requirement); NCCL splits them
        sub = [dist.new_group(list(range(0, half))), dist.new_group(list(range(half, world)))]
        pairs = [dist.new_group([i, i + half]) for i in range(half)]
        sub_groups = sub[rank // half]
        pair_groups = pairs[rank % half]
    for name in a.configs.split(","):
        if name == "cfg2d":
            shape = (8192, 8192)
        else:
            shape = (8192, 65536)
        src = [partial(d, shape) for d in mine]
        acc = torch.empty(shape, dtype=torch.float32, device="cuda")
        s16 = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
        rows = None
        if name == "cfg2d":
            cols = shape[1] // V
            dst = [torch.empty((shape[0], cols), dtype=torch.bfloat16, device="cuda") for _ in mine]
            packed = torch.empty((world, per, shape[0], cols), dtype=torch.bfloat16, device="cuda")
            recv = torch.empty((per, shape[0], cols), dtype=torch.bfloat16, device="cuda")
        elif name == "cfg3a":
            dst = [torch.empty(shape, dtype=torch.bfloat16, device="cuda") for _ in mine]
        else:  # cfg3b: rows 5:3 over subgroups {0..3}, {4..7}, 4 devices each
            b0 = shape[0] * 5 // 8
            rows = [(i * b0 // 4, (i + 1) * b0 // 4) for i in range(4)] + \
                   [(b0 + i * (shape[0] - b0) // 4, b0 + (i + 1) * (shape[0] - b0) // 4) for i in range(4)]
            dst = [torch.empty((rows[d][1] - rows[d][0], shape[1]), dtype=torch.bfloat16, device="cuda")
                   for d in mine]
            rank_rows = [(rows[r * per][0], rows[(r + 1) * per - 1][1]) for r in range(world)]

        def pre_reduce():
            acc.copy_(src[0])  # local pre-reduction, ascending device id, fp32, one rounding
            for x in src[1:]:
                acc.add_(x)
            s16.copy_(acc)

        def collective():
            if name == "cfg2d":
                dist.reduce_scatter_tensor(recv, packed.view(world, -1), op=dist.ReduceOp.SUM)
            elif name == "cfg3a" and a.hierarchical:
                # AR{0..3}, AR{4..7} on the subgroups' GPUs, then SplitAllReduce between the
                # subgroups (c {0,4}), every receiver pair (i, i + N/2) at once
                dist.all_reduce(s16, op=dist.ReduceOp.SUM, group=sub_groups)
                dist.all_reduce(s16, op=dist.ReduceOp.SUM, group=pair_groups)
            elif name == "cfg3a":
                dist.all_reduce(s16, op=dist.ReduceOp.SUM)
            else:
                for r in range(world):
                    lo, hi = rank_rows[r]
                    dist.reduce(s16[lo:hi], dst=r, op=dist.ReduceOp.SUM)

        def step():
            pre_reduce()
            if name == "cfg2d":
                packed.copy_(s16.view(shape[0], world, per, cols).permute(1, 2, 0, 3))
                dist.reduce_scatter_tensor(recv, packed.view(world, -1), op=dist.ReduceOp.SUM)
                for i, d in enumerate(dst):
                    d.copy_(recv[i])
            elif name == "cfg3a":
                collective()
                for d in dst:
                    d.copy_(s16)
            else:
                for r in range(world):
                    lo, hi = rank_rows[r]
                    dist.reduce(s16[lo:hi], dst=r, op=dist.ReduceOp.SUM)
                for i, d in enumerate(mine):
                    dst[i].copy_(s16[rows[d][0]:rows[d][1]])

        for _ in range(a.warmup):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(a.steps):
            step()
        ev1.record()
        ev1.synchronize()
        ms = torch.tensor([ev0.elapsed_time(ev1) / a.steps], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        # the NCCL collective alone (same buffers, no local pre-reduction / copies)
        torch.cuda.synchronize()
        dist.barrier()
        ev0.record()
        for _ in range(a.steps):
            collective()
        ev1.record()
        ev1.synchronize()
        coll = torch.tensor([ev0.elapsed_time(ev1) / a.steps], device="cuda")
        dist.all_reduce(coll, op=dist.ReduceOp.MAX)
        step()  # restore a correct result for the check below
        torch.cuda.synchronize()
        # exactness on the integer grid: every destination box equals the logical sum
        full = torch.zeros(shape, dtype=torch.float32, device="cuda")
        for d in range(V):
            full += partial(d, shape).float()
        ok = True
        for i, d in enumerate(mine):
            if name == "cfg2d":
                want = full[:, d * cols:(d + 1) * cols]
            elif name == "cfg3a":
                want = full
            else:
                want = full[rows[d][0]:rows[d][1]]
            ok = ok and bool(torch.equal(dst[i].float(), want))
        okt = torch.tensor([1.0 if ok else 0.0], device="cuda")
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        db = torch.tensor([float(sum(x.numel() for x in dst) * 2)], device="cuda")
        dist.all_reduce(db, op=dist.ReduceOp.SUM)  # destination-resident bytes, all ranks
        dst_bytes = db.item()
        if rank == 0:
            print(json.dumps({"workload": name, "n_gpus": world,
                              "transport": "nccl collectives (torch.distributed)" +
                                           (", hierarchical sub-communicators" if a.hierarchical else ""),
                              "ms": ms.item(), "collective_only_ms": coll.item(),
                              "GB/s": dst_bytes / (ms.item() * 1e-3) / 1e9,
                              "verified_exact_grid": okt.item() == 1.0, "nccl": torch.cuda.nccl.version()}),
                  flush=True)
        del src, acc, s16, dst, full
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
