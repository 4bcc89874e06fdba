"""NVLink-native library all-reduces for cfg3a's cross-GPU step:
PyTorch symmetric memory on NVSwitch -- `multimem_all_reduce_` (NVLS: the switch
reduces, `multimem.ld_reduce`), `two_shot_all_reduce_`, `one_shot_all_reduce` --
beside NCCL's `all_reduce`, on the 1 GiB bf16 buffer every GPU holds after its
local pre-reduction (cfg3a: AR{0..3}, AR{4..7} + SplitAllReduce = the sum of all
8 partials on every device).

    torchrun --nproc-per-node N tools/symm_mem_baseline.py

Reduction order is the switch's / the library's, not the oracle's: on the
integer grid the result is exact (checked), on real data it differs by rounding
(tolerance, not bit-exactness; the product path keeps its fixed order).  Prints
one JSON line per variant (rank 0): ms per all-reduce (CUDA events, max over
ranks), bus GB/s (2(P-1)/P * bytes / time), exactness; "unavailable" with the
reason when the op or NVLS is missing.
"""
import json
import os

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    group = dist.group.WORLD
    n = 8192 * 65536  # 1 GiB of bf16
    steps = 10

    def grid(seed):
        g = torch.Generator(device="cuda")
        g.manual_seed(seed)
        return torch.randint(-4, 4, (n,), generator=g, device="cuda", dtype=torch.int32).to(torch.bfloat16)

    want = torch.zeros(n, dtype=torch.float32, device="cuda")
    for r in range(world):
        want += grid(100 + r).float()

    def run(name, make_buf, op):
        try:
            buf = make_buf()
            src = grid(100 + rank)
            for _ in range(2):
                buf.copy_(src)
                op(buf)
            torch.cuda.synchronize()
            ok = bool(torch.equal(buf.float(), want))
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                op(buf)  # values grow; timing only
            e1.record()
            e1.synchronize()
            ms = torch.tensor([e0.elapsed_time(e1) / steps], device="cuda")
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            okt = torch.tensor([1.0 if ok else 0.0], device="cuda")
            dist.all_reduce(okt, op=dist.ReduceOp.MIN)
            rec = {"variant": name, "n_gpus": world, "ms": ms.item(),
                   "bus_gbs": 2 * (world - 1) / world * n * 2 / (ms.item() * 1e-3) / 1e9,
                   "exact_on_grid": okt.item() == 1.0}
        except Exception as e:  # the op, NVLS or symmetric memory missing on this build / box
            rec = {"variant": name, "n_gpus": world, "unavailable": repr(e)[:300]}
        if rank == 0:
            print(json.dumps(rec), flush=True)
        dist.barrier()

    run("nccl all_reduce", lambda: torch.empty(n, dtype=torch.bfloat16, device="cuda"),
        lambda b: dist.all_reduce(b))
    try:
        import torch.distributed._symmetric_memory as symm_mem
        symm_mem.enable_symm_mem_for_group(group.group_name)

        def symm_buf():
            t = symm_mem.empty(n, dtype=torch.bfloat16, device="cuda")
            symm_mem.rendezvous(t, group.group_name)
            return t
        ops = torch.ops.symm_mem
        run("symm_mem multimem_all_reduce_ (NVLS)", symm_buf,
            lambda b: ops.multimem_all_reduce_(b, "sum", group.group_name))
        run("symm_mem two_shot_all_reduce_", symm_buf,
            lambda b: ops.two_shot_all_reduce_(b, "sum", group.group_name))
    except Exception as e:
        if rank == 0:
            print(json.dumps({"variant": "symm_mem", "unavailable": repr(e)[:300]}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
