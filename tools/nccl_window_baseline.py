"""NCCL symmetric memory windows (`ncclCommWindowRegister`):
all-reduce of bf16 buffers allocated with `ncclMemAlloc` and registered as
NCCL_WIN_COLL_SYMMETRIC windows -- which lets NCCL 2.27+ pick its symmetric
(NVLink/NVLS) kernels -- against the same all-reduce on plain `cudaMalloc`
buffers, for message sizes from 1 MiB to cfg3a's 1 GiB, on one communicator.

    torchrun --nproc-per-node N tools/nccl_window_baseline.py

Calls the NCCL that PyTorch ships (nvidia/nccl/lib/libnccl.so.2, 2.28.9)
through ctypes; the unique id travels over a gloo group.  One JSON line per
(size, buffer kind) on rank 0: ms per all-reduce (CUDA events, max over
ranks) and bus GB/s; "unavailable" when registration fails.
"""
import ctypes
import json
import os

import torch
import torch.distributed as dist


def load_nccl():
    import nvidia.nccl
    base = nvidia.nccl.__path__[0]
    return ctypes.CDLL(os.path.join(base, "lib", "libnccl.so.2"))


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    nccl = load_nccl()
    uid = ctypes.create_string_buffer(128)
    if rank == 0:
        assert nccl.ncclGetUniqueId(uid) == 0
    obj = [uid.raw]
    dist.broadcast_object_list(obj, src=0)
    uid = ctypes.create_string_buffer(obj[0], 128)

    class UniqueId(ctypes.Structure):
        _fields_ = [("internal", ctypes.c_char * 128)]

    u = UniqueId()
    ctypes.memmove(ctypes.addressof(u), uid, 128)
    comm = ctypes.c_void_p()
    nccl.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, UniqueId, ctypes.c_int]
    assert nccl.ncclCommInitRank(ctypes.byref(comm), world, u, rank) == 0
    nccl.ncclAllReduce.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_void_p, ctypes.c_void_p]
    stream = torch.cuda.Stream()
    BF16, SUM = 9, 0
    for mib in (1, 32, 256, 1024):
        nbytes = mib << 20
        count = nbytes // 2
        for kind in ("cudaMalloc", "ncclMemAlloc + symmetric window"):
            rec = {"bytes": nbytes, "buffer": kind, "n_gpus": world}
            try:
                if kind == "cudaMalloc":
                    t = torch.zeros(count, dtype=torch.bfloat16, device="cuda")
                    ptr = ctypes.c_void_p(t.data_ptr())
                    win = None
                else:
                    ptr = ctypes.c_void_p()
                    r = nccl.ncclMemAlloc(ctypes.byref(ptr), ctypes.c_size_t(nbytes))
                    if r != 0:
                        raise RuntimeError(f"ncclMemAlloc -> {r}")
                    win = ctypes.c_void_p()
                    r = nccl.ncclCommWindowRegister(comm, ptr, ctypes.c_size_t(nbytes), ctypes.byref(win), 1)
                    if r != 0:
                        raise RuntimeError(f"ncclCommWindowRegister -> {r}")
                    torch.cuda.synchronize()
                s = ctypes.c_void_p(stream.cuda_stream)
                for _ in range(3):
                    assert nccl.ncclAllReduce(ptr, ptr, count, BF16, SUM, comm, s) == 0
                stream.synchronize()
                dist.barrier()
                steps = 20 if mib < 1024 else 8
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    e0.record()
                    for _ in range(steps):
                        nccl.ncclAllReduce(ptr, ptr, count, BF16, SUM, comm, s)
                    e1.record()
                e1.synchronize()
                ms = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64)
                dist.all_reduce(ms, op=dist.ReduceOp.MAX)
                rec.update(ms=ms.item(), bus_gbs=2 * (world - 1) / world * nbytes / (ms.item() * 1e-3) / 1e9)
                if win is not None:
                    nccl.ncclCommWindowDeregister(comm, win)
                    nccl.ncclMemFree(ptr)
            except Exception as e:
                rec["unavailable"] = repr(e)[:200]
            if rank == 0:
                print(json.dumps(rec), flush=True)
            dist.barrier()
    nccl.ncclCommDestroy(comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
