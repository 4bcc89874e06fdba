"""NVLink hardware counters of one multi-GPU program launch, read with ncu on ONE
rank while the other ranks run unprofiled.

ncu must not wrap a multi-rank command whose kernels wait on each other (kernel
replay would re-run a device barrier against peers that do not replay), so this
tool compiles the program with HS_PROG_SEPARATE_BARRIERS: cross-rank barriers are
their own 1-CTA launches, and the data kernels (`box_phase*`) have no waits.  The
profiled rank opens a cudaProfilerStart/Stop window around `--runs` steps; the
launcher (tools/nvlink_ncu_capture.sh) runs that rank under

    ncu --profile-from-start off -k regex:box_phase --metrics <nvl/dram/time> ...

and the other ranks plainly.  Replays of a pull kernel re-read the peer's HBM
(idempotent); pushed stores rewrite identical bytes.  Each rank prints the
compiled program's per-phase byte accounting (JSON) so the counters can be
compared with the algorithmic NVLink bytes.

    RANK=r WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=29555 \
        python tools/nvlink_ncu_capture.py --workload cfg2e --flags 16789504
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def log(msg):
    print(f"[{time.time():.3f}] {msg}", file=sys.stderr, flush=True)


def main():
    import torch
    import torch.distributed as dist

    from paper_2504_20490_b200 import hshard as H
    from paper_2504_20490_b200 import workloads as W
    from paper_2504_20490_b200.executor import (HS_PROG_SEPARATE_BARRIERS, Context, Program,
                                                ShardLayout)
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2e")
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--runs", type=int, default=1)
    ap.add_argument("--arena-gb", type=float, default=6.0)
    ap.add_argument("--profiled-rank", type=int, default=0)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    log(f"rank {rank}: process group up")
    ctx = Context(int(a.arena_gb * (1 << 30)), rank=rank, world=world, gpu=rank)
    w = W.by_name(a.workload)
    _, s, d, shp = w.transitions[0]
    plan = H.classify(s, d, shp, w.dtype)
    lay = ShardLayout(ctx, plan, w.n_virtual)
    lay.fill_src(3, "grid")
    flags = a.flags | HS_PROG_SEPARATE_BARRIERS
    prog = Program(ctx, plan, lay, flags)
    stream = torch.cuda.Stream()
    for _ in range(a.warmup):
        prog.run(stream.cuda_stream)
    stream.synchronize()
    ctx.sync()
    dist.barrier()
    log(f"rank {rank}: warm, {a.runs} profiled run(s)")
    for _ in range(a.runs):
        prog.run(stream.cuda_stream)
    stream.synchronize()
    ctx.sync()
    log(f"rank {rank}: runs done")
    dist.barrier()
    # the profiled rank's replays leave its outputs as the last replay wrote them
    # (identical bytes); the other ranks verify theirs
    bad = lay.verify_dst(3) if rank != a.profiled_rank else None
    log(f"rank {rank}: verified {bad}")
    st = prog.stats()
    print(json.dumps({"rank": rank, "world": world, "workload": a.workload, "flags": flags,
                      "verify_bad": bad, "profiled": rank == a.profiled_rank,
                      "phases": st.get("phases"), "phase_kernels": st.get("phase_kernels"),
                      "phase_bytes": st.get("phase_bytes"),
                      "nvlink_in": st.get("nvlink_in"), "nvlink_out": st.get("nvlink_out"),
                      "hbm_read": st.get("hbm_read"), "hbm_write": st.get("hbm_write")}),
          flush=True)
    dist.barrier()
    prog.close()
    ctx.close()
    log(f"rank {rank}: closed")


if __name__ == "__main__":
    main()
