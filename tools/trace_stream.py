"""Per-CTA timeline of a streamed multi-GPU program (debug tool).

    HS_TRACE=1 torchrun --nproc-per-node 2 tools/trace_stream.py cfg2e [flags]

Every TMA launch records, per CTA, %globaltimer at start / end, items taken,
the time spent waiting for ready flags, and when it first took an item of
the second (waiting) queue.  Prints one JSON summary per rank.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    from paper_2504_20490_b200 import hshard as H
    from paper_2504_20490_b200 import workloads as W
    from paper_2504_20490_b200.executor import Context, Program, ShardLayout

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(rank)
    ctx = Context(40 << 30, rank=rank, world=world, gpu=rank)
    w = W.by_name(sys.argv[1])
    flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    t, s, d, shp = w.transitions[0]
    plan = H.classify(s, d, shp, w.dtype)
    lay = ShardLayout(ctx, plan, w.n_virtual)
    lay.fill_src(1, "grid")
    prog = Program(ctx, plan, lay, flags)
    for _ in range(10):
        prog.run()
    ctx.sync()
    dist.barrier()
    prog.run()
    ctx.sync()
    st = prog.stats()
    n = st["trace_ctas"]
    tr = np.frombuffer(ctx.read(st["trace_off"], n * 64), dtype=np.uint64).reshape(n, 8).astype(np.int64)
    t0 = tr[:, 0].min()
    us = lambda x: round(float(x) / 1e3, 1)
    out = {"rank": rank, "flags": flags, "streamed": st["streamed"], "ctas": n}
    for role, name in [(1, "first"), (0, "second")]:
        m = tr[:, 7] == role
        if not m.any():
            continue
        ends = tr[m, 1] - t0
        out[name] = {"n": int(m.sum()), "end_us": [us(ends.min()), us(np.median(ends)), us(ends.max())],
                     "items": [int(tr[m, 2].min()), int(np.median(tr[m, 2])), int(tr[m, 2].max())],
                     "wait_us_total_median": us(np.median(tr[m, 3])),
                     "waits_spun_median": float(np.median(tr[m, 4])),
                     "first_second_queue_us": [us(x - t0) for x in np.percentile(tr[m, 5][tr[m, 5] > 0], [0, 50, 100])]
                     if (tr[m, 5] > 0).any() else None}
    print(json.dumps(out), flush=True)
    prog.close()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
