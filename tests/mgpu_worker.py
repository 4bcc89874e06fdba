"""Multi-GPU parity worker, launched by tests/test_multi_gpu.py under
``torchrun --nproc-per-node N``.  One process per GPU; every virtual device
lives on rank v // (n_virtual / N).  For each case the executor runs on all
ranks (peer-memory pulls over NVLink + device barriers) and each rank checks
its own destination shards bit-exactly against the CPU oracle.
Prints one JSON line per rank: {"rank": r, "ok": bool, "cases": [...]}.
"""
import json
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    from oracle import executor as ox
    from paper_2504_20490_b200 import hshard as H
    from paper_2504_20490_b200 import workloads as W
    from paper_2504_20490_b200.executor import Context, Program, ShardLayout

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # HS_TEST_RANKS may oversubscribe the GPUs (8 ranks on a 4-GPU box, two per
    # GPU) to exercise 8-rank IPC, barriers and partitions where only 4 GPUs exist
    local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    ctx = Context(8 << 30, rank=rank, world=world, gpu=local)
    flag_sets = [int(x) for x in os.environ.get("HS_MGPU_FLAGS", "0,14,1").split(",")]
    if any(f & 2048 for f in flag_sets):
        ctx.init_nccl()
    results, ok = [], True

    def run_case(name, plan, n_virtual, src_of, dtype, mode):
        nonlocal ok
        mark = ctx.alloc(0)
        lay = ShardLayout(ctx, plan, n_virtual)
        for flags in flag_sets:
            # run 1 on other values, run 2 (flag epoch 2) on the checked ones:
            # a consumer that does not wait for this run's producers reads
            # run 1's relays and fails the comparison
            lay.fill_src(12, mode)
            try:
                prog = Program(ctx, plan, lay, flags)
            except H.HshardError as e:
                if e.code != "UnsupportedOp":
                    raise
                results.append({"case": name, "flags": flags, "skipped": str(e)[:200]})  # variant not applicable
                dist.barrier()
                continue
            prog.run()
            ctx.sync()
            dist.barrier()
            lay.fill_src(11, mode)
            lay.clear_dst()
            ctx.barrier()  # hs_ctx_barrier: a device barrier between the runs as well
            ctx.sync()
            dist.barrier()
            prog.run()
            ctx.sync()
            want = src_of()
            bad = []
            for (slot, dev), rec in lay.local("dst").items():
                got = lay.read("dst", slot, dev)
                if not np.array_equal(got.view(np.uint8), want[(slot, dev)].view(np.uint8)):
                    bad.append(dev)
            st = prog.stats()
            results.append({"case": name, "flags": flags, "bad": bad, "nvlink_in": st["nvlink_in"],
                            "nvlink_out": st["nvlink_out"], "hbm_write": st["hbm_write"],
                            "streamed": st.get("streamed", 0), "tasks": st["tasks"]})
            ok = ok and not bad
            prog.close()
            dist.barrier()
        ctx.reset(mark)

    try:
        for wname, shape in [("cfg1A", (256, 64)), ("cfg1B", (256, 64)), ("cfg1D", (256, 64)),
                             ("cfg2e", (64, 256)), ("cfg2b", (64, 256)), ("cfg3b", (64, 512)),
                             ("cfg3a", (64, 512)), ("cfg3c", (60, 35))]:
            w = W.by_name(wname)
            _, src, dst, _ = w.transitions[0]
            dtype = w.dtype
            try:
                plan = H.classify(src, dst, shape, dtype)
            except H.HshardError:
                continue

            def src_of(src=src, shape=shape, dtype=dtype, plan=plan):
                s = ox.scatter(src, shape, dtype, 11, 0, "real")
                out = ox.execute_plan(plan.json(), s, dtype)
                return {(0, d): a for d, a in out.items()}
            run_case(wname, plan, w.n_virtual, src_of, dtype, "real")

        # a small graph switch (first 9 Llama-7B-shaped params, scaled down)
        entries = []
        for tid, s, d, shp in W.config4().transitions[:10]:
            shp = tuple(max(8, x // 64) for x in shp)
            entries.append((tid, s, d, shp))
        plan = H.plan_switch(entries, "bf16")

        def sw_src():
            src = {}
            for tid, s, d, shp in entries:
                for dev, a in ox.scatter(s, shp, "bf16", 11, tid, "real").items():
                    src[(tid, dev)] = a
            out = ox.execute_switch(plan.json(), entries, src, "bf16")
            slot = {tid: i for i, (tid, _, _, _) in enumerate(entries)}
            return {(slot[tid], dev): a for (tid, dev), a in out.items()}
        run_case("switch-mini", plan, 8, sw_src, "bf16", "real")
    except Exception:
        ok = False
        results.append({"error": traceback.format_exc()})
    out = os.environ.get("HS_MGPU_OUT")
    line = json.dumps({"rank": rank, "ok": ok, "cases": results})
    if out:
        with open(f"{out}.{rank}", "w") as f:
            f.write(line + "\n")
    else:
        print(line, flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
