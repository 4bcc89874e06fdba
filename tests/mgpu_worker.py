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
sys.path.insert(0, os.path.join(ROOT, "tests"))


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
    if world > torch.cuda.device_count():  # ranks share GPUs: no spinning in folded barriers
        os.environ["HS_SEPARATE_BARRIERS"] = "1"  # read by the library at its first compile
    dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    full = os.environ.get("HS_MGPU_FULL") == "1"
    ctx = Context((40 if full else 8) << 30, rank=rank, world=world, gpu=local)
    flag_sets = [int(x) for x in os.environ.get("HS_MGPU_FLAGS", "0,14,1").split(",")]
    if any(f & 2048 for f in flag_sets):
        ctx.init_nccl()
    results, ok = [], True

    def run_case(name, plan, n_virtual, src_of, dtype, mode):
        nonlocal ok
        mark = ctx.alloc(0)
        lay = ShardLayout(ctx, plan, n_virtual)
        lay_holder[:] = [lay]
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

    def full_size_cases():
        """BASELINE reduction configs at FULL size with real-valued payloads; rank 0 runs
        the native CPU executor (oracle/_ref/ref_tool N) into a shared directory and
        every rank byte-compares its own destination shards with it."""
        import tempfile

        import native_ref
        shared = os.environ["HS_MGPU_OUT"] + ".native"
        for wname in os.environ.get("HS_MGPU_FULL_CASES", "cfg2e,cfg3b,cfg2a").split(","):
            w = W.by_name(wname)
            _, src, dst, shape = w.transitions[0]
            plan = H.classify(src, dst, shape, w.dtype)
            d = f"{shared}.{wname}"
            if rank == 0:
                os.makedirs(d, exist_ok=True)
                native_ref.run(src, dst, shape, w.dtype, 11, "real", 0, d)
            dist.barrier()

            def src_of(d=d, w=w):
                out = {}
                for (slot, dev), rec in lay_holder[0].local("dst").items():
                    out[(slot, dev)] = np.fromfile(os.path.join(d, f"dev{dev}.bin"),
                                                   dtype=native_ref.NP[w.dtype]).reshape(rec["ext"])
                return out
            lay_holder.clear()
            run_case(f"{wname}-full", plan, w.n_virtual, src_of, w.dtype, "real")

    def host_path_case():
        """hs_prog_run_host / run_host_async with DIFFERENT inputs every step and no
        host-side barrier between steps: peers read this rank's sources over NVLink,
        so a step's H2D must not overwrite them before every rank has finished the
        previous run (program.cpp run_host)."""
        w = W.by_name("cfg2e")
        _, src, dst, _ = w.transitions[0]
        shape = (256, 1024)
        plan = H.classify(src, dst, shape, w.dtype)
        seeds = [21, 22, 23, 24, 25]
        srcs = {s_: ox.scatter(src, shape, w.dtype, s_, 0, "real") for s_ in seeds}
        wants = {s_: ox.execute_plan(plan.json(), srcs[s_], w.dtype) for s_ in seeds}
        bad = []
        mark = ctx.alloc(0)
        lays = [ShardLayout(ctx, plan, w.n_virtual) for _ in range(2)]
        progs = [Program(ctx, plan, lay) for lay in lays]
        local_src = {k: v for k, v in lays[0].local("src").items()}
        dst_bufs = [{k: np.empty(rec["ext"], dtype=np.uint16) for k, rec in lay.local("dst").items()}
                    for lay in lays]
        host_src = {s_: {k: np.ascontiguousarray(srcs[s_][k[1]]) for k in local_src} for s_ in seeds}
        dist.barrier()
        for s_ in seeds:  # synchronous path, back to back
            progs[0].run_host(host_src[s_], dst_bufs[0])
            for k, a in dst_bufs[0].items():
                if not np.array_equal(a, wants[s_][k[1]]):
                    bad.append(("sync", s_, k[1]))
        ctx.sync()
        dist.barrier()
        h2d, comp, d2h = (torch.cuda.Stream(device=local) for _ in range(3))
        for i, s_ in enumerate(seeds):  # pipelined: two programs, inputs change every step
            progs[i % 2].run_host_async(host_src[s_], dst_bufs[i % 2], h2d.cuda_stream, comp.cuda_stream,
                                        d2h.cuda_stream)
            if i >= 1:  # the previous step's outputs: complete once d2h has drained them
                d2h.synchronize()
                prev = seeds[i - 1]
                for k, a in dst_bufs[(i - 1) % 2].items():
                    if not np.array_equal(a, wants[prev][k[1]]):
                        bad.append(("async", prev, k[1]))
        d2h.synchronize()
        for k, a in dst_bufs[(len(seeds) - 1) % 2].items():
            if not np.array_equal(a, wants[seeds[-1]][k[1]]):
                bad.append(("async", seeds[-1], k[1]))
        ctx.sync()
        for p_ in progs:
            p_.close()
        dist.barrier()
        ctx.reset(mark)
        results.append({"case": "host-path", "flags": 0, "bad": bad, "nvlink_in": 0, "nvlink_out": 0})
        return not bad

    def pointer_case():
        """hs_prog_compile_ptrs at N > 1: every rank's shards are its own torch tensors;
        peers' buffers are mapped through hs_ipc_export / hs_ipc_import
        (executor.exchange_pointers); results bit-exact vs the oracle."""
        from paper_2504_20490_b200.executor import PointerLayout, block_map, exchange_pointers
        bad = []
        for wname, shape in [("cfg2e", (128, 512)), ("cfg1C", (256, 64)), ("cfg3a", (64, 256))]:
            w = W.by_name(wname)
            _, src, dst, _ = w.transitions[0]
            plan = H.classify(src, dst, shape, w.dtype)
            vmap = block_map(w.n_virtual, world)
            ref = ox.scatter(src, shape, w.dtype, 31, 0, "real")
            want = ox.execute_plan(plan.json(), ref, w.dtype)
            tdt = {"bf16": torch.int16, "f32": torch.float32}[w.dtype]
            keep, mine = [], {}
            for d, a in ref.items():
                if vmap[d] == rank:
                    t = torch.from_numpy(a.view(np.int16) if w.dtype == "bf16" else a).to(f"cuda:{local}")
                    keep.append(t)
                    mine[("src", 0, d)] = t.data_ptr()
            outs = {}
            for d, a in want.items():
                if vmap[d] == rank:
                    t = torch.zeros(a.shape, dtype=tdt, device=f"cuda:{local}")
                    keep.append(t)
                    outs[d] = t
                    mine[("dst", 0, d)] = t.data_ptr()
            torch.cuda.synchronize()
            ptrs = exchange_pointers(ctx, mine)
            lay = PointerLayout(w.n_virtual, 1, {(sl, d): p for (k, sl, d), p in ptrs.items() if k == "src"},
                                {(sl, d): p for (k, sl, d), p in ptrs.items() if k == "dst"}, vmap)
            prog = Program(ctx, plan, lay)
            prog.run(torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            ctx.sync()
            for d, t in outs.items():
                if not np.array_equal(t.cpu().numpy().view(np.uint8), want[d].view(np.uint8)):
                    bad.append((wname, d))
            dist.barrier()  # peers finished reading my buffers before they go
            prog.close()
            del keep, outs
        results.append({"case": "pointers", "flags": 0, "bad": bad, "nvlink_in": 0, "nvlink_out": 0})
        return not bad

    def cycle_case():
        """executor.StrategyCycle across GPUs: the cfg5 4-strategy cycle (shapes / 32) twice,
        with the default variant (PUSH_ALL at N > 1) and with flags 0, step k+1 planned and
        compiled while step k runs (the pipelined pattern); every state verified on-device
        on every rank, the second round served from the plan/program cache."""
        from paper_2504_20490_b200.executor import StrategyCycle
        steps = [[(tid, s, d, tuple(max(8, v // 32) for v in shp)) for tid, s, d, shp in W.config5(x).transitions]
                 for x in W.CONFIG5_CYCLE]
        bad = []
        cyc_flags = os.environ.get("HS_MGPU_CYCLE_FLAGS")  # exploration: variants to cycle with
        for flags in ([int(x) for x in cyc_flags.split(",")] if cyc_flags else (None, 0)):
            mark = ctx.alloc(0)
            cyc = StrategyCycle(ctx, steps, "bf16", 8, flags)
            try:
                cyc.states[0].fill(7)
                ctx.sync()
                dist.barrier()
                for rnd in range(2):
                    prog, info = cyc.prepare(0)
                    if info["program_cached"] != (rnd == 1):
                        bad.append(("cache", flags, rnd))
                    sync_prepare = os.environ.get("HS_MGPU_CYCLE_SYNC") == "1"  # exploration
                    for k in range(len(steps)):
                        if sync_prepare and k > 0:
                            prog = cyc.prepare(k)[0]
                        prog.run()  # enqueues only: the next step compiles meanwhile
                        nxt = cyc.prepare(k + 1)[0] if k + 1 < len(steps) and not sync_prepare else None
                        ctx.sync()
                        dist.barrier()
                        b = cyc.states[k + 1].verify(7)
                        if b:
                            bad.append((cyc.flags, rnd, k, b))
                        prog = nxt
            finally:
                dist.barrier()
                cyc.close()
                ctx.reset(mark)
        results.append({"case": "strategy-cycle", "flags": -1, "bad": bad, "nvlink_in": 0, "nvlink_out": 0})
        return not bad

    def random_cases():
        """Random plans of every step kind and dtype (tests/golden/gen_cases.rand_pair,
        the same seeded list on every rank), 10 virtual devices block-mapped onto the
        ranks, each through every flag set, bit-exact vs the oracle on each rank."""
        import random as _random

        from gen_cases import rand_pair, zero_width
        rng = _random.Random(2026)
        dtypes = ["bf16", "f32", "f64", "i32", "i64"]
        done = 0
        tries = 0
        while done < int(os.environ.get("HS_MGPU_RANDOM_N", "60")) and tries < 5000:
            tries += 1
            src, dst, shape = rand_pair(rng)
            dtype = dtypes[tries % len(dtypes)]
            if zero_width(src, shape) or zero_width(dst, shape):
                continue
            try:
                plan = H.classify(src, dst, shape, dtype)
                ox.execute_plan(plan.json(), ox.scatter(src, shape, dtype, 11, 0, "grid"), dtype)
            except (H.HshardError, ox.OracleError):
                continue
            mode = "real" if dtype in ("bf16", "f32", "f64") else "grid"

            def src_of(src=src, shape=shape, dtype=dtype, plan=plan, mode=mode):
                s_ = ox.scatter(src, shape, dtype, 11, 0, mode)
                out = ox.execute_plan(plan.json(), s_, dtype)
                return {(0, d): a for d, a in out.items()}
            run_case(f"rand{done}", plan, 10, src_of, dtype, mode)
            done += 1

    lay_holder = []
    try:
        if os.environ.get("HS_MGPU_RANDOM") == "1":
            random_cases()
            raise StopIteration
        if full:
            full_size_cases()
            raise StopIteration
        if not host_path_case():
            ok = False
        if not pointer_case():
            ok = False
        if not cycle_case():
            ok = False
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
    except StopIteration:
        pass
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
