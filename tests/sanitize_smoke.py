"""Small executor workloads for compute-sanitizer (memcheck / racecheck /
synccheck): the fused TMA kernel (cfg2e shape), the register path (unaligned
boxes), TMA bulk stores and small items, back-to-back runs with programmatic
dependent launch, a switch plan (device-expanded records), fill and verify
kernels.  Exit code 0 = all results correct."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import executor as ox  # noqa: E402
from paper_2504_20490_b200 import hshard as H, workloads as W  # noqa: E402
from paper_2504_20490_b200.executor import Context, Program, ShardLayout  # noqa: E402

ctx = Context(1 << 30)
cases = []
w = W.config2("e")
cases.append((w.transitions[0][1], w.transitions[0][2], (256, 512), "bf16"))
cases.append(("hsize=1 hdim=-1 [(0,1,2){0:3}]", "hsize=1 hdim=-1 [(1,2,0){-1:3}]", (12, 10), "f32"))
cases.append(("hsize=2 hdim=-2 [(0,1){0:2}; (2,3){0:2}]", "hsize=2 hdim=-1 [(0,1){0:2}; (2,3){0:2}]", (36, 20), "f64"))
bad = 0
for src, dst, shape, dt in cases:
    plan = H.classify(src, dst, shape, dt)
    for flags in (0, 14, (1 << 25) | (1 << 27)):
        mark = ctx.alloc(0)
        lay = ShardLayout(ctx, plan, 8)
        lay.fill_src(5, "real" if dt != "i32" else "grid")
        prog = Program(ctx, plan, lay, flags)
        for _ in range(3):  # back to back: programmatic dependent launch between runs
            prog.run()
        ctx.sync()
        want = ox.execute_plan(plan.json(), ox.scatter(src, shape, dt, 5, 0, "real"), dt)
        for (slot, dev) in lay.dst:
            bad += not np.array_equal(lay.read("dst", slot, dev), want[dev])
        prog.close()
        ctx.reset(mark)
entries = [(t, s, d, tuple(max(8, x // 64) for x in sh)) for t, s, d, sh in W.config4().transitions[:12]]
plan = H.plan_switch(entries, "bf16")
lay = ShardLayout(ctx, plan, 8)
lay.fill_src(6, "grid")
Program(ctx, plan, lay).run()
ctx.sync()
bad += lay.verify_dst(6) != 0
print("sanitize smoke:", "ok" if not bad else f"{bad} mismatches")
sys.exit(1 if bad else 0)
