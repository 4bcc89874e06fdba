"""Test helper: drive oracle/_ref/ref_tool's native-dtype CPU executor (command N,
oracle/native_exec.inc) and read its destination shards back as numpy arrays.

Test infrastructure only (the checker): the reference planner's plan executed
with per-row memcpy and fp32 accumulation in ascending device-id order, one
rounding per plan phase -- the numpy oracle's semantics, native and threaded so
it finishes BASELINE-size plans in seconds.
"""
from __future__ import annotations

import json
import os
import subprocess
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
NP = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64, "bf16": np.uint16}


def available() -> bool:
    return os.access(REF_TOOL, os.X_OK)


def run(src: str, dst: str, shape, dtype: str, seed: int, mode: str = "grid", threads: int = 0,
        outdir: str | None = None, reps: int = 1, warmup: int = 0, bw: str = "u"):
    """-> (json summary, {dev: flat storage array} or None when outdir is None)."""
    threads = threads or (os.cpu_count() or 1)
    cmd = (f"N|{dtype}|{','.join(str(int(s)) for s in shape)}|{bw}|{src}|{dst}|{seed}|{mode}|"
           f"{reps}|{threads}|{warmup}|{outdir or '-'}\n")
    out = subprocess.run([REF_TOOL], input=cmd, capture_output=True, text=True, timeout=3600)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else "{}"
    j = json.loads(line)
    if "error" in j or out.returncode:
        raise RuntimeError(f"ref_tool N failed: {j} {out.stderr[-500:]}")
    shards = None
    if outdir:
        shards = {int(d): np.fromfile(os.path.join(outdir, f"dev{d}.bin"), dtype=NP[dtype])
                  for d in j["shards"]}
    return j, shards


def shards(src, dst, shape, dtype, seed, mode="grid", threads=0):
    """Convenience: run in a temporary directory and return {dev: flat array}."""
    with tempfile.TemporaryDirectory(dir=os.environ.get("HS_NATIVE_TMP")) as d:
        _, s = run(src, dst, shape, dtype, seed, mode, threads, d)
        return s
