"""Multi-GPU executor parity (one process per GPU, peer-memory pulls over NVLink).

Launches tests/mgpu_worker.py under torchrun on every visible GPU (2 or more);
each rank checks its destination shards bit-exactly against the CPU oracle for
configs 1-3 (reduced sizes) and a mini graph switch, in the default, baseline
and forced-fusion program modes.  Skipped with fewer than 2 GPUs.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _release_parent_gpu_memory():
    import gc
    gc.collect()  # closes Contexts / Programs whose owners are gone (their arenas are cudaMalloc'd)
    try:
        import torch
        if torch.cuda.is_initialized():
            torch.cuda.empty_cache()
    except Exception:
        pass


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
# flag sets (HS_PROG_*); "fine:" = streamed programs cut into ~1 KB chunks so
# the small cases exercise many ready flags per run
@pytest.mark.parametrize("flags", ["0,14,1", "16,17,32,48", "128,256,480", "512,1024,1152", "2048,2062",
                                   "4096,4128,8192,12288", "fine:0,32,512,1024,8192", "16384,16896",
                                   "ce3:16384,16896", "32768,32769,32896",
                                   # STATIC_LOCAL | PULL_MID | NO_STREAM, without / with BULK_STORE
                                   "16789504,50343936",
                                   # barriers as separate launches (default: folded into kernels)
                                   "67108864,67121152",
                                   # TMA bulk stores (to peers when pushed): alone, NO_SHARE, fan-out once
                                   "33554432,33554560,33587200",
                                   # NVLink / local items interleaved: alone, keep-local relays, pull-mid
                                   "536870912,536875520,536883200",
                                   # remote mid rows half relayed before the barrier, half pulled
                                   # after it: alone, with static dealing, streamed, interleaved
                                   "1073745920,1090523136,1073741824,1610616832,1627394048",
                                   # 60 random plans of every kind and dtype through several variants
                                   "random:0,14,1,12288,536870912,1073745920,1610616832",
                                   # BASELINE reduction configs at FULL size, real-valued payloads,
                                   # vs the native CPU executor: default, plain, pull-mid, fused
                                   "full:0,14,12288,1"])
def test_multi_gpu_parity(tmp_path, flags):
    n = int(os.environ.get("HS_TEST_RANKS", min(_gpus(), 8)))  # > GPUs: ranks share GPUs
    port = 29517 + sum(map(ord, flags)) % 300
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tests", "mgpu_worker.py")]
    out = os.path.join(tmp_path, "mgpu")
    env = dict(os.environ, HS_MGPU_OUT=out, HS_MGPU_FLAGS=flags.split(":")[-1])
    if flags.startswith("fine:"):
        env["HS_STREAM_CHUNK_KB"] = "1"
    if flags.startswith("full:"):
        env["HS_MGPU_FULL"] = "1"
    if flags.startswith("random:"):
        env["HS_MGPU_RANDOM"] = "1"
    if flags.startswith("ce3:"):  # copy-engine relays in 3 chunks (uneven row cuts)
        env["HS_CE_CHUNKS"] = "3"
    _release_parent_gpu_memory()  # earlier GPU tests of this pytest process may hold GPU 0 memory
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1800, cwd=ROOT, env=env)
    if res.returncode:  # every rank's own error line first (torchrun prints the root cause last)
        errs = [l for l in res.stderr.splitlines() if "Error" in l and "[rank" in l]
        raise AssertionError("\n".join(errs[:20]) + "\n---\n" + res.stderr[-2000:])
    lines = []
    for r in range(n):
        with open(f"{out}.{r}") as f:
            lines.append(json.loads(f.read()))
    assert len(lines) == n, (res.stdout[-2000:], res.stderr[-2000:])
    for l in lines:  # one summary line per (rank, case, flags): committed as the parity log
        for c in l["cases"]:
            print(f"rank {l['rank']}/{n} " + json.dumps({k: c.get(k) for k in ("case", "flags", "bad", "skipped",
                                                                            "nvlink_in", "nvlink_out", "streamed")
                                                      if k in c}))
    bad_ranks = [json.dumps(l)[:3000] for l in lines if not l["ok"]]
    assert not bad_ranks, "\n".join(bad_ranks)
    # every byte pulled over NVLink by one rank is served by another
    for case in {c["case"] for c in lines[0]["cases"] if "case" in c}:
        for flags in {c["flags"] for c in lines[0]["cases"] if c.get("case") == case}:
            rows = [c for l in lines for c in l["cases"]
                    if c.get("case") == case and c["flags"] == flags and "skipped" not in c]
            assert sum(c["nvlink_in"] for c in rows) == sum(c["nvlink_out"] for c in rows)
