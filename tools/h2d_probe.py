"""Probe: pinned host -> device copy rate with 1, 2 and 4 concurrent streams
(6 x 128 MiB, cfg2e's per-step input), and device -> host (192 MiB).  Decides
whether the host-buffer path should spread its copies over several streams."""
import json
import time

import torch


def rate(nstreams, n=6, mib=128, reps=5, d2h=False):
    host = [torch.empty(mib << 20, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
    dev = [torch.empty(mib << 20, dtype=torch.uint8, device="cuda") for _ in range(n)]
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    for _ in range(2):
        for i in range(n):
            with torch.cuda.stream(streams[i % nstreams]):
                (host[i].copy_(dev[i], non_blocking=True) if d2h else dev[i].copy_(host[i], non_blocking=True))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        for i in range(n):
            with torch.cuda.stream(streams[i % nstreams]):
                (host[i].copy_(dev[i], non_blocking=True) if d2h else dev[i].copy_(host[i], non_blocking=True))
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    return n * (mib << 20) / dt / 1e9


out = {f"h2d_{k}_streams_GBs": rate(k) for k in (1, 2, 4)}
out.update({f"d2h_{k}_streams_GBs": rate(k, d2h=True) for k in (1, 2)})
print(json.dumps(out))
