"""Probe: which NVML NVLink counters move, and by how much, for a known peer copy.
Copies 4 GiB GPU0 -> GPU1 (torch, copy engines) and prints every NVLink
throughput / byte counter's delta on both GPUs.  Run on a >=2-GPU box."""
import time

import pynvml as nv
import torch

NAMES = [n for n in dir(nv) if n.startswith("NVML_FI_DEV_NVLINK") and
         any(k in n for k in ("THROUGHPUT", "RCV_BYTES", "XMIT_BYTES"))]


def read(h):
    out, errs = {}, {}
    for name in NAMES:
        fid = getattr(nv, name)
        for scope in (0xFFFFFFFF, 0):
            try:
                v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            except Exception as e:
                errs[name] = repr(e)[:80]
                continue
            if v.nvmlReturn == 0:
                out[(name, scope)] = v.value.ullVal
            else:
                errs[(name, scope)] = v.nvmlReturn
    return out, errs


nv.nvmlInit()
hs = [nv.nvmlDeviceGetHandleByIndex(i) for i in range(2)]
print("fields", NAMES)
a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
b = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:1")
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
before = [read(h) for h in hs]
print("errors", before[0][1])
for _ in range(4):
    b.copy_(a)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
time.sleep(1.0)
after = [read(h) for h in hs]
for g in range(2):
    for k in sorted(after[g][0]):
        d = after[g][0][k] - before[g][0].get(k, 0)
        print(g, k, d, round(d / (4 << 30), 4))
try:
    print("util", nv.nvmlDeviceGetNvLinkUtilizationCounter(hs[0], 0, 0))
except Exception as e:
    print("util err", e)
