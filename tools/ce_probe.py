"""Probe: copy-engine peer copies over NVLink, alone and concurrent with an
HBM-bound kernel on the same GPUs (one process, two GPUs)."""
import torch, time
assert torch.cuda.device_count() >= 2
a = torch.empty(64 << 20, dtype=torch.uint8, device="cuda:0")
b = torch.empty(64 << 20, dtype=torch.uint8, device="cuda:1")
big0 = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0"); big0b = torch.empty_like(big0)
big1 = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:1"); big1b = torch.empty_like(big1)
print("p2p", torch.cuda.can_device_access_peer(0, 1))
cs = torch.cuda.Stream(device="cuda:0")
def t_copy(n=10):
    torch.cuda.synchronize("cuda:0"); torch.cuda.synchronize("cuda:1")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        e0.record(cs)
        for _ in range(n): b.copy_(a, non_blocking=True)
        e1.record(cs)
    e1.synchronize()
    return e0.elapsed_time(e1) / n
def t_hbm(n=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream("cuda:0")
    e0.record(s)
    for _ in range(n): big0b.copy_(big0)
    e1.record(s)
    return e0, e1, n
for _ in range(3): t_copy(2)
ms = t_copy(); print(f"CE push 64 MiB alone: {ms:.3f} ms = {64*2**20/ms/1e6:.0f} GB/s")
# concurrent: HBM copy kernel on cuda:0 while CE copies
torch.cuda.synchronize("cuda:0")
e0, e1, n = t_hbm(20)
ms2 = t_copy(20)
e1.synchronize()
hb = e0.elapsed_time(e1) / n
print(f"concurrent: CE {ms2:.3f} ms = {64*2**20/ms2/1e6:.0f} GB/s; HBM copy 1 GiB {hb:.3f} ms = {2*2**30/hb/1e6:.0f} GB/s")
torch.cuda.synchronize("cuda:0")
e0, e1, n = t_hbm(20); e1.synchronize(); hb0 = e0.elapsed_time(e1)/n
print(f"HBM copy alone {hb0:.3f} ms = {2*2**30/hb0/1e6:.0f} GB/s")
