"""HBM bandwidth by read:write mix (torch kernels, CUDA events), to bound
write-heavy plans such as cfg1A (64 MiB read, 256 MiB written).

    python tools/hbm_mix_probe.py
"""
import json

import torch


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters / 1e3


def main():
    GiB = 1 << 30
    out = {}
    big = torch.empty(GiB // 2, dtype=torch.int16, device="cuda")
    t = timed(lambda: big.fill_(1))
    out["write_only_fill_1GiB"] = GiB / t / 1e9
    t = timed(lambda: big.zero_())
    out["write_only_memset_1GiB"] = GiB / t / 1e9
    a = torch.empty(GiB // 4, dtype=torch.int16, device="cuda")
    b = torch.empty_like(a)
    t = timed(lambda: b.copy_(a))
    out["copy_512MiB_1to1"] = 2 * a.numel() * 2 / t / 1e9
    for fan in (2, 4):
        src = torch.empty(GiB // 2 // fan // 2, dtype=torch.int16, device="cuda")  # fan x src = 512 MiB
        dst = torch.empty((fan, src.numel()), dtype=torch.int16, device="cuda")
        t = timed(lambda: dst.copy_(src.unsqueeze(0).expand(fan, -1)))
        out[f"fanout_1to{fan}_write512MiB"] = (src.numel() * 2 * (1 + fan)) / t / 1e9
    print(json.dumps({k: round(v, 1) for k, v in out.items()}))


if __name__ == "__main__":
    main()
