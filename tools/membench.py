"""Memory-hierarchy microbenchmarks on one B200 (torch kernels, CUDA-event timed).

Used to size the L2-resident decode design: read+write bandwidth of an
in-place update as a function of the working-set size (L2 vs HBM), and the
bandwidth of 512-byte-row random gathers vs contiguous copies.
"""
import json
import sys

import torch


def timed(fn, iters=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters / 1e3


out = {}
for mb in (8, 16, 32, 48, 64, 80, 96, 112, 128, 160, 256, 1024, 2048):
    x = torch.rand(mb * 2**20 // 8, dtype=torch.float64, device="cuda")
    t = timed(lambda: x.mul_(1.0))
    out[f"inplace_{mb}MB_GBps"] = round(2 * x.numel() * 8 / t / 1e9, 1)
for mb in (64, 1024):
    rows = mb * 2**20 // 512
    src = torch.rand(rows, 64, dtype=torch.float64, device="cuda")
    idx = torch.randperm(rows, device="cuda")
    dst = torch.empty_like(src)
    t = timed(lambda: torch.index_select(src, 0, idx, out=dst))
    out[f"gather512_{mb}MB_GBps"] = round(2 * src.numel() * 8 / t / 1e9, 1)
    t = timed(lambda: dst.copy_(src))
    out[f"copy_{mb}MB_GBps"] = round(2 * src.numel() * 8 / t / 1e9, 1)
print(json.dumps(out))
