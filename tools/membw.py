#!/usr/bin/env python
"""Write-only / copy bandwidth on this GPU (torch fill / copy kernels), for the store-path roofline.
    python tools/membw.py"""
import statistics

import torch

flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")


def timed(fn, clean, reps=10):
    ts = []
    for _ in range(reps):
        flush.zero_()
        if clean:
            flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


for mb in (64, 1024):
    n = mb << 18
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    for clean in (False, True):
        tw = timed(lambda: x.fill_(1.0), clean)
        tc = timed(lambda: y.copy_(x), clean)
        print(f"{mb:5d} MiB  L2 {'clean' if clean else 'dirty'}:  fill {n * 4 / tw / 1e6:7.0f} GB/s   "
              f"copy (r+w) {2 * n * 4 / tc / 1e6:7.0f} GB/s")
