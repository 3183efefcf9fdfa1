#!/usr/bin/env python
"""Host (CPU) time per enqueued step of a config, without and with the bench's NVML clock sampler
running -- if it exceeds the GPU time in front of the step (the L2 flush), the GPU idles inside the
timed region. python tools/host_cost.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1811_06378_b200 as fht  # noqa: E402
import synth  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = synth.CONFIGS[cid]
t = torch.from_numpy(synth.batch(cid)).cuda()
outs = {}
aux = torch.cuda.Stream()
plan = fht.angle_plan(c["h"], c["w"], c["theta_min"], c["theta_max"]) if c["mode"] == "range" else None
step = bench.make_step(fht, cid, c, t, outs, plan, aux)
for _ in range(10):
    step()
torch.cuda.synchronize()
for label, sampler in (("plain", None), ("with NVML sampler", bench.ClockSampler(0))):
    if sampler:
        sampler.__enter__()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__(None, None, None)
    print(f"config {cid} {label}: {(t1 - t0) / n * 1e6:.1f} us host time per step call")
