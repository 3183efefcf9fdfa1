#!/usr/bin/env python
"""Per-quadrant pass times on a config's image (which quadrant slots are the long pole).
    python tools/quadtime.py [config]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1811_06378_b200 as fht  # noqa: E402
import synth  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
t = torch.from_numpy(synth.batch(cid)).cuda()
flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
for q in range(4):
    out = {}

    def step(ev=None):
        out["h"] = fht.quadrant(t, q, out=out.get("h"), events=ev)
        return out["h"].launches

    n = step()
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    rows = []
    for _ in range(20):
        flush.zero_()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        for e in evs:  # materialise the cudaEvent_t handles the library records into
            e.record()
        step(evs)
        torch.cuda.synchronize()
        rows.append([evs[k].elapsed_time(evs[k + 1]) * 1e3 for k in range(n)])
    med = [statistics.median(r[k] for r in rows) for k in range(n)]
    print(f"quadrant {q}: " + "  ".join(f"k{k} {m:7.2f} us" for k, m in enumerate(med)))
