"""Per-item timeline of the pipelined kernel (debug hook FHT_PIPE_TRACE_PTR): where does the time go --
dequeue-to-ready waits, item durations by kind, SM occupancy over time.

    python tools/pipe_trace.py [--config 5|2|3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1811_06378_b200 as fht
import synth


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    args = ap.parse_args()
    cc = synth.CONFIGS[args.config]
    t = torch.from_numpy(synth.batch(args.config)).cuda()
    N = 1 << 20
    tr = torch.zeros(N * 4, dtype=torch.int64, device="cuda")
    os.environ["FHT_PIPE_TRACE_PTR"] = str(tr.data_ptr())
    os.environ["FHT_PIPE_TRACE_N"] = str(N)
    os.environ["FHT_PIPE_DEBUG"] = "1"
    pair = args.config in (2, 5)
    for _ in range(3):
        tr.zero_()
        if pair:
            h, s = fht.full(t, pair=True)
        else:
            h = fht.full(t)
        torch.cuda.synchronize()
    r = tr.view(N, 4).cpu().numpy()
    n = int((r[:, 2] > 0).sum())
    r = r[:n]
    t0 = r[:, 0].min()
    deq, rdy, end = (r[:, 0] - t0) / 1e3, (r[:, 1] - t0) / 1e3, (r[:, 2] - t0) / 1e3
    kind = (r[:, 3] >> 24) & 0xff
    sm = r[:, 3] >> 32
    print(f"{cc['name']}: {n} items, span {end.max():.1f} us")
    for k, nm in ((1, "pass1"), (2, "pass2")):
        m = kind == k
        if m.any():
            w = rdy[m] - deq[m]
            d = end[m] - rdy[m]
            print(f"  {nm}: {m.sum()} items, wait mean {w.mean():.2f} us (p90 {np.percentile(w, 90):.2f}, max {w.max():.1f}), "
                  f"work mean {d.mean():.2f} us (p10 {np.percentile(d, 10):.2f}, p90 {np.percentile(d, 90):.2f})")
    # gaps between consecutive items of a CTA are not visible (no CTA id); time buckets of kinds in flight
    edges = np.linspace(0, end.max(), 21)
    for a, b in zip(edges[:-1], edges[1:]):
        act1 = ((kind == 1) & (rdy < b) & (end > a)).sum()
        act2 = ((kind == 2) & (rdy < b) & (end > a)).sum()
        wt = ((deq < b) & (rdy > a)).sum()
        print(f"  [{a:7.1f},{b:7.1f}) us: pass1 active {act1:5d}  pass2 active {act2:5d}  waiting {wt:5d}")
    print("  SMs used:", len(np.unique(sm)))


if __name__ == "__main__":
    main()
