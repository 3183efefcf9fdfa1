"""C2 pass-2 cost with one vs two destinations (Hough only / fhtshift only / both)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1811_06378_b200 as fht
t = torch.from_numpy(synth.batch(int(sys.argv[1]) if len(sys.argv) > 1 else 2)).cuda()
flush = torch.empty(128 << 20, device="cuda")
for name, kw in (("plain", {}), ("shifted", {"shifted": True}), ("pair", {"pair": True})):
    out = {}
    def step(ev=None):
        r = fht.full(t, events=ev, **kw)
        return r if not isinstance(r, tuple) else r[0]
    h = step(); n = h.launches
    for _ in range(5): step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n + 1)] for _ in range(20)]
    for r in evs:
        for e in r: e.record()
    ts = []
    for i in range(20):
        flush.zero_(); step(evs[i])
    torch.cuda.synchronize()
    p1 = statistics.mean(evs[i][0].elapsed_time(evs[i][1]) for i in range(20)) * 1e3
    p2 = statistics.mean(evs[i][1].elapsed_time(evs[i][2]) for i in range(20)) * 1e3
    print(f"{name:8s} p1 {p1:7.1f} us  p2 {p2:7.1f} us")
