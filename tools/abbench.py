#!/usr/bin/env python
"""A/B timing of alternative libfht builds on the same GPU in one process each, interleaved.

    python tools/abbench.py LIB1.so LIB2.so@FHT_X=0 ... [--configs 2,5] [--rounds 3]

Every round runs each library's step for each config in a fresh subprocess (FHT_LIB=...), so
the builds see the same box, clocks and thermal state; prints per-kernel means.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, statistics, sys
sys.path.insert(0, os.environ["ROOT"])
import torch, synth
import paper_1811_06378_b200 as fht
cid = int(sys.argv[1])
c = synth.CONFIGS[cid]
imgs = synth.batch(cid)
t = torch.from_numpy(imgs).cuda()
outs = {}
aux = (torch.cuda.Stream(priority=int(os.environ.get("AB_AUX_PRIO", "0"))) if os.environ.get("AB_AUX") == "1" else None)
plan = fht.angle_plan(c["h"], c["w"], c["theta_min"], c["theta_max"]) if c["mode"] == "range" else None
def step(ev=None):
    if c["mode"] == "full":
        if cid in (2, 5):
            outs["h"], outs["s"] = fht.full(t, pair=True, out=outs.get("h"), out_shifted=outs.get("s"), events=ev,
                                            aux_stream=None if ev else aux)
        else:
            outs["h"] = fht.full(t, out=outs.get("h"), events=ev, aux_stream=None if ev else aux)
    elif c["mode"] == "range":
        outs["h"], outs["s"] = fht.angle_range(t, plan, pair=True, out=outs.get("h"), out_shifted=outs.get("s"), events=ev)
    else:
        outs["h"] = fht.quadrant(t, 0, out=outs.get("h"), events=ev)
    return outs["h"].launches
_probe = torch.cuda.Event(enable_timing=True)
_probe.record()
n = step([_probe])  # launches as the events-timed loop runs them (no stream split)
flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
def do_flush():
    flush.zero_()  # > L2 write; AB_FLUSH=rw adds a read pass so the L2 is cold AND clean (no dirty write-back)
    if os.environ.get("AB_FLUSH") == "rw":
        flush.sum()
for _ in range(5): step()
torch.cuda.synchronize()
steps = 30 if cid in (1, 2) else 8
evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n + 1)] for _ in range(steps)]
for r in evs:
    for e in r: e.record()
torch.cuda.synchronize()
for i in range(steps):
    do_flush()
    step(evs[i])
torch.cuda.synchronize()
tot = statistics.mean(evs[i][0].elapsed_time(evs[i][n]) for i in range(steps))
# whole-step time with NO events between the kernels (programmatic dependent launch can overlap)
e0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
e1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
for i in range(steps):
    do_flush()
    e0[i].record()
    step()
    e1[i].record()
torch.cuda.synchronize()
whole = statistics.mean(e0[i].elapsed_time(e1[i]) for i in range(steps))
ks = [statistics.mean(evs[i][k].elapsed_time(evs[i][k + 1]) for i in range(steps)) for k in range(n)]
first = 1 if c["mode"] == "range" else 0
p1 = sum(ks[k] for k in range(first, n) if (k - first) % 2 == 0)
p2 = sum(ks[k] for k in range(first, n) if (k - first) % 2 == 1)
print(json.dumps({"step_us": tot * 1e3, "p1_us": p1 * 1e3, "p2_us": p2 * 1e3, "whole_us": whole * 1e3}))
'''


def main():
    args = sys.argv[1:]
    cfgs = [2, 5]
    rounds = 3
    if "--configs" in args:
        i = args.index("--configs")
        cfgs = [int(x) for x in args[i + 1].split(",")]
        del args[i:i + 2]
    if "--rounds" in args:
        i = args.index("--rounds")
        rounds = int(args[i + 1])
        del args[i:i + 2]
    if "--flush" in args:  # w (default): write 512 MiB; rw: write then read 512 MiB
        i = args.index("--flush")
        os.environ["AB_FLUSH"] = args[i + 1]
        del args[i:i + 2]
    libs = args
    res = {}
    for r in range(rounds):
        for lib in libs:
            for cid in cfgs:
                # LIB@K=V,K2=V2: the same library under extra environment variables (runtime switches)
                path, _, kv = lib.partition("@")
                extra = dict(x.split("=", 1) for x in kv.split(",") if x)
                env = dict(os.environ, FHT_LIB=os.path.abspath(path), ROOT=ROOT, **extra)
                try:
                    out = subprocess.run([sys.executable, "-c", CHILD, str(cid)], env=env, capture_output=True,
                                         text=True, timeout=180)
                except subprocess.TimeoutExpired:
                    print("TIMEOUT", lib, cid)
                    continue
                try:
                    d = json.loads(out.stdout.strip().splitlines()[-1])
                except Exception:
                    print("FAIL", lib, cid, out.stderr[-500:])
                    continue
                res.setdefault((lib, cid), []).append(d)
    for (lib, cid), ds in sorted(res.items()):
        m = {k: sum(d[k] for d in ds) / len(ds) for k in ds[0]}
        mn = {k: min(d[k] for d in ds) for k in ds[0]}
        print(f"C{cid} {os.path.basename(lib):40s} step {m['step_us']:9.1f} us (min {mn['step_us']:9.1f})  "
              f"p1 {m['p1_us']:9.1f}  p2 {m['p2_us']:9.1f}  | no inter-kernel events: {m['whole_us']:9.1f} us")


if __name__ == "__main__":
    main()
