#!/usr/bin/env python
"""Pass overlap by stream priority (C5): the chunked schedule runs pass 1 of chunk k+1 on the auxiliary
stream beside pass 2 of chunk k; with the auxiliary stream at a HIGHER priority the block scheduler hands
freed SM slots to pass-1 CTAs first, so the two passes interleave instead of meeting only at the tails.
Each case runs in a fresh process (env differs); whole-step CUDA events on the caller's stream.

    python tools/prio_ab.py [--config 5] [--rounds 2]
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
cid = int(sys.argv[1]); prio = int(sys.argv[2]); single = sys.argv[3] == "1"
c = synth.CONFIGS[cid]
t = torch.from_numpy(synth.batch(cid)).cuda()
aux = torch.cuda.Stream(priority=prio)
o = {}
def step():
    if single:
        o["s"] = fht.full(t, shifted=True, out_shifted=o.get("s"), aux_stream=aux)
    else:
        o["h"], o["s"] = fht.full(t, pair=True, out=o.get("h"), out_shifted=o.get("s"), aux_stream=aux)
for _ in range(4): step()
torch.cuda.synchronize()
ts = []
for _ in range(12):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); step(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(json.dumps({"ms": statistics.median(ts), "min": min(ts)}))
'''

CASES = [
    ("one_chunk", {}, 0),
    ("chunk1_prio0", {"FHT_SCRATCH_BUDGET_MB": "60"}, 0),
    ("chunk1_prio_hi", {"FHT_SCRATCH_BUDGET_MB": "60"}, -5),
    ("chunk2_prio_hi", {"FHT_SCRATCH_BUDGET_MB": "140"}, -5),
    ("chunk4_prio_hi", {"FHT_SCRATCH_BUDGET_MB": "280"}, -5),
    ("chunk8_prio_hi", {"FHT_SCRATCH_BUDGET_MB": "560"}, -5),
    ("split_stagger_prio0", {"FHT_SPLIT_BATCH": "1", "FHT_SPLIT_STAGGER": "1"}, 0),
    ("split_stagger_prio_hi", {"FHT_SPLIT_BATCH": "1", "FHT_SPLIT_STAGGER": "1"}, -5),
    ("split_prio_hi", {"FHT_SPLIT_BATCH": "1"}, -5),
]


def main():
    cfg = "5"
    rounds = 2
    if "--config" in sys.argv:
        cfg = sys.argv[sys.argv.index("--config") + 1]
    if "--rounds" in sys.argv:
        rounds = int(sys.argv[sys.argv.index("--rounds") + 1])
    cases = CASES
    if "--cases" in sys.argv:
        want = sys.argv[sys.argv.index("--cases") + 1].split(",")
        cases = [c for c in CASES if c[0] in want]
    res = {}
    for r in range(rounds):
        for single in ("0", "1"):
            for name, env, prio in cases:
                e = dict(os.environ, ROOT=ROOT, **env)
                out = subprocess.run([sys.executable, "-c", CHILD, cfg, str(prio), single], env=e,
                                     capture_output=True, text=True)
                key = f"{name}{'_single' if single == '1' else ''}"
                try:
                    v = json.loads(out.stdout.strip().splitlines()[-1])
                except Exception:
                    v = {"err": (out.stderr or out.stdout)[-300:]}
                res.setdefault(key, []).append(v)
                print(r, key, v, flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
