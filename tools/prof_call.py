"""One benched call of a config, a few times (for ncu): python tools/prof_call.py --config 5 [--reps 3]."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1811_06378_b200 as fht
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--single", action="store_true")
args = ap.parse_args()
cc = synth.CONFIGS[args.config]
t = torch.from_numpy(synth.batch(args.config)).cuda()
o = {}
for _ in range(args.reps):
    if cc["mode"] == "full" and args.config in (2, 5) and not args.single:
        o["h"], o["s"] = fht.full(t, pair=True, out=o.get("h"), out_shifted=o.get("s"))
    elif cc["mode"] == "full" and args.config in (2, 5):
        o["s"] = fht.full(t, shifted=True, out_shifted=o.get("s"))
    elif cc["mode"] == "full":
        o["h"] = fht.full(t, out=o.get("h"))
    elif cc["mode"] == "range":
        o["h"], o["s"] = fht.angle_range(t, cc["theta_min"], cc["theta_max"], pair=True, out=o.get("h"), out_shifted=o.get("s"))
    else:
        o["h"] = fht.quadrant(t, fht.QA, out=o.get("h"))
torch.cuda.synchronize()
print("ok", cc["name"])
