"""A/B of the pipelined kernel (fht_pipe.cuh) against the two-launch path on the benched calls, same
process and box: FHT_PIPE=0/1 (and FHT_PIPE_D / FHT_PIPE_NBUF / FHT_PIPE_UNIT_MB variants), CUDA events
around back-to-back steps, L2 flushed between steps for working sets below 2x L2.

    python tools/pipe_ab.py [--configs 5,2,3] [--steps 20]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1811_06378_b200 as fht
import synth

# (name, environment, auxiliary stream: None = no aux stream, else its priority (0 default, -1 high, 1 low... torch
# uses lower numbers for higher priority))
VARIANTS = {
    "pipe": [("two-launch", {"FHT_PIPE": "0"}, 0), ("pipe D2 N4", {"FHT_PIPE": "1"}, 0),
             ("pipe D1 N3", {"FHT_PIPE": "1", "FHT_PIPE_D": "1", "FHT_PIPE_NBUF": "3"}, 0),
             ("pipe D3 N5", {"FHT_PIPE": "1", "FHT_PIPE_D": "3", "FHT_PIPE_NBUF": "5"}, 0)],
    "chunks": [("one chunk", {}, None), ("70 MB chunks (1 image)", {"FHT_SCRATCH_BUDGET_MB": "70"}, None),
               ("140 MB chunks (2 images)", {"FHT_SCRATCH_BUDGET_MB": "140"}, None),
               ("280 MB chunks (4 images)", {"FHT_SCRATCH_BUDGET_MB": "280"}, None),
               ("70 MB chunks + aux", {"FHT_SCRATCH_BUDGET_MB": "70"}, 0),
               ("140 MB chunks + aux", {"FHT_SCRATCH_BUDGET_MB": "140"}, 0)],
    "split": [("merged (no aux)", {}, None), ("split", {"FHT_SPLIT_BATCH": "1"}, 0), ("split stagger", {"FHT_SPLIT_STAGGER": "1", "FHT_SPLIT_BATCH": "1"}, 0),
              ("split stagger, aux high prio", {"FHT_SPLIT_STAGGER": "1", "FHT_SPLIT_BATCH": "1"}, -1),
              ("split, aux high prio", {"FHT_SPLIT_BATCH": "1"}, -1)],
}
KEYS = ("FHT_PIPE", "FHT_PIPE_D", "FHT_PIPE_NBUF", "FHT_PIPE_UNIT_MB", "FHT_SPLIT_STAGGER", "FHT_SCRATCH_BUDGET_MB", "FHT_SPLIT_BATCH")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="5,2,3")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--single", action="store_true", help="C2/C5 write only the fhtshift-ed image")
    ap.add_argument("--set", default="pipe", choices=sorted(VARIANTS))
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = torch.empty(512 << 18, dtype=torch.float32, device=dev)
    out = {}
    for cid in [int(c) for c in args.configs.split(",")]:
        cc = synth.CONFIGS[cid]
        t = torch.from_numpy(synth.batch(cid)).to(dev)
        small = t.numel() * t.element_size() * 9 < 2 * torch.cuda.get_device_properties(dev).L2_cache_size
        res = {}
        for name, env, prio in VARIANTS[args.set]:
            aux = None if prio is None else torch.cuda.Stream(priority=prio)
            for k in KEYS:
                os.environ.pop(k, None)
            os.environ.update(env)
            o = {}

            def step():
                if cc["mode"] == "full" and cid in (2, 5) and not args.single:
                    o["h"], o["s"] = fht.full(t, pair=True, out=o.get("h"), out_shifted=o.get("s"), aux_stream=aux)
                elif cc["mode"] == "full" and cid in (2, 5):
                    o["s"] = fht.full(t, shifted=True, out_shifted=o.get("s"), aux_stream=aux)
                elif cc["mode"] == "full":
                    o["h"] = fht.full(t, out=o.get("h"), aux_stream=aux)
                else:
                    o["h"] = fht.quadrant(t, fht.QA, out=o.get("h"))
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            ms = []
            for _ in range(args.steps):
                if small:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                step()
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            # bit-identical outputs across variants
            sig = [float(v.storage.double().sum().item()) for v in o.values()]
            res[name] = {"ms_median": statistics.median(ms), "ms_min": min(ms), "checksum": sig}
            print(cc["name"], name, res[name], flush=True)
            del o
            torch.cuda.empty_cache()
        out[cc["name"]] = res
        del t
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
