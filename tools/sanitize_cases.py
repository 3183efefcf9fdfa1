"""Small invocations of every kernel for compute-sanitizer: k_p1 / k_p2 (all four slots,
u8 / i32 / f32, the R = 6 tiles, the persistent pass 1 k_p1p, the range loaders), k_fhtshift, k_fold, k_range_tables, the peaks
kernels and the v1 kernels of degenerate frames. Exits 0 when every call ran (results are checked by
the GPU test suite, not here).

    compute-sanitizer --tool {memcheck|racecheck|synccheck|initcheck} python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1811_06378_b200 as fht
from synth import random_image


def main():
    dev = torch.device("cuda:0")
    n = 0
    for shape, dt in [((48, 40), "f32"), ((64, 64), "u8"), ((33, 17), "i32"), ((128, 72), "f32"), ((2, 9), "f32")]:
        t = torch.from_numpy(random_image(shape, dt, seed=1)).to(dev)
        h, s = fht.full(t, pair=True)                 # 4-slot merged pass pair, fused fhtshift
        fht.fhtshift(h)
        fht.full(t, layout="concat", shifted=True)
        if min(shape) >= 8:                          # (pads other than Hp need the v2 tiling)
            fht.quadrant(t, fht.QC, pad=3, pair=True)    # fold path
            fht.quadrant(t, fht.QB, pad=shape[0] + 5)    # direct pad path
        fht.peaks(h, 8)
        n += 7
    t = torch.from_numpy(random_image((256, 256), "f32", seed=2)).to(dev)
    fht.full(t, pair=True, aux_stream=torch.cuda.Stream())   # two-stream orientation split
    # R = 6 pass-1 tiles (K = 11: 6 + 5) on a narrow image
    t = torch.from_numpy(random_image((2048, 24), "f32", seed=3)).to(dev)
    fht.quadrant(t, fht.QA, pair=True)
    u = torch.from_numpy(random_image((2048, 24), "u8", seed=4)).to(dev)
    fht.quadrant(u, fht.QB)
    # persistent pass 1 (k_p1p): 64-row strips of a 4-byte image, all four slots (two transposed), two images
    t = torch.from_numpy(np.stack([random_image((2048, 2048), "f32", seed=6 + b) for b in range(2)])).to(dev)
    fht.full(t, pair=True)
    n += 1
    # persistent u8 pass 1 (k_p1p8): 16-row strips, all four slots, three images
    u = torch.from_numpy(np.stack([random_image((512, 512), "u8", seed=9 + b) for b in range(3)])).to(dev)
    fht.full(u, pair=True)
    n += 1
    # §4 range in the persistent pass 1 (64-row strips)
    t = torch.from_numpy(random_image((2048, 1200), "f32", seed=10)).to(dev)
    fht.angle_range(t, 5.0, 30.0, pair=True)
    n += 1
    # §4 range: scaled (TMA gather loader, alpha >= 1), alpha < 1 gather, pruned, horizontal
    t = torch.from_numpy(random_image((96, 80), "f32", seed=5)).to(dev)
    fht.angle_range(t, -15.0, 15.0, pair=True)
    fht.angle_range(t, -80.0, 80.0)
    fht.angle_range(t, fht.angle_plan(96, 80, -15, 15, pruned=True), pair=True)
    r = fht.angle_range(t, fht.angle_plan(96, 80, -20, 20, horizontal=True))
    fht.fhtshift(r)
    n += 9
    torch.cuda.synchronize()
    print(f"sanitize cases ok ({n} calls)")


if __name__ == "__main__":
    main()
