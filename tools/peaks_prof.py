#!/usr/bin/env python
"""Run fht.peaks on config 3's Hough planes a few times (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1811_06378_b200 as fht  # noqa: E402
import synth  # noqa: E402

h = fht.full(torch.from_numpy(synth.batch(3)).cuda())
for _ in range(3):
    out = fht.peaks(h, 16)
torch.cuda.synchronize()
print("ok")
