#!/usr/bin/env python
"""Host time per fht.full call on config 5's batch: with / without the auxiliary stream, and the
cost of the Python layer alone (descriptors etc.) vs the C call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1811_06378_b200 as fht  # noqa: E402
import synth  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
t = torch.from_numpy(synth.batch(cid)).cuda()
aux = torch.cuda.Stream()
h, s = fht.full(t, pair=True)
ws = torch.empty(fht.workspace_bytes(fht.FHT_MODE_FULL, fht._image(t)[0], None), dtype=torch.uint8, device="cuda")
for label, a in (("aux", aux), ("no aux", None)):
    for _ in range(5):
        fht.full(t, pair=True, out=h, out_shifted=s, workspace=ws, aux_stream=a)
    torch.cuda.synchronize()
    n = 50
    t0 = time.perf_counter()
    for _ in range(n):
        fht.full(t, pair=True, out=h, out_shifted=s, workspace=ws, aux_stream=a)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"config {cid} {label}: host {(t1 - t0) / n * 1e6:.1f} us per call; wall incl. GPU {(t2 - t0) / n * 1e6:.1f} us")
