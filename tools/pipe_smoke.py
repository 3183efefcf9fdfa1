"""Quick pipelined-kernel check: a 1024^2 f32 full transform (4 units) against the two-launch path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1811_06378_b200 as fht
from synth import random_image

t = torch.from_numpy(random_image((1024, 1024), "f32", seed=1)).cuda()
os.environ["FHT_PIPE"] = "0"
a, sa = fht.full(t, pair=True)
torch.cuda.synchronize()
os.environ["FHT_PIPE"] = "1"
b, sb = fht.full(t, pair=True)
torch.cuda.synchronize()
print("launches", a.launches, b.launches, "equal", torch.equal(a.storage, b.storage), torch.equal(sa.storage, sb.storage))
if not torch.equal(a.storage, b.storage):
    d = (a.view - b.view).abs()
    print("diff cells", int((d > 0).sum()), "per quadrant", [(int((d[0, q] > 0).sum())) for q in range(4)])
