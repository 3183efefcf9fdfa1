import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_06378_b200 as F
from synth import random_image
h, w, dt, q = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
img = random_image((h, w), dt, seed=1)
t = torch.from_numpy(img).cuda()
r = F.quadrant(t, q)
torch.cuda.synchronize()
print("ok", h, w, dt, q, r.launches)
