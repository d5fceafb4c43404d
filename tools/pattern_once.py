"""One generic pattern build on configs[4] (for ncu captures of the pattern kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dev = torch.device("cuda:0")
c, e = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
ed = torch.from_numpy(e).to(dev)
for _ in range(2):
    vb.P1Plan(ed, c.shape[1])
torch.cuda.synchronize()
print("ok")
