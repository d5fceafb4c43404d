"""Driver for ncu captures of the class-variant assembly on a BASELINE mesh
(kuhn128 = configs[4] by default): builds the plan, then runs the kernel --reps times."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--mesh", default="kuhn128")
ap.add_argument("--variant", default="class")
a = ap.parse_args()
c, e = synth.cube_kuhn_p1(128, jitter=0.05, seed=0) if a.mesh == "kuhn128" else synth.square_p1(2048, 0.1, 0)
dev = torch.device("cuda:0")
cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
plan = vb.P1Plan(ed, c.shape[1])
plan.classes()
K, M, _, _ = vb.fem_p1_assemble(cd, ed, plan, variant=a.variant)
for _ in range(a.reps):
    vb.fem_p1_assemble(cd, ed, plan, variant=a.variant, K=K, M=M)
torch.cuda.synchronize()
print("done")
