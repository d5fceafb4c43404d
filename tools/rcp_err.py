"""Relative max-norm error of the class / block variants against the exact-order path (config 5)."""
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dev = torch.device("cuda:0")
c, e = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
plan = vb.P1Plan(ed, c.shape[1], scatter_map=False)
Kx, Mx = vb.fem_p1_assemble_exact(cd, ed, plan)
for v in ("class", "block"):
    K, M, _, _ = vb.fem_p1_assemble(cd, ed, plan, variant=v)
    print("%s %s relmax K %.2e M %.2e" % (os.environ.get("VB_LIBVB", "default"), v,
                                         ((K - Kx).abs().max() / Kx.abs().max()).item(),
                                         ((M - Mx).abs().max() / Mx.abs().max()).item()))
