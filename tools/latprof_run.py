"""Per-CTA cycle counts of the lattice kernel (needs the VB_LAT_PROF variant: tools/build_variant.py latprof -DVB_LAT_PROF)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dims = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (128, 128, 128)
dev = torch.device("cuda:0")
c, e = synth.box_kuhn_p1(*dims, jitter=0.05, seed=0)
cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
plan = vb.P1Plan(ed, c.shape[1], scatter_map=False, gather_plan=False)
assert plan.lattice(ed, dims=dims), plan.lattice_reason
for i in range(3):
    vb.fem_p1_assemble_lattice(cd, plan)
    torch.cuda.synchronize()
    print("RUN", i, dims, "tiles", plan.lattice_tiles, flush=True)
