"""Time fem_p1_assemble_coef (NEXT-1) on the paper's 3D level-7 mesh, both variants."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

c, e = synth.cube_kuhn_p1(128, jitter=0.0, flip=(0, 0, 1))
dev = torch.device("cuda:0")
cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
plan = vb.P1Plan(ed, c.shape[1])
cf = (1.0, (1.0, 1.0, 1.0))
tag = os.path.basename(os.environ.get("VB_LIBVB", "default"))
for gqo in (1, 2):
    for mode, name in ((vb.VB_ASSEMBLE_GATHER, "gather"), (vb.VB_ASSEMBLE_ATOMIC, "atomic")):
        K, M = vb.fem_p1_assemble_coef(cd, ed, plan, gqo=gqo, cK=cf, cM=cf, mode=mode)[:2]
        for _ in range(3):
            vb.fem_p1_assemble_coef(cd, ed, plan, gqo=gqo, cK=cf, cM=cf, mode=mode, K=K, M=M)
        s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(20):
            vb.fem_p1_assemble_coef(cd, ed, plan, gqo=gqo, cK=cf, cM=cf, mode=mode, K=K, M=M)
        t.record()
        torch.cuda.synchronize()
        print("%-14s gqo=%d %-6s %.4f ms" % (tag, gqo, name, s.elapsed_time(t) / 20), flush=True)
