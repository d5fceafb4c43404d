"""Time fem_p1_pattern (count + fill, both plans) on the config-5 mesh."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

c, e = synth.cube_kuhn_p1(128)
ed = torch.from_numpy(e).cuda()
vb.P1Plan(ed, c.shape[1])
torch.cuda.synchronize()
for label, sm, gp in (("both plans", True, True), ("gather plan only", False, True), ("pattern only", False, False)):
    t = time.perf_counter()
    for _ in range(10):
        vb.P1Plan(ed, c.shape[1], scatter_map=sm, gather_plan=gp)
    torch.cuda.synchronize()
    print("pattern %s: %.2f ms" % (label, (time.perf_counter() - t) / 10 * 1e3))
