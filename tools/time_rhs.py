"""NEXT-2 load vector (fem_p1_rhs) on the config-5 mesh, gqo = 2."""
import os
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dev = torch.device("cuda:0")
c, e = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
plan = vb.P1Plan(ed, c.shape[1], scatter_map=False)
fq = torch.rand((4, e.shape[1]), dtype=torch.float64, device=dev)
f = lambda: vb.fem_p1_rhs(cd, ed, fq, plan=plan, gqo=2)  # noqa: E731
for _ in range(3):
    f()
s = torch.cuda.current_stream()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = []
for _ in range(5):
    a.record(s)
    for _ in range(10):
        f()
    b.record(s)
    b.synchronize()
    out.append(a.elapsed_time(b) / 10)
print("%s rhs config5: %.4f ms" % (os.environ.get("VB_LIBVB", "default"), statistics.median(out)))
