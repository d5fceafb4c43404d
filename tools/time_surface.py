"""config 3: vb_tri_surface on the level-10 icosphere (L2 flushed between reps)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dev = torch.device("cuda:0")
xyz, tri = synth.icosphere(10, perturb=0.01, seed=0)
xd, td = torch.from_numpy(xyz).to(dev), torch.from_numpy(tri).to(dev)
out = vb.vb_tri_surface(xd, td)
flush = torch.empty(2 * 132644864 // 4, dtype=torch.float32, device=dev)
s = torch.cuda.current_stream()
res = []
for _ in range(3):
    vb.vb_tri_surface(xd, td, out=out, work=out["work"])
for _ in range(15):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    vb.vb_tri_surface(xd, td, out=out, work=out["work"])
    b.record(s)
    b.synchronize()
    res.append(a.elapsed_time(b))
F, V = tri.shape[1], xyz.shape[1]
ms = statistics.median(res)
print("%s surface L10: %.4f ms, %.0f GB/s ALG" % (os.environ.get("VB_LIBVB", "default"), ms, (F * 68 + V * 24) / ms / 1e6))
