"""vb_create_coords3D alone on the config-5 mesh: coords3D + vectors3D, vectors3D only (ALG bytes, GB/s)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dev = torch.device("cuda:0")
coords, elems = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
cd, ed = torch.from_numpy(coords).to(dev), torch.from_numpy(elems).to(dev)
nn, ne = coords.shape[1], elems.shape[1]
flush = torch.empty(2 * 132644864 // 4, dtype=torch.float32, device=dev)
s = torch.cuda.current_stream()
for name, kw, nbytes in (("both", {}, ne * (16 + 96 + 72) + nn * 24), ("vectors3D", dict(want_coords3D=False), ne * (16 + 72) + nn * 24)):
    out = []
    for _ in range(3):
        vb.vb_create_coords3D(cd, ed, **kw)
    for _ in range(15):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        vb.vb_create_coords3D(cd, ed, **kw)
        b.record(s)
        b.synchronize()
        out.append(a.elapsed_time(b))
    ms = statistics.median(out)
    print("%s create_coords3D %-9s: %.4f ms, %.0f GB/s ALG" % (os.environ.get("VB_LIBVB", "default")[-12:], name, ms, nbytes / ms / 1e6))
