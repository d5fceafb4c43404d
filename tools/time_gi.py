"""GI alone on the config-5 volume integral (4 points, scalar) and the L10 surface flux (1 point, 3-vector)."""
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dev = torch.device("cuda:0")


def tm(fn, reps=20):
    for _ in range(3):
        fn()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = []
    for _ in range(5):
        a.record(s)
        for _ in range(reps):
            fn()
        b.record(s)
        b.synchronize()
        out.append(a.elapsed_time(b) / reps)
    return statistics.median(out)


ne = 12582912
fip = torch.rand((4, 1, ne), dtype=torch.float64, device=dev)
sz = torch.rand(ne, dtype=torch.float64, device=dev)
w = np.full(4, 0.25)
val, work = vb.vb_gi(fip, w, sz)
ms = tm(lambda: vb.vb_gi(fip, w, sz, value=val, work=work))
print("GI d=1 nip=4 N=%d: %.4f ms, %.0f GB/s" % (ne, ms, ne * 40 / ms / 1e6))
F = 20971520
fip3 = torch.rand((1, 3, F), dtype=torch.float64, device=dev)
nr = torch.rand((3, F), dtype=torch.float64, device=dev)
sz3 = torch.rand(F, dtype=torch.float64, device=dev)
val3, work3 = vb.vb_gi(fip3, [1.0], sz3, normals=nr)
ms = tm(lambda: vb.vb_gi(fip3, [1.0], sz3, normals=nr, value=val3, work=work3))
print("GI d=3 nip=1 normals N=%d: %.4f ms, %.0f GB/s" % (F, ms, F * 56 / ms / 1e6))
