"""Config-4 (2048^2 square) and config-5 class-variant timing (A/B of libvb builds via VB_LIBVB)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dev = torch.device("cuda:0")
for name, (c, e) in (("config4", synth.square_p1(2048, jitter=0.1, seed=0)),
                     ("config5", synth.cube_kuhn_p1(128, jitter=0.05, seed=0))):
    cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
    plan = vb.P1Plan(ed, c.shape[1], scatter_map=False)
    K = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
    M = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
    f = lambda: vb.fem_p1_assemble(cd, ed, plan, K=K, M=M, variant="class")  # noqa: E731
    for _ in range(5):
        f()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = []
    for _ in range(5):
        a.record(s)
        for _ in range(20):
            f()
        b.record(s)
        b.synchronize()
        out.append(a.elapsed_time(b) / 20)
    print("%s %s class %.4f ms" % (os.environ.get("VB_LIBVB", "default"), name, statistics.median(out)))
