"""Time the atomic (north-star scatter) assembly on configs[4] and configs[3] and check it against the class variant."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dev = torch.device("cuda:0")


def t(fn, reps=10):
    for _ in range(3):
        fn()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


for name, (c, e) in (("configs[4] 3D", synth.cube_kuhn_p1(128, jitter=0.05, seed=0)),
                     ("configs[3] 2D", synth.square_p1(2048, jitter=0.1, seed=0))):
    cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
    plan = vb.P1Plan(ed, c.shape[1])
    K = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
    M = torch.empty_like(K)
    ms = t(lambda: vb.fem_p1_assemble(cd, ed, plan, mode=vb.VB_ASSEMBLE_ATOMIC, K=K, M=M))
    Kc, Mc, _, _ = vb.fem_p1_assemble(cd, ed, plan, variant="class")
    rk = ((K - Kc).abs().max() / Kc.abs().max()).item()
    rm = ((M - Mc).abs().max() / Mc.abs().max()).item()
    print("%s atomic %.4f ms (%.3g elements/s); relmax vs class K %.2e M %.2e" % (name, ms, e.shape[1] / ms * 1e3, rk, rm))
