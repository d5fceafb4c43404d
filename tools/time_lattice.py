"""Time the lattice kernel against the class kernel on configs[4] (CUDA events, 20 reps)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dev = torch.device("cuda:0")
c, e = synth.cube_kuhn_p1(n, jitter=0.05, seed=0)
cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
plan = vb.P1Plan(ed, c.shape[1], scatter_map=False)
assert plan.lattice(ed), plan.lattice_reason
K = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
M = torch.empty_like(K)


def t(fn, reps=20):
    """back-to-back launches (as bench.py's timed steps), one event pair per launch"""
    for _ in range(3):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    out = [a.elapsed_time(b) for a, b in ev]
    if os.environ.get("VB_TIMES"):
        print(" ".join("%.4f" % x for x in out))
    return statistics.median(out), min(out)


tl = t(lambda: vb.fem_p1_assemble_lattice(cd, plan, K=K, M=M))
Kl, Ml = K.clone(), M.clone()
tc = t(lambda: vb.fem_p1_assemble_classes(cd, plan, K=K, M=M))
rk = ((Kl - K).abs().max() / K.abs().max()).item()
rm = ((Ml - M).abs().max() / M.abs().max()).item()
alg = c.shape[1] * 24 + e.size * 4 + 2 * plan.nnz * 8
lat_b = c.shape[1] * 24 + 2 * plan.nnz * 8 + (c.shape[1] + 1) * 4
print("n=%d tiles=%d lattice %.4f ms (min %.4f) class %.4f ms; relmax K %.2e M %.2e; ALG frac %.3f, lattice-bytes frac %.3f"
      % (n, plan.lattice_tiles, tl[0], tl[1], tc[0], rk, rm, alg / tl[0] / 1e6 / 6552.3, lat_b / tl[0] / 1e6 / 6552.3))
