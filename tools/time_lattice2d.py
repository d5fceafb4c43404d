"""Time the 2D lattice kernel against the class kernel on configs[3] (CUDA events, L2 flushed between reps)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
dev = torch.device("cuda:0")
c, e = synth.square_p1(n, jitter=0.1, seed=0)
cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
plan = vb.P1Plan(ed, c.shape[1], scatter_map=False)
assert plan.lattice(ed), plan.lattice_reason
K = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
M = torch.empty_like(K)
FLUSH = os.environ.get("VB_FLUSH", "1") == "1"
flush = torch.empty(2 * 132644864 // 4, dtype=torch.float32, device=dev)


def t(fn, reps=20):
    for _ in range(3):
        fn()
    out = []
    for _ in range(reps):
        if FLUSH:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out), min(out)


tl = t(lambda: vb.fem_p1_assemble_lattice(cd, plan, K=K, M=M))
Kl, Ml = K.clone(), M.clone()
tc = t(lambda: vb.fem_p1_assemble_classes(cd, plan, K=K, M=M))
rk = ((Kl - K).abs().max() / K.abs().max()).item()
rm = ((Ml - M).abs().max() / M.abs().max()).item()
alg = c.shape[1] * 16 + e.size * 4 + 2 * plan.nnz * 8
print("n=%d segments=%d lattice2d %.4f ms (min %.4f) class %.4f ms; relmax K %.2e M %.2e; ALG frac %.3f"
      % (n, plan.lattice_tiles, tl[0], tl[1], tc[0], rk, rm, alg / tl[0] / 1e6 / 6527.1))
