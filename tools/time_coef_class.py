"""NEXT-1 (paper tab:KM_P1_3D level 7 / tab:KM_P1_2D level 11 with --dim 2: c = e^{sum x}, gqo = 2): class vs block."""
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402


def tm(fn, reps=10):
    s = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


dev = torch.device("cuda:0")
if "--dim" in sys.argv and sys.argv[sys.argv.index("--dim") + 1] == "2":
    c, e = synth.square_crossed_p1(2 ** 11)
else:
    c, e = synth.cube_kuhn_p1(128, jitter=0.0, flip=(0, 0, 1))
cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
plan = vb.P1Plan(ed, c.shape[1], scatter_map=False)
plan.classes()
print("class coverage", plan.class_coverage(), plan.class_stats)
K = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
M = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
res = {}
for v in ("class", "block"):
    ms = tm(lambda: vb.fem_p1_assemble_coef(cd, ed, plan, gqo=2, K=K, M=M, variant=v))
    res[v] = (K.clone(), M.clone())
    print("NEXT-1 variant %s: %.4f ms (%.2f G tets/s)" % (v, ms, e.shape[1] / ms / 1e6))
(K1, M1), (K2, M2) = res["class"], res["block"]
print("class vs block relmax K %.2e M %.2e" % (((K1 - K2).abs().max() / K2.abs().max()).item(),
                                               ((M1 - M2).abs().max() / M2.abs().max()).item()))
