import os, sys
sys.path.insert(0, "/root/repo")
import torch, synth
from paper_2404_16039_b200 import vb
c, e = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
dev = torch.device("cuda:0")
cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
plan = vb.P1Plan(ed, c.shape[1])
tag = os.path.basename(os.environ.get("VB_LIBVB", "default"))
if tag.startswith("pack32"):  # noqa
    plan.node_elem_slot16 = plan.node_elem_slot   # this build reads 32-bit words with the compact budget
K, M, _, _ = vb.fem_p1_assemble(cd, ed, plan)
for compact in (False, True):
    for _ in range(3):
        vb.fem_p1_assemble(cd, ed, plan, K=K, M=M, compact=compact)
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(30):
        vb.fem_p1_assemble(cd, ed, plan, K=K, M=M, compact=compact)
    t.record(); torch.cuda.synchronize()
    print(tag, "compact" if compact else "wide", "%.4f ms" % (s.elapsed_time(t) / 30))
