import os, sys
sys.path.insert(0, "/root/repo")
import torch, synth
from paper_2404_16039_b200 import vb
c, e = synth.p2_from_p1(*synth.cube_kuhn_p1(64, jitter=0.0, flip=(0, 0, 1)))
dev = torch.device("cuda:0")
cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
plan = vb.Plan(ed, c.shape[1])
K, M, _, _ = vb.fem_p2_assemble(cd, ed, plan, mode=vb.VB_ASSEMBLE_GATHER)
for _ in range(3):
    vb.fem_p2_assemble(cd, ed, plan, K=K, M=M, mode=vb.VB_ASSEMBLE_GATHER)
torch.cuda.synchronize()
