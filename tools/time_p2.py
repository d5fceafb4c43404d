"""Time fem_p2_assemble on the paper's 3D level-6 P2 mesh: full (atomics) vs
local matrices only (element compute + local stores, no atomics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

c, e = synth.p2_from_p1(*synth.cube_kuhn_p1(64, jitter=0.0, flip=(0, 0, 1)))
dev = torch.device("cuda:0")
cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
plan = vb.Plan(ed, c.shape[1])
tag = os.path.basename(os.environ.get("VB_LIBVB", "default"))


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, u = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    u.record()
    torch.cuda.synchronize()
    return s.elapsed_time(u) / reps


K, M, _, _ = vb.fem_p2_assemble(cd, ed, plan)
print("%s P2 L6 (ne=%d): global K+M %.3f ms" % (tag, e.shape[1], t(lambda: vb.fem_p2_assemble(cd, ed, plan, K=K, M=M))))
G = vb.VB_ASSEMBLE_GATHER
print("%s P2 L6: gather K+M %.3f ms" % (tag, t(lambda: vb.fem_p2_assemble(cd, ed, plan, K=K, M=M, mode=G))))
print("%s P2 L6: K only %.3f ms" % (tag, t(lambda: vb.fem_p2_assemble(cd, ed, plan, want_M=False, K=K))))
print("%s P2 L6: local only %.3f ms" % (tag, t(lambda: vb.fem_p2_assemble(cd, ed, plan, want_K=False, want_M=False, want_local=True))))
