"""Small driver for ncu captures of the secondary kernels (config 2 page ops,
config 3 surface, NEXT-2 rhs): each op runs 4 times on the BASELINE shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dev = torch.device("cuda:0")
N = 1 << 20
A = torch.from_numpy(synth.normal_pages(4, 4, N, stream=10)).to(dev)
B = torch.from_numpy(synth.normal_pages(4, 4, N, stream=11)).to(dev)
X, _ = synth.inverse_pages(4, N, seed=0)
Xd = torch.from_numpy(X).to(dev)
xyz, tri = synth.icosphere(10, perturb=0.01, seed=0)
xd, td = torch.from_numpy(xyz).to(dev), torch.from_numpy(tri).to(dev)
for _ in range(4):
    vb.vb_page_mtimes(A, B)
    vb.vb_page_inv(Xd)
    vb.vb_tri_surface(xd, td)
torch.cuda.synchronize()
print("ok")
