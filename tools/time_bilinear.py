import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2404_16039_b200 import vb
dev = torch.device("cuda:0"); ne = 12582912
Kl = torch.from_numpy(synth.normal_pages(4, 4, ne, stream=10)).to(dev)
u = torch.from_numpy(synth.normal_pages(4, 1, ne, stream=11)).to(dev)
s = vb.vb_page_bilinear(u, Kl, u)
for _ in range(3): vb.vb_page_bilinear(u, Kl, u, s=s)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); a.record()
for _ in range(10): vb.vb_page_bilinear(u, Kl, u, s=s)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
print("bilinear 4x4 over %d pages: %.3f ms, %.0f GB/s" % (ne, ms, (16 + 4 + 4 + 1) * 8 * ne / ms / 1e6))
