import sys; sys.path.insert(0,'/root/repo')
import torch, synth
from paper_2404_16039_b200 import vb
dev=torch.device('cuda:0'); N=1<<20
for n in (2,3,4):
    A=torch.from_numpy(synth.normal_pages(n,n,N,stream=10)).to(dev)
    Z=vb.vb_page_transpose(A)
    for _ in range(3): vb.vb_page_transpose(A, Z=Z)
    flush=torch.empty(256<<20, dtype=torch.uint8, device=dev)
    ts=[]
    for _ in range(20):
        flush.zero_(); s=torch.cuda.Event(enable_timing=True); t=torch.cuda.Event(enable_timing=True)
        s.record(); vb.vb_page_transpose(A, Z=Z); t.record(); t.synchronize(); ts.append(s.elapsed_time(t))
    ts.sort(); ms=ts[10]; print(n, "%.4f ms  %.0f GB/s"%(ms, 16*n*n*N/ms/1e6))
