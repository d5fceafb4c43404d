import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2404_16039_b200 import vb
dev = torch.device("cuda:0"); N = 1 << 20
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for n in (2, 3, 4):
    X = torch.from_numpy(synth.inverse_pages(n, N, seed=0)[0]).to(dev)
    Xi, det, _ = vb.vb_page_inv(X)
    fs = torch.zeros(1, dtype=torch.int64, device=dev)
    for flag in (None, fs):
        ts = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); vb.vb_page_inv(X, Xinv=Xi, det=det, first_singular=flag); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b))
        ms = sorted(ts)[10]
        print("inv n=%d flag=%s: %.4f ms, %.0f GB/s" % (n, flag is not None, ms, (2 * n * n + 1) * 8 * N / ms / 1e6))
