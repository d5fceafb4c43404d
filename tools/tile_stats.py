"""Tile plan statistics and tile-vs-class timing on config 5 (or --n N Kuhn cube / --dim 2 square)."""
import argparse
import statistics
import sys
import time

import numpy as np
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


ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--dim", type=int, default=3)
args = ap.parse_args()
dev = torch.device("cuda:0")
if args.dim == 3:
    c, e = synth.cube_kuhn_p1(args.n, jitter=0.05, seed=0)
else:
    c, e = synth.square_p1(args.n, jitter=0.1, seed=0)
cd, ed = torch.from_numpy(c).to(dev), torch.from_numpy(e).to(dev)
plan = vb.P1Plan(ed, c.shape[1], scatter_map=False)
torch.cuda.synchronize()
t0 = time.perf_counter()
ok = plan.tiles(cd, ed)
torch.cuda.synchronize()
print("tile plan ms %.2f ok %s %s" % ((time.perf_counter() - t0) * 1e3, ok, plan.tile_reason))
print("stats (entries, max elems/tile, max nodes/tile, max colors, reason, T):", plan.tile_stats,
      "entries/element %.3f" % (plan.tile_stats[0] / e.shape[1]))
meta = plan.tile_meta.cpu().numpy()
cols = plan.tile_colors.cpu().numpy()
ncol = meta[:, 2]
print("colors per tile: hist", np.bincount(ncol).tolist())
T = meta.shape[0]
per_color = np.concatenate([np.diff(cols[t, :ncol[t] + 1]) for t in range(0, T, max(1, T // 2000))])
print("entries per color: mean %.1f min %d max %d" % (per_color.mean(), per_color.min(), per_color.max()))
print("local nodes per tile: mean %.1f; entries per tile mean %.1f" % (meta[:, 1].mean(),
                                                                      (cols[np.arange(T), ncol] - cols[:, 0]).mean()))
K = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
M = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
for v in ("tile", "class"):
    ms = tm(lambda: vb.fem_p1_assemble(cd, ed, plan, K=K, M=M, variant=v))
    print("variant %s: %.4f ms  (%.1f G el/s)" % (v, ms, e.shape[1] / ms / 1e6))
Kt = torch.empty_like(K)
Mt = torch.empty_like(M)
vb.fem_p1_assemble(cd, ed, plan, K=Kt, M=Mt, variant="tile")
vb.fem_p1_assemble(cd, ed, plan, K=K, M=M, variant="class")
print("tile vs class relmax K %.2e M %.2e" % (((Kt - K).abs().max() / K.abs().max()).item(),
                                              ((Mt - M).abs().max() / M.abs().max()).item()))
