"""Break the config-5 end-to-end step into its parts (host wall clock, device synced):
H2D of coords+elems, D2H of row_ptr/col_idx/K/M, both copies concurrently on two
streams, plan build, assembly."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    return sorted(ts)[len(ts) // 2]


c, e = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
dev = torch.device("cuda:0")
hc, he = torch.from_numpy(c).pin_memory(), torch.from_numpy(e).pin_memory()
cd, ed = hc.to(dev), he.to(dev)
plan = vb.P1Plan(ed, c.shape[1])
K, M, _, _ = vb.fem_p1_assemble(cd, ed, plan)
outs = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in
        (("rp", plan.row_ptr), ("ci", plan.col_idx), ("K", K), ("M", M))}
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def h2d():
    cd.copy_(hc, non_blocking=True)
    ed.copy_(he, non_blocking=True)


def d2h():
    outs["rp"].copy_(plan.row_ptr, non_blocking=True)
    outs["ci"].copy_(plan.col_idx, non_blocking=True)
    outs["K"].copy_(K, non_blocking=True)
    outs["M"].copy_(M, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        h2d()
    with torch.cuda.stream(s2):
        d2h()


mb_in = (c.nbytes + e.nbytes) / 1e6
mb_out = sum(v.numel() * v.element_size() for v in outs.values()) / 1e6
t_h2d, t_d2h, t_both = wall(h2d), wall(d2h), wall(both)
print("H2D %.1f MB: %.2f ms (%.1f GB/s)" % (mb_in, t_h2d, mb_in / t_h2d))
print("D2H %.1f MB: %.2f ms (%.1f GB/s)" % (mb_out, t_d2h, mb_out / t_d2h))
print("H2D || D2H: %.2f ms" % t_both)
print("plan (count+fill, gather plan): %.2f ms" % wall(lambda: vb.P1Plan(ed, c.shape[1], scatter_map=False)))
print("plan (count+fill, both plans): %.2f ms" % wall(lambda: vb.P1Plan(ed, c.shape[1])))
print("assemble gather: %.3f ms" % wall(lambda: vb.fem_p1_assemble(cd, ed, plan, K=K, M=M)))

# ---- the bench's two-stream e2e pipeline with event timestamps per phase
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
outs2 = [{k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in outs.items()} for _ in range(2)]
live = [None, None]
evlog = []


hostlog = []


def e2e_step(i):
    j = i % 2
    s = streams[j]
    h = [time.perf_counter()]
    s.synchronize()
    h.append(time.perf_counter())
    live[j] = None
    o = outs2[j]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    with torch.cuda.stream(s):
        ev[0].record(s)
        c2 = hc.to(dev, non_blocking=True)
        e2 = he.to(dev, non_blocking=True)
        ev[1].record(s)
        h.append(time.perf_counter())
        p2 = vb.P1Plan(e2, c.shape[1], scatter_map=False)
        h.append(time.perf_counter())
        ev[2].record(s)
        K2, M2, _, _ = vb.fem_p1_assemble(c2, e2, p2)
        ev[3].record(s)
        o["rp"].copy_(p2.row_ptr, non_blocking=True)
        o["ci"].copy_(p2.col_idx, non_blocking=True)
        o["K"].copy_(K2, non_blocking=True)
        o["M"].copy_(M2, non_blocking=True)
        ev[4].record(s)
    h.append(time.perf_counter())
    hostlog.append(h)
    live[j] = (c2, e2, p2, K2, M2)
    evlog.append(ev)


for i in range(2):
    e2e_step(i)
torch.cuda.synchronize()
evlog.clear()
hostlog.clear()
base = torch.cuda.Event(enable_timing=True)
base.record()
t = time.perf_counter()
base.synchronize()
t = time.perf_counter()
for i in range(8):
    e2e_step(i)
torch.cuda.synchronize()
print("e2e pipeline: %.2f ms/step" % ((time.perf_counter() - t) * 1e3 / 8))
for i, ev in enumerate(evlog):
    ts = [base.elapsed_time(x) for x in ev[:5]]
    hh = [(x - t) * 1e3 for x in hostlog[i]]
    print("  host: enter %.1f  synced %.1f  h2d-enq %.1f  plan-ret %.1f  ret %.1f" % tuple(hh))
    print("step %d: start %.1f  h2d %.2f  plan %.2f  asm %.2f  d2h %.2f  (end %.1f)" %
          (i, ts[0], ts[1] - ts[0], ts[2] - ts[1], ts[3] - ts[2], ts[4] - ts[3], ts[4]))
