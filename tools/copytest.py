"""Two-stream pipeline stall probe: per step on stream j: H2D, work, D2H; then a
host sync in the middle of the work (as fem_p1_pattern's count phase does)."""
import sys
import time

import torch

dev = torch.device("cuda:0")
mode = sys.argv[1] if len(sys.argv) > 1 else "sync"
in_h = torch.empty(250 * 2**20, dtype=torch.uint8).pin_memory()
outs = [torch.empty(600 * 2**20, dtype=torch.uint8).pin_memory() for _ in range(2)]
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
live = [None, None]
log = []
hlog = []


def step(i):
    j = i % 2
    s = streams[j]
    h = [time.perf_counter()]
    s.synchronize()
    h.append(time.perf_counter())
    live[j] = None
    h.append(time.perf_counter())
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with torch.cuda.stream(s):
        ev[0].record(s)
        h.append(time.perf_counter())
        d = in_h.to(dev, non_blocking=True)
        h.append(time.perf_counter())
        ev[1].record(s)
        torch.cuda._sleep(3_000_000)
        if mode == "sync":
            s.synchronize()
        elif mode == "mapped":
            pass
        torch.cuda._sleep(3_000_000)
        big = torch.empty(600 * 2**20, dtype=torch.uint8, device=dev)
        ev[2].record(s)
        outs[j].copy_(big, non_blocking=True)
        ev[3].record(s)
    h.append(time.perf_counter())
    live[j] = (d, big)
    log.append(ev)
    hlog.append(h)


for i in range(2):
    step(i)
torch.cuda.synchronize()
log.clear()
hlog.clear()
base = torch.cuda.Event(enable_timing=True)
base.record()
base.synchronize()
t = time.perf_counter()
for i in range(6):
    step(i)
torch.cuda.synchronize()
print(mode, "%.2f ms/step" % ((time.perf_counter() - t) * 1e3 / 6))
for i, ev in enumerate(log):
    ts = [base.elapsed_time(x) for x in ev]
    print("  host", " ".join("%.1f" % ((x - t) * 1e3) for x in hlog[i]))
    print("  step %d start %.1f h2d %.2f work %.2f d2h %.2f" % (i, ts[0], ts[1] - ts[0], ts[2] - ts[1], ts[3] - ts[2]))
