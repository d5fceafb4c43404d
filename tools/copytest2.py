"""Pipeline probe with dedicated upload / download streams (copy engines per
direction) and event hand-offs to two alternating compute streams."""
import time

import torch

dev = torch.device("cuda:0")
in_h = torch.empty(250 * 2**20, dtype=torch.uint8).pin_memory()
outs = [torch.empty(600 * 2**20, dtype=torch.uint8).pin_memory() for _ in range(2)]
up, down = torch.cuda.Stream(), torch.cuda.Stream()
comp = [torch.cuda.Stream(), torch.cuda.Stream()]
done = [None, None]
log = []
live = [None, None]


def step(i):
    j = i % 2
    if done[j] is not None:
        done[j].synchronize()          # slot j's previous download finished (host buffers free)
    live[j] = None
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with torch.cuda.stream(up):
        ev[0].record(up)
        d = in_h.to(dev, non_blocking=True)
        ev[1].record(up)
    comp[j].wait_event(ev[1])
    with torch.cuda.stream(comp[j]):
        torch.cuda._sleep(3_000_000)
        big = torch.empty(600 * 2**20, dtype=torch.uint8, device=dev)
        ev[2].record(comp[j])
    down.wait_event(ev[2])
    with torch.cuda.stream(down):
        outs[j].copy_(big, non_blocking=True)
        ev[3].record(down)
    d.record_stream(comp[j])
    big.record_stream(down)
    done[j] = ev[3]
    live[j] = (d, big)
    log.append(ev)


for i in range(2):
    step(i)
torch.cuda.synchronize()
log.clear()
base = torch.cuda.Event(enable_timing=True)
base.record()
base.synchronize()
t = time.perf_counter()
for i in range(6):
    step(i)
torch.cuda.synchronize()
print("up/down streams: %.2f ms/step" % ((time.perf_counter() - t) * 1e3 / 6))
for i, ev in enumerate(log):
    ts = [base.elapsed_time(x) for x in ev]
    print("  step %d start %.1f h2d %.2f work-end %.2f d2h-end %.2f" % (i, ts[0], ts[1] - ts[0], ts[2], ts[3]))
