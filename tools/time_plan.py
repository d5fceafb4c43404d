"""Time the one-time plans on configs[4]: lattice plan (element check + closed-form pattern) vs the generic pattern."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dev = torch.device("cuda:0")
c, e = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
ed = torch.from_numpy(e).to(dev)
nn = c.shape[1]


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


print("lattice plan (for_lattice) %.3f ms; generic pattern only %.3f ms; generic + plans %.3f ms"
      % (t(lambda: vb.P1Plan.for_lattice(ed, nn)), t(lambda: vb.P1Plan(ed, nn, scatter_map=False, gather_plan=False)),
         t(lambda: vb.P1Plan(ed, nn))))
