"""Timing of the class variant (fem_p1_assemble_classes) against the 32-row
block variant of the gather assembly on the BASELINE meshes, plus the class
plan's build time and coverage.  Checks the two variants agree (relmax).

usage: python tools/time_class.py [--reps 50] [--meshes kuhn128,square2048]"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

MESHES = {
    "kuhn128": lambda: synth.cube_kuhn_p1(128, jitter=0.05, seed=0),
    "square2048": lambda: synth.square_p1(2048, jitter=0.1, seed=0),
    "delaunay3d_64": lambda: synth.delaunay_p1(3, 64, seed=0),
}


def timed(fn, reps):
    for _ in range(3):
        fn()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    t.record()
    torch.cuda.synchronize()
    return s.elapsed_time(t) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--meshes", default="kuhn128,square2048")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    for name in a.meshes.split(","):
        c, e = MESHES[name]()
        cd = torch.from_numpy(c).to(dev)
        ed = torch.from_numpy(e).to(dev)
        plan = vb.P1Plan(ed, c.shape[1])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan.classes()
        torch.cuda.synchronize()
        t_cls = (time.perf_counter() - t0) * 1e3
        plan.class_rows = None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan.classes()
        torch.cuda.synchronize()
        t_cls2 = (time.perf_counter() - t0) * 1e3
        Kb, Mb, _, _ = vb.fem_p1_assemble(cd, ed, plan, variant="block")
        Kc, Mc, _, _ = vb.fem_p1_assemble(cd, ed, plan, variant="class")
        torch.cuda.synchronize()
        rk = ((Kc - Kb).abs().max() / Kb.abs().max()).item()
        rm = ((Mc - Mb).abs().max() / Mb.abs().max()).item()
        tb = timed(lambda: vb.fem_p1_assemble(cd, ed, plan, variant="block", K=Kb, M=Mb), a.reps)
        tc = timed(lambda: vb.fem_p1_assemble(cd, ed, plan, variant="class", K=Kc, M=Mc), a.reps)
        ne = e.shape[1]
        alg = 8 * c.size + 4 * e.size + 16 * plan.nnz
        print("%-14s ne=%9d nnz=%9d classes=%d groups=%d coverage=%.4f plan %.1f ms (first %.1f) | block %.4f ms | "
              "class %.4f ms (%.1f Gelem/s, ALG %.0f GB/s) | relmax K %.2e M %.2e"
              % (name, ne, plan.nnz, plan.class_stats[1], plan.class_stats[0], plan.class_coverage(), t_cls2, t_cls,
                 tb, tc, ne / tc * 1e-6, alg / tc * 1e-6, rk, rm), flush=True)


if __name__ == "__main__":
    main()
