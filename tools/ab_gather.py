"""A/B timing of the gather assembly on structured and unstructured meshes.

usage: VB_LIBVB=tools/variants/<name>.so python tools/ab_gather.py [--reps 30]
Meshes are cached under /tmp/vb_ab (scratch, same gpurun call only)."""
import argparse
import os
import sys

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
    "delaunay2d_1024": lambda: synth.delaunay_p1(2, 1024, seed=0),
}


def load(name):
    path = "/tmp/vb_ab/%s.npz" % name
    if os.path.exists(path):
        z = np.load(path)
        return z["c"], z["e"]
    c, e = MESHES[name]()
    os.makedirs("/tmp/vb_ab", exist_ok=True)
    np.savez(path, c=c, e=e)
    return c, e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--meshes", default=",".join(MESHES))
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    tag = os.path.basename(os.environ.get("VB_LIBVB", "default"))
    for name in a.meshes.split(","):
        c, e = load(name)
        cd = torch.from_numpy(c).to(dev)
        ed = torch.from_numpy(e).to(dev)
        plan = vb.P1Plan(ed, c.shape[1])
        out = {}
        for mode, mname in ((vb.VB_ASSEMBLE_GATHER, "gather"), (vb.VB_ASSEMBLE_ATOMIC, "atomic")):
            K, M, _, _ = vb.fem_p1_assemble(cd, ed, plan, mode=mode)
            for _ in range(3):
                vb.fem_p1_assemble(cd, ed, plan, mode=mode, K=K, M=M)
            s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            for _ in range(a.reps):
                vb.fem_p1_assemble(cd, ed, plan, mode=mode, K=K, M=M)
            t.record()
            torch.cuda.synchronize()
            out[mname] = s.elapsed_time(t) / a.reps
        L = np.diff(plan.row_ptr.cpu().numpy())
        print("%-14s %-16s ne=%9d nnz=%9d rowmean=%.2f gather %.4f ms atomic %.4f ms (%.2f Gelem/s)"
              % (tag, name, e.shape[1], plan.nnz, L.mean(), out["gather"], out["atomic"],
                 e.shape[1] / out["gather"] * 1e-6), flush=True)


if __name__ == "__main__":
    main()
