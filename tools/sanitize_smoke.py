"""Every libvb entry point on small inputs (for compute-sanitizer runs, one tool per call)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dev = torch.device("cuda:0")


def g(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


for n in (2, 3, 4):
    A = g(synth.normal_pages(n, n, 1001, stream=1))
    B = g(synth.normal_pages(n, n, 1001, stream=2))
    vb.vb_page_mtimes(A, B, True, False)
    vb.vb_page_transpose(A)
    vb.vb_page_det(A)
    vb.vb_page_inv(A, first_singular=torch.zeros(1, dtype=torch.int64, device=dev))
    vb.vb_page_bilinear(g(synth.normal_pages(n, 1, 1001)), A, g(synth.normal_pages(n, 1, 1001, stream=3)))
vb.vb_page_cross(g(synth.normal_pages(3, 1, 777)), g(synth.normal_pages(3, 1, 777, stream=5)))
xyz, tri = synth.icosphere(3)
vb.vb_tri_surface(g(xyz), g(tri))
for dim, (c, e) in ((2, synth.square_p1(20)), (3, synth.cube_kuhn_p1(6)), (2, synth.square_crossed_p1(9))):
    cd, ed = g(c), g(e)
    plan = vb.P1Plan(ed, c.shape[1])
    for mode in (vb.VB_ASSEMBLE_GATHER, vb.VB_ASSEMBLE_ATOMIC):
        vb.fem_p1_assemble(cd, ed, plan, mode=mode, want_local=True)
        vb.fem_p1_assemble_coef(cd, ed, plan, mode=mode, gqo=2)
    for variant in ("class", "block", "tile"):
        vb.fem_p1_assemble(cd, ed, plan, variant=variant)
        vb.fem_p1_assemble_coef(cd, ed, plan, gqo=2, variant=variant)
    vb.fem_p1_assemble_exact(cd, ed, plan)
    lam, w = vb.vb_quad_rule(dim, 2)
    vb.fem_p1_rhs(cd, ed, torch.ones((len(w), e.shape[1]), dtype=torch.float64, device=dev), plan=plan)
    vb.vb_create_coords3D(cd, ed)
torch.cuda.synchronize()
print("sanitize smoke ok")

# round 2: lattice plans and kernels (3D: sizes with packed tiles and several bands; 2D: several segments)
for dims in ((33, 14, 5), (7, 7, 7)):
    c, e = synth.box_kuhn_p1(*dims, jitter=0.05, seed=1)
    plan = vb.P1Plan.for_lattice(g(e), c.shape[1], dims=dims)
    assert plan is not None
    vb.fem_p1_assemble(g(c), g(e), plan, degenerate=torch.zeros(1, dtype=torch.int64, device=dev))
    p2 = vb.P1Plan(g(e), c.shape[1], scatter_map=False, gather_plan=False)
    assert p2.lattice(g(e), dims=dims)
for dims in ((70, 45), (5, 3)):
    c, e = synth.rect_p1(*dims, jitter=0.1, seed=1, flip=1)
    plan = vb.P1Plan(g(e), c.shape[1], scatter_map=False, gather_plan=False)
    assert plan.lattice(g(e), dims=dims), plan.lattice_reason
    vb.fem_p1_assemble_lattice(g(c), plan, degenerate=torch.zeros(1, dtype=torch.int64, device=dev))
torch.cuda.synchronize()
print("lattice ok")
