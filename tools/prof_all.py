"""Runs every kernel family of libvb once (after a warm-up) on the BASELINE shapes,
for one ncu metric capture of all of them (tools/ncu_all.sh):
config 2 page ops (n = 2, 3, 4), config 3 surface, config 5 pattern + assembly
(gather / atomic, c = 1 and NEXT-1 coefficients), config 4 2D assembly, NEXT-2
load vector, NEXT-3 P2 (level 6, both variants), coords3D gather, bilinear."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dev = torch.device("cuda:0")
N = 1 << 20


def twice(fn):
    fn()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("measured")
    fn()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()


for n in (2, 3, 4):
    A = torch.from_numpy(synth.normal_pages(n, n, N, stream=10)).to(dev)
    B = torch.from_numpy(synth.normal_pages(n, n, N, stream=11)).to(dev)
    X = torch.from_numpy(synth.inverse_pages(n, N, seed=0)[0]).to(dev)
    twice(lambda: vb.vb_page_mtimes(A, B))
    twice(lambda: vb.vb_page_transpose(A))
    twice(lambda: vb.vb_page_det(A))
    twice(lambda: vb.vb_page_inv(X))
a3 = torch.from_numpy(synth.normal_pages(3, 1, N, stream=10)).to(dev)
b3 = torch.from_numpy(synth.normal_pages(3, 1, N, stream=11)).to(dev)
twice(lambda: vb.vb_page_cross(a3, b3))
xyz, tri = synth.icosphere(10, perturb=0.01, seed=0)
xd, td = torch.from_numpy(xyz).to(dev), torch.from_numpy(tri).to(dev)
twice(lambda: vb.vb_tri_surface(xd, td))
del xd, td

c5, e5 = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
cd, ed = torch.from_numpy(c5).to(dev), torch.from_numpy(e5).to(dev)
# fused simplex geometry (sizes alone, normals alone, both)
twice(lambda: vb.vb_simplex_geometry(cd, ed, want_normals=False))
twice(lambda: vb.vb_simplex_geometry(cd, ed, want_meass=False))
twice(lambda: vb.vb_simplex_geometry(cd, ed))
twice(lambda: vb.P1Plan(ed, c5.shape[1]))
plan = vb.P1Plan(ed, c5.shape[1])
K = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
M = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
plan.classes()
plan.tiles(cd, ed)
# round 2: the lattice plan (element check + closed-form pattern) and the headline kernel
twice(lambda: vb.P1Plan.for_lattice(ed, c5.shape[1]))
assert plan.lattice(ed)
for mode, variant in ((vb.VB_ASSEMBLE_GATHER, "lattice"), (vb.VB_ASSEMBLE_GATHER, "class"), (vb.VB_ASSEMBLE_GATHER, "block"),
                      (vb.VB_ASSEMBLE_GATHER, "tile"), (vb.VB_ASSEMBLE_ATOMIC, None)):
    twice(lambda: vb.fem_p1_assemble(cd, ed, plan, mode=mode, K=K, M=M, variant=variant))
    if variant not in ("tile", "lattice"):
        twice(lambda: vb.fem_p1_assemble_coef(cd, ed, plan, gqo=2, mode=mode, K=K, M=M, variant=variant))
twice(lambda: vb.fem_p1_assemble_exact(cd, ed, plan))


def tile_plan():
    plan.tile_ok = None
    plan.tiles(cd, ed)


twice(tile_plan)
twice(lambda: vb.vb_create_coords3D(cd, ed))
fq = torch.ones((4, e5.shape[1]), dtype=torch.float64, device=dev)
twice(lambda: vb.fem_p1_rhs(cd, ed, fq, plan=plan, gqo=2))
Kl = torch.from_numpy(synth.normal_pages(4, 4, e5.shape[1], stream=10)).to(dev)
u = torch.from_numpy(synth.normal_pages(4, 1, e5.shape[1], stream=11)).to(dev)
twice(lambda: vb.vb_page_bilinear(u, Kl, u))
# NEXT-4 GI: the volume integral of rho = x1^2 + x2^2 (4 points) on the config-5 mesh
lam, wq = vb.vb_quad_rule(3, 2)
c3, v3 = vb.vb_create_coords3D(cd, ed)
Xip = vb.vb_page_mtimes(c3, torch.from_numpy(lam.reshape(len(wq), 4, 1).copy()).to(dev))
gsz = vb.vb_page_det(v3).abs_() / 6.0
gfip = (Xip[:, 0] ** 2 + Xip[:, 1] ** 2).unsqueeze(1).contiguous()
del c3, v3, Xip
twice(lambda: vb.vb_gi(gfip, wq * 6.0, gsz))
del gfip, gsz
del plan, K, M, cd, ed, Kl, u, fq

c4, e4 = synth.square_p1(2048, jitter=0.1, seed=0)
cd4, ed4 = torch.from_numpy(c4).to(dev), torch.from_numpy(e4).to(dev)
p4 = vb.P1Plan(ed4, c4.shape[1])
assert p4.lattice(ed4)
for mode, variant in ((vb.VB_ASSEMBLE_GATHER, "lattice"), (vb.VB_ASSEMBLE_GATHER, "class"), (vb.VB_ASSEMBLE_GATHER, "block"),
                      (vb.VB_ASSEMBLE_GATHER, "tile"), (vb.VB_ASSEMBLE_ATOMIC, None)):
    twice(lambda: vb.fem_p1_assemble(cd4, ed4, p4, mode=mode, variant=variant))
del p4, cd4, ed4
# NEXT-1 2D: the crossed-diagonal square of tab:KM_P1_2D, level 11
cq, eq = synth.square_crossed_p1(2 ** 11)
cdq, edq = torch.from_numpy(cq).to(dev), torch.from_numpy(eq).to(dev)
pq = vb.P1Plan(edq, cq.shape[1], scatter_map=False)
for variant in ("class", "block"):
    twice(lambda: vb.fem_p1_assemble_coef(cdq, edq, pq, gqo=2, variant=variant))
del pq, cdq, edq

c2, e2 = synth.p2_from_p1(*synth.cube_kuhn_p1(64, jitter=0.0, flip=(0, 0, 1)))
cd2, ed2 = torch.from_numpy(c2).to(dev), torch.from_numpy(e2).to(dev)
p2 = vb.Plan(ed2, c2.shape[1])
for mode in (vb.VB_ASSEMBLE_GATHER, vb.VB_ASSEMBLE_ATOMIC):
    twice(lambda: vb.fem_p2_assemble(cd2, ed2, p2, mode=mode))
print("ok")
