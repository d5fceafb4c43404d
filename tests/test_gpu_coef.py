"""GPU parity of the coefficient-weighted P1 assembly (NEXT-1,
fem_p1_assemble_coef) against the oracle, both variants, and reproduction on
the GPU of the paper's printed error columns (Tables tab:KM_P1_2D and
tab:KM_P1_3D) -- including the 3D level-7 row, which is the size of
configs[4] (129^3 nodes, 12.58M tets)."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2404_16039_b200 import vb

pytestmark = pytest.mark.gpu
# (mode, gather variant): the row-class kernel (3D, gqo = 2, c_K = c_M; other cases
# fall back to the blocks), the 32-row blocks, the atomic scatter
MODES = [(vb.VB_ASSEMBLE_GATHER, "class"), (vb.VB_ASSEMBLE_GATHER, "block"), (vb.VB_ASSEMBLE_ATOMIC, None)]
MODE_IDS = ["class", "block", "atomic"]
# 0: the paper's e^{x+y+z}; 1: c_K != c_M (exponentials at the points); 2: c_K == c_M
# non-trivial (per-vertex factor path of the gather kernel for gqo = 2)
COEFS = [((1.0, (1.0, 1.0, 1.0)), (1.0, (1.0, 1.0, 1.0))),
         ((2.5, (0.3, -0.7, 0.45)), (0.6, (-1.0, 0.2, 0.9))),
         ((1.7, (0.9, -1.3, 0.4)), (1.7, (0.9, -1.3, 0.4)))]


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    return torch.device("cuda:0")


def g(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def h(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def relmax(got, ref):
    return np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300)


@pytest.mark.parametrize("mode", MODES, ids=MODE_IDS)
@pytest.mark.parametrize("gqo", [1, 2])
@pytest.mark.parametrize("coef", [0, 1, 2])
@pytest.mark.parametrize("kind", ["2d", "3d", "2d-crossed"])
def test_coef_assembly_parity(dev, kind, coef, gqo, mode):
    if kind == "2d":
        coords, elems = synth.square_p1(24, jitter=0.1, seed=3)
    elif kind == "2d-crossed":
        coords, elems = synth.square_crossed_p1(16)
    else:
        coords, elems = synth.cube_kuhn_p1(7, jitter=0.05, seed=3)
    cK, cM = COEFS[coef]
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    Ko, Mo = oracle.p1_assemble_coef(coords, elems, rp, ci, gqo=gqo, cK=cK, cM=cM)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, nn)
    K, M, Kl, Ml = vb.fem_p1_assemble_coef(cd, ed, plan, gqo=gqo, cK=cK, cM=cM, mode=mode[0], variant=mode[1],
                                           want_local=True)
    assert relmax(h(K), Ko) <= 1e-12
    assert relmax(h(M), Mo) <= 1e-12
    # local matrices vs the oracle element routine on a few elements
    Kl, Ml = h(Kl), h(Ml)
    for e in (0, 7, elems.shape[1] - 1):
        Ke, Me = oracle.p1_local_coef(coords[:, elems[:, e]], gqo=gqo, cK=cK, cM=cM)
        assert relmax(Kl[:, :, e].T, Ke) <= 1e-12 and relmax(Ml[:, :, e].T, Me) <= 1e-12


def test_coef_one_equals_plain_assembly(dev):
    coords, elems = synth.cube_kuhn_p1(9, jitter=0.05, seed=1)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, coords.shape[1])
    K1, M1, _, _ = vb.fem_p1_assemble(cd, ed, plan)
    K, M, _, _ = vb.fem_p1_assemble_coef(cd, ed, plan, gqo=2, cK=(1.0, (0, 0, 0)), cM=(1.0, (0, 0, 0)))
    assert relmax(h(K), h(K1)) <= 1e-13 and relmax(h(M), h(M1)) <= 1e-13


def quad_form(rp, ci, vals, u):
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    return math.fsum(u[rows] * vals * u[ci])


def printed_close(x, printed):
    e = math.floor(math.log10(abs(printed)))
    return abs(x - printed) <= 0.5 * 10 ** (e - 2) * 1.0001


@pytest.mark.parametrize("dim,level", [(2, 7), (2, 9), (2, 11), (3, 5), (3, 7)])
def test_paper_tables_on_gpu(dev, golden, dim, level):
    """e_K, e_M of the paper's P1 tables from GPU-assembled K, M (gather
    variant, the configuration bench.py times)."""
    gd = golden("paper_tables_p1.json")
    if dim == 2:
        coords, elems = synth.square_crossed_p1(2 ** level)
        row = [r for r in gd["p1_2d"] if r["level"] == level][0]
        v = np.sin(np.pi * coords[0]) * np.sin(np.pi * coords[1])
        IK, IM = gd["I_K_2d"], gd["I_M_2d"]
    else:
        coords, elems = synth.cube_kuhn_p1(2 ** level, jitter=0.0, flip=(0, 0, 1))
        row = [r for r in gd["p1_3d"] if r["level"] == level][0]
        v = np.cos(np.pi * coords[0]) * np.cos(np.pi * coords[1]) * np.cos(np.pi * coords[2])
        IK, IM = gd["I_K_3d"], gd["I_M_3d"]
    assert coords.shape[1] == row["size"]
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, coords.shape[1], scatter_map=False)
    K, M, _, _ = vb.fem_p1_assemble_coef(cd, ed, plan, gqo=2)
    rp, ci = h(plan.row_ptr), h(plan.col_idx)
    assert printed_close(abs(quad_form(rp, ci, h(K), v) - IK), row["e_K"])
    assert printed_close(abs(quad_form(rp, ci, h(M), v) - IM), row["e_M"])
    if dim == 3:
        # the default (row classes for these meshes) against the 32-row blocks on every entry
        assert plan.class_coverage() >= 0.9
        K2, M2, _, _ = vb.fem_p1_assemble_coef(cd, ed, plan, gqo=2, variant="block")
        assert relmax(h(K), h(K2)) <= 1e-12 and relmax(h(M), h(M2)) <= 1e-12
