"""GPU parity of NEXT-2: the load vector (fem_p1_rhs, both variants), the page
bilinear form (vb_page_bilinear = avtamav) and the element energies
J_{1,k} = 1/2 u_k^T K_k u_k composed from vb_create_coords3D (dim = 1 gather of
a nodal vector), fem_p1_assemble's K3D and vb_page_bilinear (eq:Jk_comps)."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2404_16039_b200 import vb

pytestmark = pytest.mark.gpu


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


def test_quad_rule_matches_oracle():
    for dim in (2, 3):
        for gqo in (1, 2):
            lam, w = vb.vb_quad_rule(dim, gqo)
            lo, wo = oracle.quad_rule(dim, gqo)
            assert np.max(np.abs(lam - lo)) <= 2.3e-16 and np.max(np.abs(w - wo)) <= 1e-17   # 1 ulp


@pytest.mark.parametrize("mode", [vb.VB_ASSEMBLE_GATHER, vb.VB_ASSEMBLE_ATOMIC])
@pytest.mark.parametrize("dim,gqo", [(2, 1), (2, 2), (3, 1), (3, 2)])
def test_rhs_parity(dev, dim, gqo, mode):
    coords, elems = synth.square_p1(40, jitter=0.1, seed=5) if dim == 2 else synth.cube_kuhn_p1(9, jitter=0.05, seed=5)
    lam, w = oracle.quad_rule(dim, gqo)
    xq = np.einsum("qa,cae->qce", lam, coords[:, elems])
    fq = np.ascontiguousarray(np.exp(xq.sum(1)) * np.cos(3 * xq[:, 0]))
    bo, b2o = oracle.p1_rhs(coords, elems, fq, gqo=gqo)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, coords.shape[1], scatter_map=False)
    b, b2 = vb.fem_p1_rhs(cd, ed, g(fq, dev), plan=plan, gqo=gqo, mode=mode)
    assert relmax(h(b), bo) <= 1e-12
    assert relmax(h(b2), b2o) <= 1e-12


@pytest.mark.parametrize("mode", [vb.VB_ASSEMBLE_GATHER, vb.VB_ASSEMBLE_ATOMIC])
@pytest.mark.parametrize("dim", [2, 3])
def test_rhs_odd_element_count_scalar_path(dev, dim, mode):
    """An odd element count takes the one-element-per-thread kernel (the paired kernel needs even planes):
    same parity bar, and b2D equals the paired kernel's on the shared elements bit for bit."""
    coords, elems = synth.delaunay_p1(dim, 14 if dim == 2 else 8, seed=3)
    if elems.shape[1] % 2 == 0:
        elems = np.ascontiguousarray(elems[:, :-1])
    ne = elems.shape[1]
    assert ne % 2 == 1
    lam, w = oracle.quad_rule(dim, 2)
    xq = np.einsum("qa,cae->qce", lam, coords[:, elems])
    fq = np.ascontiguousarray(np.exp(xq.sum(1)) * np.cos(3 * xq[:, 0]))
    bo, b2o = oracle.p1_rhs(coords, elems, fq, gqo=2)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, coords.shape[1], scatter_map=False)
    b, b2 = vb.fem_p1_rhs(cd, ed, g(fq, dev), plan=plan, gqo=2, mode=mode)
    assert relmax(h(b), bo) <= 1e-12 and relmax(h(b2), b2o) <= 1e-12
    ev = np.ascontiguousarray(elems[:, :ne - 1])                       # even count: the paired kernel
    fv = np.ascontiguousarray(fq[:, :ne - 1])
    pe = vb.P1Plan(g(ev, dev), coords.shape[1], scatter_map=False)
    _, b2e = vb.fem_p1_rhs(cd, g(ev, dev), g(fv, dev), plan=pe, gqo=2, mode=mode)
    assert np.array_equal(h(b2e), h(b2)[:, :ne - 1])


def test_rhs_gather_is_bitwise_reproducible(dev):
    coords, elems = synth.cube_kuhn_p1(12, jitter=0.05, seed=6)
    lam, w = oracle.quad_rule(3, 2)
    fq = np.ascontiguousarray(np.einsum("qa,cae->qce", lam, coords[:, elems]).sum(1))
    cd, ed, fd = g(coords, dev), g(elems, dev), g(fq, dev)
    plan = vb.P1Plan(ed, coords.shape[1], scatter_map=False)
    b1, _ = vb.fem_p1_rhs(cd, ed, fd, plan=plan)
    b2, _ = vb.fem_p1_rhs(cd, ed, fd, plan=plan)
    assert np.array_equal(h(b1), h(b2))


@pytest.mark.parametrize("n,m", [(1, 1), (2, 3), (3, 3), (4, 4), (4, 2)])
def test_bilinear_parity(dev, n, m):
    N = 4099
    A = synth.normal_pages(n, 1, N, stream=80)
    Mx = synth.normal_pages(n, m, N, stream=81)
    B = synth.normal_pages(m, 1, N, stream=82)
    s = h(vb.vb_page_bilinear(g(A, dev), g(Mx, dev), g(B, dev)))
    assert relmax(s, oracle.page_bilinear(A, Mx, B)) <= 1e-12
    Ai = synth.integer_pages(n, 1, N, seed=83)
    Mi = synth.integer_pages(n, m, N, seed=84)
    Bi = synth.integer_pages(m, 1, N, seed=85)
    assert np.array_equal(h(vb.vb_page_bilinear(g(Ai, dev), g(Mi, dev), g(Bi, dev))), oracle.page_bilinear(Ai, Mi, Bi))
    Ms = synth.normal_pages(n, m, 1, stream=86)                       # broadcast single matrix (ld = 0)
    assert relmax(h(vb.vb_page_bilinear(g(A, dev), g(Ms, dev), g(B, dev))), oracle.page_bilinear(A, Ms, B)) <= 1e-12


def test_element_energies_compose(dev):
    """J_{1,k} = 1/2 u_k^T K_k u_k (eq:Jk_comps) on the GPU; sum_k J_{1,k} = 1/2 u^T K u."""
    coords, elems = synth.cube_kuhn_p1(10, jitter=0.05, seed=7)
    u = np.cos(np.pi * coords[0]) * np.sin(np.pi * coords[1]) + coords[2]
    cd, ed, ud = g(coords, dev), g(elems, dev), g(u[None, :], dev)
    plan = vb.P1Plan(ed, coords.shape[1])
    K, M, K3, M3 = vb.fem_p1_assemble(cd, ed, plan, want_local=True)
    uk, _ = vb.vb_create_coords3D(ud, ed, want_vectors3D=False)           # (nv, 1, ne): u restricted to elements
    uk = uk.reshape(1, 4, -1).contiguous()
    J1k = 0.5 * h(vb.vb_page_bilinear(uk, K3, uk))
    J2k = 0.5 * h(vb.vb_page_bilinear(uk, M3, uk))
    K3o, M3o = oracle.p1_local_all(coords, elems)
    uko = np.ascontiguousarray(u[elems][None])
    assert relmax(J1k, 0.5 * oracle.page_bilinear(uko, K3o, uko)) <= 1e-12
    assert relmax(J2k, 0.5 * oracle.page_bilinear(uko, M3o, uko)) <= 1e-12
    rp, ci = h(plan.row_ptr), h(plan.col_idx)
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    uKu = math.fsum(u[rows] * h(K) * u[ci])
    assert abs(math.fsum(J1k) - 0.5 * uKu) <= 1e-12 * abs(uKu)
