"""GPU parity of the 2D element-once lattice assembly (fem_plan_lattice2d +
fem_p1_assemble_lattice2d) against the CPU oracle through the C ABI: K and M
within 1e-12 relative max-norm on rectangles whose sizes straddle the kernel's
x segments (31 nodes) and short warp ranges, both cell diagonals, shuffled
element and vertex order, K-only / M-only outputs, bitwise reproducibility,
refusal of other meshes, the unjittered 5-point stencil, and every entry of the
full configs[3] matrices against the full oracle assembly."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2404_16039_b200 import vb

pytestmark = pytest.mark.gpu
TOL = 1e-12


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


def run(coords, elems, dev, dims, **kw):
    plan = vb.P1Plan(g(elems, dev), coords.shape[1], scatter_map=False, gather_plan=False)
    assert plan.lattice(g(elems, dev), dims=dims), plan.lattice_reason
    K, M = vb.fem_p1_assemble_lattice(g(coords, dev), plan, **kw)
    return plan, K, M


@pytest.mark.parametrize("dims", [(2, 1), (2, 2), (3, 5), (29, 3), (30, 2), (31, 4), (32, 3), (61, 2), (62, 7), (63, 5),
                                  (5, 40), (33, 100), (100, 33), (7, 700), (200, 150)])
@pytest.mark.parametrize("flip", [0, 1])
def test_lattice2d_vs_oracle(dev, dims, flip):
    coords, elems = synth.rect_p1(*dims, jitter=0.1, seed=2, flip=flip)
    rp, ci = oracle.p1_pattern(elems, coords.shape[1])
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    plan, K, M = run(coords, elems, dev, dims)
    assert np.array_equal(h(plan.row_ptr), rp) and np.array_equal(h(plan.col_idx), ci)
    assert relmax(h(K), Ko) <= TOL
    assert relmax(h(M), Mo) <= TOL


def test_lattice2d_shuffled_elements_and_vertices(dev):
    coords, elems = synth.rect_p1(40, 23, jitter=0.1, seed=4)
    rng = np.random.default_rng(0)
    elems = elems[:, rng.permutation(elems.shape[1])]
    for e in range(elems.shape[1]):
        elems[:, e] = elems[rng.permutation(3), e]
    elems = np.ascontiguousarray(elems)
    rp, ci = oracle.p1_pattern(elems, coords.shape[1])
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    _, K, M = run(coords, elems, dev, (40, 23))
    assert relmax(h(K), Ko) <= TOL and relmax(h(M), Mo) <= TOL


def test_lattice2d_unjittered_five_point_stencil(dev):
    """Unjittered right triangles: interior rows of K are (4, -1, -1, -1, -1) with exact zeros on the diagonal
    neighbours (the oracle's pin), M row sums h^2."""
    n = 48
    coords, elems = synth.rect_p1(n, n, jitter=0.0)
    plan, K, M = run(coords, elems, dev, (n, n))
    rp, ci, K = h(plan.row_ptr), h(plan.col_idx), h(K)
    v = 10 + (n + 1) * 17
    row = dict(zip(ci[rp[v]:rp[v + 1]], K[rp[v]:rp[v + 1]]))
    assert abs(row[v] - 4.0) <= 1e-13
    for w in (v - 1, v + 1, v - (n + 1), v + (n + 1)):
        assert abs(row[w] + 1.0) <= 1e-13
    for w in (v + n + 2, v - n - 2):
        assert abs(row[w]) <= 1e-13
    assert abs(h(M).sum() - 1.0) <= 1e-12


def test_lattice2d_k_only_m_only_and_reproducible(dev):
    coords, elems = synth.rect_p1(70, 45, jitter=0.1, seed=1)
    plan, K, M = run(coords, elems, dev, (70, 45))
    cd = g(coords, dev)
    K2, none = vb.fem_p1_assemble_lattice(cd, plan, want_M=False)
    none2, M2 = vb.fem_p1_assemble_lattice(cd, plan, want_K=False)
    assert none is None and none2 is None
    assert torch.equal(K, K2) and torch.equal(M, M2)
    for _ in range(3):
        K3, M3 = vb.fem_p1_assemble_lattice(cd, plan)
        assert torch.equal(K, K3) and torch.equal(M, M3)
    # unaligned outputs take the plain-store path: same bits
    buf = torch.empty(2 * plan.nnz + 3, dtype=torch.float64, device=dev)
    Ku, Mu = buf[1:1 + plan.nnz], buf[plan.nnz + 2:2 * plan.nnz + 2]
    vb.fem_p1_assemble_lattice(cd, plan, K=Ku, M=Mu)
    assert torch.equal(K, Ku) and torch.equal(M, Mu)


def test_lattice2d_refuses_other_meshes_and_falls_back(dev):
    coords, elems = synth.rect_p1(12, 9, jitter=0.1, seed=0)
    bad = elems.copy()
    bad[:, 5] = bad[:, 6]
    plan = vb.P1Plan(g(bad, dev), coords.shape[1])
    assert not plan.lattice(g(bad, dev), dims=(12, 9)) and "triangle" in plan.lattice_reason
    c2, e2 = synth.square_crossed_p1(8)          # 4 triangles per cell: not this lattice
    p2 = vb.P1Plan(g(e2, dev), c2.shape[1])
    assert not p2.lattice(g(e2, dev))
    rp, ci = oracle.p1_pattern(e2, c2.shape[1])
    Ko, Mo = oracle.p1_assemble(c2, e2, rp, ci)
    K, M, _, _ = vb.fem_p1_assemble(g(c2, dev), g(e2, dev), p2)   # falls back to the class / block variants
    assert relmax(h(K), Ko) <= TOL and relmax(h(M), Mo) <= TOL


def test_full_size_configs3_every_entry_vs_oracle(dev):
    coords, elems = synth.square_p1(2048, jitter=0.1, seed=0)
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    plan = vb.P1Plan(g(elems, dev), nn, scatter_map=False, gather_plan=False)
    assert plan.lattice(g(elems, dev))
    K, M, _, _ = vb.fem_p1_assemble(g(coords, dev), g(elems, dev), plan)   # variant None -> 2D lattice
    assert relmax(h(K), Ko) <= TOL and relmax(h(M), Mo) <= TOL


@pytest.mark.parametrize("layout", ["aos", "aos4"])
def test_lattice2d_strided_coords_through_the_abi(dev, layout):
    """coords strided as in vb_create_coords3D (node-major xy pairs, padded xy__ records) through the C ABI,
    with the degenerate counter requested (its pass reads the same strides)."""
    coords, elems = synth.rect_p1(45, 31, jitter=0.1, seed=6, flip=1)
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    plan = vb.P1Plan(g(elems, dev), nn, scatter_map=False, gather_plan=False)
    assert plan.lattice(g(elems, dev), dims=(45, 31))
    if layout == "aos":
        cbuf, ns = g(np.ascontiguousarray(coords.T), dev), 2
    else:
        pad = np.zeros((nn, 4))
        pad[:, :2] = coords.T
        cbuf, ns = g(pad, dev), 4
    K = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
    M = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
    cnt = torch.full((1,), -1, dtype=torch.int64, device=dev)
    vb._check(vb.lib().fem_p1_assemble_lattice2d(nn, vb._ptr(cbuf), ns, 1, vb._ptr(plan.row_ptr), plan.nnz,
                                                 vb._ptr(plan.lattice_plan), 45, 31, plan.lattice_flips, vb._ptr(K),
                                                 vb._ptr(M), vb._ptr(cnt), None))
    assert relmax(h(K), Ko) <= TOL and relmax(h(M), Mo) <= TOL
    assert int(h(cnt)[0]) == 0


@pytest.mark.parametrize("dims,flip", [((2, 1), 0), ((31, 4), 1), ((62, 7), 0), ((33, 100), 1), ((200, 150), 0)])
def test_lattice2d_pattern_closed_form_bit_exact(dev, dims, flip):
    """fem_lattice2d_pattern (P1Plan.for_lattice in 2D) against the oracle's pattern built from shuffled elements;
    K, M assembled on that plan against the oracle."""
    coords, elems = synth.rect_p1(*dims, jitter=0.1, seed=3, flip=flip)
    rng = np.random.default_rng(2)
    elems = np.ascontiguousarray(elems[:, rng.permutation(elems.shape[1])])
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    plan = vb.P1Plan.for_lattice(g(elems, dev), nn, dims=dims)
    assert plan is not None and plan.nnz == int(rp[-1])
    assert np.array_equal(h(plan.row_ptr), rp) and np.array_equal(h(plan.col_idx), ci)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    K, M, _, _ = vb.fem_p1_assemble(g(coords, dev), g(elems, dev), plan)
    assert relmax(h(K), Ko) <= TOL and relmax(h(M), Mo) <= TOL
    bad = elems.copy()
    bad[:, 0] = bad[:, 1]
    assert vb.P1Plan.for_lattice(g(bad, dev), nn, dims=dims) is None
