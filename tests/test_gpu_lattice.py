"""GPU parity of the element-once Kuhn-lattice assembly (fem_plan_lattice +
fem_p1_assemble_lattice, the headline kernel) against the CPU oracle through
the C ABI: K and M within 1e-12 relative max-norm (BASELINE.json north_star)
on boxes whose sizes straddle the kernel's tile edges (x segments of 32/31
nodes, y bands of 12/11 lines, packed short segments, one-layer z ranges),
every cell diagonal, shuffled element and vertex order, K-only / M-only
outputs, bitwise reproducibility, refusal of non-lattice meshes (and the
fallback of fem_p1_assemble), and every entry of the full configs[4] matrices
against the full oracle assembly."""
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


def lattice_run(coords, elems, dev, dims=None, **kw):
    nn = coords.shape[1]
    plan = vb.P1Plan(g(elems, dev), nn, scatter_map=False, gather_plan=False)
    assert plan.lattice(g(elems, dev), dims=dims), plan.lattice_reason
    K, M = vb.fem_p1_assemble_lattice(g(coords, dev), plan, **kw)
    return plan, K, M


@pytest.mark.parametrize("dims", [(2, 2, 1), (2, 2, 2), (3, 4, 5), (7, 7, 7), (29, 2, 3), (30, 3, 2), (31, 2, 2),
                                  (32, 2, 3), (61, 2, 2), (62, 3, 1), (63, 2, 1), (2, 11, 3), (3, 12, 2), (2, 23, 2),
                                  (4, 24, 3), (5, 40, 2), (12, 13, 14), (70, 25, 3), (124, 3, 2),
                                  (2, 2, 300), (95, 23, 9), (31, 12, 40), (64, 56, 20)])
def test_lattice_vs_oracle(dev, dims):
    coords, elems = synth.box_kuhn_p1(*dims, jitter=0.05, seed=3)
    rp, ci = oracle.p1_pattern(elems, coords.shape[1])
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    plan, K, M = lattice_run(coords, elems, dev, dims=dims)
    assert np.array_equal(h(plan.row_ptr), rp) and np.array_equal(h(plan.col_idx), ci)
    assert relmax(h(K), Ko) <= TOL
    assert relmax(h(M), Mo) <= TOL


@pytest.mark.parametrize("flip", [(0, 0, 1), (0, 1, 0), (1, 0, 0), (1, 1, 0), (0, 1, 1), (1, 1, 1)])
def test_lattice_every_diagonal(dev, flip):
    coords, elems = synth.box_kuhn_p1(9, 14, 5, jitter=0.05, seed=1, flip=flip)
    rp, ci = oracle.p1_pattern(elems, coords.shape[1])
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    plan, K, M = lattice_run(coords, elems, dev, dims=(9, 14, 5))
    assert relmax(h(K), Ko) <= TOL and relmax(h(M), Mo) <= TOL


def test_lattice_shuffled_elements_and_vertices(dev):
    coords, elems = synth.cube_kuhn_p1(8, jitter=0.05, seed=2)
    rng = np.random.default_rng(7)
    order = rng.permutation(elems.shape[1])
    e2 = elems[:, order]
    for e in range(e2.shape[1]):
        e2[:, e] = e2[rng.permutation(4), e]
    rp, ci = oracle.p1_pattern(e2, coords.shape[1])
    Ko, Mo = oracle.p1_assemble(coords, e2, rp, ci)
    plan, K, M = lattice_run(coords, e2, dev)
    assert relmax(h(K), Ko) <= TOL and relmax(h(M), Mo) <= TOL


def test_lattice_unjittered_kuhn_row(dev):
    # SURVEY §8(c) pin 6 on the GPU: interior row = 6h diagonal, -h at the 6 axis neighbours, 0 elsewhere
    n = 6
    coords, elems = synth.cube_kuhn_p1(n, jitter=0.0)
    plan, K, M = lattice_run(coords, elems, dev)
    rp, ci, Kh, Mh = h(plan.row_ptr), h(plan.col_idx), h(K), h(M)
    hh = 1.0 / n
    v = 3 + (n + 1) * (3 + (n + 1) * 3)
    row = dict(zip(ci[rp[v]:rp[v + 1]], Kh[rp[v]:rp[v + 1]]))
    assert abs(row[v] - 6 * hh) < 1e-14
    for d in (1, n + 1, (n + 1) ** 2):
        assert abs(row[v + d] + hh) < 1e-14 and abs(row[v - d] + hh) < 1e-14
    others = [x for c, x in row.items() if c not in (v, v + 1, v - 1, v + n + 1, v - n - 1, v + (n + 1) ** 2,
                                                      v - (n + 1) ** 2)]
    assert len(others) == 8 and max(abs(x) for x in others) < 1e-15
    assert abs(Mh[rp[v]:rp[v + 1]].sum() - hh ** 3) < 1e-15


def test_lattice_k_only_m_only_and_reproducible(dev):
    coords, elems = synth.box_kuhn_p1(34, 13, 4, jitter=0.05, seed=4)
    plan, K, M = lattice_run(coords, elems, dev, dims=(34, 13, 4))
    Kh, Mh = h(K), h(M)
    _, K2, M2 = lattice_run(coords, elems, dev, dims=(34, 13, 4))
    assert np.array_equal(h(K2), Kh) and np.array_equal(h(M2), Mh)   # bitwise run to run
    cd = g(coords, dev)
    Ko, Mn = vb.fem_p1_assemble_lattice(cd, plan, want_M=False)
    assert Mn is None and np.array_equal(h(Ko), Kh)
    Kn, Mo = vb.fem_p1_assemble_lattice(cd, plan, want_K=False)
    assert Kn is None and np.array_equal(h(Mo), Mh)
    # K, M that are not 16-byte aligned take the plain-store path of every tile: the same bits
    buf = torch.empty(2 * plan.nnz + 3, dtype=torch.float64, device=dev)
    Ku, Mu = buf[1:1 + plan.nnz], buf[plan.nnz + 2:2 * plan.nnz + 2]
    assert Ku.data_ptr() % 16 == 8
    vb.fem_p1_assemble_lattice(cd, plan, K=Ku, M=Mu)
    assert np.array_equal(h(Ku), Kh) and np.array_equal(h(Mu), Mh)


def test_lattice_refuses_other_meshes_and_fem_p1_assemble_falls_back(dev):
    coords, elems = synth.cube_kuhn_p1(5, jitter=0.05, seed=0)
    nn = coords.shape[1]
    # (a) one element replaced by a non-Kuhn tetrahedron of the same nodes (the pattern changes too)
    bad = elems.copy()
    bad[3, 7] = bad[3, 7] + 1
    plan = vb.P1Plan(g(bad, dev), nn)
    assert not plan.lattice(g(bad, dev)) and plan.lattice_reason
    rp, ci = oracle.p1_pattern(bad, nn)
    Ko, Mo = oracle.p1_assemble(coords, bad, rp, ci)
    K, M, _, _ = vb.fem_p1_assemble(g(coords, dev), g(bad, dev), plan)   # variant None: falls back
    assert relmax(h(K), Ko) <= TOL and relmax(h(M), Mo) <= TOL
    # (b) one Kuhn tetrahedron listed twice (another dropped)
    dup = elems.copy()
    dup[:, 11] = dup[:, 10]
    plan = vb.P1Plan(g(dup, dev), nn)
    assert not plan.lattice(g(dup, dev))
    # (c) renumbered nodes: same mesh, not lattice numbering
    c2, e2 = synth.permute_mesh(coords, elems, seed=1)
    plan = vb.P1Plan(g(e2, dev), nn)
    assert not plan.lattice(g(e2, dev))
    # (d) wrong dims
    plan = vb.P1Plan(g(elems, dev), nn)
    assert not plan.lattice(g(elems, dev), dims=(4, 5, 6))
    # (e) lattices thinner than the kernel's column order allows (nx or ny = 1): refused, fallback exact
    for dims in ((1, 1, 1), (1, 4, 3), (5, 1, 2)):
        c1, e1 = synth.box_kuhn_p1(*dims, jitter=0.05, seed=5)
        plan = vb.P1Plan(g(e1, dev), c1.shape[1])
        assert not plan.lattice(g(e1, dev), dims=dims)
        rp1, ci1 = oracle.p1_pattern(e1, c1.shape[1])
        Ko1, Mo1 = oracle.p1_assemble(c1, e1, rp1, ci1)
        K1, M1, _, _ = vb.fem_p1_assemble(g(c1, dev), g(e1, dev), plan)
        assert relmax(h(K1), Ko1) <= TOL and relmax(h(M1), Mo1) <= TOL


def test_lattice_plan_abi_errors(dev):
    L = vb.lib()
    import ctypes as C
    wb, pi = C.c_size_t(0), C.c_int64(0)
    stats = (C.c_int64 * 4)()
    assert L.fem_plan_lattice(8, 6, None, 6, None, None, 0, 0, 1, 1, None, C.byref(wb), None, C.byref(pi), stats,
                              None) == -1
    assert L.fem_p1_assemble_lattice(9, None, 1, 9, None, 0, None, 1, 1, 1, 0, None, None, None, None) == -1


@pytest.mark.parametrize("dims,flip", [((2, 2, 1), (0, 0, 0)), ((3, 4, 5), (0, 1, 0)), ((31, 2, 2), (1, 0, 0)),
                                       ((12, 13, 14), (0, 0, 1)), ((33, 25, 3), (1, 1, 0)), ((7, 7, 7), (1, 1, 1))])
def test_lattice_pattern_closed_form_bit_exact(dev, dims, flip):
    """fem_lattice_pattern (the stencil written directly) against the oracle's pattern built from the elements,
    for every orientation, shuffled elements; then K, M assembled on that plan against the oracle."""
    coords, elems = synth.box_kuhn_p1(*dims, jitter=0.05, seed=5, flip=flip)
    rng = np.random.default_rng(1)
    elems = np.ascontiguousarray(elems[:, rng.permutation(elems.shape[1])])
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    plan = vb.P1Plan.for_lattice(g(elems, dev), nn, dims=dims)
    assert plan is not None
    assert plan.nnz == int(rp[-1])
    assert np.array_equal(h(plan.row_ptr), rp) and np.array_equal(h(plan.col_idx), ci)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    K, M, _, _ = vb.fem_p1_assemble(g(coords, dev), g(elems, dev), plan)
    assert relmax(h(K), Ko) <= TOL and relmax(h(M), Mo) <= TOL


def test_lattice_pattern_refuses_non_lattices(dev):
    coords, elems = synth.cube_kuhn_p1(6, jitter=0.05, seed=0)
    bad = elems.copy()
    bad[:, 7] = bad[:, 8]                      # one element twice, one missing
    assert vb.P1Plan.for_lattice(g(bad, dev), coords.shape[1]) is None
    cd, ed = synth.delaunay_p1(3, 6, seed=1)
    assert vb.P1Plan.for_lattice(g(ed, dev), cd.shape[1]) is None


def test_full_size_configs4_every_entry_vs_oracle(dev):
    # BASELINE configs[4] in bench.py's launch configuration: all 31.8 M entries of K and M vs the full oracle
    coords, elems = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    plan = vb.P1Plan(g(elems, dev), nn, scatter_map=False, gather_plan=False)
    assert np.array_equal(h(plan.row_ptr), rp) and np.array_equal(h(plan.col_idx), ci)
    assert plan.lattice(g(elems, dev))
    K, M, _, _ = vb.fem_p1_assemble(g(coords, dev), g(elems, dev), plan)   # variant None -> lattice
    assert relmax(h(K), Ko) <= TOL
    assert relmax(h(M), Mo) <= TOL
    # bench.py's plan: the closed-form pattern, bit-identical, and the same K, M bits on it
    fast = vb.P1Plan.for_lattice(g(elems, dev), nn)
    assert fast is not None and np.array_equal(h(fast.row_ptr), rp) and np.array_equal(h(fast.col_idx), ci)
    K2, M2, _, _ = vb.fem_p1_assemble(g(coords, dev), g(elems, dev), fast)
    assert torch.equal(K2, K) and torch.equal(M2, M)


def _collapse(coords, elems, a, b):
    """Move node a onto node b: exactly the elements holding both have det = 0 (a zero edge vector)."""
    c = coords.copy()
    c[:, a] = c[:, b]
    return c, int(np.sum(np.any(elems == a, axis=0) & np.any(elems == b, axis=0)))


def test_degenerate_element_counter(dev):
    """The optional counter of elements outside the domain of the inverse (det tjac = 0) of
    fem_p1_assemble (block and atomic calls), of the 3D lattice kernel and of the 2D lattice kernel: zero on the
    jittered meshes, and the number of elements that hold both ends of a collapsed edge otherwise -- whichever
    edge of the element collapses (with contracted cofactors some of them leave a rounding residual instead of
    an exact 0: the rule counts identical vertices too), the same number from every kernel."""
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    coords, elems = synth.box_kuhn_p1(9, 14, 5, jitter=0.05, seed=2)
    nx1, nxy = 10, 10 * 15
    a = 4 + nx1 * 6 + nxy * 2                        # an interior node
    ed = g(elems, dev)
    plan = vb.P1Plan(ed, coords.shape[1])
    assert plan.lattice(ed, dims=(9, 14, 5))
    cases = [(coords, 0)]
    for u, v in ((a, a + 1 + nx1 + nxy), (a, a + 1), (a + 1, a + 1 + nx1), (a + nx1, a + nx1 + nxy),
                 (a + 1, a + 1 + nx1 + nxy), (a, a + nx1 + nxy)):      # diagonal, axis edges, face diagonals
        cases.append(_collapse(coords, elems, u, v))
        assert cases[-1][1] in (4, 6, 8)
    for cc, want in cases:
        for kw in (dict(variant="lattice"), dict(variant="block"), dict(variant="class"), dict(variant="tile"),
                   dict(mode=vb.VB_ASSEMBLE_ATOMIC)):
            cnt.fill_(-1)
            vb.fem_p1_assemble(g(cc, dev), ed, plan, degenerate=cnt, **kw)
            assert int(h(cnt)[0]) == want, (kw, want)
    for flip in (0, 1):
        c2, e2 = synth.rect_p1(40, 23, jitter=0.1, seed=1, flip=flip)
        e2d = g(e2, dev)
        p2 = vb.P1Plan(e2d, c2.shape[1])
        assert p2.lattice(e2d, dims=(40, 23))
        a2 = 17 + 41 * 9
        cases2 = [(c2, 0), _collapse(c2, e2, a2, a2 + 1), _collapse(c2, e2, a2, a2 + 41),
                  _collapse(c2, e2, a2 + (1 if flip else 0), a2 + 41 + (0 if flip else 1))]
        for cc, want in cases2:
            assert want in (0, 2)
            for kw in (dict(variant="lattice"), dict(variant="block")):
                cnt.fill_(-1)
                vb.fem_p1_assemble(g(cc, dev), e2d, p2, degenerate=cnt, **kw)
                assert int(h(cnt)[0]) == want, (flip, kw, want)
