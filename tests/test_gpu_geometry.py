"""NEXT-4: the paper's tetrahedral geometry workloads as compositions of the
page-wise primitives on the GPU (§3.2):
  meass = amdet(vectors3D)/factorial(dim), meas = norm(meass, 1)
  normals3D = amsm(amt(aminv(vectors3D)), normalsRef)
parity against the same compositions of oracle functions, plus geometric
pins: the volumes of a cube triangulation sum to 1, every normal is
orthogonal to its face's edges, and the paper's worked example."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2404_16039_b200 import vb

pytestmark = pytest.mark.gpu
NORMALS_REF = np.array([[-1, 0, 0, 1], [0, -1, 0, 1], [0, 0, -1, 1]], dtype=np.float64)


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


def gpu_volumes_normals(cd, ed, dev):
    _, v3 = vb.vb_create_coords3D(cd, ed, want_coords3D=False)           # vectors3D: 3 x 3 pages
    meass = vb.vb_page_det(v3) / 6.0
    vinv, _, _ = vb.vb_page_inv(v3, want_det=False)
    nref = g(NORMALS_REF.T[:, :, None], dev)                             # 3 x 4 single object (ld = 0)
    normals = vb.vb_page_mtimes(vb.vb_page_transpose(vinv), nref)        # 3 x 4 pages
    return meass, normals


@pytest.mark.parametrize("n", [3, 16])
def test_volumes_and_normals_parity(dev, n):
    coords, elems = synth.cube_kuhn_p1(n, jitter=0.05, seed=9)
    meass, normals = gpu_volumes_normals(g(coords, dev), g(elems, dev), dev)
    _, v3 = oracle.create_coords3D(coords, elems)
    meass_o = oracle.page_det(v3) / 6.0
    vinv_o, _ = oracle.page_inv(v3)
    normals_o = oracle.page_mtimes(oracle.page_transpose(vinv_o), np.ascontiguousarray(NORMALS_REF.T[:, :, None]))
    assert relmax(h(meass), meass_o) <= 1e-12
    N = h(normals)
    per_page = np.max(np.abs(N - normals_o), axis=(0, 1)) / np.max(np.abs(normals_o), axis=(0, 1))
    assert np.max(per_page) <= 1e-10
    assert abs(math.fsum(np.abs(h(meass))) - 1.0) <= 1e-12                 # meas = norm(meass, 1) = |cube|
    # normal of face j is orthogonal to the face's edges (vectors from the last node)
    X = coords[:, elems]                                                    # 3 x 4 x ne
    faces = [(1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)]                    # face opposite vertex j of normalsRef's order
    nrm = N                                                                 # (4, 3, ne): nrm[j] = column j = normal j
    for j in range(4):
        p, q, r = faces[j]
        for a, b in ((p, q), (q, r)):
            edge = X[:, b, :] - X[:, a, :]
            dot = np.abs(np.einsum("ce,ce->e", nrm[j], edge))
            assert np.max(dot / (np.linalg.norm(nrm[j], axis=0) * np.linalg.norm(edge, axis=0))) < 1e-12


def test_paper_example_on_gpu(dev, golden):
    gd = golden("paper_tet_example.json")
    nodes = np.array(gd["nodes"], dtype=np.float64)
    meass, normals = gpu_volumes_normals(g(nodes.T, dev), g(np.arange(4, dtype=np.int32)[:, None], dev), dev)
    assert h(meass)[0] == -25.0 / 64.0
    expect = np.array([[x[0] / x[1] for x in row] for row in gd["normals3D"]])
    assert np.max(np.abs(h(normals)[:, :, 0].T - expect)) <= 1e-15


# ------------------------------------------------------------------ fused: vb_simplex_geometry
def check_fused(coords, elems, dev, meass_t=None, normals_t=None):
    m, N = vb.vb_simplex_geometry(g(coords, dev), g(elems, dev), meass=meass_t, normals=normals_t)
    m_o, N_o = oracle.simplex_geometry(coords, elems)
    assert relmax(h(m), m_o) <= 1e-12
    Nh = h(N)
    per_page = np.max(np.abs(Nh - N_o), axis=(0, 1)) / np.max(np.abs(N_o), axis=(0, 1))
    assert np.max(per_page) <= 1e-10
    return h(m), Nh


@pytest.mark.parametrize("n", [1, 3, 16, 21])
def test_fused_geometry_3d_parity(dev, n):
    coords, elems = synth.cube_kuhn_p1(n, jitter=0.05, seed=9)          # n = 21: 55566 tets, several blocks
    m, _ = check_fused(coords, elems, dev)
    assert abs(math.fsum(np.abs(m)) - 1.0) <= 1e-12


@pytest.mark.parametrize("n", [1, 5, 64])
def test_fused_geometry_2d_parity(dev, n):
    coords, elems = synth.square_p1(n, jitter=0.05, seed=2)
    m, _ = check_fused(coords, elems, dev)
    assert abs(math.fsum(np.abs(m)) - 1.0) <= 1e-12


@pytest.mark.parametrize("dim", [2, 3])
def test_fused_geometry_odd_counts_and_unaligned_planes_same_bits(dev, dim):
    """An odd element count (the last element takes the scalar tail) and output planes that are not
    16-byte aligned (the scalar path) give the same bits as the 128-bit path."""
    if dim == 3:
        coords, elems = synth.delaunay_p1(3, 9, seed=4)
    else:
        coords, elems = synth.delaunay_p1(2, 15, seed=4)
    for ne in (elems.shape[1], elems.shape[1] - 1, 1, 2, 3):
        el = np.ascontiguousarray(elems[:, :ne])
        m0, N0 = check_fused(coords, el, dev)
        buf_m = torch.full((ne + 3,), 7.0, dtype=torch.float64, device=dev)
        buf_n = torch.full(((dim + 1) * dim * ne + 3,), 7.0, dtype=torch.float64, device=dev)
        m1, N1 = vb.vb_simplex_geometry(g(coords, dev), g(el, dev), meass=buf_m[1:1 + ne],
                                        normals=buf_n[1:1 + (dim + 1) * dim * ne].view(dim + 1, dim, ne))
        assert np.array_equal(h(m1), m0) and np.array_equal(h(N1), N0)
        assert float(buf_m[0]) == 7.0 and float(buf_m[ne + 1]) == 7.0   # nothing written outside
        assert float(buf_n[0]) == 7.0 and float(buf_n[-2]) == 7.0
        m2, _ = vb.vb_simplex_geometry(g(coords, dev), g(el, dev), want_normals=False)
        _, N2 = vb.vb_simplex_geometry(g(coords, dev), g(el, dev), want_meass=False)
        assert np.array_equal(h(m2), m0) and np.array_equal(h(N2), N0)


def test_fused_geometry_equals_the_page_chain(dev):
    """The fused call and the chain of page calls agree entry by entry (both within rounding of the oracle)."""
    coords, elems = synth.cube_kuhn_p1(8, jitter=0.05, seed=1)
    cd, ed = g(coords, dev), g(elems, dev)
    m, N = vb.vb_simplex_geometry(cd, ed)
    m_c, N_c = gpu_volumes_normals(cd, ed, dev)
    assert relmax(h(m), h(m_c)) <= 1e-14
    assert relmax(h(N), h(N_c)) <= 1e-12


def test_fused_geometry_paper_example(dev, golden):
    gd = golden("paper_tet_example.json")
    nodes = np.array(gd["nodes"], dtype=np.float64)
    m, N = vb.vb_simplex_geometry(g(nodes.T, dev), g(np.arange(4, dtype=np.int32)[:, None], dev))
    assert h(m)[0] == -25.0 / 64.0
    expect = np.array([[x[0] / x[1] for x in row] for row in gd["normals3D"]])
    assert np.max(np.abs(h(N)[:, :, 0].T - expect)) <= 1e-15


def test_fused_geometry_empty_and_degenerate(dev):
    coords, elems = synth.cube_kuhn_p1(2, jitter=0.0, seed=0)
    m, N = vb.vb_simplex_geometry(g(coords, dev), g(elems[:, :0], dev))
    assert m.numel() == 0 and N.numel() == 0
    el = elems.copy()
    el[1, 0] = el[0, 0]                                                   # a collapsed edge: det = 0
    m, N = vb.vb_simplex_geometry(g(coords, dev), g(el, dev))
    assert h(m)[0] == 0.0 and not np.all(np.isfinite(h(N)[:, :, 0]))
    assert np.all(np.isfinite(h(N)[:, :, 1:]))


def test_fused_geometry_full_size_configs4_every_element(dev):
    """BASELINE configs[4] mesh (12.58 M tets) in the launch configuration bench.py times: every size and
    every normal against the oracle's chain."""
    coords, elems = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
    m, N = vb.vb_simplex_geometry(g(coords, dev), g(elems, dev))
    m_o, N_o = oracle.simplex_geometry(coords, elems)
    assert relmax(h(m), m_o) <= 1e-12
    Nh = h(N)
    per_page = np.max(np.abs(Nh - N_o), axis=(0, 1)) / np.max(np.abs(N_o), axis=(0, 1))
    assert np.max(per_page) <= 1e-10
    assert abs(math.fsum(np.abs(h(m))) - 1.0) <= 1e-11


@pytest.mark.parametrize("dim", [2, 3])
def test_fused_geometry_strided_coords_through_the_c_abi(dev, dim):
    """coords addressed as coords[c*comp_stride + v*node_stride]: AoS (node_stride = dim) and padded AoS
    (node_stride = 4) through the C ABI give the same bits as the SoA layout; ldn > ne leaves the gap untouched."""
    import ctypes as C
    coords, elems = synth.delaunay_p1(dim, 10 if dim == 2 else 7, seed=6)
    nn, ne = coords.shape[1], elems.shape[1]
    m0, N0 = vb.vb_simplex_geometry(g(coords, dev), g(elems, dev))
    ed = g(elems, dev)
    L = vb.lib()
    for ns in (dim, 4):
        aos = np.zeros((nn, ns))
        aos[:, :dim] = coords.T
        ad = g(aos, dev)
        ldn = ne + 6
        m = torch.full((ne,), 7.0, dtype=torch.float64, device=dev)
        N = torch.full(((dim + 1) * dim, ldn), 7.0, dtype=torch.float64, device=dev)
        rc = L.vb_simplex_geometry(dim, ne, C.c_void_p(ad.data_ptr()), ns, 1, C.c_void_p(ed.data_ptr()), ne,
                                   C.c_void_p(m.data_ptr()), C.c_void_p(N.data_ptr()), ldn, None)
        assert rc == 0, L.vb_last_error()
        assert np.array_equal(h(m), h(m0))
        Nh = h(N)
        assert np.array_equal(Nh[:, :ne].reshape(dim + 1, dim, ne), h(N0))
        assert np.all(Nh[:, ne:] == 7.0)
