"""GPU parity of the page-wise kernels (a1-a5, a7) against the CPU oracle,
through the C ABI.  Bar (BASELINE.json north_star): integer-valued pages and
pure data movement bit-exact; fp64 pages within 1e-12 relative max-norm over
the array; inverses within 1e-10 relative per page for cond <= 1e4."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2404_16039_b200 import vb

pytestmark = pytest.mark.gpu

SIZES = [1, 2, 17, 1000, 4099]


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


# ---------------------------------------------------------------- a1 mtimes
@pytest.mark.parametrize("tX,tY", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("n", [2, 3, 4])
@pytest.mark.parametrize("N", SIZES)
def test_mtimes_square_float(dev, n, N, tX, tY):
    A = synth.normal_pages(n, n, N, stream=50)
    B = synth.normal_pages(n, n, N, stream=51)
    Z = h(vb.vb_page_mtimes(g(A, dev), g(B, dev), tX, tY))
    assert relmax(Z, oracle.page_mtimes(A, B, tX, tY)) <= 1e-12


@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (2, 3, 4), (4, 1, 3), (3, 4, 1), (1, 4, 1), (4, 4, 4), (3, 2, 3)])
@pytest.mark.parametrize("tX,tY", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_mtimes_integer_bitwise(dev, m, k, n, tX, tY):
    N = 1003
    xr, xc = (k, m) if tX else (m, k)
    yr, yc = (n, k) if tY else (k, n)
    X = synth.integer_pages(xr, xc, N, seed=8)
    Y = synth.integer_pages(yr, yc, N, seed=9)
    Z = h(vb.vb_page_mtimes(g(X, dev), g(Y, dev), tX, tY))
    assert np.array_equal(Z, oracle.page_mtimes(X, Y, tX, tY))


def test_mtimes_broadcast_single_objects(dev):
    """amsm (ldy=0), smamt (ldx=0, tY), svamt (ldx=0, tX, tY) -- P:404-409."""
    N = 777
    X = synth.normal_pages(3, 4, N, stream=52)
    S = synth.normal_pages(4, 2, 1, stream=53)
    assert relmax(h(vb.vb_page_mtimes(g(X, dev), g(S, dev))), oracle.page_mtimes(X, S)) <= 1e-12
    Sm = synth.normal_pages(2, 4, 1, stream=54)
    assert relmax(h(vb.vb_page_mtimes(g(Sm, dev), g(X, dev), False, True)),
                  oracle.page_mtimes(Sm, X, False, True)) <= 1e-12
    sv = synth.normal_pages(4, 1, 1, stream=55)
    assert relmax(h(vb.vb_page_mtimes(g(sv, dev), g(X, dev), True, True)),
                  oracle.page_mtimes(sv, X, True, True)) <= 1e-12


def test_mtimes_padded_ld_and_odd_offsets(dev):
    """ld > npages (padding) and a misaligned (odd-offset) view take the scalar path."""
    N, L = 1001, 1030
    A = synth.normal_pages(3, 3, N, stream=56)
    B = synth.normal_pages(3, 3, N, stream=57)
    Ap = np.zeros((3, 3, L)); Ap[:, :, :N] = A
    Bp = np.zeros((3, 3, L + 1)); Bp[:, :, 1:N + 1] = B            # view starting at an odd offset
    Ad, Bd = g(Ap, dev), g(Bp, dev)
    Zd = torch.full((3, 3, L), np.nan, dtype=torch.float64, device=dev)
    rc = vb.lib().vb_page_mtimes(N, C.c_void_p(Ad.data_ptr()), 3, 3, L, 0,
                                 C.c_void_p(Bd.data_ptr() + 8), 3, 3, L + 1, 1,
                                 C.c_void_p(Zd.data_ptr()), L, vb._stream())
    assert rc == 0
    Z = h(Zd)
    assert relmax(Z[:, :, :N], oracle.page_mtimes(A, B, 0, 1)) <= 1e-12
    assert np.all(np.isnan(Z[:, :, N:]))                             # padding untouched


# ---------------------------------------------------------------- a2 transpose
@pytest.mark.parametrize("r,c", [(1, 1), (2, 2), (3, 3), (4, 4), (2, 3), (4, 1), (3, 4)])
@pytest.mark.parametrize("N", [1, 17, 4099])
def test_transpose_bitwise(dev, r, c, N):
    X = synth.normal_pages(r, c, N, stream=58)
    assert np.array_equal(h(vb.vb_page_transpose(g(X, dev))), oracle.page_transpose(X))


# ---------------------------------------------------------------- a3 det
@pytest.mark.parametrize("n", [1, 2, 3, 4])
@pytest.mark.parametrize("N", SIZES)
def test_det(dev, n, N):
    X = synth.normal_pages(n, n, N, stream=59)
    assert relmax(h(vb.vb_page_det(g(X, dev))), oracle.page_det(X)) <= 1e-12


@pytest.mark.parametrize("n", [2, 3, 4])
def test_det_integer_bitwise(dev, n):
    X = synth.integer_pages(n, n, 5000, seed=10, bound=9)
    assert np.array_equal(h(vb.vb_page_det(g(X, dev))), oracle.page_det(X))


def test_det_paper_example(dev, golden):
    gd = golden("paper_tet_example.json")
    V = np.array(gd["vectors3D_times4"], dtype=np.float64) / 4.0
    d = h(vb.vb_page_det(g(V.T[:, :, None], dev)))[0]
    assert d == -75.0 / 32.0


# ---------------------------------------------------------------- a4 inverse
@pytest.mark.parametrize("n", [1, 2, 3, 4])
@pytest.mark.parametrize("N", SIZES)
def test_inverse_per_page(dev, n, N):
    X, _ = synth.inverse_pages(n, N, seed=4)
    Xi, d, fs = vb.vb_page_inv(g(X, dev), first_singular=torch.zeros(1, dtype=torch.int64, device=dev))
    Xo, do = oracle.page_inv(X)
    got = h(Xi)
    per_page = np.max(np.abs(got - Xo), axis=(0, 1)) / np.max(np.abs(Xo), axis=(0, 1))
    assert np.max(per_page) <= 1e-10
    assert relmax(h(d), do) <= 1e-12
    assert int(h(fs)[0]) == N                                            # none singular


def test_inverse_unimodular_bitwise_and_singular_flag(dev):
    rng = np.random.default_rng(3)
    for n in (2, 3, 4):
        L = np.tril(rng.integers(-2, 3, size=(999, n, n)), -1) + np.eye(n, dtype=np.int64)
        U = np.triu(rng.integers(-2, 3, size=(999, n, n)), 1) + np.eye(n, dtype=np.int64)
        A = np.matmul(L, U).astype(np.float64)
        A[37] = 0.0
        A[37, 0, 0] = 1.0                                                 # singular page
        A[500, :, 1] = A[500, :, 0]                                       # singular page (equal columns)
        X = np.ascontiguousarray(A.transpose(2, 1, 0))
        fs = torch.zeros(1, dtype=torch.int64, device=dev)
        Xi, d, fs = vb.vb_page_inv(g(X, dev), first_singular=fs)
        Xo, do = oracle.page_inv(X)
        got = h(Xi)
        ok = np.ones(999, dtype=bool)
        ok[[37, 500]] = False
        assert np.array_equal(got[:, :, ok], Xo[:, :, ok])
        assert np.array_equal(h(d), do)
        assert int(h(fs)[0]) == 37


def test_paper_normals_composition(dev, golden):
    """amsm(amt(aminv(vectors3D)), normalsRef) on the GPU."""
    gd = golden("paper_tet_example.json")
    nodes = np.array(gd["nodes"], dtype=np.float64)
    coords = g(nodes.T, dev)
    elems = g(np.arange(4, dtype=np.int32)[:, None], dev)
    c3, v3 = vb.vb_create_coords3D(coords, elems)
    vinv, _, _ = vb.vb_page_inv(v3)
    nref = g(np.array(gd["normalsRef"], dtype=np.float64).T[:, :, None], dev)
    normals = h(vb.vb_page_mtimes(vb.vb_page_transpose(vinv), nref))[:, :, 0].T
    expect = np.array([[x[0] / x[1] for x in row] for row in gd["normals3D"]])
    assert np.max(np.abs(normals - expect)) <= 1e-15


# ---------------------------------------------------------------- a5 cross
@pytest.mark.parametrize("N", SIZES)
def test_cross(dev, N):
    A = synth.normal_pages(3, 1, N, stream=60)
    B = synth.normal_pages(3, 1, N, stream=61)
    assert relmax(h(vb.vb_page_cross(g(A, dev), g(B, dev))), oracle.page_cross(A, B)) <= 1e-12
    Ai = synth.integer_pages(3, 1, N, seed=12)
    Bi = synth.integer_pages(3, 1, N, seed=13)
    assert np.array_equal(h(vb.vb_page_cross(g(Ai, dev), g(Bi, dev))), oracle.page_cross(Ai, Bi))


# ---------------------------------------------------------------- a7 gather
@pytest.mark.parametrize("dim", [2, 3])
def test_create_coords3D_bitwise(dev, dim):
    coords, elems = synth.square_p1(9) if dim == 2 else synth.cube_kuhn_p1(5)
    c3, v3 = vb.vb_create_coords3D(g(coords, dev), g(elems, dev))
    oc3, ov3 = oracle.create_coords3D(coords, elems)
    assert np.array_equal(h(c3), oc3) and np.array_equal(h(v3), ov3)


@pytest.mark.parametrize("dim", [2, 3])
def test_create_coords3D_odd_count_and_surface_faces_bitwise(dev, dim):
    """Odd element counts take the one-element-per-thread kernel, even ones the paired 128-bit kernel; also the
    3 x 3 x |F_b| form for boundary faces (nv = 3 in 3D).  All bitwise equal to the oracle."""
    coords, elems = synth.delaunay_p1(dim, 12 if dim == 2 else 7, seed=2)
    for ne in (elems.shape[1], elems.shape[1] - 1, 1, 2):
        el = np.ascontiguousarray(elems[:, :ne])
        c3, v3 = vb.vb_create_coords3D(g(coords, dev), g(el, dev))
        oc3, ov3 = oracle.create_coords3D(coords, el)
        assert np.array_equal(h(c3), oc3) and np.array_equal(h(v3), ov3)
        _, v3b = vb.vb_create_coords3D(g(coords, dev), g(el, dev), want_coords3D=False)
        assert np.array_equal(h(v3b), ov3)
    if dim == 3:
        xyz, tri = synth.icosphere(3, perturb=0.01, seed=0)
        for nf in (tri.shape[1], tri.shape[1] - 1):
            t = np.ascontiguousarray(tri[:, :nf])
            c3, v3 = vb.vb_create_coords3D(g(xyz, dev), g(t, dev))
            oc3, ov3 = oracle.create_coords3D(xyz, t)
            assert np.array_equal(h(c3), oc3) and np.array_equal(h(v3), ov3)


def test_create_coords3D_full_size_configs4(dev):
    """The configs[4] mesh (12.58 M tets) in the launch configuration bench.py times, every entry."""
    coords, elems = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
    c3, v3 = vb.vb_create_coords3D(g(coords, dev), g(elems, dev))
    oc3, ov3 = oracle.create_coords3D(coords, elems)
    assert np.array_equal(h(c3), oc3)
    del c3, oc3
    assert np.array_equal(h(v3), ov3)


# ---------------------------------------------------------------- full size (config 2)
@pytest.mark.parametrize("n", [2, 3, 4])
def test_config2_full_size(dev, n):
    """BASELINE configs[1]: N = 2^20 pages, the launch configuration bench.py times."""
    N = 1 << 20
    A = synth.normal_pages(n, n, N, stream=10)
    B = synth.normal_pages(n, n, N, stream=11)
    Ad, Bd = g(A, dev), g(B, dev)
    for tX, tY in ((0, 0), (0, 1), (1, 0)):
        assert relmax(h(vb.vb_page_mtimes(Ad, Bd, tX, tY)), oracle.page_mtimes(A, B, tX, tY)) <= 1e-12
    assert np.array_equal(h(vb.vb_page_transpose(Ad)), oracle.page_transpose(A))
    assert relmax(h(vb.vb_page_det(Ad)), oracle.page_det(A)) <= 1e-12
    X, _ = synth.inverse_pages(n, N, seed=0)
    Xi, d, _ = vb.vb_page_inv(g(X, dev))
    Xo, do = oracle.page_inv(X)
    per_page = np.max(np.abs(h(Xi) - Xo), axis=(0, 1)) / np.max(np.abs(Xo), axis=(0, 1))
    assert np.max(per_page) <= 1e-10
