"""Pins of the P1 FEM oracle (O8-O11) against what the paper and the
mathematics fix (SURVEY.md §8(c) "Pins for K and M"): hand values, an
independent facet-normal formula for the element stiffness, exact quadrature
for the mass, brute-force dense adjacency and assembly, closed-form nnz,
K 1 = 0, sum(M) = |Omega|, u^T K u = |a|^2 |Omega| for linear u, the
5-point stencil on the unjittered square and O(h^2) convergence."""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth


def frac_mat(m, scale):
    return np.array(m, dtype=np.float64) / scale


# ------------------------------------------------------- independent formulas
def facet_normals(X):
    """Area-weighted OUTWARD normals N_a of the facet opposite vertex a
    (no Jacobian inverse).  X: (dim, nv).  Returns (dim, nv), |T|."""
    dim, nv = X.shape
    N = np.zeros((dim, nv))
    if dim == 2:
        for a in range(3):
            p, q = X[:, (a + 1) % 3], X[:, (a + 2) % 3]
            t = q - p
            n = np.array([t[1], -t[0]])
            if np.dot(n, X[:, a] - p) > 0:
                n = -n
            N[:, a] = n
        e1, e2 = X[:, 1] - X[:, 0], X[:, 2] - X[:, 0]
        vol = abs(e1[0] * e2[1] - e1[1] * e2[0]) / 2.0
    else:
        for a in range(4):
            o = [b for b in range(4) if b != a]
            p, q, r = X[:, o[0]], X[:, o[1]], X[:, o[2]]
            n = 0.5 * np.cross(q - p, r - p)
            if np.dot(n, X[:, a] - p) > 0:
                n = -n
            N[:, a] = n
        e = X[:, 1:] - X[:, :1]
        vol = abs(np.dot(e[:, 0], np.cross(e[:, 1], e[:, 2]))) / 6.0
    return N, vol


def ke_facet(X):
    """grad phi_a = -N_a / (d |T|)  =>  K_ab = N_a . N_b / (d^2 |T|)."""
    N, vol = facet_normals(X)
    d = X.shape[0]
    return (N.T @ N) / (d * d * vol), vol


def me_quadrature(X):
    """Exact degree-2 quadrature of phi_a phi_b (phi_a = barycentric lambda_a).
    2D: edge midpoints, weights |T|/3.  3D: 4-point rule a=0.5854101966249685,
    b=0.1381966011250105, weights |T|/4."""
    dim = X.shape[0]
    _, vol = facet_normals(X)
    if dim == 2:
        pts = [np.array(p) for p in ([0.5, 0.5, 0.0], [0.0, 0.5, 0.5], [0.5, 0.0, 0.5])]
        w = vol / 3.0
    else:
        a, b = (5.0 + 3.0 * math.sqrt(5.0)) / 20.0, (5.0 - math.sqrt(5.0)) / 20.0
        pts = [np.array([a if i == j else b for i in range(4)]) for j in range(4)]
        w = vol / 4.0
    return sum(w * np.outer(p, p) for p in pts)


# ------------------------------------------------------- local matrices (O9)
def test_reference_triangle_and_tet_hand_values(golden):
    g = golden("derived_local_matrices.json")
    t = g["ref_triangle"]
    K, M = oracle.p1_local(np.array(t["X"], dtype=np.float64))
    assert np.array_equal(K, frac_mat(t["K_times2"], 2.0))
    assert np.max(np.abs(M - frac_mat(t["M_times24"], 24.0))) <= 1e-17
    t = g["ref_tet"]
    K, M = oracle.p1_local(np.array(t["X"], dtype=np.float64))
    assert np.max(np.abs(K - frac_mat(t["K_times6"], 6.0))) <= 1e-16
    assert np.max(np.abs(M - frac_mat(t["M_times120"], 120.0))) <= 1e-17


def test_paper_tet_local_stiffness(golden):
    g = golden("derived_local_matrices.json")["paper_tet"]
    nodes = np.array(golden("paper_tet_example.json")["nodes"], dtype=np.float64)
    K, M = oracle.p1_local(np.ascontiguousarray(nodes.T))
    vol = float(Fraction(*g["volume"]))
    assert np.max(np.abs(K - frac_mat(g["K_times144"], 144.0))) <= 2e-16
    assert abs(np.sum(M) - vol) <= 1e-16


@pytest.mark.parametrize("dim", [2, 3])
def test_local_matrices_vs_facet_formula_and_quadrature(dim):
    rng = np.random.default_rng(11)
    for _ in range(200):
        X = rng.normal(size=(dim, dim + 1))
        K, M = oracle.p1_local(X)
        Kf, vol = ke_facet(X)
        if vol < 1e-3:
            continue
        assert np.max(np.abs(K - Kf)) <= 1e-12 * np.max(np.abs(Kf))
        assert np.max(np.abs(M - me_quadrature(X))) <= 1e-14 * vol
        assert np.array_equal(K, K.T)                     # pin 9: bitwise symmetric


def test_local_all_pages_match_single_element():
    coords, elems = synth.cube_kuhn_p1(2, jitter=0.05, seed=0)
    K3, M3 = oracle.p1_local_all(coords, elems)
    for e in (0, 5, 17, 47):
        K, M = oracle.p1_local(coords[:, elems[:, e]])
        assert np.array_equal(K3[:, :, e].T, K)
        assert np.array_equal(M3[:, :, e].T, M)


# ------------------------------------------------------- pattern (O10)
def brute_pattern(elems, nn):
    adj = np.zeros((nn, nn), dtype=bool)
    for e in range(elems.shape[1]):
        v = elems[:, e]
        adj[np.ix_(v, v)] = True
    rows, cols = np.nonzero(adj)
    row_ptr = np.zeros(nn + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    return np.cumsum(row_ptr).astype(np.int32), cols.astype(np.int32)


@pytest.mark.parametrize("mesh", ["sq3", "sq5", "cube2", "cube3"])
def test_pattern_vs_dense_brute_force(mesh):
    if mesh.startswith("sq"):
        coords, elems = synth.square_p1(int(mesh[2:]))
    else:
        coords, elems = synth.cube_kuhn_p1(int(mesh[4:]))
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    brp, bci = brute_pattern(elems, nn)
    assert np.array_equal(rp, brp) and np.array_equal(ci, bci)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_pattern_closed_form_nnz(n):
    _, e2 = synth.square_p1(n)
    nn2 = (n + 1) ** 2
    rp, ci = oracle.p1_pattern(e2, nn2)
    assert rp[-1] == nn2 + 2 * (2 * n * (n + 1) + n * n)
    _, e3 = synth.cube_kuhn_p1(n)
    nn3 = (n + 1) ** 3
    rp3, ci3 = oracle.p1_pattern(e3, nn3)
    assert rp3[-1] == nn3 + 2 * (3 * n * (n + 1) ** 2 + 3 * n * n * (n + 1) + n ** 3)
    if n >= 3:
        lens2 = np.diff(rp).reshape(n + 1, n + 1)
        assert np.all(lens2[1:-1, 1:-1] == 7)
        lens3 = np.diff(rp3).reshape(n + 1, n + 1, n + 1)
        assert np.all(lens3[1:-1, 1:-1, 1:-1] == 15)
    for a, b in ((rp, ci), (rp3, ci3)):
        for r in range(len(a) - 1):
            seg = b[a[r]:a[r + 1]]
            assert np.all(np.diff(seg) > 0) and r in seg        # sorted, diagonal present


# ------------------------------------------------------- assembly (O11)
def assemble(coords, elems):
    rp, ci = oracle.p1_pattern(elems, coords.shape[1])
    K, M = oracle.p1_assemble(coords, elems, rp, ci)
    return rp, ci, K, M


def csr_matvec(rp, ci, v, u):
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    out = np.zeros(len(rp) - 1)
    np.add.at(out, rows, v * u[ci])
    return out


@pytest.mark.parametrize("dim,n", [(2, 8), (2, 32), (3, 4), (3, 8)])
def test_assembly_invariants(dim, n):
    if dim == 2:
        coords, elems = synth.square_p1(n, jitter=0.1, seed=0)
        a = np.array([1.0, 2.0])
    else:
        coords, elems = synth.cube_kuhn_p1(n, jitter=0.05, seed=0)
        a = np.array([1.0, 2.0, 3.0])
    rp, ci, K, M = assemble(coords, elems)
    nn = coords.shape[1]
    Kinf = np.max(np.abs(K))
    assert np.max(np.abs(csr_matvec(rp, ci, K, np.ones(nn)))) <= 1e-13 * Kinf      # K 1 = 0
    assert abs(math.fsum(M) - 1.0) <= 1e-13                                          # sum M = |Omega|
    u = a @ coords
    uKu = math.fsum(u * csr_matvec(rp, ci, K, u))
    assert abs(uKu - float(a @ a)) <= 1e-12 * float(a @ a)                          # |a|^2 |Omega|
    Ku = csr_matvec(rp, ci, K, u)
    idx = np.arange(nn)
    grid = [(idx // (n + 1) ** k) % (n + 1) for k in range(dim)]
    inner = np.all([(g > 0) & (g < n) for g in grid], axis=0)
    assert np.max(np.abs(Ku[inner])) <= 1e-12 * Kinf                                  # patch test
    # symmetry: K[i,j] == K[j,i] bitwise (same products, same order), same for M
    rows = np.repeat(np.arange(nn), np.diff(rp))
    key = rows.astype(np.int64) * nn + ci
    tkey = ci.astype(np.int64) * nn + rows
    perm = np.searchsorted(key, tkey)
    assert np.array_equal(K[perm], K) and np.array_equal(M[perm], M)


@pytest.mark.parametrize("dim,n", [(2, 3), (3, 2)])
def test_assembly_vs_dense_brute_force_independent_formulas(dim, n):
    if dim == 2:
        coords, elems = synth.square_p1(n, jitter=0.1, seed=4)
    else:
        coords, elems = synth.cube_kuhn_p1(n, jitter=0.05, seed=4)
    nn = coords.shape[1]
    Kd = np.zeros((nn, nn))
    Md = np.zeros((nn, nn))
    for e in range(elems.shape[1]):
        v = elems[:, e]
        X = coords[:, v]
        Ke, _ = ke_facet(X)
        Kd[np.ix_(v, v)] += Ke
        Md[np.ix_(v, v)] += me_quadrature(X)
    rp, ci, K, M = assemble(coords, elems)
    rows = np.repeat(np.arange(nn), np.diff(rp))
    assert np.max(np.abs(K - Kd[rows, ci])) <= 1e-13 * np.max(np.abs(Kd))
    assert np.max(np.abs(M - Md[rows, ci])) <= 1e-13 * np.max(np.abs(Md))
    mask = np.zeros((nn, nn), dtype=bool)
    mask[rows, ci] = True
    assert not np.any(Kd[~mask]) and not np.any(Md[~mask])


def test_unjittered_square_stencil_bitwise():
    """5-point stencil (4, -1, -1, -1, -1) and 0 on the split diagonal, bitwise
    (h = 1/32 keeps every intermediate dyadic); M_ii = h^2/2, M_ij = h^2/12."""
    n = 32
    h = 1.0 / n
    coords, elems = synth.square_p1(n, jitter=0.0)
    rp, ci, K, M = assemble(coords, elems)
    n1 = n + 1
    for (i, j) in [(5, 7), (16, 16), (1, 30), (30, 1)]:
        v = i + n1 * j
        seg = slice(rp[v], rp[v + 1])
        cols = ci[seg]
        vals = dict(zip(cols.tolist(), K[seg].tolist()))
        mvals = dict(zip(cols.tolist(), M[seg].tolist()))
        assert len(cols) == 7
        assert vals[v] == 4.0
        for w in (v - 1, v + 1, v - n1, v + n1):
            assert vals[w] == -1.0
        for w in (v - n1 - 1, v + n1 + 1):                      # SW-NE diagonal neighbours
            assert vals[w] == 0.0
        assert abs(mvals[v] - h * h / 2) <= 1e-18 and abs(mvals[v + 1] - h * h / 12) <= 1e-19
    # edge row (i = 0 side, interior j): 2, -1/2, -1/2, -1, 0
    v = 0 + n1 * 10
    vals = dict(zip(ci[rp[v]:rp[v + 1]].tolist(), K[rp[v]:rp[v + 1]].tolist()))
    assert vals[v] == 2.0 and vals[v + 1] == -1.0 and vals[v - n1] == -0.5 and vals[v + n1] == -0.5
    # corners on the split diagonal: 1, -1/2, -1/2, 0 ; other corners 1, -1/2, -1/2
    v = 0
    vals = dict(zip(ci[rp[v]:rp[v + 1]].tolist(), K[rp[v]:rp[v + 1]].tolist()))
    assert vals == {0: 1.0, 1: -0.5, n1: -0.5, n1 + 1: 0.0}
    v = n
    vals = dict(zip(ci[rp[v]:rp[v + 1]].tolist(), K[rp[v]:rp[v + 1]].tolist()))
    assert vals == {n - 1: -0.5, n: 1.0, n + n1: -0.5}


def test_unjittered_kuhn_interior_row():
    n = 8
    h = 1.0 / n
    coords, elems = synth.cube_kuhn_p1(n, jitter=0.0)
    rp, ci, K, M = assemble(coords, elems)
    n1 = n + 1
    v = 4 + n1 * (3 + n1 * 5)
    seg = slice(rp[v], rp[v + 1])
    vals = dict(zip(ci[seg].tolist(), K[seg].tolist()))
    assert abs(vals[v] - 6 * h) <= 1e-15
    for w in (v - 1, v + 1, v - n1, v + n1, v - n1 * n1, v + n1 * n1):
        assert abs(vals[w] + h) <= 1e-15
    others = [x for c, x in vals.items() if c not in (v, v - 1, v + 1, v - n1, v + n1, v - n1 * n1, v + n1 * n1)]
    assert len(others) == 8 and max(abs(x) for x in others) <= 1e-15
    assert abs(math.fsum(M[seg]) - h ** 3) <= 1e-18


@pytest.mark.parametrize("dim", [2, 3])
def test_row_mask_restriction_is_bitwise_subset(dim):
    coords, elems = (synth.square_p1(6) if dim == 2 else synth.cube_kuhn_p1(3))
    nn = coords.shape[1]
    rp, ci, K, M = assemble(coords, elems)
    mask = np.zeros(nn, dtype=np.uint8)
    mask[::5] = 1
    Kr, Mr = oracle.p1_assemble(coords, elems, rp, ci, row_mask=mask)
    rows = np.repeat(np.arange(nn), np.diff(rp))
    sel = mask[rows] == 1
    assert np.array_equal(Kr[sel], K[sel]) and np.array_equal(Mr[sel], M[sel])


def test_convergence_of_quadratic_forms_2d():
    """u = sin(pi x) sin(pi y): u^T K u -> pi^2/2, u^T M u -> 1/4 at O(h^2)
    (c = 1 analog of the paper's I_K, I_M checks)."""
    eK, eM = [], []
    for n in (8, 16, 32):
        coords, elems = synth.square_p1(n, jitter=0.0)
        rp, ci, K, M = assemble(coords, elems)
        u = np.sin(np.pi * coords[0]) * np.sin(np.pi * coords[1])
        eK.append(abs(u @ csr_matvec(rp, ci, K, u) - np.pi ** 2 / 2))
        eM.append(abs(u @ csr_matvec(rp, ci, M, u) - 0.25))
    for e in (eK, eM):
        assert 3.5 < e[0] / e[1] < 4.5 and 3.5 < e[1] / e[2] < 4.5


def test_jittered_meshes_keep_orientation():
    """Jitter (<= 0.1h in 2D, 0.05h in 3D) never inverts an element."""
    for (c0, e0), (c1, e1) in (((synth.square_p1(16, 0.0)), synth.square_p1(16, 0.1)),
                               ((synth.cube_kuhn_p1(6, 0.0)), synth.cube_kuhn_p1(6, 0.05))):
        def signs(c, e):
            X = c[:, e]                     # (dim, nv, ne)
            J = X[:, 1:, :] - X[:, :1, :]
            return np.sign(np.linalg.det(J.transpose(2, 0, 1)))
        assert np.array_equal(signs(c0, e0), signs(c1, e1))


@pytest.mark.parametrize("dim,n", [(2, 12), (3, 5)])
def test_delaunay_invariants_and_numbering_independence(dim, n):
    """Unstructured (Delaunay) meshes: K 1 = 0, sum M = |Omega|, u^T K u =
    |a|^2 for linear u, and the assembled operator does not depend on node,
    element or vertex numbering (same entries after relabelling)."""
    coords, elems = synth.delaunay_p1(dim, n, seed=2)
    nn = coords.shape[1]
    rp, ci, K, M = assemble(coords, elems)
    Kinf = np.max(np.abs(K))
    assert np.max(np.abs(csr_matvec(rp, ci, K, np.ones(nn)))) <= 1e-13 * Kinf
    assert abs(math.fsum(M) - 1.0) <= 1e-13
    a = np.arange(1.0, dim + 1.0)
    u = a @ coords
    assert abs(math.fsum(u * csr_matvec(rp, ci, K, u)) - float(a @ a)) <= 1e-12 * float(a @ a)
    c2, e2 = synth.permute_mesh(coords, elems, seed=3)
    rp2, ci2, K2, M2 = assemble(c2, e2)
    # node map old -> new from the coordinates (all distinct)
    new_of_old = np.lexsort(c2[::-1])[np.argsort(np.lexsort(coords[::-1]))]
    assert np.array_equal(c2[:, new_of_old], coords)
    D1 = np.zeros((nn, nn)), np.zeros((nn, nn))
    rows = np.repeat(np.arange(nn), np.diff(rp))
    rows2 = np.repeat(np.arange(nn), np.diff(rp2))
    for D, v in zip(D1, (K, M)):
        D[new_of_old[rows], new_of_old[ci]] = v
    assert np.max(np.abs(D1[0][rows2, ci2] - K2)) <= 1e-13 * Kinf
    assert np.max(np.abs(D1[1][rows2, ci2] - M2)) <= 1e-13 * np.max(M)
    assert np.count_nonzero(np.diff(rp2)) == nn and len(ci2) == len(ci)


def test_rect_p1_generator_and_oracle_invariants():
    """synth.rect_p1 (inputs of the 2D lattice tests): flip = 0 on a square is square_p1's mesh bit for bit; on
    rectangles and for both diagonals the oracle's K has zero row sums, sum(M) = the area nx ny / m^2, the
    closed-form nnz of the 7-point stencil, and every triangle is positively oriented or consistently
    negative (no inverted element after the jitter)."""
    c0, e0 = synth.square_p1(9, jitter=0.1, seed=3)
    c1, e1 = synth.rect_p1(9, 9, jitter=0.1, seed=3, flip=0)
    assert np.array_equal(c0, c1) and np.array_equal(e0, e1)
    for (nx, ny), flip in (((7, 4), 0), ((7, 4), 1), ((3, 11), 1)):
        coords, elems = synth.rect_p1(nx, ny, jitter=0.1, seed=1, flip=flip)
        nn = (nx + 1) * (ny + 1)
        assert coords.shape == (2, nn) and elems.shape == (3, 2 * nx * ny)
        rp, ci = oracle.p1_pattern(elems, nn)
        # self + 2 axis neighbours per axis + the two diagonal neighbours along the split diagonal
        nnz = nn + 2 * (nx * (ny + 1) + ny * (nx + 1)) + 2 * nx * ny
        assert int(rp[-1]) == nnz
        K, M = oracle.p1_assemble(coords, elems, rp, ci)
        rows = np.repeat(np.arange(nn), np.diff(rp))
        assert np.max(np.abs(np.bincount(rows, weights=K, minlength=nn))) <= 1e-12
        m = max(nx, ny)
        assert abs(M.sum() - nx * ny / m ** 2) <= 1e-13
        x = coords[:, elems]                      # (2, 3, ne)
        det = (x[0, 1] - x[0, 0]) * (x[1, 2] - x[1, 0]) - (x[1, 1] - x[1, 0]) * (x[0, 2] - x[0, 0])
        assert np.all(det > 0) or np.all(det < 0)
