"""Pins of the page-wise oracle (O2-O6, O8) against things other than itself:
library routines it does not call, exact integer arithmetic, an independent
determinant definition (Leibniz), and the paper's worked example.
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth


def to_mats(P):
    """SoA (cols, rows, N) -> (N, rows, cols) numpy matrices."""
    return np.ascontiguousarray(P.transpose(2, 1, 0))


def to_pages(A):
    return np.ascontiguousarray(A.transpose(2, 1, 0))


def frac(v):
    return Fraction(v[0], v[1])


# ---------------------------------------------------------------- mtimes (O2)
@pytest.mark.parametrize("tX,tY", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (2, 2, 2), (3, 3, 3), (4, 4, 4), (2, 3, 4), (4, 1, 3), (3, 4, 1)])
def test_mtimes_integer_pages_exact_vs_numpy(tX, tY, m, k, n):
    N = 37
    xr, xc = (k, m) if tX else (m, k)
    yr, yc = (n, k) if tY else (k, n)
    X = synth.integer_pages(xr, xc, N, seed=1)
    Y = synth.integer_pages(yr, yc, N, seed=2)
    Z = oracle.page_mtimes(X, Y, tX, tY)
    A = to_mats(X).astype(np.int64)
    B = to_mats(Y).astype(np.int64)
    if tX:
        A = A.transpose(0, 2, 1)
    if tY:
        B = B.transpose(0, 2, 1)
    ref = np.matmul(A, B).astype(np.float64)
    assert np.array_equal(to_mats(Z), ref)


def test_mtimes_broadcast_single_object():
    """ld = 0 is the copy map (eq:copy): amsm / smamt."""
    N = 19
    X = synth.integer_pages(3, 4, N, seed=3)
    S = synth.integer_pages(4, 2, 1, seed=4)
    Z = oracle.page_mtimes(X, S)                       # amsm: X_k * S
    ref = np.matmul(to_mats(X), to_mats(S)[0])
    assert np.array_equal(to_mats(Z), ref)
    Sm = synth.integer_pages(2, 4, 1, seed=5)
    Z3 = oracle.page_mtimes(Sm, X, tX=False, tY=True)  # smamt: S * X_k^T
    ref3 = np.matmul(to_mats(Sm)[0], to_mats(X).transpose(0, 2, 1))
    assert np.array_equal(to_mats(Z3), ref3)


def test_amtam_spec_example(golden):
    g = golden("spec_amtam_example.json")
    P = to_pages(np.array(g["amx"], dtype=np.float64)[None])   # one 2x3 page
    Z = oracle.page_mtimes(P, P, tX=True, tY=False)
    assert np.array_equal(to_mats(Z)[0], np.array(g["result"], dtype=np.float64))


def test_mtimes_transpose_identity_bitwise():
    """(AB)^T == B^T A^T bitwise: same products, same summation order."""
    N = 101
    A = synth.normal_pages(3, 4, N, stream=20)
    B = synth.normal_pages(4, 2, N, stream=21)
    AB_T = oracle.page_transpose(oracle.page_mtimes(A, B))
    BtAt = oracle.page_mtimes(B, A, tX=True, tY=True)
    assert np.array_equal(AB_T, BtAt)


def test_mtimes_float_vs_numpy():
    N = 1000
    for n in (2, 3, 4):
        A = synth.normal_pages(n, n, N, stream=22)
        B = synth.normal_pages(n, n, N, stream=23)
        Z = oracle.page_mtimes(A, B, False, True)
        ref = np.matmul(to_mats(A), to_mats(B).transpose(0, 2, 1))
        assert np.max(np.abs(to_mats(Z) - ref)) <= 1e-14 * np.max(np.abs(ref))


# ---------------------------------------------------------------- transpose (O3)
def test_transpose_involution_and_numpy():
    X = synth.normal_pages(3, 4, 17, stream=24)
    T = oracle.page_transpose(X)
    assert T.shape == (3, 4, 17)
    assert np.array_equal(to_mats(T), to_mats(X).transpose(0, 2, 1))
    assert np.array_equal(oracle.page_transpose(T), X)


# ---------------------------------------------------------------- det (O4)
def leibniz(M):
    n = len(M)
    s = 0
    for perm in itertools.permutations(range(n)):
        inv = sum(1 for i in range(n) for j in range(i + 1, n) if perm[i] > perm[j])
        p = 1
        for i in range(n):
            p *= M[i][perm[i]]
        s += -p if inv % 2 else p
    return s


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_det_integer_pages_exact_vs_leibniz(n):
    N = 200
    X = synth.integer_pages(n, n, N, seed=7, bound=9)
    d = oracle.page_det(X)
    mats = to_mats(X).astype(np.int64)
    for k in range(N):
        assert d[k] == float(leibniz(mats[k].tolist()))


def test_det_paper_example(golden):
    g = golden("paper_tet_example.json")
    V = np.array(g["vectors3D_times4"], dtype=np.float64) / 4.0
    d = oracle.page_det(np.ascontiguousarray(V.T[:, :, None]))[0]
    assert d / 6.0 == float(frac(g["det_over_6"]))      # -25/64, exact in binary
    assert d == float(Fraction(-75, 32))


def test_det_identity_triangular_and_multiplicative():
    N = 500
    for n in (2, 3, 4):
        I = np.tile(np.eye(n)[:, :, None], (1, 1, 5))
        assert np.all(oracle.page_det(I) == 1.0)
        A = to_mats(synth.normal_pages(n, n, N, stream=30))
        U = np.triu(A)
        d = oracle.page_det(to_pages(U))
        ref = np.prod(np.diagonal(U, axis1=1, axis2=2), axis=1)
        assert np.allclose(d, ref, rtol=1e-14, atol=0)
        B = to_mats(synth.normal_pages(n, n, N, stream=31))
        dA = oracle.page_det(to_pages(A))
        dB = oracle.page_det(to_pages(B))
        dAB = oracle.page_det(oracle.page_mtimes(to_pages(A), to_pages(B)))
        scale = np.abs(dA * dB) + 1e-300
        assert np.max(np.abs(dAB - dA * dB) / np.maximum(scale, 1e-3)) < 1e-11
        assert np.allclose(dA, np.linalg.det(A), rtol=1e-11, atol=1e-13)


# ---------------------------------------------------------------- inverse (O5)
def unimodular(n, N, rng):
    """Products of unit lower and unit upper integer triangular matrices."""
    L = np.tril(rng.integers(-2, 3, size=(N, n, n)), -1) + np.eye(n, dtype=np.int64)
    U = np.triu(rng.integers(-2, 3, size=(N, n, n)), 1) + np.eye(n, dtype=np.int64)
    return np.matmul(L, U)


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_inv_unimodular_exact(n):
    rng = np.random.default_rng(5)
    A = unimodular(n, 300, rng)
    Ainv, d = oracle.page_inv(to_pages(A.astype(np.float64)))
    assert np.all(d == 1.0)
    Ai = to_mats(Ainv)
    assert np.array_equal(Ai, np.rint(Ai))                 # integer inverse
    assert np.array_equal(np.matmul(A, Ai.astype(np.int64)), np.broadcast_to(np.eye(n, dtype=np.int64), A.shape))


@pytest.mark.parametrize("n", [2, 3, 4])
def test_inv_multiply_back_and_numpy(n):
    X, _ = synth.inverse_pages(n, 2000, seed=3)
    Xi, d = oracle.page_inv(X)
    A = to_mats(X)
    Ai = to_mats(Xi)
    cond = np.linalg.cond(A)
    I = np.eye(n)
    err_r = np.max(np.abs(np.matmul(A, Ai) - I), axis=(1, 2))
    err_l = np.max(np.abs(np.matmul(Ai, A) - I), axis=(1, 2))
    assert np.all(err_r <= 1e-13 * cond) and np.all(err_l <= 1e-13 * cond)
    ref = np.linalg.inv(A)
    rel = np.max(np.abs(Ai - ref), axis=(1, 2)) / np.max(np.abs(ref), axis=(1, 2))
    assert np.all(rel <= 1e-14 * cond)
    assert np.allclose(d, np.linalg.det(A), rtol=1e-12)


def test_paper_normals_example(golden):
    """normals3D = amsm(amt(aminv(vectors3D)), normalsRef)."""
    g = golden("paper_tet_example.json")
    nodes = np.array(g["nodes"], dtype=np.float64)             # rows N1..N4
    coords = np.ascontiguousarray(nodes.T)                      # (3, 4)
    elems = np.arange(4, dtype=np.int32)[:, None]
    c3, v3 = oracle.create_coords3D(coords, elems)
    assert np.array_equal(to_mats(v3)[0], np.array(g["vectors3D_times4"]) / 4.0)
    vinv, d = oracle.page_inv(v3)
    nref = np.ascontiguousarray(np.array(g["normalsRef"], dtype=np.float64).T[:, :, None])
    normals = oracle.page_mtimes(oracle.page_transpose(vinv), nref)
    expect = np.array([[float(frac(x)) for x in row] for row in g["normals3D"]])
    assert np.max(np.abs(to_mats(normals)[0] - expect)) <= 1e-15


def test_create_coords3D_paper_nodes_and_fancy_index(golden):
    """coords3D(:, a, e) = coords(elems(e, a), :) (Code coords3D).  Pins: the paper's
    tetrahedron N1..N4 gathered by the identity element gives back the node matrix, by a
    permuted element the permuted node matrix; on random meshes numpy fancy indexing (independent of
    the oracle's loops) gives every plane, and vectors3D = coords3D(:, a) - coords3D(:, end)."""
    g = golden("paper_tet_example.json")
    nodes = np.array(g["nodes"], dtype=np.float64)             # rows N1..N4
    coords = np.ascontiguousarray(nodes.T)                      # (3, 4)
    c3, _ = oracle.create_coords3D(coords, np.arange(4, dtype=np.int32)[:, None])
    # page layout (a, c, e): entry (c, a) of the dim x nv page is coordinate c of vertex a
    assert c3.shape == (4, 3, 1)
    assert np.array_equal(c3[:, :, 0], nodes)
    perm = np.array([2, 0, 3, 1], dtype=np.int32)
    c3p, v3p = oracle.create_coords3D(coords, perm[:, None])
    assert np.array_equal(c3p[:, :, 0], nodes[perm])
    assert np.array_equal(v3p[:, :, 0], nodes[perm][:3] - nodes[perm][3])
    rng = np.random.default_rng(11)
    for dim, nv, nn, ne in [(2, 3, 50, 333), (3, 4, 70, 1001), (3, 3, 40, 257), (3, 10, 90, 129)]:
        coords = rng.standard_normal((dim, nn))
        elems = rng.integers(0, nn, size=(nv, ne)).astype(np.int32)
        c3, v3 = oracle.create_coords3D(coords, elems)
        ref = coords.T[elems]                                   # (nv, ne, dim)
        assert np.array_equal(c3, ref.transpose(0, 2, 1))
        assert np.array_equal(v3, (ref[:-1] - ref[-1]).transpose(0, 2, 1))


# ---------------------------------------------------------------- cross (O6)
def test_cross_basis_and_numpy():
    e = np.eye(3)
    A = np.ascontiguousarray(e[None])                # pages e1, e2, e3 -> shape (1,3,3)
    B = np.ascontiguousarray(e[:, [1, 2, 0]][None])  # pages e2, e3, e1
    Cc = oracle.page_cross(A, B)
    assert np.array_equal(Cc[0].T, e[[2, 0, 1]])      # e1xe2=e3, e2xe3=e1, e3xe1=e2
    N = 1000
    a = synth.normal_pages(3, 1, N, stream=40)
    b = synth.normal_pages(3, 1, N, stream=41)
    c = oracle.page_cross(a, b)
    ref = np.cross(a[0].T, b[0].T).T
    assert np.max(np.abs(c[0] - ref)) <= 1e-15 * np.max(np.abs(ref)) * 4
    # a.(a x b) = 0 and Lagrange's identity
    dot = np.sum(a[0] * c[0], axis=0)
    assert np.max(np.abs(dot)) < 1e-13
    lhs = np.sum(c[0] ** 2, 0) + np.sum(a[0] * b[0], 0) ** 2
    rhs = np.sum(a[0] ** 2, 0) * np.sum(b[0] ** 2, 0)
    assert np.allclose(lhs, rhs, rtol=1e-13)


def test_cross_equals_cofactor_columns():
    """A13: cof(V) = det(V) V^{-T}; its columns are crosses of V's columns."""
    V, _ = synth.inverse_pages(3, 500, seed=9)
    Vi, d = oracle.page_inv(V)
    cof = to_mats(oracle.page_transpose(Vi)) * d[:, None, None]
    cols = [np.ascontiguousarray(V[j][None]) for j in range(3)]   # column j of each page
    for j in range(3):
        c = oracle.page_cross(cols[(j + 1) % 3], cols[(j + 2) % 3])[0]
        assert np.max(np.abs(c.T - cof[:, :, j])) < 1e-12
