"""Pins of the NEXT-2 oracle functions: avtamav (page bilinear form) and the
P1 load vector of Code rhs_vectorP1, against independent definitions."""
import math

import numpy as np
import pytest

import oracle
import synth


def to_mats(P):
    return np.ascontiguousarray(P.transpose(2, 1, 0))


@pytest.mark.parametrize("n,m", [(1, 1), (2, 3), (3, 3), (4, 2), (4, 4)])
def test_bilinear_integer_exact_vs_numpy(n, m):
    N = 301
    A = synth.integer_pages(n, 1, N, seed=20)
    Mx = synth.integer_pages(n, m, N, seed=21)
    B = synth.integer_pages(m, 1, N, seed=22)
    s = oracle.page_bilinear(A, Mx, B)
    ref = np.einsum("ki,kij,kj->k", to_mats(A)[:, :, 0].astype(np.int64), to_mats(Mx).astype(np.int64),
                    to_mats(B)[:, :, 0].astype(np.int64))
    assert np.array_equal(s, ref.astype(np.float64))


def test_bilinear_identity_is_dot_bitwise():
    """avtamav(a, I, b) == avtav(a, b) bitwise."""
    N = 500
    a = synth.normal_pages(3, 1, N, stream=70)
    b = synth.normal_pages(3, 1, N, stream=71)
    I = np.ascontiguousarray(np.tile(np.eye(3)[:, :, None], (1, 1, N)))
    s = oracle.page_bilinear(a, I, b)
    dot = oracle.page_mtimes(a, b, tX=True)[0, 0]                 # avtav
    assert np.array_equal(s, dot)


def dense_mass_exact(coords, elems):
    """Independent c = 1 mass matrix: exact integrals int phi_a phi_b = |T|(1+d_ab)/((d+1)(d+2))
    with |T| from numpy determinants."""
    dim, nn = coords.shape
    X = coords[:, elems]
    vol = np.abs(np.linalg.det((X[:, 1:, :] - X[:, :1, :]).transpose(2, 1, 0))) / math.factorial(dim)
    Md = np.zeros((nn, nn))
    loc = (np.ones((dim + 1, dim + 1)) + np.eye(dim + 1)) / ((dim + 1) * (dim + 2))
    for e in range(elems.shape[1]):
        v = elems[:, e]
        Md[np.ix_(v, v)] += vol[e] * loc
    return Md


@pytest.mark.parametrize("dim", [2, 3])
def test_rhs_of_a_p1_function_is_mass_times_nodal_values(dim):
    """For f in the P1 space, int f phi_i = (M f~)_i exactly with a degree-2 rule."""
    coords, elems = synth.square_p1(6, jitter=0.1, seed=2) if dim == 2 else synth.cube_kuhn_p1(3, jitter=0.05, seed=2)
    rng = np.random.default_rng(4)
    ft = rng.normal(size=coords.shape[1])
    lam, w = oracle.quad_rule(dim, 2)
    fq = lam @ ft[elems]                                  # f at the points: sum_a lam_qa f~_a
    b, b2 = oracle.p1_rhs(coords, elems, fq, gqo=2)
    ref = dense_mass_exact(coords, elems) @ ft
    assert np.max(np.abs(b - ref)) <= 1e-14 * np.max(np.abs(ref))
    assert b2.shape == elems.shape
    bb = np.zeros_like(b)
    np.add.at(bb, elems.ravel(), b2.ravel())               # accumarray of the local contributions
    assert np.max(np.abs(bb - b)) <= 1e-15 * np.max(np.abs(b))


@pytest.mark.parametrize("dim,gqo", [(2, 1), (2, 2), (3, 1), (3, 2)])
def test_rhs_constant_and_total(dim, gqo):
    """f = c: b_i = c sum_{T ∋ i} |T|/(d+1) and sum b = c |Omega| = c."""
    coords, elems = synth.square_p1(7, jitter=0.1) if dim == 2 else synth.cube_kuhn_p1(4, jitter=0.05)
    lam, w = oracle.quad_rule(dim, gqo)
    fq = np.full((len(w), elems.shape[1]), 2.5)
    b, b2 = oracle.p1_rhs(coords, elems, fq, gqo=gqo)
    assert abs(math.fsum(b) - 2.5) <= 1e-13
    X = coords[:, elems]
    vol = np.abs(np.linalg.det((X[:, 1:, :] - X[:, :1, :]).transpose(2, 1, 0))) / math.factorial(dim)
    ref = np.zeros(coords.shape[1])
    np.add.at(ref, elems.ravel(), np.tile(vol, dim + 1) * 2.5 / (dim + 1))
    assert np.max(np.abs(b - ref)) <= 1e-15


def test_rhs_converges_to_exact_integral():
    """sum_i b_i v_i -> int f v for smooth f, v (O(h^2)): f = e^{x+y}, v = sin(pi x) sin(pi y)."""
    errs = []
    exact = (math.pi * (math.e + 1) / (1 + math.pi ** 2)) ** 2
    for n in (16, 32, 64):
        coords, elems = synth.square_p1(n, jitter=0.0)
        lam, w = oracle.quad_rule(2, 2)
        xq = np.einsum("qa,cae->qce", lam, coords[:, elems])
        fq = np.exp(xq.sum(1))
        b, _ = oracle.p1_rhs(coords, elems, fq)
        v = np.sin(np.pi * coords[0]) * np.sin(np.pi * coords[1])
        errs.append(abs(math.fsum(b * v) - exact))
    assert 3.5 < errs[0] / errs[1] < 4.5 and 3.5 < errs[1] / errs[2] < 4.5
