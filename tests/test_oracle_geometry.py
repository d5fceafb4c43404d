"""Pins of oracle.simplex_geometry (meass = amdet(vectors3D)/d!, normals3D =
amsm(amt(aminv(vectors3D)), normalsRef)) against things other than itself: the paper's worked
example in exact fractions, the identities normals_j . v_k = -delta_jk and sum_j normals_j = 0
(V^{-T} normalsRef with normalsRef = [-I | 1]), |normal_j| = area of face j / (d |T|), volumes of
a partition summing to the box, and numpy.linalg on random simplices."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth


def test_paper_example_exact(golden):
    gd = golden("paper_tet_example.json")
    nodes = np.array(gd["nodes"], dtype=np.float64)
    meass, normals = oracle.simplex_geometry(nodes.T, np.arange(4, dtype=np.int32)[:, None])
    assert Fraction(meass[0]) == Fraction(*gd["det_over_6"])       # -25/64
    expect = np.array([[Fraction(*x) for x in row] for row in gd["normals3D"]], dtype=object)
    got = normals[:, :, 0].T                                        # rows = components, columns = normals
    for c in range(3):
        for j in range(4):
            assert abs(got[c, j] - float(expect[c, j])) <= 1e-15


@pytest.mark.parametrize("dim", [2, 3])
def test_identities_and_numpy_on_random_simplices(dim):
    rng = np.random.default_rng(5 + dim)
    ne = 200
    coords = rng.uniform(-1.0, 2.0, size=(dim, (dim + 1) * ne))
    elems = rng.permutation((dim + 1) * ne).astype(np.int32).reshape(dim + 1, ne)
    meass, normals = oracle.simplex_geometry(coords, elems)
    X = coords[:, elems]                                            # dim x (dim+1) x ne
    V = X[:, :dim, :] - X[:, dim:, :]                               # vectors from the LAST node
    fact = 2.0 if dim == 2 else 6.0
    for e in range(ne):
        Ve = V[:, :, e]
        assert abs(meass[e] - np.linalg.det(Ve) / fact) <= 1e-13 * max(1.0, abs(meass[e]))
        N = normals[:, :, e].T                                      # dim x (dim+1)
        ref = np.linalg.inv(Ve).T @ oracle.NORMALS_REF[dim]
        assert np.max(np.abs(N - ref)) <= 1e-10 * np.max(np.abs(ref))
        # normals_j . v_k = -delta_jk for j < dim; the last normal is minus the sum of the others
        D = N[:, :dim].T @ Ve
        assert np.max(np.abs(D + np.eye(dim))) <= 1e-9
        assert np.max(np.abs(N.sum(axis=1))) <= 1e-10 * np.max(np.abs(N))
        # |normal_j| = (size of face j) / (d |T|): face j is opposite local node j
        for j in range(dim + 1):
            f = [k for k in range(dim + 1) if k != j]
            if dim == 3:
                area = 0.5 * np.linalg.norm(np.cross(X[:, f[1], e] - X[:, f[0], e], X[:, f[2], e] - X[:, f[0], e]))
            else:
                area = np.linalg.norm(X[:, f[1], e] - X[:, f[0], e])
            assert abs(np.linalg.norm(N[:, j]) - area / (dim * abs(meass[e]))) <= 1e-9 * np.linalg.norm(N[:, j])
            # and it points away from node j
            assert np.dot(N[:, j], X[:, j, e] - X[:, f[0], e]) < 0.0


def test_partition_of_a_box():
    coords, elems = synth.cube_kuhn_p1(5, jitter=0.05, seed=3)
    meass, _ = oracle.simplex_geometry(coords, elems)
    assert abs(np.sum(np.abs(meass)) - 1.0) <= 1e-13                # meas = norm(meass, 1)
    c2, e2 = synth.square_p1(7, jitter=0.05, seed=4)
    a2, _ = oracle.simplex_geometry(c2, e2)
    assert abs(np.sum(np.abs(a2)) - 1.0) <= 1e-13
