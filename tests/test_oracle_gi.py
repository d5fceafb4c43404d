"""Pins of the oracle's GI (Code GI; NEXT-4 volume and surface
integrals) against closed forms and an independent surface formula."""
import math

import numpy as np

import oracle
import synth


def points(coords, elems, lam):
    """Quadrature points x_q = sum_a lam[q, a] x_a of every element: (nip, dim, ne)."""
    X = coords[:, elems]                      # (dim, nv, ne)
    return np.einsum("qa,cae->qce", lam, X)


def volumes(coords, elems):
    dim = coords.shape[0]
    X = coords[:, elems]
    J = np.stack([X[:, r + 1] - X[:, 0] for r in range(dim)])   # (dim rows, dim cols, ne)
    return np.abs(np.linalg.det(np.moveaxis(J, -1, 0))) / math.factorial(dim)


def gi_scalar(coords, elems, f, gqo=2):
    dim = coords.shape[0]
    lam, w = oracle.quad_rule(dim, gqo)
    w = np.asarray(w) * math.factorial(dim)        # GI averages over the points (reading B20)
    Xq = points(coords, elems, np.asarray(lam))
    fip = f(Xq)[:, None, :]                        # (nip, 1, ne)
    return oracle.gi(fip, w, volumes(coords, elems))


def test_volume_integrals_exact_for_quadratics():
    """Kuhn cube (boundary not jittered: Omega is the unit cube): the degree-2
    rule integrates quadratics exactly (P:717-735 rho = x1^2 + x2^2)."""
    c, e = synth.cube_kuhn_p1(6, jitter=0.05, seed=3)
    assert abs(gi_scalar(c, e, lambda X: np.ones(X.shape[::2])) - 1.0) <= 1e-13
    assert abs(gi_scalar(c, e, lambda X: X[:, 0] ** 2 + X[:, 1] ** 2) - 2.0 / 3.0) <= 1e-13
    assert abs(gi_scalar(c, e, lambda X: X[:, 0] * X[:, 1]) - 0.25) <= 1e-13
    c2, e2 = synth.square_p1(9, jitter=0.1, seed=3)
    assert abs(gi_scalar(c2, e2, lambda X: X[:, 0] ** 2 + 3 * X[:, 0] * X[:, 1]) - (1 / 3 + 3 / 4)) <= 1e-13


def test_smooth_integrand_converges():
    """A non-polynomial density, int sin(pi x1) sin(pi x2) sin(pi x3) = (2/pi)^3:
    the error falls by >= 4x per refinement (degree-2 rule, O(h^2) or better)."""
    ref = (2.0 / math.pi) ** 3
    errs = []
    for n in (4, 8, 16):
        c, e = synth.cube_kuhn_p1(n, jitter=0.0)
        f = lambda X: np.sin(np.pi * X[:, 0]) * np.sin(np.pi * X[:, 1]) * np.sin(np.pi * X[:, 2])  # noqa: E731
        errs.append(abs(gi_scalar(c, e, f) - ref))
    assert errs[0] > errs[1] > errs[2] and errs[2] < 1e-3
    assert errs[0] / errs[1] > 3.5 and errs[1] / errs[2] > 3.5


def test_surface_flux_equals_enclosed_volume():
    """Surface integral with outer normals (GI with normals): the flux
    of F = x/3 through a closed triangulated surface is its enclosed volume (the
    centroid rule is exact for a linear field on flat faces), equal to the
    divergence-theorem volume of the surface routine; a constant field has zero
    flux."""
    xyz, tri = synth.icosphere(3, perturb=0.01, seed=2)
    n, nh, area, vol = oracle.tri_surface(xyz, tri)
    cen = xyz[:, tri].mean(axis=1)                 # (3, F)
    fip = (cen / 3.0)[None, :, :]                  # (1, 3, F)
    flux = oracle.gi(fip, [1.0], area, normals=nh)
    assert abs(flux - vol) <= 1e-13 * abs(vol)
    const = np.tile(np.array([[0.3], [-1.2], [0.7]]), (1, tri.shape[1]))[None]
    assert abs(oracle.gi(const, [1.0], area, normals=nh)) <= 1e-13 * area.sum()


def test_gi_brute_force_small():
    rng = np.random.default_rng(7)
    fip = rng.standard_normal((3, 2, 5))
    w = rng.random(3)
    sz = rng.random(5)
    nrm = rng.standard_normal((2, 5))
    ref = sum(sz[e] * sum(sum(w[q] * fip[q, c, e] for q in range(3)) * nrm[c, e] for c in range(2)) for e in range(5))
    assert abs(oracle.gi(fip, w, sz, normals=nrm) - ref) <= 1e-14 * max(1.0, abs(ref))
