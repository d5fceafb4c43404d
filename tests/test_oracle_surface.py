"""Pins of the surface-geometry oracle (O7, config 3) against closed forms of
the icosahedron, the divergence theorem's limit 4*pi/3, Heron's formula and
an independent triple-product volume formula."""
import math

import numpy as np

import oracle
import synth


def test_icosahedron_closed_forms(golden):
    g = golden("icosahedron.json")
    xyz, tri = synth.icosphere(0, perturb=0.0)
    n, nh, area, vol = oracle.tri_surface(xyz, tri)
    a = 4.0 / math.sqrt(10.0 + 2.0 * math.sqrt(5.0))
    assert abs(vol - (5.0 / 12.0) * (3.0 + math.sqrt(5.0)) * a ** 3) < 1e-14
    assert abs(vol - g["volume"]) < 1e-14
    assert abs(math.fsum(area) - g["area"]) < 1e-14
    assert abs(math.fsum(area) - 5.0 * math.sqrt(3.0) * a * a) < 1e-14


def test_closed_surface_normals_sum_to_zero_and_units():
    xyz, tri = synth.icosphere(3, perturb=0.01, seed=0)
    n, nh, area, vol = oracle.tri_surface(xyz, tri)
    tot = np.array([math.fsum(n[d]) for d in range(3)])
    assert np.max(np.abs(tot)) < 1e-14 * np.sum(np.abs(n))
    assert np.allclose(np.sum(nh * nh, 0), 1.0, rtol=0, atol=1e-15)
    assert np.allclose(area, 0.5 * np.sqrt(np.sum(n * n, 0)), rtol=0, atol=0)


def test_area_vs_heron_and_volume_vs_triple_product():
    xyz, tri = synth.icosphere(4, perturb=0.01, seed=3)
    n, nh, area, vol = oracle.tri_surface(xyz, tri)
    A = xyz[:, tri[0]]
    B = xyz[:, tri[1]]
    Cc = xyz[:, tri[2]]
    la = np.sqrt(np.sum((B - Cc) ** 2, 0))
    lb = np.sqrt(np.sum((A - Cc) ** 2, 0))
    lc = np.sqrt(np.sum((A - B) ** 2, 0))
    s = 0.5 * (la + lb + lc)
    heron = np.sqrt(s * (s - la) * (s - lb) * (s - lc))
    assert np.max(np.abs(area - heron) / heron) < 1e-9          # Heron is ill-conditioned; loose
    trip = np.einsum("ij,ij->j", A, np.cross(B.T, Cc.T).T) / 6.0
    assert abs(vol - math.fsum(trip)) < 1e-14 * abs(vol)
    # orientation: every face normal points away from the origin
    assert np.all(np.einsum("ij,ij->j", nh, (A + B + Cc) / 3.0) > 0)


def test_volume_converges_to_ball_volume():
    errs = []
    for level in (2, 3, 4, 5):
        xyz, tri = synth.icosphere(level, perturb=0.0)
        _, _, area, vol = oracle.tri_surface(xyz, tri)
        errs.append(4.0 * math.pi / 3.0 - vol)
    ratios = [errs[i] / errs[i + 1] for i in range(3)]
    assert all(e > 0 for e in errs)
    assert all(3.8 < r < 4.2 for r in ratios)                    # O(h^2)
    assert abs(errs[-1] - 2.27e-3) < 0.01e-3                      # SURVEY §8(c) surface pin (iii)
