"""GPU GI (Code GI; NEXT-4 volume and surface integrals P:717-899):
parity with the oracle on random page batches, and the paper's volume-integral
pipeline (create_coords3D -> amsm -> rho -> GI, Code volume_integral) and a
surface flux on the GPU against closed forms, up to the configs[4] / configs[2]
sizes."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2404_16039_b200 import vb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    return torch.device("cuda:0")


def g(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


@pytest.mark.parametrize("d,nip,N", [(1, 1, 1), (1, 4, 1000), (3, 1, 777), (3, 11, 5000), (2, 3, 200003), (1, 16, 7)])
def test_gi_parity(dev, d, nip, N):
    rng = np.random.default_rng(d * 100 + nip)
    fip = rng.standard_normal((nip, d, N))
    w = rng.random(nip)
    sz = rng.random(N)
    nrm = rng.standard_normal((d, N)) if d > 1 or nip == 4 else None
    ref = oracle.gi(fip, w, sz, normals=nrm)
    scale = float(np.sum(sz * np.abs(fip).sum(axis=(0, 1))) * max(1.0, np.abs(nrm).max() if nrm is not None else 1.0))
    val, work = vb.vb_gi(g(fip, dev), w, g(sz, dev), normals=g(nrm, dev) if nrm is not None else None)
    got = val.item()
    assert abs(got - ref) <= 1e-13 * scale
    val2, _ = vb.vb_gi(g(fip, dev), w, g(sz, dev), normals=g(nrm, dev) if nrm is not None else None, work=work)
    assert val2.item() == got                                    # fixed-shape reduction


def test_gi_errors(dev):
    fip = torch.zeros((2, 3, 10), dtype=torch.float64, device=dev)
    with pytest.raises(vb.VbError, match="normals"):
        vb.vb_gi(fip, [0.5, 0.5], torch.ones(10, dtype=torch.float64, device=dev))
    val, _ = vb.vb_gi(torch.zeros((1, 1, 0), dtype=torch.float64, device=dev), [1.0],
                      torch.zeros(0, dtype=torch.float64, device=dev))
    assert val.item() == 0.0


def volume_integral(dev, coords, elems, rho, gqo=2):
    """Code volume_integral on the GPU: coords3D, X_ip = amsm(coords3D, ip),
    rho(X_ip) (the user's function, torch elementwise), sizes = |amdet(vectors3D)| / d!, GI."""
    dim = coords.shape[0]
    lam, w = oracle.quad_rule(dim, gqo)
    ip = torch.from_numpy(np.ascontiguousarray(np.asarray(lam)[:, :, None])).to(dev)   # (nip, nv, 1): nv x nip page
    c3, v3 = vb.vb_create_coords3D(g(coords, dev), g(elems, dev))
    Xip = vb.vb_page_mtimes(c3, ip)                                # (nip, dim, ne)
    sizes = vb.vb_page_det(v3).abs_() / math.factorial(dim)
    fip = rho(Xip).unsqueeze(1).contiguous()                       # (nip, 1, ne)
    val, _ = vb.vb_gi(fip, np.asarray(w) * math.factorial(dim), sizes)
    return val.item()


@pytest.mark.parametrize("n", [6, 128])
def test_volume_integral_pipeline(dev, n):
    """rho = x1^2 + x2^2 over the unit cube: 2/3 exactly for the degree-2
    rule, on a jittered Kuhn cube up to the configs[4] mesh (12.58M tets)."""
    c, e = synth.cube_kuhn_p1(n, jitter=0.05, seed=0)
    val = volume_integral(dev, c, e, lambda X: X[:, 0] ** 2 + X[:, 1] ** 2)
    assert abs(val - 2.0 / 3.0) <= 1e-12
    if n == 6:
        ref = oracle.gi(*_oracle_inputs(c, e))
        assert abs(val - ref) <= 1e-13


def _oracle_inputs(c, e):
    lam, w = oracle.quad_rule(3, 2)
    X = c[:, e]
    Xq = np.einsum("qa,cae->qce", np.asarray(lam), X)
    J = np.stack([X[:, r + 1] - X[:, 0] for r in range(3)])
    sizes = np.abs(np.linalg.det(np.moveaxis(J, -1, 0))) / 6.0
    return (Xq[:, 0] ** 2 + Xq[:, 1] ** 2)[:, None, :], np.asarray(w) * 6.0, sizes


@pytest.mark.parametrize("level", [3, 10])
def test_surface_flux_pipeline(dev, level):
    """Flux of F = x/3 through the perturbed icosphere with the outer unit normals
    and areas of vb_tri_surface and the centroid rule: the enclosed volume (the
    same surface's divergence-theorem volume), up to the configs[2] mesh."""
    xyz, tri = synth.icosphere(level, perturb=0.01, seed=0)
    xd, td = g(xyz, dev), g(tri, dev)
    o = vb.vb_tri_surface(xd, td)
    c3, _ = vb.vb_create_coords3D(xd, td, want_vectors3D=False)   # (3, 3, F): vertices of each face
    third = torch.full((1, 3, 1), 1.0 / 9.0, dtype=torch.float64, device=dev)   # centroid / 3
    fip = vb.vb_page_mtimes(c3, third)                            # (1, 3, F): F(centroid) = centroid / 3
    val, _ = vb.vb_gi(fip, [1.0], o["area"], normals=o["nhat"])
    vol = o["volume"].item()
    assert abs(val.item() - vol) <= 1e-12 * abs(vol)
