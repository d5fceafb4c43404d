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
