"""Synthetic meshes with the shapes of the paper's workloads (no method arithmetic).

Recipes (BASELINE.json configs; restated in DESIGN.md):

* ``square_p1(n)`` -- unit square, n x n cells, node id = i + (n+1) j at
  (i/n, j/n); cell (i, j) taken x-fastest, split along the SW-NE diagonal into
  (v00, v10, v11) and (v00, v11, v01) (counter-clockwise).  Configs 1 and 4
  (P:1082-1096 use unit-square meshes).
* ``cube_kuhn_p1(n)`` -- unit cube, n^3 cells, node id = i + (n+1)(j + (n+1)k);
  cell x-fastest; 6 Kuhn tetrahedra per cell, one per axis permutation p in
  lexicographic order: v0, v0+e_p0, v0+e_p0+e_p1, v0+(1,1,1).  Config 5; the
  node counts (2^L+1)^3 match P:1113-1125.
* jitter: one U[-1,1) draw per node and coordinate (stream 1, index
  v*dim + c, node-id order, drawn for every node) scaled by amp*h and applied
  to interior nodes only, so the domain stays the exact unit square / cube.
* ``icosphere(level)`` -- the 12-vertex icosahedron normalised to r = 1,
  ``level`` rounds of 1 -> 4 midpoint subdivision (midpoints re-normalised to
  r = 1 every round, new vertex ids in order of first creation while scanning
  faces in order and edges (a,b), (b,c), (c,a)), then radius 1 + amp*U[-1,1)
  per vertex (stream 2).  Config 3.
"""
import numpy as np

from .rng import uniform_pm1

JITTER_STREAM = 1
RADIUS_STREAM = 2


def square_counts(n):
    nn = (n + 1) ** 2
    ne = 2 * n * n
    return nn, ne


def cube_counts(n):
    nn = (n + 1) ** 3
    ne = 6 * n ** 3
    return nn, ne


def icosphere_counts(level):
    f = 20 * 4 ** level
    v = 10 * 4 ** level + 2
    return v, f


def _interior_mask(idx_per_axis, n):
    m = np.ones(idx_per_axis[0].shape, dtype=bool)
    for ia in idx_per_axis:
        m &= (ia > 0) & (ia < n)
    return m


def square_p1(n, jitter=0.1, seed=0):
    """Return (coords (2, nn) float64, elems (3, ne) int32)."""
    n1 = n + 1
    v = np.arange(n1 * n1, dtype=np.int64)
    i = v % n1
    j = v // n1
    coords = np.empty((2, n1 * n1), dtype=np.float64)
    coords[0] = i / n
    coords[1] = j / n
    if jitter:
        r = uniform_pm1(seed, JITTER_STREAM, 2 * n1 * n1).reshape(n1 * n1, 2)
        inner = _interior_mask((i, j), n)
        h = 1.0 / n
        coords[0, inner] += jitter * h * r[inner, 0]
        coords[1, inner] += jitter * h * r[inner, 1]
    c = np.arange(n * n, dtype=np.int64)
    ci = c % n
    cj = c // n
    v00 = ci + n1 * cj
    v10 = v00 + 1
    v01 = v00 + n1
    v11 = v01 + 1
    elems = np.empty((3, 2 * n * n), dtype=np.int32)
    elems[:, 0::2] = np.stack([v00, v10, v11])
    elems[:, 1::2] = np.stack([v00, v11, v01])
    return coords, elems


def rect_p1(nx, ny, jitter=0.1, seed=0, flip=0):
    """square_p1's recipe on nx x ny cells of side h = 1/max(nx, ny): node id = i + (nx+1) j, cells x-fastest, two
    triangles per cell along the diagonal (0,0)-(1,1) (flip = 0: (v00, v10, v11), (v00, v11, v01)) or
    (1,0)-(0,1) (flip = 1: (v00, v10, v01), (v10, v11, v01)); interior nodes jittered by jitter * h."""
    m = max(nx, ny)
    nx1 = nx + 1
    nn = nx1 * (ny + 1)
    v = np.arange(nn, dtype=np.int64)
    i, j = v % nx1, v // nx1
    coords = np.empty((2, nn), dtype=np.float64)
    coords[0], coords[1] = i / m, j / m
    if jitter:
        r = uniform_pm1(seed, JITTER_STREAM, 2 * nn).reshape(nn, 2)
        inner = (i > 0) & (i < nx) & (j > 0) & (j < ny)
        coords[0, inner] += jitter / m * r[inner, 0]
        coords[1, inner] += jitter / m * r[inner, 1]
    c = np.arange(nx * ny, dtype=np.int64)
    v00 = c % nx + nx1 * (c // nx)
    v10, v01 = v00 + 1, v00 + nx1
    v11 = v01 + 1
    elems = np.empty((3, 2 * nx * ny), dtype=np.int32)
    if flip:
        elems[:, 0::2] = np.stack([v00, v10, v01])
        elems[:, 1::2] = np.stack([v10, v11, v01])
    else:
        elems[:, 0::2] = np.stack([v00, v10, v11])
        elems[:, 1::2] = np.stack([v00, v11, v01])
    return coords, elems


_KUHN_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def cube_kuhn_p1(n, jitter=0.05, seed=0, flip=(0, 0, 0)):
    """Return (coords (3, nn) float64, elems (4, ne) int32).

    ``flip`` picks the cell diagonal shared by the 6 Kuhn tets: axis d is walked
    from the cell's far side when flip[d] = 1.  flip = (0, 0, 0) is the
    (0,0,0)-(1,1,1) diagonal of BASELINE configs[4]; flip = (0, 0, 1) (the
    (0,0,1)-(1,1,0) diagonal) reproduces the error columns of the paper's 3D P1
    table (tab:KM_P1_3D) -- see tests/golden/paper_tables_p1.json."""
    return box_kuhn_p1(n, n, n, jitter=jitter, seed=seed, flip=flip)


def box_kuhn_p1(nx, ny, nz, jitter=0.05, seed=0, flip=(0, 0, 0)):
    """cube_kuhn_p1 on the box [0, nx/m] x [0, ny/m] x [0, nz/m], m = max(nx, ny, nz)
    (cells of side h = 1/m): node id = i + (nx+1)(j + (ny+1)k), cells x-fastest,
    6 Kuhn tets per cell in lexicographic path order, the same jitter recipe
    (one draw per node and coordinate in id order, interior nodes only)."""
    nx1, ny1, nz1 = nx + 1, ny + 1, nz + 1
    nn = nx1 * ny1 * nz1
    m = max(nx, ny, nz)
    v = np.arange(nn, dtype=np.int64)
    i = v % nx1
    j = (v // nx1) % ny1
    k = v // (nx1 * ny1)
    coords = np.empty((3, nn), dtype=np.float64)
    coords[0] = i / m
    coords[1] = j / m
    coords[2] = k / m
    if jitter:
        r = uniform_pm1(seed, JITTER_STREAM, 3 * nn).reshape(nn, 3)
        inner = (i > 0) & (i < nx) & (j > 0) & (j < ny) & (k > 0) & (k < nz)
        h = 1.0 / m
        for c in range(3):
            coords[c, inner] += jitter * h * r[inner, c]
    c = np.arange(nx * ny * nz, dtype=np.int64)
    ci = c % nx
    cj = (c // nx) % ny
    ck = c // (nx * ny)
    fl = [int(bool(f)) for f in flip]
    v0 = (ci + fl[0]) + nx1 * ((cj + fl[1]) + ny1 * (ck + fl[2]))
    step = (1 - 2 * fl[0], nx1 * (1 - 2 * fl[1]), nx1 * ny1 * (1 - 2 * fl[2]))
    elems = np.empty((4, 6 * nx * ny * nz), dtype=np.int32)
    for t, p in enumerate(_KUHN_PERMS):
        a1 = v0 + step[p[0]]
        a2 = a1 + step[p[1]]
        a3 = a2 + step[p[2]]
        elems[:, t::6] = np.stack([v0, a1, a2, a3])
    return coords, elems


def square_crossed_p1(n):
    """Unit square, n x n cells, each split into 4 triangles by its centre node
    (the paper's 2D meshes: (n+1)^2 + n^2 nodes).  Corner node id
    i + (n+1) j at (i/n, j/n); centre of cell (i, j) (x-fastest) has id
    (n+1)^2 + i + n j; cell triangles (v00, v10, m), (v10, v11, m), (v11, v01, m),
    (v01, v00, m) in that order.  Returns (coords (2, nn), elems (3, 4n^2))."""
    n1 = n + 1
    v = np.arange(n1 * n1, dtype=np.int64)
    c = np.arange(n * n, dtype=np.int64)
    ci, cj = c % n, c // n
    coords = np.concatenate([np.stack([(v % n1) / n, (v // n1) / n]),
                             np.stack([(ci + 0.5) / n, (cj + 0.5) / n])], axis=1)
    v00 = ci + n1 * cj
    v10, v01 = v00 + 1, v00 + n1
    v11 = v01 + 1
    m = n1 * n1 + c
    elems = np.empty((3, 4 * n * n), dtype=np.int32)
    for t, (a, b) in enumerate(((v00, v10), (v10, v11), (v11, v01), (v01, v00))):
        elems[:, t::4] = np.stack([a, b, m])
    return coords, elems


P2_EDGES = {2: ((0, 1), (1, 2), (0, 2)),
            3: ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))}


def p2_from_p1(coords, elems):
    """P2 mesh from a P1 mesh (the paper's "additional vertices located at the
    midpoints of the edges"): midpoint nodes appended after the
    vertices, ids in order of first creation scanning elements in order and each
    element's edges in the canonical order P2_EDGES (2D edges
    (1,2),(2,3),(1,3) -> local nodes 4,5,6; 3D (1,2),(1,3),(1,4),(2,3),(2,4),(3,4)
    -> 5..10).  Returns (coords (dim, nn + n_edges), elems (nlb, ne) int32)."""
    dim, nn = coords.shape
    pairs = P2_EDGES[dim]
    e64 = elems.astype(np.int64)
    E = np.stack([np.stack([e64[a], e64[b]], 1) for a, b in pairs], 1).reshape(-1, 2)
    key = np.minimum(E[:, 0], E[:, 1]) * nn + np.maximum(E[:, 0], E[:, 1])
    _, first, inv = np.unique(key, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    mid = nn + rank[inv].reshape(-1, len(pairs))
    ue = E[first[order]]
    coords2 = np.concatenate([coords, 0.5 * (coords[:, ue[:, 0]] + coords[:, ue[:, 1]])], axis=1)
    elems2 = np.concatenate([elems, mid.T.astype(np.int32)], axis=0)
    return np.ascontiguousarray(coords2), np.ascontiguousarray(elems2)


_PHI = (1.0 + 5.0 ** 0.5) / 2.0
_ICO_V = np.array([
    [-1, _PHI, 0], [1, _PHI, 0], [-1, -_PHI, 0], [1, -_PHI, 0],
    [0, -1, _PHI], [0, 1, _PHI], [0, -1, -_PHI], [0, 1, -_PHI],
    [_PHI, 0, -1], [_PHI, 0, 1], [-_PHI, 0, -1], [-_PHI, 0, 1]], dtype=np.float64)
_ICO_F = np.array([
    [0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
    [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
    [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
    [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)


def _normalise_rows(x):
    return x / np.sqrt((x * x).sum(axis=1, keepdims=True))


def icosphere(level, perturb=0.01, seed=0):
    """Return (xyz (3, V) float64, tri (3, F) int32)."""
    verts = _normalise_rows(_ICO_V.copy())
    faces = _ICO_F.copy()
    for _ in range(level):
        nv = verts.shape[0]
        a, b, c = faces[:, 0], faces[:, 1], faces[:, 2]
        e = np.stack([np.stack([a, b], 1), np.stack([b, c], 1), np.stack([c, a], 1)], 1).reshape(-1, 2)
        key = np.minimum(e[:, 0], e[:, 1]) * nv + np.maximum(e[:, 0], e[:, 1])
        uniq, first, inv = np.unique(key, return_index=True, return_inverse=True)
        order = np.argsort(first, kind="stable")          # unique edges by first creation
        rank = np.empty_like(order)
        rank[order] = np.arange(order.size)
        mid_id = nv + rank[inv]                           # id of midpoint of each face edge
        ue = e[first[order]]
        mids = _normalise_rows(0.5 * (verts[ue[:, 0]] + verts[ue[:, 1]]))
        verts = np.concatenate([verts, mids], 0)
        m = mid_id.reshape(-1, 3)
        ab, bc, ca = m[:, 0], m[:, 1], m[:, 2]
        faces = np.stack([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
                          np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)], 1).reshape(-1, 3)
    if perturb:
        r = 1.0 + perturb * uniform_pm1(seed, RADIUS_STREAM, verts.shape[0])
        verts = verts * r[:, None]
    xyz = np.ascontiguousarray(verts.T)
    tri = np.ascontiguousarray(faces.T.astype(np.int32))
    return xyz, tri


DELAUNAY_STREAM = 3
PERMUTE_STREAM = 4


def delaunay_p1(dim, n, jitter=0.35, seed=0):
    """Unstructured P1 mesh: the (n+1)^dim grid of the unit square / cube with
    every node moved by jitter*h*U[-1,1) per coordinate (stream 3, boundary
    nodes kept on their faces), triangulated by scipy's Delaunay (Qhull).  Row
    lengths then follow the Delaunay degree distribution (3D: mean ~15.5, many
    rows above 16) instead of the fixed Kuhn/square stencils."""
    from scipy.spatial import Delaunay

    n1 = n + 1
    axes = np.meshgrid(*([np.arange(n1)] * dim), indexing="ij")
    idx = np.stack([a.ravel(order="F") for a in axes])          # x fastest
    nn = idx.shape[1]
    d = uniform_pm1(seed, DELAUNAY_STREAM, nn * dim).reshape(nn, dim).T
    inner = (idx > 0) & (idx < n)                               # per coordinate
    coords = (idx + np.where(inner, jitter * d, 0.0)) / n
    tri = Delaunay(coords.T, qhull_options="Qbb Qc Qz Q12" if dim == 3 else "Qbb Qc Qz")
    elems = np.ascontiguousarray(tri.simplices.T.astype(np.int32))
    return np.ascontiguousarray(coords), elems


def permute_mesh(coords, elems, seed=0):
    """Relabel nodes, reorder elements and rotate each element's vertex list by
    seeded random permutations (stream 4): the same mesh in another numbering,
    so nothing may rely on the generators' locality or ordering."""
    nv, ne = elems.shape
    nn = coords.shape[1]
    keys = uniform_pm1(seed, PERMUTE_STREAM, nn + ne + ne)
    new_of_old = np.empty(nn, dtype=np.int64)
    new_of_old[np.argsort(keys[:nn], kind="stable")] = np.arange(nn)
    c2 = np.empty_like(coords)
    c2[:, new_of_old] = coords
    order = np.argsort(keys[nn:nn + ne], kind="stable")
    rot = (np.floor((keys[nn + ne:] + 1.0) * 0.5 * nv).astype(np.int64) % nv)[order]
    e2 = new_of_old[elems[:, order]]
    rows = (np.arange(nv)[:, None] + rot[None, :]) % nv
    e2 = np.take_along_axis(e2, rows, axis=0)
    return np.ascontiguousarray(c2), np.ascontiguousarray(e2.astype(np.int32))
