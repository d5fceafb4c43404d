"""GPU parity of the P1 assembly path (a6-a17) against the CPU oracle through
the C ABI: the CSR pattern and the scatter plans bit-exact, K/M within 1e-12
relative max-norm (BASELINE.json north_star), the deterministic variant
bitwise reproducible, plus edge cases (empty mesh, isolated nodes, a single
element, rows longer than the fast-path capacity) and full-size checks of
configs 3-5 on sampled rows / faces in the launch configuration bench.py times."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2404_16039_b200 import vb

pytestmark = pytest.mark.gpu
# (mode, gather variant): row classes, 32-row blocks, element-once tiles (falls
# back to blocks outside its limits), atomic scatter
MODES = [(vb.VB_ASSEMBLE_GATHER, "class"), (vb.VB_ASSEMBLE_GATHER, "block"), (vb.VB_ASSEMBLE_GATHER, "tile"),
         (vb.VB_ASSEMBLE_ATOMIC, None)]
MODE_IDS = ["class", "block", "tile", "atomic"]


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


def mesh(kind, n, seed=0):
    if kind == "2d":
        return synth.square_p1(n, jitter=0.1, seed=seed)
    return synth.cube_kuhn_p1(n, jitter=0.05, seed=seed)


def expected_elem2nnz(elems, rp, ci):
    nv, ne = elems.shape
    out = np.empty((nv * nv, ne), dtype=np.int64)
    for a in range(nv):
        r = elems[a].astype(np.int64)
        for b in range(nv):
            c = elems[b]
            # position of c within row r of the oracle's CSR
            lo = rp[r].astype(np.int64)
            hi = rp[r + 1].astype(np.int64)
            pos = np.empty(ne, dtype=np.int64)
            for e in range(ne):
                pos[e] = lo[e] + np.searchsorted(ci[lo[e]:hi[e]], c[e])
            out[a * nv + b] = pos
    return out


# ---------------------------------------------------------------- pattern + plans
@pytest.mark.parametrize("kind,n", [("2d", 1), ("2d", 7), ("2d", 32), ("3d", 1), ("3d", 4), ("3d", 9)])
def test_pattern_and_plans_bit_exact(dev, kind, n):
    coords, elems = mesh(kind, n)
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    plan = vb.P1Plan(g(elems, dev), nn)
    assert np.array_equal(h(plan.row_ptr), rp)
    assert np.array_equal(h(plan.col_idx), ci)
    assert np.array_equal(h(plan.elem2nnz), expected_elem2nnz(elems, rp, ci))
    # gather plan: incidences of each node, ascending e, with the right slots
    nptr, nel, nsl = h(plan.node_elem_ptr), h(plan.node_elem), h(plan.node_elem_slot).view(np.uint32)
    nv = elems.shape[0]
    for v in range(0, nn, max(1, nn // 97)):
        inc = nel[nptr[v]:nptr[v + 1]]
        e, a = inc >> 2, inc & 3
        assert np.all(np.diff(e) > 0) and np.all(elems[a, e] == v)
        assert len(inc) == np.count_nonzero(elems == v)
        for k, (ee, aa) in enumerate(zip(e, a)):
            sl = nsl[nptr[v] + k]
            others = [b for b in range(nv) if b != aa]
            assert ci[rp[v] + (sl & 0xFF)] == v                          # byte 0: the diagonal
            for j, b in enumerate(others):
                assert ci[rp[v] + ((sl >> (8 * (j + 1))) & 0xFF)] == elems[b, ee]


# ---------------------------------------------------------------- assembly
@pytest.mark.parametrize("mode", MODES, ids=MODE_IDS)
@pytest.mark.parametrize("kind,n", [("2d", 1), ("2d", 32), ("2d", 50), ("3d", 1), ("3d", 6), ("3d", 11)])
def test_assembly_parity(dev, kind, n, mode):
    coords, elems = mesh(kind, n, seed=1)
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, nn)
    K, M, Kl, Ml = vb.fem_p1_assemble(cd, ed, plan, mode=mode[0], variant=mode[1], want_local=True)
    assert relmax(h(K), Ko) <= 1e-12
    assert relmax(h(M), Mo) <= 1e-12
    K3o, M3o = oracle.p1_local_all(coords, elems)
    assert relmax(h(Kl), K3o) <= 1e-12 and relmax(h(Ml), M3o) <= 1e-12


@pytest.mark.parametrize("variant", ["class", "block", "tile"])
def test_gather_variant_bitwise_reproducible(dev, variant):
    coords, elems = mesh("3d", 12, seed=2)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, coords.shape[1])
    K1, M1, _, _ = vb.fem_p1_assemble(cd, ed, plan, mode=vb.VB_ASSEMBLE_GATHER, variant=variant)
    K1, M1 = h(K1), h(M1)
    for _ in range(3):
        K2, M2, _, _ = vb.fem_p1_assemble(cd, ed, plan, mode=vb.VB_ASSEMBLE_GATHER, variant=variant)
        assert np.array_equal(h(K2), K1) and np.array_equal(h(M2), M1)


@pytest.mark.parametrize("kind,n,permute", [("3d", 1, False), ("3d", 9, False), ("3d", 9, True), ("2d", 40, False),
                                            ("delaunay2", 30, True)])
def test_tile_plan(dev, kind, n, permute):
    """fem_plan_tiles: the tiles' owned rows partition the rows; each tile holds
    exactly the elements with a vertex in it, with local ids that map back to
    the element's vertices; the slots point at the right CSR columns; the halo
    is ascending; within a color no two entries update the same (row, slot)."""
    if kind == "delaunay2":
        coords, elems = synth.delaunay_p1(2, n, seed=3)
    else:
        coords, elems = mesh(kind, n, seed=3)
    if permute:
        coords, elems = synth.permute_mesh(coords, elems, seed=6)
    nn = coords.shape[1]
    nv, ne = elems.shape
    rp, ci = oracle.p1_pattern(elems, nn)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, nn)
    assert plan.tiles(cd, ed), plan.tile_reason
    meta, nodes, rows = h(plan.tile_meta), h(plan.tile_nodes), h(plan.tile_rows)
    cols, ent = h(plan.tile_colors), h(plan.tile_elems).view(np.uint32)
    T = (nn + vb.TILE_ROWS - 1) // vb.TILE_ROWS
    assert plan.tile_stats[5] == T and plan.tile_stats[2] <= vb.TILE_NLOC
    owned = np.concatenate([nodes[t, :meta[t, 0]] for t in range(T)])
    assert np.array_equal(np.sort(owned), np.arange(nn))
    tile_of = np.empty(nn, dtype=np.int64)
    for t in range(T):
        tile_of[nodes[t, :meta[t, 0]]] = t
    total = 0
    for t in range(T):
        nown, nloc, ncol, e0 = meta[t]
        tn = nodes[t, :nloc]
        assert np.all(np.diff(tn[nown:]) > 0) and not np.any(tile_of[tn[nown:]] == t)
        for i in range(nown):
            v = tn[i]
            lo, info = rows[t, i]
            assert lo == rp[v] and (info & 0xFF) == rp[v + 1] - rp[v] and ci[lo + (info >> 8)] == v
        assert cols[t, 0] == e0
        E = ent[cols[t, 0]:cols[t, ncol]]
        total += len(E)
        loc = np.stack([E[:, 0] & 0xFFFF, E[:, 0] >> 16, E[:, 1] & 0xFFFF, E[:, 1] >> 16])[:nv]
        verts = tn[loc]                                            # (nv, entries) global vertex ids
        want = elems[:, np.any(tile_of[elems] == t, axis=0)]
        assert sorted(map(tuple, verts.T)) == sorted(map(tuple, want.T))
        sb = E[:, 2].astype(np.uint64) | (E[:, 3].astype(np.uint64) << np.uint64(32))
        for c in range(ncol):
            seen = set()
            for k in range(cols[t, c] - e0, cols[t, c + 1] - e0):
                for a in range(nv):
                    if loc[a, k] >= nown:
                        continue
                    others = [b for b in range(nv) if b != a]
                    for j, b in enumerate(others):
                        sl = int((sb[k] >> np.uint64(4 * (nv - 1) * a + 4 * j)) & np.uint64(15))
                        assert ci[rp[verts[a, k]] + sl] == verts[b, k]
                        key = (int(loc[a, k]), sl)
                        assert key not in seen
                        seen.add(key)
    assert total == plan.tile_stats[0]


@pytest.mark.parametrize("kind,n,permute", [("2d", 20, False), ("3d", 6, False), ("delaunay3", 7, True),
                                            ("delaunay2", 30, False), ("fan", 40, False)])
def test_exact_order_bitwise_equals_oracle(dev, kind, n, permute):
    """fem_p1_assemble_exact (SURVEY §8(c) bitwise mode) reproduces the oracle bit
    for bit on jittered and unstructured meshes: the same definition, the same
    operation order, IEEE round-to-nearest without contraction on both sides."""
    if kind.startswith("delaunay"):
        coords, elems = synth.delaunay_p1(int(kind[-1]), n, seed=8)
    elif kind == "fan":
        coords, elems = fan_mesh(n, 3)
    else:
        coords, elems = mesh(kind, n, seed=8)
    if permute:
        coords, elems = synth.permute_mesh(coords, elems, seed=9)
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, nn)
    K, M = vb.fem_p1_assemble_exact(cd, ed, plan)
    assert np.array_equal(h(K).view(np.uint64), Ko.view(np.uint64))
    assert np.array_equal(h(M).view(np.uint64), Mo.view(np.uint64))
    # M only, K only
    _, M2 = vb.fem_p1_assemble_exact(cd, ed, plan, want_K=False)
    K2, _ = vb.fem_p1_assemble_exact(cd, ed, plan, want_M=False)
    assert np.array_equal(h(M2), h(M)) and np.array_equal(h(K2), h(K))


def test_tile_plan_refuses_long_rows(dev):
    coords, elems = fan_mesh(40)
    plan = vb.P1Plan(g(elems, dev), coords.shape[1])
    assert not plan.tiles(g(coords, dev), g(elems, dev)) and "longer than 16" in plan.tile_reason


def test_class_rows_wider_than_the_c1_kernel(dev):
    """The crossed-diagonal square: its 9-entry vertex rows form classes (2D plan
    budget 12) that the c = 1 class kernel (8 columns) assembles in place; the
    auto choice then takes the blocks; both match the oracle."""
    coords, elems = synth.square_crossed_p1(12)
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, nn)
    plan.classes()
    assert plan.class_stats[3] == 9 and plan.class_coverage() >= 0.9
    assert not vb._use_classes(plan, None) and vb._use_classes(plan, None, coef=True)
    for variant in ("class", None):
        K, M, _, _ = vb.fem_p1_assemble(cd, ed, plan, variant=variant)
        assert relmax(h(K), Ko) <= 1e-12 and relmax(h(M), Mo) <= 1e-12


def signature(v, rp, nptr, nsl):
    return (int(rp[v + 1] - rp[v]), tuple(int(x) for x in nsl[nptr[v]:nptr[v + 1]]))


@pytest.mark.parametrize("kind,n", [("2d", 9), ("3d", 1), ("3d", 7), ("3d", 10), ("delaunay3", 6), ("crossed", 12)])
def test_row_classes_plan(dev, kind, n):
    """fem_plan_classes: class_rows is a permutation of the rows; every group is
    up to 32 rows of one class, all with the signature of the class's first
    row (row length and plan words, checked here word by word on the host);
    mixed rows are the last groups; Kuhn cubes put >= 90 % of rows in classes."""
    if kind == "delaunay3":
        coords, elems = synth.delaunay_p1(3, n, seed=0)
    elif kind == "crossed":
        coords, elems = synth.square_crossed_p1(n)
    else:
        coords, elems = mesh(kind, n)
    nn = coords.shape[1]
    plan = vb.P1Plan(g(elems, dev), nn)
    plan.classes()
    rows, groups = h(plan.class_rows)[:nn], h(plan.groups)
    assert np.array_equal(np.sort(rows), np.arange(nn))
    rp, nptr, nsl = h(plan.row_ptr), h(plan.node_elem_ptr), h(plan.node_elem_slot).view(np.uint32)
    assert groups[0, 0] == 0 and np.all(groups[1:, 0] == groups[:-1, 0] + groups[:-1, 1])
    assert groups[-1, 0] + groups[-1, 1] == nn
    assert np.all((groups[:, 1] >= 1) & (groups[:, 1] <= 32))
    seen_mixed = False
    in_classes = 0
    lmax = 0
    for pos, cnt, head, _ in groups:
        if head < 0:
            seen_mixed = True
            continue
        assert not seen_mixed                        # mixed rows come last
        ref = signature(head, rp, nptr, nsl)
        assert ref[0] <= (15 if elems.shape[0] == 4 else 12)
        lmax = max(lmax, ref[0])
        for v in rows[pos:pos + cnt]:
            assert signature(v, rp, nptr, nsl) == ref
        in_classes += cnt
    assert plan.class_stats[0] == len(groups) and plan.class_stats[2] == in_classes
    assert plan.class_stats[3] == lmax
    if kind in ("2d", "3d") and n >= 9:
        assert plan.class_coverage() >= 0.9


def test_unjittered_square_stencil_bitwise_on_gpu(dev):
    coords, elems = synth.square_p1(32, jitter=0.0)
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    Ko, _ = oracle.p1_assemble(coords, elems, rp, ci)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, nn)
    for mode in MODES:
        K, _, _, _ = vb.fem_p1_assemble(cd, ed, plan, mode=mode[0], variant=mode[1])
        assert np.array_equal(h(K), Ko)           # dyadic values: exact in any order


def test_invariants_on_gpu_output(dev):
    coords, elems = mesh("3d", 10, seed=5)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, coords.shape[1])
    K, M, _, _ = vb.fem_p1_assemble(cd, ed, plan)
    rp, ci, K, M = h(plan.row_ptr), h(plan.col_idx), h(K), h(M)
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    Kone = np.zeros(len(rp) - 1)
    np.add.at(Kone, rows, K)
    assert np.max(np.abs(Kone)) <= 1e-13 * np.max(np.abs(K))
    assert abs(math.fsum(M) - 1.0) <= 1e-13
    a = np.array([1.0, 2.0, 3.0])
    u = a @ coords
    Ku = np.zeros(len(rp) - 1)
    np.add.at(Ku, rows, K * u[ci])
    assert abs(math.fsum(u * Ku) - 14.0) <= 1e-12 * 14.0


# ---------------------------------------------------------------- edge cases
def test_empty_mesh_and_isolated_nodes(dev):
    # no elements at all
    ed = torch.zeros((4, 0), dtype=torch.int32, device=dev)
    plan = vb.P1Plan(ed, 5)
    assert plan.nnz == 0 and np.array_equal(h(plan.row_ptr), np.zeros(6, dtype=np.int32))
    cd = torch.zeros((3, 5), dtype=torch.float64, device=dev)
    for mode in MODES:
        vb.fem_p1_assemble(cd, ed, plan, mode=mode[0], variant=mode[1])
    # one element plus isolated nodes (empty rows)
    coords = np.zeros((3, 9))
    coords[:, [2, 5, 6, 8]] = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=np.float64).T
    elems = np.array([[2], [5], [6], [8]], dtype=np.int32)
    rp, ci = oracle.p1_pattern(elems, 9)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    plan = vb.P1Plan(g(elems, dev), 9)
    assert np.array_equal(h(plan.row_ptr), rp) and np.array_equal(h(plan.col_idx), ci)
    for mode in MODES:
        K, M, _, _ = vb.fem_p1_assemble(g(coords, dev), g(elems, dev), plan, mode=mode[0], variant=mode[1])
        assert relmax(h(K), Ko) <= 1e-12 and relmax(h(M), Mo) <= 1e-12


def fan_mesh(k, fans=1):
    """`fans` centre nodes (ids 0..fans-1), each surrounded by its own k-gon of
    triangles, so row c has k+1 entries.  Several fans put more than the
    shared-memory budget of CSR entries into the first CTA's row range."""
    t = 2 * np.pi * np.arange(k) / k
    nn = fans * (k + 1)
    coords = np.zeros((2, nn))
    el = []
    for f in range(fans):
        ring = fans + f * k + np.arange(k)
        coords[0, f] = 3.0 * f
        coords[0, ring] = 3.0 * f + np.cos(t)
        coords[1, ring] = np.sin(t)
        i = np.arange(k)
        el.append(np.stack([np.full(k, f), ring[i], ring[(i + 1) % k]]))
    return coords, np.ascontiguousarray(np.concatenate(el, axis=1).astype(np.int32))


@pytest.mark.parametrize("k,fans", [(100, 1), (200, 1), (200, 8)])
def test_long_rows_fallback_paths(dev, k, fans):
    """Rows longer than the 64-entry fast path (pattern fallback) and a CTA whose
    CSR range exceeds the shared-memory budget (in-place gather)."""
    coords, elems = fan_mesh(k, fans)
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    plan = vb.P1Plan(g(elems, dev), nn)
    assert np.array_equal(h(plan.row_ptr), rp) and np.array_equal(h(plan.col_idx), ci)
    for mode in MODES:
        K, M, _, _ = vb.fem_p1_assemble(g(coords, dev), g(elems, dev), plan, mode=mode[0], variant=mode[1])
        assert relmax(h(K), Ko) <= 1e-12 and relmax(h(M), Mo) <= 1e-12


def test_rows_over_255_need_the_scatter_map(dev):
    coords, elems = fan_mesh(300)
    nn = coords.shape[1]
    with pytest.raises(vb.VbError, match="255"):
        vb.P1Plan(g(elems, dev), nn)
    plan = vb.P1Plan(g(elems, dev), nn, gather_plan=False)
    rp, ci = oracle.p1_pattern(elems, nn)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    K, M, _, _ = vb.fem_p1_assemble(g(coords, dev), g(elems, dev), plan, mode=vb.VB_ASSEMBLE_ATOMIC)
    assert relmax(h(K), Ko) <= 1e-12 and relmax(h(M), Mo) <= 1e-12


# ---------------------------------------------------------------- full-size configs
def sampled_rows(nn, count=4000, seed=0):
    rng = np.random.default_rng(seed)
    mask = np.zeros(nn, dtype=np.uint8)
    mask[rng.choice(nn, size=count, replace=False)] = 1
    mask[[0, nn - 1]] = 1
    return mask


@pytest.mark.parametrize("cfg", ["config5", "config4"])
def test_full_size_assembly_every_entry(dev, cfg):
    """configs[4] (128^3 Kuhn, 12.58M tets) and configs[3] (2048^2 square,
    8.39M triangles): pattern bit-exact in full; every entry of K and of M of
    every variant against the oracle's full assembly (31.8M / 29.4M entries
    each).  Extra: the exact-order path is bitwise equal to the oracle on every
    entry."""
    if cfg == "config5":
        coords, elems = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
    else:
        coords, elems = synth.square_p1(2048, jitter=0.1, seed=0)
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, nn)
    assert np.array_equal(h(plan.row_ptr), rp)
    assert np.array_equal(h(plan.col_idx), ci)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    Kx, Mx = vb.fem_p1_assemble_exact(cd, ed, plan)
    assert np.array_equal(h(Kx).view(np.uint64), Ko.view(np.uint64))
    assert np.array_equal(h(Mx).view(np.uint64), Mo.view(np.uint64))
    del Kx, Mx
    variants = list(MODES) + ([(vb.VB_ASSEMBLE_GATHER, None)] if cfg == "config5" else [])   # None -> lattice in 3D
    for mode in variants:
        K, M, _, _ = vb.fem_p1_assemble(cd, ed, plan, mode=mode[0], variant=mode[1])
        K, M = h(K), h(M)
        assert relmax(K, Ko) <= 1e-12 and relmax(M, Mo) <= 1e-12    # every entry of both matrices
        assert abs(math.fsum(M) - 1.0) <= 1e-12                      # whole-matrix property


@pytest.mark.parametrize("level", [3, 6])
def test_surface_parity(dev, level):
    xyz, tri = synth.icosphere(level, perturb=0.01, seed=0)
    o = vb.vb_tri_surface(g(xyz, dev), g(tri, dev))
    n, nh, ar, vol = oracle.tri_surface(xyz, tri)
    assert relmax(h(o["n"]), n) <= 1e-12
    assert relmax(h(o["nhat"]), nh) <= 1e-12
    assert relmax(h(o["area"]), ar) <= 1e-12
    assert abs(h(o["volume"])[0] - vol) <= 1e-12 * abs(vol)
    o2 = vb.vb_tri_surface(g(xyz, dev), g(tri, dev))
    assert h(o2["volume"])[0] == h(o["volume"])[0]                     # fixed-shape reduction


def test_surface_full_size_config3(dev):
    """configs[2]: level-10 icosphere (20.97M faces), all faces compared."""
    xyz, tri = synth.icosphere(10, perturb=0.01, seed=0)
    o = vb.vb_tri_surface(g(xyz, dev), g(tri, dev))
    n, nh, ar, vol = oracle.tri_surface(xyz, tri)
    assert relmax(h(o["n"]), n) <= 1e-12
    assert relmax(h(o["nhat"]), nh) <= 1e-12
    assert relmax(h(o["area"]), ar) <= 1e-12
    assert abs(h(o["volume"])[0] - vol) <= 1e-12 * abs(vol)
    assert abs(vol - 4.0 * math.pi / 3.0) < 2e-3                     # near the unit ball (radii +-1%)


def test_surface_scalar_and_paired_paths_same_bits(dev):
    """An odd face count or an output plane that is not 16-byte aligned takes the one-face-per-thread
    kernel, everything else the paired 128-bit kernel: same n, nhat, area bit for bit, and each path's
    volume within 1e-12 of the oracle on its faces (an open surface is fine for the sum)."""
    xyz, tri = synth.icosphere(5, perturb=0.01, seed=1)
    nf = tri.shape[1]
    xd = g(xyz, dev)
    full = vb.vb_tri_surface(xd, g(tri, dev))                                   # paired path
    odd = np.ascontiguousarray(tri[:, :nf - 1])
    o = vb.vb_tri_surface(xd, g(odd, dev))                                      # odd count: scalar path
    n, nh, ar, vol = oracle.tri_surface(xyz, odd)
    for key in ("n", "nhat"):
        assert np.array_equal(h(o[key]), h(full[key])[:, :nf - 1])
    assert np.array_equal(h(o["area"]), h(full["area"])[:nf - 1])
    assert abs(h(o["volume"])[0] - vol) <= 1e-12 * abs(vol)
    buf = torch.full((3 * nf + 3,), 7.0, dtype=torch.float64, device=dev)       # n 8 bytes off: scalar path
    o3 = vb.vb_tri_surface(xd, g(tri, dev), out={"n": buf[1:1 + 3 * nf].view(3, nf)})
    assert np.array_equal(h(o3["n"]), h(full["n"])) and np.array_equal(h(o3["nhat"]), h(full["nhat"]))
    assert float(buf[0]) == 7.0 and float(buf[3 * nf + 1]) == 7.0
    _, _, _, vol_full = oracle.tri_surface(xyz, tri)
    assert abs(h(o3["volume"])[0] - vol_full) <= 1e-12 * abs(vol_full)
    assert abs(h(full["volume"])[0] - vol_full) <= 1e-12 * abs(vol_full)


# ---------------------------------------------------------------- unstructured meshes
@pytest.mark.parametrize("permute", [False, True])
@pytest.mark.parametrize("dim,n", [(2, 40), (3, 7), (3, 13)])
def test_delaunay_meshes_parity(dev, dim, n, permute):
    """Delaunay meshes (3D: ~30% of rows longer than the 16-column per-lane
    arrays, so staged blocks mix smem rows and in-place rows), optionally in a
    random node/element/vertex numbering."""
    coords, elems = synth.delaunay_p1(dim, n, seed=4)
    if permute:
        coords, elems = synth.permute_mesh(coords, elems, seed=5)
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    plan = vb.P1Plan(g(elems, dev), nn)
    assert np.array_equal(h(plan.row_ptr), rp) and np.array_equal(h(plan.col_idx), ci)
    assert np.array_equal(h(plan.elem2nnz), expected_elem2nnz(elems, rp, ci))
    for mode in MODES:
        K, M, _, _ = vb.fem_p1_assemble(g(coords, dev), g(elems, dev), plan, mode=mode[0], variant=mode[1])
        assert relmax(h(K), Ko) <= 1e-12 and relmax(h(M), Mo) <= 1e-12
    for cK, cM in (((2.0, (0.4, -0.3, 0.2)), (0.5, (-0.6, 0.1, 0.8))),
                   ((1.3, (0.7, 0.2, -0.5)), (1.3, (0.7, 0.2, -0.5)))):
        Ko, Mo = oracle.p1_assemble_coef(coords, elems, rp, ci, gqo=2, cK=cK, cM=cM)
        for mode in MODES:
            K, M = vb.fem_p1_assemble_coef(g(coords, dev), g(elems, dev), plan, gqo=2, cK=cK, cM=cM, mode=mode[0])[:2]
            assert relmax(h(K), Ko) <= 1e-12 and relmax(h(M), Mo) <= 1e-12


@pytest.mark.parametrize("kind,n", [("3d", 5), ("2d", 20)])
def test_fill_phase_without_count_state(dev, kind, n):
    """The fill phase reuses the count phase's lists when it gets the count
    phase's work buffer; given a different (zeroed) work buffer it rebuilds them
    and must produce identical plans."""
    import ctypes as C
    coords, elems = mesh(kind, n, seed=3)
    nn = coords.shape[1]
    ed = g(elems, dev)
    ref = vb.P1Plan(ed, nn)
    L = vb.lib()
    nv, ne = elems.shape
    sz, nnz = C.c_size_t(0), C.c_int64(0)
    vb._check(L.fem_p1_pattern(nv - 1, nn, ne, None, ne, None, C.byref(sz), None, None, 0, None, None, None, None,
                               None, None))
    w1 = torch.empty(sz.value, dtype=torch.uint8, device=dev)
    w2 = torch.zeros(sz.value, dtype=torch.uint8, device=dev)
    rp = torch.empty(nn + 1, dtype=torch.int32, device=dev)
    vb._check(L.fem_p1_pattern(nv - 1, nn, ne, vb._ptr(ed), ne, vb._ptr(w1), C.byref(sz), vb._ptr(rp), None, 0, None,
                               None, None, None, C.byref(nnz), None))
    k = int(nnz.value)
    ci = torch.zeros(k + 4, dtype=torch.int32, device=dev)
    e2n = torch.empty((nv * nv, ne), dtype=torch.int32, device=dev)
    nptr = torch.empty(nn + 1, dtype=torch.int32, device=dev)
    nel = torch.empty(nv * ne, dtype=torch.int32, device=dev)
    nsl = torch.zeros(nv * ne + 4, dtype=torch.int32, device=dev)
    vb._check(L.fem_p1_pattern(nv - 1, nn, ne, vb._ptr(ed), ne, vb._ptr(w2), C.byref(sz), vb._ptr(rp), vb._ptr(ci),
                               k + 4, vb._ptr(e2n), vb._ptr(nptr), vb._ptr(nel), vb._ptr(nsl), C.byref(nnz), None))
    assert np.array_equal(h(rp), h(ref.row_ptr)) and np.array_equal(h(ci)[:k], h(ref.col_idx))
    assert np.array_equal(h(e2n), h(ref.elem2nnz))
    assert np.array_equal(h(nptr), h(ref.node_elem_ptr)) and np.array_equal(h(nel), h(ref.node_elem))
    assert np.array_equal(h(nsl)[:nv * ne], h(ref.node_elem_slot)[:nv * ne])


@pytest.mark.parametrize("kind", ["kuhn", "kuhn-permuted", "delaunay", "fan"])
def test_gather_budgets_and_plan_stats(dev, kind):
    """fem_plan_stats reports the block maxima; the gather kernel gives the same
    bits with the wide and the compact shared-memory budget (packed 16-bit plan
    words), also for a random numbering whose blocks may exceed the compact
    budget; the packed form refuses rows of more than 16 entries."""
    if kind == "kuhn":
        coords, elems = synth.cube_kuhn_p1(9, jitter=0.05, seed=6)
    elif kind == "kuhn-permuted":
        coords, elems = synth.permute_mesh(*synth.cube_kuhn_p1(9, jitter=0.05, seed=6), seed=7)
    elif kind == "delaunay":
        coords, elems = synth.delaunay_p1(3, 9, seed=6)
    else:
        coords, elems = fan_mesh(40, fans=3)
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    plan = vb.P1Plan(g(elems, dev), nn)
    L = np.diff(rp)
    nptr = h(plan.node_elem_ptr)
    nb = (nn + 31) // 32
    blk = [min(32 * (b + 1), nn) for b in range(nb)]
    exp = (int(L.max()), max(int(rp[e] - rp[32 * b]) for b, e in enumerate(blk)),
           max(int(nptr[e] - nptr[32 * b]) for b, e in enumerate(blk)))
    assert plan.stats == exp
    if kind == "kuhn":
        assert plan.compact
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    cd, ed = g(coords, dev), g(elems, dev)
    if L.max() > 16:
        assert not plan.compact
        with pytest.raises(vb.VbError, match="16"):
            plan.pack_slots()
        budgets = (False,)
    else:
        budgets = (False, True)
    out = []
    for compact in budgets:
        K, M, _, _ = vb.fem_p1_assemble(cd, ed, plan, compact=compact, variant="block")
        K, M = h(K), h(M)
        assert relmax(K, Ko) <= 1e-12 and relmax(M, Mo) <= 1e-12
        out.append((K, M))
        cf = (1.3, (0.7, 0.2, -0.5))
        Kc, Mc, _, _ = vb.fem_p1_assemble_coef(cd, ed, plan, gqo=2, cK=cf, cM=cf, compact=compact, variant="block")
        Kco, Mco = oracle.p1_assemble_coef(coords, elems, rp, ci, gqo=2, cK=cf, cM=cf)
        assert relmax(h(Kc), Kco) <= 1e-12 and relmax(h(Mc), Mco) <= 1e-12
    for K, M in out[1:]:
        assert np.array_equal(out[0][0], K) and np.array_equal(out[0][1], M)


@pytest.mark.parametrize("layout", ["aos", "aos4", "wide_elems"])
def test_strided_coords_and_elem_ld_through_the_abi(dev, layout):
    """The C ABI's strided addressing: coords[c*comp_stride + v*node_stride]
    (AoS: stride dim; padded AoS: stride 4) and elems[a*elem_ld + e] with
    elem_ld > ne, in both assembly variants, against the SoA result."""
    import ctypes as C
    coords, elems = synth.cube_kuhn_p1(6, jitter=0.05, seed=8)
    dim, nn = coords.shape
    nv, ne = elems.shape
    rp, ci = oracle.p1_pattern(elems, nn)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    plan = vb.P1Plan(g(elems, dev), nn)
    node_stride, comp_stride, eld = 1, nn, ne
    if layout == "aos":
        cbuf = g(np.ascontiguousarray(coords.T), dev)                         # (nn, 3)
        node_stride, comp_stride = dim, 1
    elif layout == "aos4":
        pad = np.zeros((nn, 4))
        pad[:, :dim] = coords.T
        cbuf = g(pad, dev)
        node_stride, comp_stride = 4, 1
    else:
        cbuf = g(coords, dev)
    if layout == "wide_elems":
        eld = ne + 37
        wide = np.full((nv, eld), -1, dtype=np.int32)
        wide[:, :ne] = elems
        ebuf = g(wide, dev)
    else:
        ebuf = g(elems, dev)
    L = vb.lib()
    for mode in (vb.VB_ASSEMBLE_GATHER, vb.VB_ASSEMBLE_ATOMIC):
        K = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
        M = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
        vb._check(L.fem_p1_assemble(dim, nn, ne, vb._ptr(cbuf), node_stride, comp_stride, vb._ptr(ebuf), eld,
                                    vb._ptr(plan.row_ptr), vb._ptr(plan.col_idx), plan.nnz, vb._ptr(plan.elem2nnz),
                                    vb._ptr(plan.node_elem_ptr), vb._ptr(plan.node_elem),
                                    vb._ptr(plan.node_elem_slot), vb._ptr(K), vb._ptr(M), None, None, mode,
                                    vb._ptr(vb._work16(dev)), vb._wb(), None, None))
        assert relmax(h(K), Ko) <= 1e-12 and relmax(h(M), Mo) <= 1e-12
    # the class variant with the same strided coordinates
    plan.classes()
    K = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
    M = torch.empty(plan.nnz, dtype=torch.float64, device=dev)
    vb._check(L.fem_p1_assemble_classes(dim, nn, vb._ptr(cbuf), node_stride, comp_stride, vb._ptr(plan.row_ptr),
                                        vb._ptr(plan.col_idx), plan.nnz, vb._ptr(plan.node_elem_ptr),
                                        vb._ptr(plan.node_elem_slot), vb._ptr(plan.class_rows), vb._ptr(plan.groups),
                                        plan.groups.shape[0], vb._ptr(K), vb._ptr(M), vb._ptr(vb._work16(dev)),
                                        vb._wb(), None))
    assert relmax(h(K), Ko) <= 1e-12 and relmax(h(M), Mo) <= 1e-12
    # the class coefficient path (its per-node factor pass reads the strided coordinates too)
    cb = (C.c_double * 3)(0.7, -0.4, 0.9)
    Kco, Mco = oracle.p1_assemble_coef(coords, elems, rp, ci, gqo=2, cK=(1.3, (0.7, -0.4, 0.9)),
                                       cM=(1.3, (0.7, -0.4, 0.9)))
    work = torch.empty(2 * nn + 2, dtype=torch.float64, device=dev)   # factors + the group counter
    vb._check(L.fem_p1_assemble_classes_coef(dim, nn, vb._ptr(cbuf), node_stride, comp_stride, vb._ptr(plan.row_ptr),
                                             vb._ptr(plan.col_idx), plan.nnz, vb._ptr(plan.node_elem_ptr),
                                             vb._ptr(plan.node_elem_slot), vb._ptr(plan.class_rows),
                                             vb._ptr(plan.groups), plan.groups.shape[0], 2, 1.3, C.cast(cb, C.c_void_p),
                                             vb._ptr(work), vb._ptr(K), vb._ptr(M), None))
    assert relmax(h(K), Kco) <= 1e-12 and relmax(h(M), Mco) <= 1e-12
    # the lattice variant with the same strided coordinates
    lp = vb.P1Plan(g(elems, dev), nn, scatter_map=False, gather_plan=False)
    assert lp.lattice(g(elems, dev))
    vb._check(L.fem_p1_assemble_lattice(nn, vb._ptr(cbuf), node_stride, comp_stride, vb._ptr(lp.row_ptr), lp.nnz,
                                        vb._ptr(lp.lattice_plan), 6, 6, 6, lp.lattice_flips, vb._ptr(K), vb._ptr(M),
                                        None, None))
    assert relmax(h(K), Ko) <= 1e-12 and relmax(h(M), Mo) <= 1e-12


@pytest.mark.parametrize("mode", MODES, ids=MODE_IDS)
@pytest.mark.parametrize("kind", ["2d", "3d"])
def test_k_only_and_m_only(dev, kind, mode):
    """One matrix requested (the other pointer NULL) through every variant, c = 1
    and, in gather mode, the coefficient path (row classes where they apply)."""
    coords, elems = mesh(kind, 7, seed=5)
    nn = coords.shape[1]
    rp, ci = oracle.p1_pattern(elems, nn)
    Ko, Mo = oracle.p1_assemble(coords, elems, rp, ci)
    cf = (1.1, (0.3, -0.6, 0.5))
    Kc, Mc = oracle.p1_assemble_coef(coords, elems, rp, ci, gqo=2, cK=cf, cM=cf)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, nn)
    K, M, _, _ = vb.fem_p1_assemble(cd, ed, plan, mode=mode[0], variant=mode[1], want_M=False)
    assert M is None and relmax(h(K), Ko) <= 1e-12
    K, M, _, _ = vb.fem_p1_assemble(cd, ed, plan, mode=mode[0], variant=mode[1], want_K=False)
    assert K is None and relmax(h(M), Mo) <= 1e-12
    if mode[1] != "tile":
        K, M, _, _ = vb.fem_p1_assemble_coef(cd, ed, plan, gqo=2, cK=cf, cM=cf, mode=mode[0], variant=mode[1],
                                             want_M=False)
        assert M is None and relmax(h(K), Kc) <= 1e-12
        K, M, _, _ = vb.fem_p1_assemble_coef(cd, ed, plan, gqo=2, cK=cf, cM=cf, mode=mode[0], variant=mode[1],
                                             want_K=False)
        assert K is None and relmax(h(M), Mc) <= 1e-12


# ---------------------------------------------------------------- ABI v2 conventions
def test_pattern_validation_mode_names_the_bad_vertex(dev):
    """fem_p1_pattern with VB_PATTERN_VALIDATE: an out-of-range vertex id is VB_ERR_ARG naming the first
    offending element and vertex (before any kernel indexes by it); valid meshes build as usual."""
    coords, elems = synth.cube_kuhn_p1(5, jitter=0.05, seed=0)
    nn = coords.shape[1]
    ok = vb.P1Plan(g(elems, dev), nn, validate=True)
    rp, ci = oracle.p1_pattern(elems, nn)
    assert np.array_equal(h(ok.row_ptr), rp) and np.array_equal(h(ok.col_idx), ci)
    for e_bad, a_bad, val in ((137, 2, nn), (22, 0, -1), (elems.shape[1] - 1, 3, nn + 5)):
        bad = elems.copy()
        bad[a_bad, e_bad] = val
        with pytest.raises(vb.VbError) as ei:
            vb.P1Plan(g(bad, dev), nn, validate=True)
        msg = str(ei.value)
        assert "VB_ERR_ARG" in msg and "vertex %d of element %d" % (a_bad, e_bad) in msg and str(val) in msg


@pytest.mark.parametrize("variant", ["class", "block", "lattice"])
def test_many_concurrent_launches_on_two_streams(dev, variant):
    """More than 64 assembly launches in flight on two streams (each with its own caller-owned work buffer
    for the dynamic block schedule): every result bitwise equal to a serial run -- the library keeps no
    per-launch state of its own (round 1's global counter ring could be reset by another launch)."""
    coords, elems = synth.cube_kuhn_p1(20, jitter=0.05, seed=1)
    cd, ed = g(coords, dev), g(elems, dev)
    plan = vb.P1Plan(ed, coords.shape[1])
    if variant == "lattice":
        assert plan.lattice(ed)
    else:
        plan.classes()
    Kr, Mr, _, _ = vb.fem_p1_assemble(cd, ed, plan, variant=variant)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    outs = []
    n = 80
    for i in range(n):
        for s in streams:
            with torch.cuda.stream(s):
                K = torch.full((plan.nnz,), float("nan"), dtype=torch.float64, device=dev)
                M = torch.full((plan.nnz,), float("nan"), dtype=torch.float64, device=dev)
                vb.fem_p1_assemble(cd, ed, plan, K=K, M=M, variant=variant)
                outs.append((K, M))
    torch.cuda.synchronize()
    assert len(outs) == 2 * n
    for K, M in outs:
        assert torch.equal(K, Kr) and torch.equal(M, Mr)
