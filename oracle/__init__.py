"""ctypes wrapper of the plain C oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2404_16039_b200`` (neither imports
the other).  Arrays are numpy, in the same SoA layouts as include/vb.h.

Functions with no independent pin are listed in DESIGN.md §Oracle; at the
time of writing every function here is pinned (tests/test_oracle_*.py).
"""
import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-shared", "-fPIC"]


def build(force=False):
    """Compile oracle.c with gcc (no GPU needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        i64, i32, d, p = C.c_int64, C.c_int, C.c_double, C.c_void_p
        sig = {
            "orc_page_mtimes": (i32, [i64, p, i32, i32, i64, i32, p, i32, i32, i64, i32, p, i64]),
            "orc_page_transpose": (i32, [i64, p, i32, i32, i64, p, i64]),
            "orc_page_det": (i32, [i64, i32, p, i64, p]),
            "orc_page_inv": (i32, [i64, i32, p, i64, p, i64, p]),
            "orc_page_cross": (i32, [i64, p, i64, p, i64, p, i64]),
            "orc_create_coords3D": (i32, [i32, i32, i64, p, i64, i64, p, i64, p, p]),
            "orc_tri_surface": (i32, [i64, p, i64, p, i64, i64, p, p, p, p]),
            "orc_p1_local": (None, [i32, p, p, p]),
            "orc_p1_local_all": (i32, [i32, i64, p, i64, i64, p, i64, p, p]),
            "orc_p1_pattern": (i64, [i32, i64, i64, p, i64, p, p]),
            "orc_p1_assemble": (i32, [i32, i64, i64, p, i64, i64, p, i64, p, p, p, p, p]),
            "orc_quad_rule": (i32, [i32, i32, p, p]),
            "orc_p1_local_coef": (i32, [i32, p, i32, d, p, d, p, p, p]),
            "orc_p1_assemble_coef": (i32, [i32, i64, i64, p, i64, i64, p, i64, p, p, i32, d, p, d, p, p, p]),
            "orc_page_bilinear": (i32, [i64, i32, i32, p, i64, p, i64, p, i64, p]),
            "orc_p1_rhs": (i32, [i32, i64, i64, p, i64, i64, p, i64, i32, p, p, p]),
            "orc_pattern": (i64, [i32, i64, i64, p, i64, p, p]),
            "orc_p2_local_coef": (i32, [i32, p, i32, d, p, d, p, p, p]),
            "orc_gi": (i32, [i64, i32, i32, p, i64, p, p, p, i64, p]),
            "orc_p2_assemble_coef": (i32, [i32, i64, i64, p, i64, i64, p, i64, p, p, i32, d, p, d, p, p, p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _check(rc, what):
    if rc != 0:
        raise ValueError("oracle %s failed with status %d" % (what, rc))


# ------------------------------------------------------------------ pages
def page_mtimes(X, Y, tX=False, tY=False, npages=None):
    """Z_k = op(X_k) op(Y_k).  X: (xc, xr, N) or (xc, xr, 1) broadcast (ld=0)."""
    X, Y = _f64(X), _f64(Y)
    xc, xr, nx = X.shape
    yc, yr, ny = Y.shape
    n = npages if npages is not None else max(nx, ny)
    m = xc if tX else xr
    q = yr if tY else yc
    Z = np.empty((q, m, n))
    ldx = 0 if nx == 1 and n != 1 else nx
    ldy = 0 if ny == 1 and n != 1 else ny
    _check(lib().orc_page_mtimes(n, _p(X), xr, xc, ldx, int(tX), _p(Y), yr, yc, ldy, int(tY), _p(Z), n), "mtimes")
    return Z


def page_transpose(X):
    X = _f64(X)
    c, r, n = X.shape
    Z = np.empty((r, c, n))
    _check(lib().orc_page_transpose(n, _p(X), r, c, n, _p(Z), n), "transpose")
    return Z


def page_det(X):
    X = _f64(X)
    n, n2, N = X.shape
    assert n == n2
    d = np.empty(N)
    _check(lib().orc_page_det(N, n, _p(X), N, _p(d)), "det")
    return d


def page_inv(X):
    """Returns (inverse pages, determinants)."""
    X = _f64(X)
    n, n2, N = X.shape
    assert n == n2
    Z = np.empty_like(X)
    d = np.empty(N)
    _check(lib().orc_page_inv(N, n, _p(X), N, _p(Z), N, _p(d)), "inv")
    return Z, d


def page_cross(A, B):
    A, B = _f64(A), _f64(B)
    assert A.shape[:2] == (1, 3) and B.shape[:2] == (1, 3)
    N = A.shape[2]
    Cc = np.empty((1, 3, N))
    _check(lib().orc_page_cross(N, _p(A), N, _p(B), N, _p(Cc), N), "cross")
    return Cc


def create_coords3D(coords, elems):
    """(coords3D (nv, dim, ne), vectors3D (nv-1, dim, ne)) -- P:514-526."""
    coords, elems = _f64(coords), _i32(elems)
    dim, nn = coords.shape
    nv, ne = elems.shape
    c3 = np.empty((nv, dim, ne))
    v3 = np.empty((nv - 1, dim, ne))
    _check(lib().orc_create_coords3D(dim, nv, ne, _p(coords), 1, nn, _p(elems), ne, _p(c3), _p(v3)), "gather")
    return c3, v3


NORMALS_REF = {   # outer normals of the reference simplex as columns (3D: P:562-570; 2D: the same construction)
    2: np.array([[-1.0, 0.0, 1.0], [0.0, -1.0, 1.0]]),
    3: np.array([[-1.0, 0.0, 0.0, 1.0], [0.0, -1.0, 0.0, 1.0], [0.0, 0.0, -1.0, 1.0]]),
}


def simplex_geometry(coords, elems):
    """Signed sizes and (not normalised) outer normals of every simplex, the paper's two scripts written out
    with the oracle's own page functions, step by step:
        [~, vectors3D] = create_coords3D(coords, elems)
        meass = amdet(vectors3D) / factorial(dim)
        normals3D = amsm(amt(aminv(vectors3D)), normalsRef)
    Returns (meass (ne,), normals3D (dim+1, dim, ne): column j of page e at [j, :, e])."""
    coords, elems = _f64(coords), _i32(elems)
    dim = coords.shape[0]
    assert elems.shape[0] == dim + 1 and dim in (2, 3)
    _, v3 = create_coords3D(coords, elems)
    fact = 2.0 if dim == 2 else 6.0
    meass = page_det(v3) / fact
    vinv, _ = page_inv(v3)
    nref = np.ascontiguousarray(NORMALS_REF[dim].T[:, :, None])   # one dim x (dim+1) object for every page (eq:copy)
    normals = page_mtimes(page_transpose(vinv), nref)
    return meass, normals


def tri_surface(xyz, tri):
    """(n (3,F), nhat (3,F), area (F,), volume float)."""
    xyz, tri = _f64(xyz), _i32(tri)
    nverts = xyz.shape[1]
    nf = tri.shape[1]
    n = np.empty((3, nf))
    nh = np.empty((3, nf))
    ar = np.empty(nf)
    vol = np.empty(1)
    _check(lib().orc_tri_surface(nf, _p(tri), nf, _p(xyz), 1, nverts, _p(n), _p(nh), _p(ar), _p(vol)), "surface")
    return n, nh, ar, float(vol[0])


# ------------------------------------------------------------------ FEM P1
def p1_local(X):
    """X: (dim, nv) vertex coordinates of one element -> (Ke, Me) nv x nv."""
    X = _f64(X)
    dim, nv = X.shape
    Ke = np.empty((nv, nv))
    Me = np.empty((nv, nv))
    lib().orc_p1_local(dim, _p(X), _p(Ke), _p(Me))
    return Ke, Me


def p1_local_all(coords, elems):
    """K3D, M3D page arrays, shape (nv, nv, ne) (entry (a,b) at [b, a, e])."""
    coords, elems = _f64(coords), _i32(elems)
    dim, nn = coords.shape
    nv, ne = elems.shape
    K3 = np.empty((nv, nv, ne))
    M3 = np.empty((nv, nv, ne))
    _check(lib().orc_p1_local_all(dim, ne, _p(coords), 1, nn, _p(elems), ne, _p(K3), _p(M3)), "local_all")
    return K3, M3


def p1_pattern(elems, nn):
    """(row_ptr (nn+1,), col_idx (nnz,)) int32."""
    elems = _i32(elems)
    nv, ne = elems.shape
    dim = nv - 1
    row_ptr = np.empty(nn + 1, dtype=np.int32)
    nnz = lib().orc_p1_pattern(dim, nn, ne, _p(elems), ne, _p(row_ptr), None)
    if nnz < 0:
        raise MemoryError("oracle pattern")
    col_idx = np.empty(max(nnz, 1), dtype=np.int32)
    nnz2 = lib().orc_p1_pattern(dim, nn, ne, _p(elems), ne, _p(row_ptr), _p(col_idx))
    assert nnz2 == nnz
    return row_ptr, col_idx[:nnz]


def p1_assemble(coords, elems, row_ptr, col_idx, row_mask=None):
    """(K, M) CSR values on the given pattern (O11)."""
    coords, elems = _f64(coords), _i32(elems)
    row_ptr, col_idx = _i32(row_ptr), _i32(col_idx)
    dim, nn = coords.shape
    nv, ne = elems.shape
    nnz = int(row_ptr[-1])
    K = np.empty(nnz)
    M = np.empty(nnz)
    mask = None
    if row_mask is not None:
        mask = np.ascontiguousarray(row_mask, dtype=np.uint8)
        assert mask.shape == (nn,)
    rc = lib().orc_p1_assemble(dim, nn, ne, _p(coords), 1, nn, _p(elems), ne,
                               _p(row_ptr), _p(col_idx), _p(K), _p(M), _p(mask))
    _check(rc, "assemble")
    return K, M


# ------------------------------------------------------------------ NEXT-1
def quad_rule(dim, gqo):
    """(lam (nip, dim+1) barycentric points, w (nip,)) of intquad(gqo, dim)."""
    lam = np.empty(64)
    w = np.empty(16)
    nip = lib().orc_quad_rule(dim, gqo, _p(lam), _p(w))
    if nip < 0:
        raise ValueError("no quadrature rule for dim=%d gqo=%d" % (dim, gqo))
    return lam[:nip * (dim + 1)].reshape(nip, dim + 1).copy(), w[:nip].copy()


def _coef(dim, c):
    a, b = c
    bb = np.zeros(3)
    bb[:dim] = np.asarray(b, dtype=np.float64)[:dim]
    return float(a), bb


def p1_local_coef(X, gqo=2, cK=(1.0, (1.0, 1.0, 1.0)), cM=(1.0, (1.0, 1.0, 1.0))):
    """Element matrices with c(x) = a * exp(b . x); X (dim, nv)."""
    X = _f64(X)
    dim, nv = X.shape
    (ka, kb), (ma, mb) = _coef(dim, cK), _coef(dim, cM)
    Ke = np.empty((nv, nv))
    Me = np.empty((nv, nv))
    _check(lib().orc_p1_local_coef(dim, _p(X), gqo, ka, _p(kb), ma, _p(mb), _p(Ke), _p(Me)), "local_coef")
    return Ke, Me


def p1_assemble_coef(coords, elems, row_ptr, col_idx, gqo=2, cK=(1.0, (1.0, 1.0, 1.0)),
                     cM=(1.0, (1.0, 1.0, 1.0))):
    coords, elems = _f64(coords), _i32(elems)
    row_ptr, col_idx = _i32(row_ptr), _i32(col_idx)
    dim, nn = coords.shape
    nv, ne = elems.shape
    (ka, kb), (ma, mb) = _coef(dim, cK), _coef(dim, cM)
    nnz = int(row_ptr[-1])
    K = np.empty(nnz)
    M = np.empty(nnz)
    _check(lib().orc_p1_assemble_coef(dim, nn, ne, _p(coords), 1, nn, _p(elems), ne, _p(row_ptr), _p(col_idx),
                                      gqo, ka, _p(kb), ma, _p(mb), _p(K), _p(M)), "assemble_coef")
    return K, M


# ------------------------------------------------------------------ NEXT-2
def page_bilinear(A, Mx, B):
    """avtamav: s_k = a_k^T M_k b_k.  A (1, n, N), Mx (m, n, N), B (1, m, N)."""
    A, Mx, B = _f64(A), _f64(Mx), _f64(B)
    m, n, _ = Mx.shape
    N = max(A.shape[-1], Mx.shape[-1], B.shape[-1])

    def ld(X):                       # eq:copy broadcast of a single object
        return 0 if (X.shape[-1] == 1 and N > 1) else X.shape[-1]
    s = np.empty(N)
    _check(lib().orc_page_bilinear(N, n, m, _p(A), ld(A), _p(Mx), ld(Mx), _p(B), ld(B), _p(s)), "bilinear")
    return s


def p1_rhs(coords, elems, fq, gqo=2):
    """(b (nn,), b2D (nv, ne)) of Code rhs_vectorP1 with f values fq (nip, ne)."""
    coords, elems, fq = _f64(coords), _i32(elems), _f64(fq)
    dim, nn = coords.shape
    nv, ne = elems.shape
    b = np.empty(nn)
    b2 = np.empty((nv, ne))
    _check(lib().orc_p1_rhs(dim, nn, ne, _p(coords), 1, nn, _p(elems), ne, gqo, _p(fq), _p(b2), _p(b)), "rhs")
    return b, b2


# ------------------------------------------------------------------ NEXT-3 (P2)
def pattern(elems, nn):
    """Topological CSR pattern for elements with any number of nodes (P2: 6 / 10)."""
    elems = _i32(elems)
    nv, ne = elems.shape
    row_ptr = np.empty(nn + 1, dtype=np.int32)
    nnz = lib().orc_pattern(nv, nn, ne, _p(elems), ne, _p(row_ptr), None)
    if nnz < 0:
        raise MemoryError("oracle pattern")
    col_idx = np.empty(max(nnz, 1), dtype=np.int32)
    assert lib().orc_pattern(nv, nn, ne, _p(elems), ne, _p(row_ptr), _p(col_idx)) == nnz
    return row_ptr, col_idx[:nnz]


def p2_local_coef(X, gqo=4, cK=(1.0, (1.0, 1.0, 1.0)), cM=(1.0, (1.0, 1.0, 1.0))):
    """P2 element matrices; X (dim, nlb) node coordinates (vertices, then edges)."""
    X = _f64(X)
    dim, nlb = X.shape
    (ka, kb), (ma, mb) = _coef(dim, cK), _coef(dim, cM)
    Ke = np.empty((nlb, nlb))
    Me = np.empty((nlb, nlb))
    _check(lib().orc_p2_local_coef(dim, _p(X), gqo, ka, _p(kb), ma, _p(mb), _p(Ke), _p(Me)), "p2_local")
    return Ke, Me


def p2_assemble_coef(coords, elems, row_ptr, col_idx, gqo=4, cK=(1.0, (1.0, 1.0, 1.0)),
                     cM=(1.0, (1.0, 1.0, 1.0))):
    coords, elems = _f64(coords), _i32(elems)
    row_ptr, col_idx = _i32(row_ptr), _i32(col_idx)
    dim, nn = coords.shape
    nlb, ne = elems.shape
    (ka, kb), (ma, mb) = _coef(dim, cK), _coef(dim, cM)
    nnz = int(row_ptr[-1])
    K = np.empty(nnz)
    M = np.empty(nnz)
    _check(lib().orc_p2_assemble_coef(dim, nn, ne, _p(coords), 1, nn, _p(elems), ne, _p(row_ptr), _p(col_idx),
                                      gqo, ka, _p(kb), ma, _p(mb), _p(K), _p(M)), "p2_assemble")
    return K, M


def gi(fip, w, sizes, normals=None):
    """Code GI: fip (nip, d, ne) page array (entry (c, q) of page e at
    [q, c, e]), w (nip,), sizes (ne,), normals (d, ne) or None.  Returns the integral."""
    fip = _f64(fip)
    nip, d, ne = fip.shape
    w, sizes = _f64(w), _f64(sizes)
    nrm = _f64(normals) if normals is not None else None
    out = np.empty(1)
    _check(lib().orc_gi(ne, d, nip, _p(fip), ne, _p(w), _p(sizes), _p(nrm) if nrm is not None else None, ne,
                        _p(out)), "gi")
    return float(out[0])
