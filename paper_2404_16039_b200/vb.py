"""Thin Python binding of libvb.so (include/vb.h) -- argument marshalling only.

Every function has the name of the C entry point it calls and runs nothing but
that call: torch is used for device memory (output allocation) and the current
CUDA stream.  There is no CPU path: if libvb.so is missing or CUDA is not
available the calls raise.

Layouts (include/vb.h): a page batch of N r x c pages is a contiguous float64
CUDA tensor of shape (c, r, N) (column-major entries, page-contiguous planes);
a single object broadcast to every page (eq:copy) is a tensor of
shape (c, r, 1) used with npages > 1 (ld = 0).  Meshes: coords (dim, nn)
float64, elems (nv, ne) int32.
"""
import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VB_LIBVB") or os.path.join(_HERE, "libvb.so")   # VB_LIBVB: A/B builds (tools/)

VB_ASSEMBLE_ATOMIC = 0
VB_ASSEMBLE_GATHER = 1
VB_GATHER_HINT_COMPACT = 0x100
VB_PATTERN_VALIDATE = 0x100   # fem_p1_pattern: dim | VB_PATTERN_VALIDATE checks every vertex id first
TILE_ROWS, TILE_NLOC, TILE_MAXC = 128, 1024, 32   # VB_TILE_ROWS, VB_TILE_NLOC, VB_TILE_MAXC


def _gather_mode(mode, plan, compact):
    """(mode, plan words): the compact-budget hint from the plan's block maxima
    (compact=None) or forced (True / False), with the packed 16-bit plan words it
    needs (packing fails for rows of more than 16 entries; blocks beyond the
    budget only cost speed)."""
    if mode != VB_ASSEMBLE_GATHER:
        return int(mode), plan.node_elem_slot
    use = getattr(plan, "compact", False) if compact is None else bool(compact)
    if not use:
        return int(mode), plan.node_elem_slot
    if getattr(plan, "node_elem_slot16", None) is None:
        plan.node_elem_slot16 = plan.pack_slots()
    return int(mode) | VB_GATHER_HINT_COMPACT, plan.node_elem_slot16

_STATUS = {0: "VB_OK", -1: "VB_ERR_ARG", -2: "VB_ERR_DIM", -3: "VB_ERR_UNSUPPORTED",
           -4: "VB_ERR_OVERFLOW", -5: "VB_ERR_WORKSPACE", -6: "VB_ERR_CUDA"}

EXPORTS = ("vb_last_error", "vb_abi_version", "vb_page_mtimes", "vb_page_transpose", "vb_page_det",
           "vb_page_inv", "vb_page_cross", "vb_create_coords3D", "vb_tri_surface", "fem_p1_pattern",
           "fem_p1_assemble", "fem_p1_assemble_coef", "vb_quad_rule", "fem_p1_rhs", "vb_page_bilinear",
           "fem_pattern", "fem_p2_assemble", "fem_plan_stats", "fem_plan_pack_slots", "fem_plan_classes",
           "fem_p1_assemble_classes", "fem_plan_tiles", "fem_p1_assemble_tiles",
           "fem_p1_assemble_exact", "fem_p1_assemble_classes_coef", "vb_gi", "fem_plan_lattice",
           "fem_p1_assemble_lattice", "fem_lattice_pattern", "fem_plan_lattice2d", "fem_p1_assemble_lattice2d", "fem_lattice2d_pattern",
           "vb_simplex_geometry")


class VbError(RuntimeError):
    def __init__(self, status, message):
        super().__init__("%s (%d): %s" % (_STATUS.get(status, "?"), status, message))
        self.status = status


_lib = None


def lib():
    """Load libvb.so (raises if it is missing -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libvb.so not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        i64, i32, d, p, sz = C.c_int64, C.c_int, C.c_double, C.c_void_p, C.POINTER(C.c_size_t)
        sig = {
            "vb_last_error": (C.c_char_p, []),
            "vb_abi_version": (i32, []),
            "vb_page_mtimes": (i32, [i64, p, i32, i32, i64, i32, p, i32, i32, i64, i32, p, i64, p]),
            "vb_page_transpose": (i32, [i64, p, i32, i32, i64, p, i64, p]),
            "vb_page_det": (i32, [i64, i32, p, i64, p, p]),
            "vb_page_inv": (i32, [i64, i32, p, i64, p, i64, p, p, d, p]),
            "vb_page_cross": (i32, [i64, p, i64, p, i64, p, i64, p]),
            "vb_create_coords3D": (i32, [i32, i32, i64, p, i64, i64, p, i64, p, p, p]),
            "vb_simplex_geometry": (i32, [i32, i64, p, i64, i64, p, i64, p, p, i64, p]),
            "vb_tri_surface": (i32, [i64, p, i64, i64, p, i64, i64, p, p, p, p, p, sz, p]),
            "fem_p1_pattern": (i32, [i32, i64, i64, p, i64, p, sz, p, p, i64, p, p, p, p,
                                     C.POINTER(C.c_int64), p]),
            "fem_p1_assemble": (i32, [i32, i64, i64, p, i64, i64, p, i64, p, p, i64, p, p, p, p,
                                      p, p, p, p, i32, p, sz, p, p]),
            "fem_p1_assemble_coef": (i32, [i32, i64, i64, p, i64, i64, p, i64, p, p, i64, p, p, p, p,
                                           i32, d, p, d, p, p, p, p, p, i32, p, sz, p, p]),
            "vb_quad_rule": (i32, [i32, i32, p, p]),
            "fem_p1_rhs": (i32, [i32, i64, i64, p, i64, i64, p, i64, i32, p, p, p, p, p, i32, p]),
            "vb_page_bilinear": (i32, [i64, i32, i32, p, i64, p, i64, p, i64, p, p]),
            "fem_plan_stats": (i32, [i64, p, p, p, C.POINTER(C.c_int64), p]),
            "fem_plan_pack_slots": (i32, [i32, i64, p, p, p, p]),
            "fem_plan_classes": (i32, [i32, i64, p, p, p, p, sz, p, p, i64, C.POINTER(C.c_int64), p]),
            "fem_p1_assemble_classes": (i32, [i32, i64, p, i64, i64, p, p, i64, p, p, p, p, i64, p, p, p, sz, p]),
            "fem_plan_tiles": (i32, [i32, i64, i64, p, i64, i64, p, i64, p, p, p, sz, p, p, p, p, p, i64,
                                     C.POINTER(C.c_int64), p]),
            "fem_p1_assemble_tiles": (i32, [i32, i64, p, i64, i64, i64, p, p, p, p, p, i32, i32, p, p, p]),
            "fem_p1_assemble_exact": (i32, [i32, i64, p, i64, i64, p, i64, p, p, p, p, p, p, p]),
            "fem_p1_assemble_classes_coef": (i32, [i32, i64, p, i64, i64, p, p, i64, p, p, p, p, i64, i32, d, p, p,
                                                   p, p, p]),
            "vb_gi": (i32, [i64, i32, i32, p, i64, p, p, p, i64, p, p, sz, p]),
            "fem_plan_lattice": (i32, [i64, i64, p, i64, p, p, i64, i32, i32, i32, p, sz, p, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int64), p]),
            "fem_p1_assemble_lattice": (i32, [i64, p, i64, i64, p, i64, p, i32, i32, i32, i32, p, p, p, p]),
            "fem_lattice_pattern": (i32, [i64, i32, i32, i32, i32, p, sz, p, p, i64, C.POINTER(C.c_int64), p]),
            "fem_plan_lattice2d": (i32, [i64, i64, p, i64, p, p, i64, i32, i32, p, sz, p, C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int64), p]),
            "fem_p1_assemble_lattice2d": (i32, [i64, p, i64, i64, p, i64, p, i32, i32, i32, p, p, p, p]),
            "fem_lattice2d_pattern": (i32, [i64, i32, i32, i32, p, sz, p, p, i64, C.POINTER(C.c_int64), p]),
            "fem_pattern": (i32, [i32, i64, i64, p, i64, p, sz, p, p, i64, p, p, p, p, C.POINTER(C.c_int64), p]),
            "fem_p2_assemble": (i32, [i32, i64, i64, p, i64, i64, p, i64, p, p, i64, p, p, p, i32, d, p, d, p,
                                      p, p, p, p, i32, p, sz, p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise VbError(rc, lib().vb_last_error().decode())


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libvb takes device tensors only (got a %s tensor)" % t.device)
    if not t.is_contiguous():
        raise ValueError("libvb takes contiguous tensors")
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _f64(t):
    if t.dtype != torch.float64:
        raise TypeError("expected float64, got %s" % t.dtype)
    return t


def _ld(t, npages):
    n = t.shape[-1]
    return 0 if (n == 1 and npages != 1) else n


# ------------------------------------------------------------------ page ops
def vb_page_mtimes(X, Y, transX=False, transY=False, Z=None, stream=None):
    """Z_k = op(X_k) op(Y_k).  X: (xcols, xrows, N|1), Y: (ycols, yrows, N|1)."""
    _f64(X), _f64(Y)
    xc, xr, nx = X.shape
    yc, yr, ny = Y.shape
    npages = max(nx, ny)
    m = xc if transX else xr
    n = yr if transY else yc
    if Z is None:
        Z = torch.empty((n, m, npages), dtype=torch.float64, device=X.device)
    _check(lib().vb_page_mtimes(npages, _ptr(X), xr, xc, _ld(X, npages), int(bool(transX)),
                                _ptr(Y), yr, yc, _ld(Y, npages), int(bool(transY)),
                                _ptr(Z), Z.shape[-1], _stream(stream)))
    return Z


def vb_page_transpose(X, Z=None, stream=None):
    _f64(X)
    c, r, n = X.shape
    if Z is None:
        Z = torch.empty((r, c, n), dtype=torch.float64, device=X.device)
    _check(lib().vb_page_transpose(n, _ptr(X), r, c, n, _ptr(Z), Z.shape[-1], _stream(stream)))
    return Z


def vb_page_det(X, det=None, stream=None):
    _f64(X)
    n, n2, N = X.shape
    if det is None:
        det = torch.empty((N,), dtype=torch.float64, device=X.device)
    _check(lib().vb_page_det(N, n if n == n2 else -1, _ptr(X), N, _ptr(det), _stream(stream)))
    return det


def vb_page_inv(X, Xinv=None, det=None, first_singular=None, sing_tol=1e-14, want_det=True, stream=None):
    """Returns (Xinv, det or None, first_singular device int64 tensor or None)."""
    _f64(X)
    n, n2, N = X.shape
    if n != n2:
        raise ValueError("vb_page_inv: pages are %dx%d, not square" % (n2, n))
    if Xinv is None:
        Xinv = torch.empty_like(X)
    if det is None and want_det:
        det = torch.empty((N,), dtype=torch.float64, device=X.device)
    _check(lib().vb_page_inv(N, n, _ptr(X), N, _ptr(Xinv), Xinv.shape[-1], _ptr(det), _ptr(first_singular),
                             float(sing_tol), _stream(stream)))
    return Xinv, det, first_singular


def vb_page_cross(A, B, Cout=None, stream=None):
    _f64(A), _f64(B)
    N = max(A.shape[-1], B.shape[-1])
    if Cout is None:
        Cout = torch.empty((1, 3, N), dtype=torch.float64, device=A.device)
    _check(lib().vb_page_cross(N, _ptr(A), _ld(A, N), _ptr(B), _ld(B, N), _ptr(Cout), N, _stream(stream)))
    return Cout


def vb_create_coords3D(coords, elems, want_coords3D=True, want_vectors3D=True, stream=None):
    dim, nn = coords.shape
    nv, ne = elems.shape
    c3 = torch.empty((nv, dim, ne), dtype=torch.float64, device=coords.device) if want_coords3D else None
    v3 = torch.empty((nv - 1, dim, ne), dtype=torch.float64, device=coords.device) if want_vectors3D else None
    _check(lib().vb_create_coords3D(dim, nv, ne, _ptr(coords), 1, nn, _ptr(elems), ne, _ptr(c3), _ptr(v3),
                                    _stream(stream)))
    return c3, v3


def vb_simplex_geometry(coords, elems, want_meass=True, want_normals=True, meass=None, normals=None, stream=None):
    """(meass (ne,), normals3D (dim+1, dim, ne)): signed sizes and outer normals of every simplex."""
    _f64(coords)
    dim, nn = coords.shape
    nv, ne = elems.shape
    if nv != dim + 1:
        raise ValueError("vb_simplex_geometry: elems must have dim+1 vertex planes")
    if want_meass and meass is None:
        meass = torch.empty((ne,), dtype=torch.float64, device=coords.device)
    if want_normals and normals is None:
        normals = torch.empty((nv, dim, ne), dtype=torch.float64, device=coords.device)
    _check(lib().vb_simplex_geometry(dim, ne, _ptr(coords), 1, nn, _ptr(elems), ne, _ptr(meass), _ptr(normals), ne,
                                     _stream(stream)))
    return meass, normals


def vb_tri_surface(xyz, tri, want_n=True, want_nhat=True, want_area=True, want_volume=True, work=None, out=None,
                   stream=None):
    """Returns dict with n (3,F), nhat (3,F), area (F,), volume (1,) device tensors."""
    _f64(xyz)
    nverts = xyz.shape[1]
    nf = tri.shape[1]
    dev = xyz.device
    o = dict(out or {})
    if want_n and "n" not in o:
        o["n"] = torch.empty((3, nf), dtype=torch.float64, device=dev)
    if want_nhat and "nhat" not in o:
        o["nhat"] = torch.empty((3, nf), dtype=torch.float64, device=dev)
    if want_area and "area" not in o:
        o["area"] = torch.empty((nf,), dtype=torch.float64, device=dev)
    if want_volume and "volume" not in o:
        o["volume"] = torch.empty((1,), dtype=torch.float64, device=dev)
    sz = C.c_size_t(0)
    vol = o.get("volume")
    _check(lib().vb_tri_surface(nf, None, nf, nverts, None, 1, nverts, None, None, None, _ptr(vol), None,
                                C.byref(sz), _stream(stream)))
    if work is None or work.numel() < sz.value:
        work = torch.empty((max(sz.value, 1),), dtype=torch.uint8, device=dev)
    sz2 = C.c_size_t(work.numel())
    _check(lib().vb_tri_surface(nf, _ptr(tri), nf, nverts, _ptr(xyz), 1, nverts, _ptr(o.get("n")),
                                _ptr(o.get("nhat")), _ptr(o.get("area")), _ptr(vol), _ptr(work), C.byref(sz2),
                                _stream(stream)))
    o["work"] = work
    return o


def vb_gi(fip, w, sizes, normals=None, value=None, work=None, stream=None):
    """Code GI: fip (nip, d, N) page array, w (nip,) host weights,
    sizes (N,), normals (d, N) or None.  Returns (value (1,) device tensor, work)."""
    _f64(fip)
    nip, d, N = fip.shape
    dev = fip.device
    if value is None:
        value = torch.empty((1,), dtype=torch.float64, device=dev)
    wb = (C.c_double * nip)(*[float(x) for x in w])
    sz = C.c_size_t(0)
    _check(lib().vb_gi(N, d, nip, None, N, C.cast(wb, C.c_void_p), None, None, N, None, None, C.byref(sz),
                       _stream(stream)))
    if work is None or work.numel() < sz.value:
        work = torch.empty((max(sz.value, 256),), dtype=torch.uint8, device=dev)
    sz2 = C.c_size_t(work.numel())
    _check(lib().vb_gi(N, d, nip, _ptr(fip), N, C.cast(wb, C.c_void_p), _ptr(sizes), _ptr(normals), N, _ptr(value),
                       _ptr(work), C.byref(sz2), _stream(stream)))
    return value, work


# ------------------------------------------------------------------ FEM P1
def _work16(dev):
    """A fresh 16-byte device buffer for one launch's block counter (the caller-owned work of the
    assembly calls); torch's stream-ordered allocator keeps it private to this launch."""
    return torch.empty((2,), dtype=torch.float64, device=dev)


def _wb(n=16):
    return C.byref(C.c_size_t(n))


def _pad4(n):
    return max(4, (n + 3) // 4 * 4)


class P1Plan:
    """CSR pattern + scatter plans of a P1 mesh (fem_p1_pattern, both phases).

    Attributes: row_ptr (nn+1), col_idx (nnz) int32; elem2nnz (nv*nv, ne) int32
    or None; node_elem_ptr (nn+1), node_elem (nv*ne) int32 and node_elem_slot
    (nv*ne) int32 (uint32 bits) or None; nnz."""

    def __init__(self, elems, nn, scatter_map=True, gather_plan=True, stream=None, validate=False):
        """validate: check every vertex id against [0, nn) first (VB_PATTERN_VALIDATE; VbError naming the
        first offending element and vertex)."""
        if elems.dtype != torch.int32:
            raise TypeError("elems must be int32")
        nv, ne = elems.shape
        self.dim, self.nn, self.ne, self.nv = nv - 1, int(nn), int(ne), nv
        dev = elems.device
        L = lib()
        sz = C.c_size_t(0)
        nnz = C.c_int64(0)
        st = _stream(stream)
        _check(L.fem_p1_pattern(self.dim, nn, ne, None, ne, None, C.byref(sz), None, None, 0, None, None, None, None,
                                None, st))
        self.work = torch.empty((max(sz.value, 16),), dtype=torch.uint8, device=dev)
        self.row_ptr = torch.empty((nn + 1,), dtype=torch.int32, device=dev)
        _check(L.fem_p1_pattern(self.dim | (VB_PATTERN_VALIDATE if validate else 0), nn, ne, _ptr(elems), ne,
                                _ptr(self.work), C.byref(sz), _ptr(self.row_ptr),
                                None, 0, None, None, None, None, C.byref(nnz), st))
        self.nnz = int(nnz.value)
        # gather mode streams col_idx / node_elem_slot in 16-byte chunks: pad to a multiple of 4 entries
        self.col_idx = torch.zeros((_pad4(self.nnz),), dtype=torch.int32, device=dev)
        self.elem2nnz = torch.empty((nv * nv, ne), dtype=torch.int32, device=dev) if scatter_map else None
        if gather_plan:
            self.node_elem_ptr = torch.empty((nn + 1,), dtype=torch.int32, device=dev)
            self.node_elem = torch.empty((max(nv * ne, 1),), dtype=torch.int32, device=dev)
            self.node_elem_slot = torch.zeros((_pad4(nv * ne),), dtype=torch.int32, device=dev)
        else:
            self.node_elem_ptr = self.node_elem = self.node_elem_slot = None
        _check(L.fem_p1_pattern(self.dim, nn, ne, _ptr(elems), ne, _ptr(self.work), C.byref(sz), _ptr(self.row_ptr),
                                _ptr(self.col_idx), self.col_idx.numel(), _ptr(self.elem2nnz), _ptr(self.node_elem_ptr),
                                _ptr(self.node_elem), _ptr(self.node_elem_slot), C.byref(nnz), st))
        self.col_idx_padded = self.col_idx
        self.col_idx = self.col_idx[:self.nnz]
        self.work = None   # the pattern workspace is not needed after the plan exists
        # block maxima -> the gather kernel's compact shared-memory budget where it fits (3D)
        stats = (C.c_int64 * 3)()
        scratch = torch.empty((16,), dtype=torch.uint8, device=dev)
        _check(L.fem_plan_stats(nn, _ptr(self.row_ptr), _ptr(self.node_elem_ptr), _ptr(scratch), stats, st))
        self.stats = tuple(int(x) for x in stats)   # (max row, max block entries, max block incidences)
        self.compact = (self.dim == 3 and gather_plan and self.stats[0] <= 15 and self.stats[1] <= 16 * 32
                        and self.stats[2] <= 25 * 32)
        self.node_elem_slot16 = self.pack_slots() if self.compact else None

    @classmethod
    def for_lattice(cls, elems, nn, dims=None, stream=None):
        """Plan of a Kuhn-lattice mesh without the generic pattern build: fem_plan_lattice verifies the
        elements (row_ptr = col_idx = NULL), fem_lattice_pattern writes the stencil pattern in closed form
        (bit-identical to fem_p1_pattern's).  dims: (nx, ny, nz), None = a cube inferred from ne.  Returns the
        plan (pattern + lattice plan; no scatter map, no gather plan), or None if the mesh is refused."""
        if elems.dtype != torch.int32:
            raise TypeError("elems must be int32")
        nv, ne = elems.shape
        if nv == 3:
            return cls._for_lattice2d(elems, nn, dims, stream)
        if nv != 4:
            return None
        if dims is None:
            n = int(round((ne / 6) ** (1.0 / 3.0))) if ne > 0 else 0
            dims = (n, n, n)
        nx, ny, nz = (int(d) for d in dims)
        if nx < 2 or ny < 2 or nz < 1 or (nx + 1) * (ny + 1) * (nz + 1) != nn or 6 * nx * ny * nz != ne:
            return None   # the kernel needs nx, ny >= 2
        self = cls.__new__(cls)
        self.dim, self.nn, self.ne, self.nv = 3, int(nn), int(ne), 4
        dev = elems.device
        L = lib()
        st = _stream(stream)
        wb, pints, nnz, pwb = C.c_size_t(0), C.c_int64(0), C.c_int64(0), C.c_size_t(0)
        stats = (C.c_int64 * 4)()
        _check(L.fem_lattice_pattern(nn, nx, ny, nz, 0, None, C.byref(pwb), None, None, 0, C.byref(nnz), st))
        self.nnz = int(nnz.value)
        _check(L.fem_plan_lattice(nn, ne, None, ne, None, None, self.nnz, nx, ny, nz, None, C.byref(wb), None,
                                  C.byref(pints), stats, st))
        work = torch.empty((max(wb.value, pwb.value, 16),), dtype=torch.uint8, device=dev)
        plan = torch.zeros((max(int(pints.value), 16),), dtype=torch.int32, device=dev)
        _check(L.fem_plan_lattice(nn, ne, _ptr(elems), elems.shape[1], None, None, self.nnz, nx, ny, nz, _ptr(work),
                                  C.byref(wb), _ptr(plan), C.byref(pints), stats, st))
        if stats[0] != 1:
            return None
        self.row_ptr = torch.empty((nn + 1,), dtype=torch.int32, device=dev)
        self.col_idx_padded = torch.zeros((_pad4(self.nnz),), dtype=torch.int32, device=dev)
        _check(L.fem_lattice_pattern(nn, nx, ny, nz, int(stats[3]) & 7, _ptr(work), C.byref(pwb), _ptr(self.row_ptr),
                                     _ptr(self.col_idx_padded), self.col_idx_padded.numel(), C.byref(nnz), st))
        self.col_idx = self.col_idx_padded[:self.nnz]
        self.elem2nnz = self.node_elem_ptr = self.node_elem = self.node_elem_slot = None
        self.node_elem_slot16, self.compact, self.work, self.stats = None, False, None, (15, 0, 0)
        self.lattice_plan, self.lattice_dims = plan, (nx, ny, nz)
        self.lattice_flips, self.lattice_tiles = int(stats[3]), int(stats[1])
        self.lattice_ok, self.lattice_reason = True, ""
        return self

    @classmethod
    def _for_lattice2d(cls, elems, nn, dims, stream):
        """for_lattice in 2D: fem_plan_lattice2d on the elements + fem_lattice2d_pattern."""
        ne = elems.shape[1]
        if dims is None:
            n = int(round((ne / 2) ** 0.5)) if ne > 0 else 0
            dims = (n, n)
        nx, ny = (int(d) for d in dims[:2])
        if nx < 2 or ny < 1 or (nx + 1) * (ny + 1) != nn or 2 * nx * ny != ne:
            return None
        self = cls.__new__(cls)
        self.dim, self.nn, self.ne, self.nv = 2, int(nn), int(ne), 3
        dev = elems.device
        L = lib()
        st = _stream(stream)
        wb, pints, nnz, pwb = C.c_size_t(0), C.c_int64(0), C.c_int64(0), C.c_size_t(0)
        stats = (C.c_int64 * 4)()
        _check(L.fem_lattice2d_pattern(nn, nx, ny, 0, None, C.byref(pwb), None, None, 0, C.byref(nnz), st))
        self.nnz = int(nnz.value)
        _check(L.fem_plan_lattice2d(nn, ne, None, ne, None, None, self.nnz, nx, ny, None, C.byref(wb), None,
                                    C.byref(pints), stats, st))
        work = torch.empty((max(wb.value, pwb.value, 16),), dtype=torch.uint8, device=dev)
        plan = torch.zeros((max(int(pints.value), 16),), dtype=torch.int32, device=dev)
        _check(L.fem_plan_lattice2d(nn, ne, _ptr(elems), elems.shape[1], None, None, self.nnz, nx, ny, _ptr(work),
                                    C.byref(wb), _ptr(plan), C.byref(pints), stats, st))
        if stats[0] != 1:
            return None
        self.row_ptr = torch.empty((nn + 1,), dtype=torch.int32, device=dev)
        self.col_idx_padded = torch.zeros((_pad4(self.nnz),), dtype=torch.int32, device=dev)
        _check(L.fem_lattice2d_pattern(nn, nx, ny, int(stats[3]) & 1, _ptr(work), C.byref(pwb), _ptr(self.row_ptr),
                                       _ptr(self.col_idx_padded), self.col_idx_padded.numel(), C.byref(nnz), st))
        self.col_idx = self.col_idx_padded[:self.nnz]
        self.elem2nnz = self.node_elem_ptr = self.node_elem = self.node_elem_slot = None
        self.node_elem_slot16, self.compact, self.work, self.stats = None, False, None, (7, 0, 0)
        self.lattice_plan, self.lattice_dims = plan, (nx, ny)
        self.lattice_flips, self.lattice_tiles = int(stats[3]), int(stats[1])
        self.lattice_ok, self.lattice_reason = True, ""
        return self

    def classes(self):
        """Row classes of the gather plan (fem_plan_classes), built once and kept:
        class_rows (nn,) int32, groups (ngroups, 4) int32, class_stats = (groups,
        classes, rows in classes).  None without a gather plan."""
        if self.node_elem_ptr is None:
            return None
        if getattr(self, "class_rows", None) is None:
            dev = self.row_ptr.device
            L = lib()
            sz = C.c_size_t(0)
            st = _stream()
            stats = (C.c_int64 * 4)()
            _check(L.fem_plan_classes(self.dim, self.nn, None, None, None, None, C.byref(sz), None, None, 0, stats,
                                      st))
            work = torch.empty((max(sz.value, 16),), dtype=torch.uint8, device=dev)
            self.class_rows = torch.empty((max(self.nn, 1),), dtype=torch.int32, device=dev)
            cap = self.nn // 32 + 1024
            while True:
                groups = torch.empty((cap, 4), dtype=torch.int32, device=dev)
                rc = L.fem_plan_classes(self.dim, self.nn, _ptr(self.row_ptr), _ptr(self.node_elem_ptr),
                                        _ptr(self.node_elem_slot), _ptr(work), C.byref(sz), _ptr(self.class_rows),
                                        _ptr(groups), cap, stats, st)
                if rc == -5 and stats[0] > cap:
                    cap = int(stats[0])
                    continue
                _check(rc)
                break
            self.groups = groups[:int(stats[0])]
            self.class_stats = tuple(int(x) for x in stats)
        return self.class_rows

    def tiles(self, coords, elems):
        """Tile plan (fem_plan_tiles), built once and kept; coords only choose the
        tiles.  Returns True, or False when the mesh is outside the tile
        variant's limits (plan.tile_reason says why)."""
        if getattr(self, "tile_ok", None) is not None:
            return self.tile_ok
        _f64(coords)
        dev = coords.device
        L = lib()
        sz = C.c_size_t(0)
        st = _stream()
        stats = (C.c_int64 * 6)()
        dim, nn = coords.shape
        ne = elems.shape[1]
        _check(L.fem_plan_tiles(self.dim, nn, ne, None, 1, nn, None, ne, None, None, None, C.byref(sz), None, None,
                                None, None, None, 0, stats, st))
        work = torch.empty((max(sz.value, 16),), dtype=torch.uint8, device=dev)
        T = (nn + TILE_ROWS - 1) // TILE_ROWS
        self.tile_meta = torch.empty((max(T, 1), 4), dtype=torch.int32, device=dev)
        self.tile_nodes = torch.empty((max(T, 1), TILE_NLOC), dtype=torch.int32, device=dev)
        self.tile_rows = torch.empty((max(T, 1), TILE_ROWS, 2), dtype=torch.int32, device=dev)
        self.tile_colors = torch.empty((max(T, 1), TILE_MAXC + 1), dtype=torch.int32, device=dev)
        cap = max(self.nv * ne, 1)
        elems_buf = torch.empty((cap, 4), dtype=torch.int32, device=dev)
        rc = L.fem_plan_tiles(self.dim, nn, ne, _ptr(coords), 1, nn, _ptr(elems), ne, _ptr(self.row_ptr),
                              _ptr(self.col_idx), _ptr(work), C.byref(sz), _ptr(self.tile_meta),
                              _ptr(self.tile_nodes), _ptr(self.tile_rows), _ptr(self.tile_colors), _ptr(elems_buf),
                              cap, stats, st)
        self.tile_stats = tuple(int(x) for x in stats)   # entries, max elems/tile, max nodes/tile, colors, reason, T
        if rc == -3:
            self.tile_ok, self.tile_reason = False, lib().vb_last_error().decode()
            self.tile_meta = self.tile_nodes = self.tile_rows = self.tile_colors = self.tile_elems = None
            return False
        _check(rc)
        self.tile_elems = elems_buf[:max(self.tile_stats[0], 1)].clone()   # keep only the used entries
        self.tile_ok, self.tile_reason = True, ""
        return True

    def lattice(self, elems, dims=None):
        """Kuhn-lattice plan (fem_plan_lattice), built once and kept: verifies that
        the mesh is an nx x ny x nz Kuhn lattice (dims; None = a cube inferred from
        ne) and that the pattern is its stencil.  Returns True, or False with
        plan.lattice_reason."""
        if getattr(self, "lattice_ok", None) is not None:
            return self.lattice_ok
        self.lattice_ok, self.lattice_reason = False, ""
        if self.dim == 2:
            return self._lattice2d(elems, dims)
        if dims is None:
            n = int(round((self.ne / 6) ** (1.0 / 3.0))) if self.ne > 0 else 0
            dims = (n, n, n)
        nx, ny, nz = (int(d) for d in dims)
        if min(nx, ny, nz) < 1 or (nx + 1) * (ny + 1) * (nz + 1) != self.nn or 6 * nx * ny * nz != self.ne:
            self.lattice_reason = "counts are not those of a %d x %d x %d Kuhn lattice" % (nx, ny, nz)
            return False
        L = lib()
        dev = self.row_ptr.device
        wb = C.c_size_t(0)
        pints = C.c_int64(0)
        st = _stream()
        stats = (C.c_int64 * 4)()
        _check(L.fem_plan_lattice(self.nn, self.ne, None, self.ne, None, None, self.nnz, nx, ny, nz, None,
                                  C.byref(wb), None, C.byref(pints), stats, st))
        work = torch.empty((max(wb.value, 16),), dtype=torch.uint8, device=dev)
        plan = torch.zeros((max(int(pints.value), 16),), dtype=torch.int32, device=dev)
        _check(L.fem_plan_lattice(self.nn, self.ne, _ptr(elems), elems.shape[1], _ptr(self.row_ptr),
                                  _ptr(self.col_idx), self.nnz, nx, ny, nz, _ptr(work), C.byref(wb), _ptr(plan),
                                  C.byref(pints), stats, st))
        reasons = {0: "", 1: "counts", 2: "element 0 is not a Kuhn tetrahedron", 3: "degenerate lattice",
                   4: "an element is not a Kuhn tetrahedron of the lattice (or appears twice)",
                   5: "the CSR pattern is not the lattice stencil"}
        if stats[0] != 1:
            self.lattice_reason = reasons.get(int(stats[2]), "refused (%d)" % stats[2])
            return False
        self.lattice_plan = plan
        self.lattice_dims = (nx, ny, nz)
        self.lattice_flips = int(stats[3])
        self.lattice_tiles = int(stats[1])
        self.lattice_ok = True
        return True

    def _lattice2d(self, elems, dims):
        """fem_plan_lattice2d: dims (nx, ny), None = a square inferred from ne."""
        if dims is None:
            n = int(round((self.ne / 2) ** 0.5)) if self.ne > 0 else 0
            dims = (n, n)
        nx, ny = (int(d) for d in dims[:2])
        if nx < 2 or ny < 1 or (nx + 1) * (ny + 1) != self.nn or 2 * nx * ny != self.ne:
            self.lattice_reason = "counts are not those of a %d x %d triangulated lattice" % (nx, ny)
            return False
        L = lib()
        dev = self.row_ptr.device
        wb, pints, st = C.c_size_t(0), C.c_int64(0), _stream()
        stats = (C.c_int64 * 4)()
        _check(L.fem_plan_lattice2d(self.nn, self.ne, None, self.ne, None, None, self.nnz, nx, ny, None, C.byref(wb),
                                    None, C.byref(pints), stats, st))
        work = torch.empty((max(wb.value, 16),), dtype=torch.uint8, device=dev)
        plan = torch.zeros((max(int(pints.value), 16),), dtype=torch.int32, device=dev)
        _check(L.fem_plan_lattice2d(self.nn, self.ne, _ptr(elems), elems.shape[1], _ptr(self.row_ptr),
                                    _ptr(self.col_idx), self.nnz, nx, ny, _ptr(work), C.byref(wb), _ptr(plan),
                                    C.byref(pints), stats, st))
        reasons = {1: "counts", 2: "element 0 is not a triangle of a cell", 3: "nx < 2",
                   4: "an element is not a triangle of the lattice (or appears twice)",
                   5: "the CSR pattern is not the lattice stencil"}
        if stats[0] != 1:
            self.lattice_reason = reasons.get(int(stats[2]), "refused (%d)" % stats[2])
            return False
        self.lattice_plan, self.lattice_dims = plan, (nx, ny)
        self.lattice_flips, self.lattice_tiles = int(stats[3]), int(stats[1])
        self.lattice_ok = True
        return True

    def class_coverage(self):
        """Fraction of rows that the class variant assembles with the uniform loop."""
        if self.classes() is None or self.nn == 0:
            return 0.0
        return self.class_stats[2] / self.nn

    def pack_slots(self):
        """The packed 16-bit plan words of the compact gather budget (fem_plan_pack_slots)."""
        n = self.nv * self.ne
        out = torch.zeros((max(8, (n + 7) // 8 * 8),), dtype=torch.int16, device=self.row_ptr.device)
        scratch = torch.empty((16,), dtype=torch.uint8, device=self.row_ptr.device)
        _check(lib().fem_plan_pack_slots(self.dim, n, _ptr(self.node_elem_slot), _ptr(out), _ptr(scratch),
                                         _stream()))
        return out


def fem_p1_pattern(elems, nn, scatter_map=True, gather_plan=True, stream=None):
    return P1Plan(elems, nn, scatter_map, gather_plan, stream)


def fem_p1_assemble_tiles(coords, plan, K=None, M=None, want_K=True, want_M=True, stream=None):
    """Tile-variant K, M (fem_p1_assemble_tiles) on a plan whose tiles() were built."""
    _f64(coords)
    dim, nn = coords.shape
    dev = coords.device
    if not getattr(plan, "tile_ok", False):
        raise ValueError("plan has no tile plan: call plan.tiles(coords, elems) first (and check it returned True)")
    K = (K if K is not None else torch.empty((plan.nnz,), dtype=torch.float64, device=dev)) if want_K else None
    M = (M if M is not None else torch.empty((plan.nnz,), dtype=torch.float64, device=dev)) if want_M else None
    _check(lib().fem_p1_assemble_tiles(dim, nn, _ptr(coords), 1, nn, plan.nnz, _ptr(plan.tile_meta),
                                       _ptr(plan.tile_nodes), _ptr(plan.tile_rows), _ptr(plan.tile_colors),
                                       _ptr(plan.tile_elems), plan.tile_stats[2], plan.tile_stats[1], _ptr(K), _ptr(M),
                                       _stream(stream)))
    return K, M


def fem_p1_assemble_lattice(coords, plan, K=None, M=None, want_K=True, want_M=True, stream=None, degenerate=None):
    """Element-once K, M on a Kuhn lattice (fem_p1_assemble_lattice); plan.lattice(elems) must be True.
    degenerate: optional device int64 tensor (1,) receiving the number of tets with det = 0."""
    _f64(coords)
    dim, nn = coords.shape
    dev = coords.device
    if not getattr(plan, "lattice_ok", False):
        raise ValueError("plan has no lattice plan: call plan.lattice(elems) first (and check it returned True)")
    K = (K if K is not None else torch.empty((plan.nnz,), dtype=torch.float64, device=dev)) if want_K else None
    M = (M if M is not None else torch.empty((plan.nnz,), dtype=torch.float64, device=dev)) if want_M else None
    if len(plan.lattice_dims) == 2:
        nx, ny = plan.lattice_dims
        _check(lib().fem_p1_assemble_lattice2d(nn, _ptr(coords), 1, nn, _ptr(plan.row_ptr), plan.nnz,
                                               _ptr(plan.lattice_plan), nx, ny, plan.lattice_flips, _ptr(K), _ptr(M),
                                               _ptr(degenerate), _stream(stream)))
        return K, M
    nx, ny, nz = plan.lattice_dims
    _check(lib().fem_p1_assemble_lattice(nn, _ptr(coords), 1, nn, _ptr(plan.row_ptr), plan.nnz,
                                         _ptr(plan.lattice_plan), nx, ny, nz, plan.lattice_flips, _ptr(K), _ptr(M),
                                         _ptr(degenerate), _stream(stream)))
    return K, M


def fem_p1_assemble_exact(coords, elems, plan, want_K=True, want_M=True, stream=None):
    """K, M in the definition's exact operation order (fem_p1_assemble_exact):
    bitwise equal to any plain IEEE fp64 evaluation of it in that order.  Slow;
    for checking.  Needs the plan's gather lists (node_elem)."""
    _f64(coords)
    dim, nn = coords.shape
    ne = elems.shape[1]
    dev = coords.device
    if plan.node_elem_ptr is None:
        raise ValueError("fem_p1_assemble_exact needs a plan with gather_plan=True")
    K = torch.empty((plan.nnz,), dtype=torch.float64, device=dev) if want_K else None
    M = torch.empty((plan.nnz,), dtype=torch.float64, device=dev) if want_M else None
    _check(lib().fem_p1_assemble_exact(dim, nn, _ptr(coords), 1, nn, _ptr(elems), ne, _ptr(plan.row_ptr),
                                       _ptr(plan.col_idx), _ptr(plan.node_elem_ptr), _ptr(plan.node_elem), _ptr(K),
                                       _ptr(M), _stream(stream)))
    return K, M


def _use_classes(plan, variant, coef=False):
    """Gather variant: "class" (row classes, fem_p1_assemble_classes), "block"
    (32-row blocks, fem_p1_assemble) or None = "class" when at least 90 % of the
    rows fall into row classes (meshes from uniform refinement) that the kernel
    keeps on chip (2D c = 1: rows of <= 8 entries), else "block"."""
    if variant not in (None, "class", "block", "tile"):
        raise ValueError("variant must be None, 'class', 'block' or 'tile'")
    if variant == "block" or plan.node_elem_ptr is None:
        return False
    if variant == "class":
        return True
    if plan.class_coverage() < 0.9:
        return False
    return coef or plan.dim == 3 or plan.class_stats[3] <= 8


def fem_p1_assemble_classes(coords, plan, K=None, M=None, want_K=True, want_M=True, stream=None):
    """Gather-variant K, M through the row classes of the plan (fem_p1_assemble_classes)."""
    _f64(coords)
    dim, nn = coords.shape
    dev = coords.device
    K = (K if K is not None else torch.empty((plan.nnz,), dtype=torch.float64, device=dev)) if want_K else None
    M = (M if M is not None else torch.empty((plan.nnz,), dtype=torch.float64, device=dev)) if want_M else None
    plan.classes()
    work = _work16(dev)
    _check(lib().fem_p1_assemble_classes(dim, nn, _ptr(coords), 1, nn, _ptr(plan.row_ptr), _ptr(plan.col_idx),
                                         plan.nnz, _ptr(plan.node_elem_ptr), _ptr(plan.node_elem_slot),
                                         _ptr(plan.class_rows), _ptr(plan.groups), plan.groups.shape[0], _ptr(K),
                                         _ptr(M), _ptr(work), _wb(), _stream(stream)))
    return K, M


def fem_p1_assemble(coords, elems, plan, mode=VB_ASSEMBLE_GATHER, want_K=True, want_M=True, want_local=False,
                    K=None, M=None, stream=None, compact=None, variant=None, degenerate=None):
    """Returns (K_vals, M_vals, K_local, M_local) (None where not requested).
    Gather mode: `variant` None (auto: lattice, else class / block as _use_classes),
    "lattice", "class", "block" or "tile".  degenerate: optional device int64 tensor (1,)
    receiving the number of degenerate elements (det = 0 as evaluated, or two identical
    vertices): every variant fills it (the class and tile calls through a counting-only
    fem_p1_assemble call)."""
    _f64(coords)
    dim, nn = coords.shape
    nv, ne = elems.shape
    dev = coords.device
    if want_K and K is None:
        K = torch.empty((plan.nnz,), dtype=torch.float64, device=dev)
    if want_M and M is None:
        M = torch.empty((plan.nnz,), dtype=torch.float64, device=dev)
    if not want_K:
        K = None
    if not want_M:
        M = None
    Kl = torch.empty((nv, nv, ne), dtype=torch.float64, device=dev) if want_local else None
    Ml = torch.empty((nv, nv, ne), dtype=torch.float64, device=dev) if want_local else None

    def count_only():   # the class and tile entry points take no counter: a counting-only call of the C entry
        if degenerate is not None:
            _check(lib().fem_p1_assemble(dim, nn, ne, _ptr(coords), 1, nn, _ptr(elems), ne, None, None, plan.nnz,
                                         None, None, None, None, None, None, None, None, VB_ASSEMBLE_ATOMIC,
                                         None, None, _ptr(degenerate), _stream(stream)))
    if (mode == VB_ASSEMBLE_GATHER and variant == "tile" and (K is not None or M is not None)
            and plan.tiles(coords, elems)):
        fem_p1_assemble_tiles(coords, plan, K=K, M=M, want_K=K is not None, want_M=M is not None, stream=stream)
        count_only()
        if want_local:
            _check(lib().fem_p1_assemble(dim, nn, ne, _ptr(coords), 1, nn, _ptr(elems), ne, None, None, plan.nnz,
                                         None, None, None, None, None, None, _ptr(Kl), _ptr(Ml), int(mode),
                                         None, None, None, _stream(stream)))
        return K, M, Kl, Ml
    if variant == "tile":
        variant = "block"   # outside the tile variant's limits (plan.tile_reason)
    if (mode == VB_ASSEMBLE_GATHER and variant in (None, "lattice") and (K is not None or M is not None)
            and plan.lattice(elems)):
        fem_p1_assemble_lattice(coords, plan, K=K, M=M, want_K=K is not None, want_M=M is not None, stream=stream,
                                degenerate=degenerate)
        if want_local:
            _check(lib().fem_p1_assemble(dim, nn, ne, _ptr(coords), 1, nn, _ptr(elems), ne, None, None, plan.nnz,
                                         None, None, None, None, None, None, _ptr(Kl), _ptr(Ml), int(mode),
                                         None, None, None, _stream(stream)))
        return K, M, Kl, Ml
    if variant == "lattice":
        variant = None   # not a Kuhn lattice (plan.lattice_reason)
    if mode == VB_ASSEMBLE_GATHER and (K is not None or M is not None) and _use_classes(plan, variant):
        fem_p1_assemble_classes(coords, plan, K=K, M=M, want_K=K is not None, want_M=M is not None, stream=stream)
        count_only()
        if want_local:
            _check(lib().fem_p1_assemble(dim, nn, ne, _ptr(coords), 1, nn, _ptr(elems), ne, None, None, plan.nnz,
                                         None, None, None, None, None, None, _ptr(Kl), _ptr(Ml), int(mode),
                                         None, None, None, _stream(stream)))
        return K, M, Kl, Ml
    gmode, words = _gather_mode(mode, plan, compact)
    work = _work16(dev)
    _check(lib().fem_p1_assemble(dim, nn, ne, _ptr(coords), 1, nn, _ptr(elems), ne, _ptr(plan.row_ptr),
                                 _ptr(plan.col_idx), plan.nnz, _ptr(plan.elem2nnz), _ptr(plan.node_elem_ptr),
                                 _ptr(plan.node_elem), _ptr(words), _ptr(K), _ptr(M), _ptr(Kl),
                                 _ptr(Ml), gmode, _ptr(work), _wb(), _ptr(degenerate), _stream(stream)))
    return K, M, Kl, Ml


def fem_p1_assemble_coef(coords, elems, plan, gqo=2, cK=(1.0, (1.0, 1.0, 1.0)), cM=(1.0, (1.0, 1.0, 1.0)),
                         mode=VB_ASSEMBLE_GATHER, want_K=True, want_M=True, want_local=False, K=None, M=None,
                         stream=None, compact=None, variant=None):
    """Coefficient-weighted K, M with c(x) = a * exp(b . x) (NEXT-1).  Returns
    (K_vals, M_vals, K_local, M_local).  Gather mode, gqo = 2, c_K = c_M:
    `variant` as _use_classes picks the row-class kernel
    (fem_p1_assemble_classes_coef) or the 32-row blocks; other cases run the
    blocks."""
    _f64(coords)
    dim, nn = coords.shape
    nv, ne = elems.shape
    dev = coords.device
    K = (K if K is not None else torch.empty((plan.nnz,), dtype=torch.float64, device=dev)) if want_K else None
    M = (M if M is not None else torch.empty((plan.nnz,), dtype=torch.float64, device=dev)) if want_M else None
    Kl = torch.empty((nv, nv, ne), dtype=torch.float64, device=dev) if want_local else None
    Ml = torch.empty((nv, nv, ne), dtype=torch.float64, device=dev) if want_local else None
    kb = (C.c_double * 3)(*[float(x) for x in list(cK[1])[:3]] + [0.0] * (3 - len(list(cK[1])[:3])))
    mb = (C.c_double * 3)(*[float(x) for x in list(cM[1])[:3]] + [0.0] * (3 - len(list(cM[1])[:3])))
    same = float(cK[0]) == float(cM[0]) and list(kb) == list(mb)
    if (mode == VB_ASSEMBLE_GATHER and int(gqo) == 2 and same and (K is not None or M is not None)
            and variant != "tile" and _use_classes(plan, variant, coef=True)):
        plan.classes()
        fac_work = torch.empty((2 * nn + 2,), dtype=torch.float64, device=dev)   # factors + the group counter
        _check(lib().fem_p1_assemble_classes_coef(dim, nn, _ptr(coords), 1, nn, _ptr(plan.row_ptr),
                                                  _ptr(plan.col_idx), plan.nnz, _ptr(plan.node_elem_ptr),
                                                  _ptr(plan.node_elem_slot), _ptr(plan.class_rows),
                                                  _ptr(plan.groups), plan.groups.shape[0], 2, float(cK[0]),
                                                  C.cast(kb, C.c_void_p), _ptr(fac_work), _ptr(K), _ptr(M),
                                                  _stream(stream)))
        if want_local:
            _check(lib().fem_p1_assemble_coef(dim, nn, ne, _ptr(coords), 1, nn, _ptr(elems), ne, None, None,
                                              plan.nnz, None, None, None, None, int(gqo), float(cK[0]),
                                              C.cast(kb, C.c_void_p), float(cM[0]), C.cast(mb, C.c_void_p), None,
                                              None, _ptr(Kl), _ptr(Ml), int(mode), None, None, None,
                                              _stream(stream)))
        return K, M, Kl, Ml
    gmode, words = _gather_mode(mode, plan, compact)
    work = _work16(dev)
    _check(lib().fem_p1_assemble_coef(dim, nn, ne, _ptr(coords), 1, nn, _ptr(elems), ne, _ptr(plan.row_ptr),
                                      _ptr(plan.col_idx), plan.nnz, _ptr(plan.elem2nnz), _ptr(plan.node_elem_ptr),
                                      _ptr(plan.node_elem), _ptr(words), int(gqo), float(cK[0]),
                                      C.cast(kb, C.c_void_p), float(cM[0]), C.cast(mb, C.c_void_p), _ptr(K), _ptr(M),
                                      _ptr(Kl), _ptr(Ml), gmode, _ptr(work), _wb(), None, _stream(stream)))
    return K, M, Kl, Ml


# ------------------------------------------------------------------ NEXT-2
def vb_quad_rule(dim, gqo):
    """(lam (nip, dim+1) numpy, w (nip,) numpy) of intquad(gqo, dim) as the kernels use it."""
    import numpy as np
    lam = np.zeros(16)
    w = np.zeros(4)
    nip = lib().vb_quad_rule(dim, gqo, lam.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p))
    if nip < 0:
        _check(nip)
    return lam[:nip * (dim + 1)].reshape(nip, dim + 1).copy(), w[:nip].copy()


def fem_p1_rhs(coords, elems, fq, plan=None, gqo=2, mode=VB_ASSEMBLE_GATHER, want_b2D=True, stream=None):
    """(b (nn,), b2D (nv, ne)) of Code rhs_vectorP1 with f values fq (nip, ne) at the
    integration points.  Gather mode needs the plan (node_elem_ptr, node_elem)."""
    _f64(coords), _f64(fq)
    dim, nn = coords.shape
    nv, ne = elems.shape
    dev = coords.device
    b = torch.empty((nn,), dtype=torch.float64, device=dev)
    b2 = torch.empty((nv, ne), dtype=torch.float64, device=dev) if (want_b2D or mode == VB_ASSEMBLE_GATHER) else None
    nptr = plan.node_elem_ptr if plan is not None else None
    nel = plan.node_elem if plan is not None else None
    _check(lib().fem_p1_rhs(dim, nn, ne, _ptr(coords), 1, nn, _ptr(elems), ne, int(gqo), _ptr(fq), _ptr(b2), _ptr(b),
                            _ptr(nptr), _ptr(nel), int(mode), _stream(stream)))
    return b, b2


def vb_page_bilinear(A, Mx, B, s=None, stream=None):
    """avtamav: s_k = a_k^T M_k b_k.  A (1, n, N|1), Mx (m, n, N|1), B (1, m, N|1)."""
    _f64(A), _f64(Mx), _f64(B)
    m, n, nm = Mx.shape
    N = max(A.shape[-1], nm, B.shape[-1])
    if s is None:
        s = torch.empty((N,), dtype=torch.float64, device=Mx.device)
    _check(lib().vb_page_bilinear(N, n, m, _ptr(A), _ld(A, N), _ptr(Mx), _ld(Mx, N), _ptr(B), _ld(B, N), _ptr(s),
                                  _stream(stream)))
    return s


# ------------------------------------------------------------------ NEXT-3 (P2)
class Plan:
    """Generic CSR pattern (fem_pattern) for elements with any node count, with
    the scatter map (elem2nnz) and / or the gather plan (node_elem_ptr,
    node_elem, node_elem_slot: ceil(nv/4) words per incidence)."""

    def __init__(self, elems, nn, scatter_map=True, gather_plan=True, stream=None):
        if elems.dtype != torch.int32:
            raise TypeError("elems must be int32")
        nv, ne = elems.shape
        self.nv, self.nn, self.ne = nv, int(nn), int(ne)
        dev = elems.device
        L = lib()
        sz = C.c_size_t(0)
        nnz = C.c_int64(0)
        st = _stream(stream)
        _check(L.fem_pattern(nv, nn, ne, None, ne, None, C.byref(sz), None, None, 0, None, None, None, None, None, st))
        work = torch.empty((max(sz.value, 16),), dtype=torch.uint8, device=dev)
        self.row_ptr = torch.empty((nn + 1,), dtype=torch.int32, device=dev)
        _check(L.fem_pattern(nv, nn, ne, _ptr(elems), ne, _ptr(work), C.byref(sz), _ptr(self.row_ptr), None, 0, None,
                             None, None, None, C.byref(nnz), st))
        self.nnz = int(nnz.value)
        col = torch.zeros((max(4, (self.nnz + 3) // 4 * 4),), dtype=torch.int32, device=dev)
        self.elem2nnz = torch.empty((nv * nv, ne), dtype=torch.int32, device=dev) if scatter_map else None
        if gather_plan:
            self.slot_words = (nv + 3) // 4
            self.node_elem_ptr = torch.empty((nn + 1,), dtype=torch.int32, device=dev)
            self.node_elem = torch.empty((max(nv * ne, 1),), dtype=torch.int32, device=dev)
            self.node_elem_slot = torch.empty((max(nv * ne * self.slot_words, 1),), dtype=torch.int32, device=dev)
        else:
            self.slot_words = 0
            self.node_elem_ptr = self.node_elem = self.node_elem_slot = None
        _check(L.fem_pattern(nv, nn, ne, _ptr(elems), ne, _ptr(work), C.byref(sz), _ptr(self.row_ptr), _ptr(col),
                             col.numel(), _ptr(self.elem2nnz), _ptr(self.node_elem_ptr), _ptr(self.node_elem),
                             _ptr(self.node_elem_slot), C.byref(nnz), st))
        self.col_idx = col[:self.nnz]


def fem_pattern(elems, nn, scatter_map=True, gather_plan=True, stream=None):
    return Plan(elems, nn, scatter_map, gather_plan, stream)


def fem_p2_assemble(coords, elems, plan, gqo=4, cK=(1.0, (1.0, 1.0, 1.0)), cM=(1.0, (1.0, 1.0, 1.0)),
                    mode=VB_ASSEMBLE_ATOMIC, want_K=True, want_M=True, want_local=False, K=None, M=None,
                    stream=None):
    """P2 stiffness / mass (NEXT-3).  mode VB_ASSEMBLE_ATOMIC (needs the plan's
    elem2nnz) or VB_ASSEMBLE_GATHER (deterministic; needs its gather plan).
    Returns (K_vals, M_vals, K_local, M_local)."""
    _f64(coords)
    dim, nn = coords.shape
    nlb, ne = elems.shape
    dev = coords.device
    K = (K if K is not None else torch.empty((plan.nnz,), dtype=torch.float64, device=dev)) if want_K else None
    M = (M if M is not None else torch.empty((plan.nnz,), dtype=torch.float64, device=dev)) if want_M else None
    Kl = torch.empty((nlb, nlb, ne), dtype=torch.float64, device=dev) if want_local else None
    Ml = torch.empty((nlb, nlb, ne), dtype=torch.float64, device=dev) if want_local else None
    kb = (C.c_double * 3)(*(list(map(float, cK[1]))[:3] + [0.0] * (3 - len(list(cK[1])[:3]))))
    mb = (C.c_double * 3)(*(list(map(float, cM[1]))[:3] + [0.0] * (3 - len(list(cM[1])[:3]))))
    L = lib()
    work, sz = None, C.c_size_t(0)
    if mode == VB_ASSEMBLE_GATHER:
        _check(L.fem_p2_assemble(dim, nn, ne, None, 1, nn, None, ne, None, None, plan.nnz, None, None, None,
                                 int(gqo), 0.0, None, 0.0, None, None, None, None, None, mode, None, C.byref(sz),
                                 None))
        work = torch.empty((max(sz.value, 16),), dtype=torch.uint8, device=dev)
    _check(L.fem_p2_assemble(dim, nn, ne, _ptr(coords), 1, nn, _ptr(elems), ne, _ptr(plan.row_ptr),
                             _ptr(plan.elem2nnz), plan.nnz, _ptr(plan.node_elem_ptr), _ptr(plan.node_elem),
                             _ptr(plan.node_elem_slot), int(gqo), float(cK[0]), C.cast(kb, C.c_void_p),
                             float(cM[0]), C.cast(mb, C.c_void_p), _ptr(K), _ptr(M), _ptr(Kl), _ptr(Ml), int(mode),
                             _ptr(work), C.byref(sz), _stream(stream)))
    return K, M, Kl, Ml
