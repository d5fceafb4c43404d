"""C-ABI contract tests that need no GPU: libvb.so loads, exports every
symbol include/vb.h declares, and argument/shape errors are reported
synchronously (before any CUDA call) with a message naming the argument."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2404_16039_b200 import _build
    _build.build()
    from paper_2404_16039_b200 import vb
    return vb.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "vb.h")).read()
    return sorted(set(re.findall(r"VB_API\s+[\w\s\*]+?\b(\w+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = declared_symbols()
    for n in ("vb_page_mtimes", "vb_page_transpose", "vb_page_det", "vb_page_inv", "vb_page_cross",
              "fem_p1_pattern", "fem_p1_assemble"):
        assert n in names


def test_library_exports_every_declared_symbol(L):
    from paper_2404_16039_b200 import vb
    out = subprocess.check_output(["nm", "-D", "--defined-only", vb.LIB_PATH]).decode()
    exported = set(re.findall(r" T (\w+)$", out, flags=re.M))
    for n in declared_symbols():
        assert n in exported, n
        assert hasattr(L, n)
    assert set(vb.EXPORTS) == set(declared_symbols())
    assert L.vb_abi_version() == 2


def test_sm100a_code_only(L):
    from paper_2404_16039_b200 import vb
    out = subprocess.check_output(["cuobjdump", "--list-elf", vb.LIB_PATH]).decode()
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


FAKE = C.c_void_p(0x1000)


def test_mtimes_dimension_errors(L):
    rc = L.vb_page_mtimes(8, FAKE, 3, 2, 8, 0, FAKE, 3, 3, 8, 0, FAKE, 8, None)
    assert rc == -2 and b"inner dimension" in L.vb_last_error()
    rc = L.vb_page_mtimes(8, FAKE, 5, 2, 8, 0, FAKE, 2, 3, 8, 0, FAKE, 8, None)
    assert rc == -3
    rc = L.vb_page_mtimes(8, FAKE, 3, 2, 4, 0, FAKE, 2, 3, 8, 0, FAKE, 8, None)
    assert rc == -1 and b"leading dimension" in L.vb_last_error()
    rc = L.vb_page_mtimes(8, None, 3, 2, 8, 0, FAKE, 2, 3, 8, 0, FAKE, 8, None)
    assert rc == -1 and b"NULL X" in L.vb_last_error()
    assert L.vb_page_mtimes(0, None, 3, 2, 0, 0, None, 2, 3, 0, 0, None, 0, None) == 0   # empty batch


def test_det_inv_transpose_cross_errors(L):
    assert L.vb_page_det(4, 5, FAKE, 4, FAKE, None) == -3
    assert L.vb_page_det(-1, 2, FAKE, 4, FAKE, None) == -1
    assert L.vb_page_inv(4, 0, FAKE, 4, FAKE, 4, None, None, 1e-14, None) == -3
    assert L.vb_page_transpose(4, FAKE, 2, 7, 4, FAKE, 4, None) == -3
    assert L.vb_page_cross(4, FAKE, 2, FAKE, 4, FAKE, 4, None) == -1


def test_simplex_geometry_argument_errors(L):
    assert L.vb_simplex_geometry(3, -1, FAKE, 1, 8, FAKE, 8, FAKE, FAKE, 8, None) == -1      # ne < 0
    assert L.vb_simplex_geometry(4, 8, FAKE, 1, 8, FAKE, 8, FAKE, FAKE, 8, None) == -3       # dim
    assert L.vb_simplex_geometry(3, 0, None, 1, 8, None, 0, None, None, 0, None) == 0        # empty: nothing to do
    assert L.vb_simplex_geometry(3, 8, FAKE, 1, 8, FAKE, 8, None, None, 8, None) == -1       # no output
    assert L.vb_simplex_geometry(3, 8, FAKE, 1, 8, FAKE, 7, FAKE, FAKE, 8, None) == -1       # elem_ld < ne
    assert L.vb_simplex_geometry(3, 8, FAKE, 1, 8, FAKE, 8, FAKE, FAKE, 7, None) == -1       # ldn < ne
    assert b"ldn" in L.vb_last_error()


def test_fem_argument_errors(L):
    nnz = C.c_int64(0)
    sz = C.c_size_t(0)
    assert L.fem_p1_pattern(4, 10, 10, FAKE, 10, None, C.byref(sz), FAKE, None, 0, None, None, None, None,
                            C.byref(nnz), None) == -3
    assert L.fem_p1_pattern(3, 10, 1 << 29, FAKE, 1 << 29, None, C.byref(sz), FAKE, None, 0, None, None, None, None,
                            C.byref(nnz), None) == -4
    # work-size query needs no GPU and grows with the mesh
    assert L.fem_p1_pattern(3, 1000, 6000, None, 6000, None, C.byref(sz), None, None, 0, None, None, None, None,
                            None, None) == 0
    small = sz.value
    assert L.fem_p1_pattern(3, 2000, 12000, None, 12000, None, C.byref(sz), None, None, 0, None, None, None, None,
                            None, None) == 0
    assert sz.value > small
    assert L.fem_p1_assemble(3, 10, 10, FAKE, 1, 10, FAKE, 10, FAKE, FAKE, 5, None, None, None, None, FAKE, None,
                             None, None, 7, None, None, None, None) == -1
    assert L.fem_p1_assemble(3, 10, 10, FAKE, 1, 10, FAKE, 10, FAKE, FAKE, 5, None, None, None, None, FAKE, None,
                             None, None, 0, None, None, None, None) == -1   # atomic mode without elem2nnz
    assert b"elem2nnz" in L.vb_last_error()


def test_assembly_work_convention(L):
    """The launch's block counter lives in caller-owned work (vb.h, fem_p1_assemble): work == NULL with
    work_bytes is a size query that does nothing else; a buffer smaller than queried is refused."""
    assert L.vb_abi_version() == 2
    sz = C.c_size_t(0)
    assert L.fem_p1_assemble(3, 10, 10, FAKE, 1, 10, FAKE, 10, FAKE, FAKE, 5, None, None, None, None, FAKE, FAKE,
                             None, None, 1, None, C.byref(sz), None, None) == 0
    assert sz.value == 16
    small = C.c_size_t(8)
    assert L.fem_p1_assemble(3, 10, 10, FAKE, 1, 10, FAKE, 10, FAKE, FAKE, 5, None, None, None, None, FAKE, FAKE,
                             None, None, 1, FAKE, C.byref(small), None, None) == -5
    sz = C.c_size_t(0)
    assert L.fem_p1_assemble_coef(3, 10, 10, FAKE, 1, 10, FAKE, 10, FAKE, FAKE, 5, None, None, None, None, 2, 1.0,
                                  None, 1.0, None, FAKE, FAKE, None, None, 1, None, C.byref(sz), None, None) == 0
    assert sz.value == 16
    sz = C.c_size_t(0)
    assert L.fem_p1_assemble_classes(3, 10, FAKE, 1, 10, FAKE, FAKE, 5, FAKE, FAKE, FAKE, FAKE, 1, FAKE, FAKE, None,
                                     C.byref(sz), None) == 0
    assert sz.value == 16
    assert L.fem_p1_assemble_classes(3, 10, FAKE, 1, 10, FAKE, FAKE, 5, FAKE, FAKE, FAKE, FAKE, 1, FAKE, FAKE, FAKE,
                                     C.byref(small), None) == -5


def test_lattice_plan_query_and_argument_errors(L):
    wb, pi = C.c_size_t(0), C.c_int64(0)
    stats = (C.c_int64 * 4)()
    # size query (no GPU): plan ints = header + 32 lane descriptors (int4) per tile + 1025 CTA range bounds
    assert L.fem_plan_lattice(129 ** 3, 6 * 128 ** 3, None, 6 * 128 ** 3, None, None, 0, 128, 128, 128, None,
                              C.byref(wb), None, C.byref(pi), stats, None) == 0
    assert wb.value > 6 * 128 ** 3 // 8 and (pi.value - 16 - 1025) % 128 == 0 and pi.value > 16 + 1025
    assert L.fem_plan_lattice(8, 6, None, 6, None, None, 0, 0, 1, 1, None, C.byref(wb), None, C.byref(pi), stats,
                              None) == -1
    # closed-form pattern: nnz of the 15-point stencil (query, no GPU) = sum over directions of the node boxes
    nz_ = C.c_int64(0)
    assert L.fem_lattice_pattern(129 ** 3, 128, 128, 128, 0, None, C.byref(wb), None, None, 0, C.byref(nz_), None) == 0
    assert nz_.value == 31802497 and wb.value > 4 * 129 ** 3
    assert L.fem_lattice_pattern(28, 2, 2, 2, 0, None, C.byref(wb), None, None, 0, C.byref(nz_), None) == -1
    # the assembly refuses inconsistent counts and lattices below the kernel's limits, before any CUDA call
    assert L.fem_p1_assemble_lattice(9, FAKE, 1, 9, FAKE, 0, FAKE, 1, 1, 1, 0, FAKE, FAKE, None, None) == -1
    assert L.fem_p1_assemble_lattice(18, FAKE, 1, 18, FAKE, 0, FAKE, 1, 2, 2, 0, FAKE, FAKE, None, None) == -1
    assert b"nx, ny >= 2" in L.vb_last_error() or b"nn" in L.vb_last_error()


def test_tile_and_exact_argument_errors(L):
    sz = C.c_size_t(0)
    stats = (C.c_int64 * 6)()
    # fem_plan_tiles: unsupported dim, NULL work_bytes, size overflow; the work-size query needs no GPU
    assert L.fem_plan_tiles(4, 10, 10, FAKE, 1, 10, FAKE, 10, FAKE, FAKE, None, C.byref(sz), None, None, None, None,
                            None, 0, stats, None) == -3
    assert L.fem_plan_tiles(3, 10, 10, FAKE, 1, 10, FAKE, 10, FAKE, FAKE, None, None, None, None, None, None,
                            None, 0, stats, None) == -1
    assert L.fem_plan_tiles(3, 1 << 30, 10, FAKE, 1, 10, FAKE, 10, FAKE, FAKE, None, C.byref(sz), None, None, None,
                            None, None, 0, stats, None) == -4
    assert L.fem_plan_tiles(3, 1000, 6000, None, 1, 1000, None, 6000, None, None, None, C.byref(sz), None, None, None,
                            None, None, 0, stats, None) == 0
    assert sz.value > 0
    # fem_p1_assemble_tiles: nloc_max beyond the node table, bad dim
    assert L.fem_p1_assemble_tiles(3, 10, FAKE, 1, 10, 5, FAKE, FAKE, FAKE, FAKE, FAKE, 4096, 10, FAKE, FAKE,
                                   None) == -1
    assert b"nloc_max" in L.vb_last_error()
    assert L.fem_p1_assemble_tiles(1, 10, FAKE, 1, 10, 5, FAKE, FAKE, FAKE, FAKE, FAKE, 10, 10, FAKE, FAKE,
                                   None) == -3
    # fem_p1_assemble_exact: bad dim, missing gather lists
    assert L.fem_p1_assemble_exact(5, 10, FAKE, 1, 10, FAKE, 10, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, None) == -3
    assert L.fem_p1_assemble_exact(3, 10, FAKE, 1, 10, FAKE, 10, FAKE, FAKE, None, None, FAKE, FAKE, None) == -1
    # nothing requested: a no-op
    assert L.fem_p1_assemble_exact(3, 10, FAKE, 1, 10, FAKE, 10, FAKE, FAKE, None, None, None, None, None) == 0
