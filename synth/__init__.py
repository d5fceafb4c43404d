"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module is the ONLY code both sides share, and it holds none of the
method's arithmetic (no products, determinants, inverses, cross products,
gradients or assembly): it only produces meshes and page batches with the
shapes, sizes and value distributions of the paper's workloads, as fixed by
BASELINE.json ``configs`` and SURVEY.md §8(d).  The recipe is restated in
DESIGN.md §"Input recipe".

Layouts produced here are the ones the C ABI consumes (include/vb.h):

* page batches: struct-of-arrays planes, entry (i, j) of page k at
  ``plane[(i + j*rows)][k]`` -> numpy array of shape (cols, rows, N), C order
  (column-major entries, page-contiguous, ld = N);
* meshes: ``coords`` shape (dim, nn) float64 (one plane per coordinate,
  node_stride = 1, comp_stride = nn); ``elems`` shape (nv, ne) int32, 0-based
  (vertex a of element e at ``elems[a, e]``, elem_ld = ne).
"""
from .rng import splitmix64_u64, uniform01, uniform_pm1, normal
from .meshes import (square_p1, rect_p1, square_crossed_p1, cube_kuhn_p1, box_kuhn_p1, icosphere, square_counts,
                     cube_counts, icosphere_counts, p2_from_p1, P2_EDGES, delaunay_p1,
                     permute_mesh)
from .pages import normal_pages, inverse_pages, integer_pages

__all__ = [
    "splitmix64_u64", "uniform01", "uniform_pm1", "normal",
    "square_p1", "rect_p1", "square_crossed_p1", "cube_kuhn_p1", "box_kuhn_p1", "icosphere",
    "square_counts", "cube_counts", "icosphere_counts", "delaunay_p1", "permute_mesh",
    "normal_pages", "inverse_pages", "integer_pages",
]
