"""B200-native page-wise fp64 linear algebra and P1 FEM assembly (arXiv 2404.16039 hot path).

The product is the C ABI in include/vb.h, implemented by libvb.so (hand-written
sm_100a CUDA kernels under csrc/).  ``vb`` is its thin Python binding.
"""
from . import vb  # noqa: F401
from .vb import (VB_ASSEMBLE_ATOMIC, VB_ASSEMBLE_GATHER, P1Plan, VbError, fem_p1_assemble,  # noqa: F401
                 fem_p1_assemble_coef,
                 fem_p1_pattern, vb_create_coords3D, vb_page_cross, vb_page_det, vb_page_inv, vb_page_mtimes,
                 vb_page_transpose, vb_tri_surface)
