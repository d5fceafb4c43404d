// NEXT-4, fused: signed sizes and outer normals of every simplex straight from coords and elems
// (P:612-627):   [~, vectors3D] = create_coords3D(coords, elems)
//                meass     = amdet(vectors3D) / factorial(dim)
//                normals3D = amsm(amt(aminv(vectors3D)), normalsRef)
// The page-op chain (vb_create_coords3D -> vb_page_det / vb_page_inv -> vb_page_transpose ->
// vb_page_mtimes) writes and re-reads vectors3D, its inverse and the transpose (544 B per tet); here one
// thread takes two consecutive elements, gathers their vertices once and writes only the results
// (16 B of indices + 8 + 96 B of output per tet), every plane with 128-bit stores.
//   V = [v_0 .. v_{d-1}], v_a = x_a - x_d (vectors from the LAST local node)
//   rows of V^{-1}: r_j = cofactor row j / det V  (3D: r_0 = v_1 x v_2 / det, r_1 = v_2 x v_0 / det,
//   r_2 = v_0 x v_1 / det), so with normalsRef = [-I | 1] column j < d of normals3D is
//   -r_j and the last column is r_0 + .. + r_{d-1}.
#include "vb_internal.cuh"

namespace vb {
namespace {

constexpr int GEO_BLOCK = 256;

template <int DIM>
__device__ __forceinline__ void simplex_one(const double (&x)[DIM + 1][DIM], double& meas,
                                            double (&nr)[DIM + 1][DIM]) {
    double v[DIM][DIM];
#pragma unroll
    for (int a = 0; a < DIM; a++)
#pragma unroll
        for (int c = 0; c < DIM; c++) v[a][c] = x[a][c] - x[DIM][c];
    double r[DIM][DIM], det;
    if constexpr (DIM == 2) {
        det = fma(v[0][0], v[1][1], -v[0][1] * v[1][0]);
        r[0][0] = v[1][1];
        r[0][1] = -v[1][0];
        r[1][0] = -v[0][1];
        r[1][1] = v[0][0];
        meas = det * 0.5;
    } else {
        r[0][0] = fma(v[1][1], v[2][2], -v[1][2] * v[2][1]);   // v_1 x v_2
        r[0][1] = fma(v[1][2], v[2][0], -v[1][0] * v[2][2]);
        r[0][2] = fma(v[1][0], v[2][1], -v[1][1] * v[2][0]);
        r[1][0] = fma(v[2][1], v[0][2], -v[2][2] * v[0][1]);   // v_2 x v_0
        r[1][1] = fma(v[2][2], v[0][0], -v[2][0] * v[0][2]);
        r[1][2] = fma(v[2][0], v[0][1], -v[2][1] * v[0][0]);
        r[2][0] = fma(v[0][1], v[1][2], -v[0][2] * v[1][1]);   // v_0 x v_1
        r[2][1] = fma(v[0][2], v[1][0], -v[0][0] * v[1][2]);
        r[2][2] = fma(v[0][0], v[1][1], -v[0][1] * v[1][0]);
        det = fma(v[0][0], r[0][0], fma(v[0][1], r[0][1], v[0][2] * r[0][2]));
        meas = det / 6.0;
    }
    const double q = 1.0 / det;
#pragma unroll
    for (int c = 0; c < DIM; c++) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < DIM; j++) {
            const double t = r[j][c] * q;
            nr[j][c] = -t;
            s += t;
        }
        nr[DIM][c] = s;
    }
}

// Resident blocks per SM: with normals 4 (64 registers, a few spilled words: configs[4] normals 0.306 -> 0.289 ms
// against 2 blocks; 3 measured slower); sizes alone (NRM = false: no cofactors kept) VB_GEO_MINB_M.
#ifndef VB_GEO_MINB
#define VB_GEO_MINB 4
#endif
#ifndef VB_GEO_MINB_M
#define VB_GEO_MINB_M 5   // 48 registers, no spills: configs[4] sizes 0.105 ms (6: 40 registers with spills 0.140; 8: 0.190)
#endif
template <int DIM, bool VEC, bool NRM>
__global__ void __launch_bounds__(GEO_BLOCK, NRM ? VB_GEO_MINB : VB_GEO_MINB_M) simplex_geometry_k(int64_t ne, const double* __restrict__ coords,
                                                                int64_t ns, int64_t cst,
                                                                const int32_t* __restrict__ elems, int64_t eld,
                                                                double* __restrict__ meass,
                                                                double* __restrict__ nrm, int64_t ldn) {
    constexpr int NV = DIM + 1;
    const int64_t npair = (ne + 1) / 2;
    const int64_t stride = (int64_t)gridDim.x * GEO_BLOCK;
    for (int64_t t = (int64_t)blockIdx.x * GEO_BLOCK + threadIdx.x; t < npair; t += stride) {
        const int64_t e0 = 2 * t;
        const bool two = e0 + 1 < ne;
        int32_t vi[2][NV];
#pragma unroll
        for (int a = 0; a < NV; a++) {
            if (VEC && two) {
                const int2 p = __ldcs(reinterpret_cast<const int2*>(elems + a * eld + e0));
                vi[0][a] = p.x;
                vi[1][a] = p.y;
            } else {
                vi[0][a] = __ldcs(elems + a * eld + e0);
                vi[1][a] = two ? __ldcs(elems + a * eld + e0 + 1) : vi[0][a];
            }
        }
        double x[2][NV][DIM];
#pragma unroll
        for (int k = 0; k < 2; k++)
#pragma unroll
            for (int a = 0; a < NV; a++)
#pragma unroll
                for (int c = 0; c < DIM; c++) x[k][a][c] = __ldg(coords + c * cst + (int64_t)vi[k][a] * ns);
        double m[2], nr[2][NV][DIM];
        simplex_one<DIM>(x[0], m[0], nr[0]);   // NRM = false: the normals are dead code
        simplex_one<DIM>(x[1], m[1], nr[1]);
        if (VEC && two) {
            if (meass) stcs2(meass + e0, make_double2(m[0], m[1]));
            if (NRM) {
#pragma unroll
                for (int j = 0; j < NV; j++)
#pragma unroll
                    for (int c = 0; c < DIM; c++)
                        stcs2(nrm + (int64_t)(c + j * DIM) * ldn + e0, make_double2(nr[0][j][c], nr[1][j][c]));
            }
        } else {
#pragma unroll
            for (int k = 0; k < 2; k++) {
                if (k == 1 && !two) break;
                if (meass) stcs(meass + e0 + k, m[k]);
                if (NRM) {
#pragma unroll
                    for (int j = 0; j < NV; j++)
#pragma unroll
                        for (int c = 0; c < DIM; c++) stcs(nrm + (int64_t)(c + j * DIM) * ldn + e0 + k, nr[k][j][c]);
                }
            }
        }
    }
}

}  // namespace
}  // namespace vb

using namespace vb;

extern "C" vb_status vb_simplex_geometry(int dim, int64_t ne, const double* coords, int64_t node_stride,
                                         int64_t comp_stride, const int32_t* elems, int64_t elem_ld, double* meass,
                                         double* normals3D, int64_t ldn, vb_stream_t stream) {
    clear_error();
    const char* fn = "vb_simplex_geometry";
    if (ne < 0) { set_error("%s: ne < 0", fn); return VB_ERR_ARG; }
    if (dim != 2 && dim != 3) { set_error("%s: dim=%d, need 2 or 3", fn, dim); return VB_ERR_UNSUPPORTED; }
    if (ne == 0) return VB_OK;
    if (!coords || !elems || (!meass && !normals3D)) { set_error("%s: NULL argument", fn); return VB_ERR_ARG; }
    if (elem_ld < ne) { set_error("%s: elem_ld < ne", fn); return VB_ERR_ARG; }
    if (normals3D && ldn < ne) { set_error("%s: ldn < ne", fn); return VB_ERR_ARG; }
    // 128-bit path: every plane starts 16-byte aligned (elems planes 8-byte aligned for the index pairs)
    const bool vec = (!meass || aligned16(meass)) && (!normals3D || (aligned16(normals3D) && (ldn & 1) == 0)) &&
                     (reinterpret_cast<uintptr_t>(elems) & 7u) == 0 && (elem_ld & 1) == 0;
    const bool nrm = normals3D != nullptr;
    const unsigned g = grid_for((ne + 1) / 2, GEO_BLOCK, nrm ? VB_GEO_MINB : VB_GEO_MINB_M);
    cudaStream_t s = cs(stream);
#define VB_GEO(D, V, N) \
    simplex_geometry_k<D, V, N><<<g, GEO_BLOCK, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, meass, normals3D, ldn)
#define VB_GEO2(D, V) \
    do { if (nrm) VB_GEO(D, V, true); else VB_GEO(D, V, false); } while (0)
    if (dim == 2) {
        if (vec) VB_GEO2(2, true); else VB_GEO2(2, false);
    } else {
        if (vec) VB_GEO2(3, true); else VB_GEO2(3, false);
    }
#undef VB_GEO2
#undef VB_GEO
    return launch_check(fn);
}
