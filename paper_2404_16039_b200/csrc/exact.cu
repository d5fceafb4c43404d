// Exact-order P1 assembly (fem_p1_assemble_exact): the verification path of
// SURVEY §8(c) "bitwise mode".  Every operation of the definition is an IEEE
// round-to-nearest fp64 operation written as an intrinsic (__dadd_rn, __dsub_rn,
// __dmul_rn, __ddiv_rn: nothing contracts to an FMA), in the order the
// definition is written out:
//   tjac = D X^T, J[r][c] = x_{r+1}[c] - x_0[c]                   (smamt)
//   det J by Laplace expansion along row 0 (cofactors of the 2x2 minors)
//                                                           (eq:det3)
//   |T| = |det J| / d!
//   Jinv[i][j] = (-1)^{i+j} minor(j, i) / det J        (adjugate, aminv)
//   G = Jinv D, D = [-1 | I], sums over l ascending               (amsm)
//   K_e[a][b] = |T| * sum_r G[r][a] G[r][b], r ascending     (amtam)
//   M_e[a][b] = (|T| / ((d+1)(d+2))) * (1 + delta_ab)
// and the duplicates of sparse(X3D(:),Y3D(:),..) are summed per
// CSR entry starting from 0 in ascending element id.  One thread per row walks
// its incidences (node_elem of fem_p1_pattern, ascending e) and finds each
// column by binary search.  The result is therefore the one any plain IEEE
// fp64 program computing the definition in that order gets, bit for bit.  It
// is slow by design (no staging, one element evaluation per incidence) and is
// used to check the fast variants over whole full-size matrices.
#include "vb_internal.cuh"

namespace vb {
namespace {

__device__ __forceinline__ double det2(double a00, double a01, double a10, double a11) {
    return __dsub_rn(__dmul_rn(a00, a11), __dmul_rn(a01, a10));
}

// Laplace expansion of a DIM x DIM matrix along row 0 (DIM = 2: the 2x2 formula)
template <int DIM>
__device__ __forceinline__ double det_laplace(const double (&a)[DIM][DIM]) {
    if constexpr (DIM == 2) {
        return det2(a[0][0], a[0][1], a[1][0], a[1][1]);
    } else {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < 3; c++) {
            const int c0 = c == 0 ? 1 : 0, c1 = c == 2 ? 1 : 2;   // the columns kept, ascending
            const double term = __dmul_rn(a[0][c], det2(a[1][c0], a[1][c1], a[2][c0], a[2][c1]));
            s = (c % 2 == 0) ? __dadd_rn(s, term) : __dsub_rn(s, term);
        }
        return s;
    }
}

// determinant of a with row r and column c removed
template <int DIM>
__device__ __forceinline__ double minor_rc(const double (&a)[DIM][DIM], int r, int c) {
    if constexpr (DIM == 2) {
        return a[1 - r][1 - c];
    } else {
        const int r0 = r == 0 ? 1 : 0, r1 = r == 2 ? 1 : 2;
        const int c0 = c == 0 ? 1 : 0, c1 = c == 2 ? 1 : 2;
        return det2(a[r0][c0], a[r0][c1], a[r1][c0], a[r1][c1]);
    }
}

template <int DIM>
__global__ void __launch_bounds__(128) assemble_exact_k(int64_t nn, const double* __restrict__ coords, int64_t ns,
                                                        int64_t cst, const int32_t* __restrict__ elems, int64_t eld,
                                                        const int32_t* __restrict__ row_ptr,
                                                        const int32_t* __restrict__ col_idx,
                                                        const int32_t* __restrict__ nptr,
                                                        const int32_t* __restrict__ nel, double* __restrict__ K,
                                                        double* __restrict__ M) {
    constexpr int NV = DIM + 1;
    constexpr double FACT = DIM == 3 ? 6.0 : 2.0;        // d!
    constexpr double MDEN = DIM == 3 ? 20.0 : 12.0;      // (d+1)(d+2)
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nn) return;
    const int lo = row_ptr[v], hi = row_ptr[v + 1];
    for (int p = lo; p < hi; p++) {
        if (K) K[p] = 0.0;
        if (M) M[p] = 0.0;
    }
    for (int i = nptr[v]; i < nptr[v + 1]; i++) {
        const int inc = nel[i];
        const int64_t e = inc >> 2;
        const int a = inc & 3;
        int32_t vid[NV];
        double X[DIM][NV];
#pragma unroll
        for (int b = 0; b < NV; b++) {
            vid[b] = elems[b * eld + e];
#pragma unroll
            for (int c = 0; c < DIM; c++) X[c][b] = coords[c * cst + (int64_t)vid[b] * ns];
        }
        double J[DIM][DIM];
#pragma unroll
        for (int r = 0; r < DIM; r++)
#pragma unroll
            for (int c = 0; c < DIM; c++) J[r][c] = __dsub_rn(X[c][r + 1], X[c][0]);
        const double detJ = det_laplace<DIM>(J);
        const double T = __ddiv_rn(fabs(detJ), FACT);
        double Ji[DIM][DIM];
#pragma unroll
        for (int r = 0; r < DIM; r++)
#pragma unroll
            for (int c = 0; c < DIM; c++) {
                double cof = minor_rc<DIM>(J, c, r);
                if ((r + c) % 2) cof = -cof;
                Ji[r][c] = __ddiv_rn(cof, detJ);
            }
        double G[DIM][NV];
#pragma unroll
        for (int r = 0; r < DIM; r++)
#pragma unroll
            for (int b = 0; b < NV; b++) {
                double s = 0.0;
#pragma unroll
                for (int l = 0; l < DIM; l++) {
                    const double dlb = b == 0 ? -1.0 : (l == b - 1 ? 1.0 : 0.0);
                    s = __dadd_rn(s, __dmul_rn(Ji[r][l], dlb));
                }
                G[r][b] = s;
            }
        const double mscale = __ddiv_rn(T, MDEN);
        for (int b = 0; b < NV; b++) {
            // position of column vid[b] in row v (present by construction of the pattern)
            int l0 = lo, l1 = hi;
            while (l0 < l1) {
                const int mid = (l0 + l1) >> 1;
                if (col_idx[mid] < vid[b]) l0 = mid + 1;
                else l1 = mid;
            }
            if (K) {
                double s = 0.0;
#pragma unroll
                for (int r = 0; r < DIM; r++) s = __dadd_rn(s, __dmul_rn(G[r][a], G[r][b]));
                K[l0] = __dadd_rn(K[l0], __dmul_rn(T, s));
            }
            if (M) M[l0] = __dadd_rn(M[l0], __dmul_rn(mscale, a == b ? 2.0 : 1.0));
        }
    }
}

}  // namespace
}  // namespace vb

using namespace vb;

extern "C" vb_status fem_p1_assemble_exact(int dim, int64_t nn, const double* coords, int64_t node_stride,
                                           int64_t comp_stride, const int32_t* elems, int64_t elem_ld,
                                           const int32_t* row_ptr, const int32_t* col_idx,
                                           const int32_t* node_elem_ptr, const int32_t* node_elem, double* K_vals,
                                           double* M_vals, vb_stream_t stream) {
    const char* fn = "fem_p1_assemble_exact";
    clear_error();
    if (dim != 2 && dim != 3) { set_error("%s: dim=%d, need 2 or 3", fn, dim); return VB_ERR_UNSUPPORTED; }
    if (nn < 0 || elem_ld < 0) { set_error("%s: negative size", fn); return VB_ERR_ARG; }
    if (nn == 0 || (!K_vals && !M_vals)) return VB_OK;
    if (!coords || !elems || !row_ptr || !col_idx || !node_elem_ptr || !node_elem) {
        set_error("%s: NULL argument", fn);
        return VB_ERR_ARG;
    }
    const unsigned g = (unsigned)((nn + 127) / 128);
    cudaStream_t s = cs(stream);
    if (dim == 3)
        assemble_exact_k<3><<<g, 128, 0, s>>>(nn, coords, node_stride, comp_stride, elems, elem_ld, row_ptr, col_idx,
                                              node_elem_ptr, node_elem, K_vals, M_vals);
    else
        assemble_exact_k<2><<<g, 128, 0, s>>>(nn, coords, node_stride, comp_stride, elems, elem_ld, row_ptr, col_idx,
                                              node_elem_ptr, node_elem, K_vals, M_vals);
    return launch_check(fn);
}
