// a7-a17: fused P1 stiffness + mass assembly (c_K = c_M = 1).
//
// Element math (Code phider P:929-947, stiffness_matrixP1 P:978-1004):
//   tjac = D X^T  (J[r][c] = x_{r+1}[c] - x_0[c]),   detJ,   |T| = |detJ| / d!
//   G = tjac^{-1} D = H / detJ  with  H = adj(tjac) D  (H_0 = -sum_b H_b)
//   K_e[a][b] = |T| G_a . G_b = (H_a . H_b) / (d! |detJ|)     (one reciprocal)
//   M_e[a][b] = |T| / ((d+1)(d+2)) (1 + delta_ab)
//
// Two ways to sum duplicates (MATLAB sparse()):
//   * assemble_atomic_k: one thread per element, 2*nv^2 fp64 RED.ADD through the
//     element-to-nnz scatter map (north_star design; order unspecified, B13);
//   * assemble_gather_k: deterministic segmented reduction, one thread per row:
//     the row's incident elements (ascending e) are evaluated, row a of K_e/M_e
//     is added into the row's slots kept in shared memory, and the CTA's
//     contiguous CSR range is written once with coalesced stores (no atomics,
//     no zero-fill, no read-modify-write of K/M in HBM).
#include "vb_internal.cuh"

namespace vb {
namespace {

template <int DIM>
struct P1 {
    static constexpr double INV_DFACT = DIM == 2 ? 0.5 : 1.0 / 6.0;
    static constexpr double MFACT = DIM == 2 ? 1.0 / 24.0 : 1.0 / 120.0;  // 1/(d! (d+1)(d+2))
};

// H = adj(tjac) D (DIM x NV) and detJ from the element's vertex coordinates x[NV][DIM].
template <int DIM>
__device__ __forceinline__ double element_H(const double (&x)[DIM + 1][DIM], double (&H)[DIM][DIM + 1]) {
    double J[DIM][DIM];
#pragma unroll
    for (int r = 0; r < DIM; r++)
#pragma unroll
        for (int c = 0; c < DIM; c++) J[r][c] = x[r + 1][c] - x[0][c];
    double det;
    if constexpr (DIM == 2) {
        // adj = [[J11, -J01], [-J10, J00]]
        H[0][1] = J[1][1];
        H[0][2] = -J[0][1];
        H[1][1] = -J[1][0];
        H[1][2] = J[0][0];
        det = fma(J[0][0], J[1][1], -J[0][1] * J[1][0]);
    } else {
        // adj(i,j) = cofactor C_ji
        H[0][1] = fma(J[1][1], J[2][2], -J[1][2] * J[2][1]);
        H[1][1] = fma(J[1][2], J[2][0], -J[1][0] * J[2][2]);
        H[2][1] = fma(J[1][0], J[2][1], -J[1][1] * J[2][0]);
        H[0][2] = fma(J[0][2], J[2][1], -J[0][1] * J[2][2]);
        H[1][2] = fma(J[0][0], J[2][2], -J[0][2] * J[2][0]);
        H[2][2] = fma(J[0][1], J[2][0], -J[0][0] * J[2][1]);
        H[0][3] = fma(J[0][1], J[1][2], -J[0][2] * J[1][1]);
        H[1][3] = fma(J[0][2], J[1][0], -J[0][0] * J[1][2]);
        H[2][3] = fma(J[0][0], J[1][1], -J[0][1] * J[1][0]);
        det = fma(J[0][0], H[0][1], fma(J[0][1], H[1][1], J[0][2] * H[2][1]));
    }
#pragma unroll
    for (int r = 0; r < DIM; r++) {
        double s = H[r][1];
#pragma unroll
        for (int b = 2; b <= DIM; b++) s += H[r][b];
        H[r][0] = -s;
    }
    return det;
}

template <int DIM>
__device__ __forceinline__ void load_element(int64_t e, const int32_t* __restrict__ elems, int64_t eld,
                                             const double* __restrict__ coords, int64_t ns, int64_t cst,
                                             int32_t (&vid)[DIM + 1], double (&x)[DIM + 1][DIM]) {
#pragma unroll
    for (int a = 0; a <= DIM; a++) vid[a] = __ldg(elems + a * eld + e);
#pragma unroll
    for (int a = 0; a <= DIM; a++)
#pragma unroll
        for (int c = 0; c < DIM; c++) x[a][c] = __ldg(coords + c * cst + (int64_t)vid[a] * ns);
}

// ------------------------------------------------------------ zero fill
__global__ void zero2_k(double* __restrict__ a, double* __restrict__ b, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (a) a[i] = 0.0;
        if (b) b[i] = 0.0;
    }
}

// ------------------------------------------------------------ atomic variant
template <int DIM>
__global__ void __launch_bounds__(256) assemble_atomic_k(int64_t ne, const double* __restrict__ coords, int64_t ns,
                                                         int64_t cst, const int32_t* __restrict__ elems, int64_t eld,
                                                         const int32_t* __restrict__ e2n, double* __restrict__ K,
                                                         double* __restrict__ M, double* __restrict__ Kl,
                                                         double* __restrict__ Ml) {
    constexpr int NV = DIM + 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += stride) {
        int32_t vid[NV];
        double x[NV][DIM], H[DIM][NV];
        load_element<DIM>(e, elems, eld, coords, ns, cst, vid, x);
        double det = element_H<DIM>(x, H);
        double adet = fabs(det);
        double s = P1<DIM>::INV_DFACT / adet;
        double m = P1<DIM>::MFACT * adet;
#pragma unroll
        for (int a = 0; a < NV; a++)
#pragma unroll
            for (int b = a; b < NV; b++) {
                double d = H[0][a] * H[0][b];
#pragma unroll
                for (int r = 1; r < DIM; r++) d = fma(H[r][a], H[r][b], d);
                double k = s * d;
                double mm = (a == b) ? 2.0 * m : m;
                int32_t pab = __ldcs(e2n + (int64_t)(a * NV + b) * ne + e);
                if (K) atomicAdd(K + pab, k);
                if (M) atomicAdd(M + pab, mm);
                if (Kl) stcs(Kl + (int64_t)(a + b * NV) * ne + e, k);
                if (Ml) stcs(Ml + (int64_t)(a + b * NV) * ne + e, mm);
                if (a != b) {
                    int32_t pba = __ldcs(e2n + (int64_t)(b * NV + a) * ne + e);
                    if (K) atomicAdd(K + pba, k);
                    if (M) atomicAdd(M + pba, mm);
                    if (Kl) stcs(Kl + (int64_t)(b + a * NV) * ne + e, k);
                    if (Ml) stcs(Ml + (int64_t)(b + a * NV) * ne + e, mm);
                }
            }
    }
}

// ------------------------------------------------------------ local matrices only
template <int DIM>
__global__ void __launch_bounds__(256) local_k(int64_t ne, const double* __restrict__ coords, int64_t ns, int64_t cst,
                                               const int32_t* __restrict__ elems, int64_t eld, double* __restrict__ Kl,
                                               double* __restrict__ Ml) {
    constexpr int NV = DIM + 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += stride) {
        int32_t vid[NV];
        double x[NV][DIM], H[DIM][NV];
        load_element<DIM>(e, elems, eld, coords, ns, cst, vid, x);
        double det = element_H<DIM>(x, H);
        double adet = fabs(det);
        double s = P1<DIM>::INV_DFACT / adet;
        double m = P1<DIM>::MFACT * adet;
#pragma unroll
        for (int a = 0; a < NV; a++)
#pragma unroll
            for (int b = a; b < NV; b++) {
                double d = H[0][a] * H[0][b];
#pragma unroll
                for (int r = 1; r < DIM; r++) d = fma(H[r][a], H[r][b], d);
                double k = s * d, mm = (a == b) ? 2.0 * m : m;
                if (Kl) { stcs(Kl + (int64_t)(a + b * NV) * ne + e, k); if (a != b) stcs(Kl + (int64_t)(b + a * NV) * ne + e, k); }
                if (Ml) { stcs(Ml + (int64_t)(a + b * NV) * ne + e, mm); if (a != b) stcs(Ml + (int64_t)(b + a * NV) * ne + e, mm); }
            }
    }
}

// ------------------------------------------------------------ gather (deterministic) variant
constexpr int GATHER_BLOCK = 128;
template <int DIM>
struct GatherCfg {
    static constexpr int SLOTS_PER_ROW = DIM == 2 ? 10 : 20;           // smem budget per row (average)
    static constexpr int CAP = GATHER_BLOCK * SLOTS_PER_ROW;          // doubles per matrix per CTA
};

// Accumulate row v (owned by this thread) into accK/accM (indices relative to
// the row start `lo`).  ACC points to shared or global memory.
template <int DIM>
__device__ __forceinline__ void gather_row(int64_t v, const double* __restrict__ coords, int64_t ns, int64_t cst,
                                           const int32_t* __restrict__ elems, int64_t eld,
                                           const int32_t* __restrict__ nptr, const int32_t* __restrict__ nelem,
                                           const uint32_t* __restrict__ nslot, double* accK, double* accM) {
    constexpr int NV = DIM + 1;
    int i0 = __ldg(nptr + v), i1 = __ldg(nptr + v + 1);
    for (int i = i0; i < i1; i++) {
        int32_t ea = __ldcs(nelem + i);
        uint32_t sl = __ldcs(nslot + i);
        int64_t e = ea >> 2;
        int a = ea & 3;
        int32_t vid[NV];
        double x[NV][DIM], H[DIM][NV];
        load_element<DIM>(e, elems, eld, coords, ns, cst, vid, x);
        double det = element_H<DIM>(x, H);
        double adet = fabs(det);
        double s = P1<DIM>::INV_DFACT / adet;
        double m = P1<DIM>::MFACT * adet;
        double h[DIM];
#pragma unroll
        for (int r = 0; r < DIM; r++) {
            double t = H[r][0];
#pragma unroll
            for (int b = 1; b < NV; b++) t = (a == b) ? H[r][b] : t;
            h[r] = s * t;
        }
#pragma unroll
        for (int b = 0; b < NV; b++) {
            double d = h[0] * H[0][b];
#pragma unroll
            for (int r = 1; r < DIM; r++) d = fma(h[r], H[r][b], d);
            int slot = (sl >> (8 * b)) & 0xff;
            if (accK) accK[slot] += d;
            if (accM) accM[slot] += (a == b) ? 2.0 * m : m;
        }
    }
}

template <int DIM>
__global__ void __launch_bounds__(GATHER_BLOCK) assemble_gather_k(int64_t nn, const double* __restrict__ coords,
                                                                  int64_t ns, int64_t cst,
                                                                  const int32_t* __restrict__ elems, int64_t eld,
                                                                  const int32_t* __restrict__ row_ptr,
                                                                  const int32_t* __restrict__ nptr,
                                                                  const int32_t* __restrict__ nelem,
                                                                  const uint32_t* __restrict__ nslot,
                                                                  double* __restrict__ K, double* __restrict__ M) {
    constexpr int CAP = GatherCfg<DIM>::CAP;
    extern __shared__ double smem[];
    double* sK = smem;
    double* sM = smem + CAP;
    for (int64_t r0 = (int64_t)blockIdx.x * GATHER_BLOCK; r0 < nn; r0 += (int64_t)gridDim.x * GATHER_BLOCK) {
        int64_t rend = r0 + GATHER_BLOCK < nn ? r0 + GATHER_BLOCK : nn;
        int32_t p0 = __ldg(row_ptr + r0), p1 = __ldg(row_ptr + rend);
        int64_t v = r0 + threadIdx.x;
        bool own = v < rend;
        if (p1 - p0 <= CAP) {
            // zero the CTA's range, accumulate per row in smem, write the range once
            for (int q = threadIdx.x; q < p1 - p0; q += GATHER_BLOCK) {
                sK[q] = 0.0;
                sM[q] = 0.0;
            }
            __syncthreads();
            if (own) {
                int lo = __ldg(row_ptr + v) - p0;
                gather_row<DIM>(v, coords, ns, cst, elems, eld, nptr, nelem, nslot, K ? sK + lo : nullptr,
                                M ? sM + lo : nullptr);
            }
            __syncthreads();
            for (int q = threadIdx.x; q < p1 - p0; q += GATHER_BLOCK) {
                if (K) stcs(K + p0 + q, sK[q]);
                if (M) stcs(M + p0 + q, sM[q]);
            }
            __syncthreads();
        } else if (own) {
            // long rows: same per-row ownership, accumulated in place in HBM
            int lo = __ldg(row_ptr + v), hi = __ldg(row_ptr + v + 1);
            for (int q = lo; q < hi; q++) {
                if (K) K[q] = 0.0;
                if (M) M[q] = 0.0;
            }
            gather_row<DIM>(v, coords, ns, cst, elems, eld, nptr, nelem, nslot, K ? K + lo : nullptr,
                            M ? M + lo : nullptr);
        }
    }
}

}  // namespace
}  // namespace vb

using namespace vb;

extern "C" vb_status fem_p1_assemble(int dim, int64_t nn, int64_t ne, const double* coords, int64_t node_stride,
                                     int64_t comp_stride, const int32_t* elems, int64_t elem_ld,
                                     const int32_t* row_ptr, const int32_t* col_idx, int64_t nnz,
                                     const int32_t* elem2nnz, const int32_t* node_elem_ptr, const int32_t* node_elem,
                                     const uint32_t* node_elem_slot, double* K_vals, double* M_vals, double* K_local,
                                     double* M_local, int mode, vb_stream_t stream) {
    clear_error();
    if (dim != 2 && dim != 3) { set_error("fem_p1_assemble: dim=%d, need 2 or 3", dim); return VB_ERR_UNSUPPORTED; }
    if (nn < 0 || ne < 0 || nnz < 0) { set_error("fem_p1_assemble: negative size"); return VB_ERR_ARG; }
    if (mode != VB_ASSEMBLE_ATOMIC && mode != VB_ASSEMBLE_GATHER) { set_error("fem_p1_assemble: unknown mode %d", mode); return VB_ERR_ARG; }
    if (ne > 0 && (!coords || !elems)) { set_error("fem_p1_assemble: NULL %s", !coords ? "coords" : "elems"); return VB_ERR_ARG; }
    if (elem_ld < ne) { set_error("fem_p1_assemble: elem_ld < ne"); return VB_ERR_ARG; }
    (void)col_idx;
    cudaStream_t s = cs(stream);
    const bool want_global = K_vals || M_vals;
    vb_status st = VB_OK;
    if (mode == VB_ASSEMBLE_ATOMIC) {
        if (want_global && (!elem2nnz || !row_ptr)) { set_error("fem_p1_assemble: atomic mode needs elem2nnz and row_ptr"); return VB_ERR_ARG; }
        if (want_global && nnz > 0) {
            zero2_k<<<grid_for(nnz, 256, 8), 256, 0, s>>>(K_vals, M_vals, nnz);
            if ((st = launch_check("fem_p1_assemble(zero)")) != VB_OK) return st;
        }
        if (ne == 0 || (!want_global && !K_local && !M_local)) return VB_OK;
        unsigned g = grid_for(ne, 256, 8);
        if (!want_global) {
            if (dim == 2) local_k<2><<<g, 256, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, K_local, M_local);
            else local_k<3><<<g, 256, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, K_local, M_local);
        } else if (dim == 2) {
            assemble_atomic_k<2><<<g, 256, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, elem2nnz, K_vals, M_vals, K_local, M_local);
        } else {
            assemble_atomic_k<3><<<g, 256, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, elem2nnz, K_vals, M_vals, K_local, M_local);
        }
        return launch_check("fem_p1_assemble(atomic)");
    }
    // gather mode
    if (want_global && (!row_ptr || !node_elem_ptr || !node_elem || !node_elem_slot)) {
        set_error("fem_p1_assemble: gather mode needs row_ptr, node_elem_ptr, node_elem, node_elem_slot");
        return VB_ERR_ARG;
    }
    if (want_global && nn > 0) {
        if (dim == 2) {
            size_t sm = 2 * GatherCfg<2>::CAP * sizeof(double);
            unsigned g = (unsigned)((nn + GATHER_BLOCK - 1) / GATHER_BLOCK);
            assemble_gather_k<2><<<g, GATHER_BLOCK, sm, s>>>(nn, coords, node_stride, comp_stride, elems, elem_ld, row_ptr,
                                                             node_elem_ptr, node_elem, node_elem_slot, K_vals, M_vals);
        } else {
            size_t sm = 2 * GatherCfg<3>::CAP * sizeof(double);
            unsigned g = (unsigned)((nn + GATHER_BLOCK - 1) / GATHER_BLOCK);
            assemble_gather_k<3><<<g, GATHER_BLOCK, sm, s>>>(nn, coords, node_stride, comp_stride, elems, elem_ld, row_ptr,
                                                             node_elem_ptr, node_elem, node_elem_slot, K_vals, M_vals);
        }
        if ((st = launch_check("fem_p1_assemble(gather)")) != VB_OK) return st;
    }
    if ((K_local || M_local) && ne > 0) {
        unsigned g = grid_for(ne, 256, 8);
        if (dim == 2) local_k<2><<<g, 256, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, K_local, M_local);
        else local_k<3><<<g, 256, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, K_local, M_local);
        if ((st = launch_check("fem_p1_assemble(local)")) != VB_OK) return st;
    }
    return VB_OK;
}
