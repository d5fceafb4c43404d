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
// One thread owns row v; a CTA owns GATHER_BLOCK consecutive rows, i.e. one
// contiguous range of the CSR arrays and one contiguous range of the gather
// plan, both staged in shared memory with coalesced loads.  The edge vectors
// f_s = x_{col(s)} - x_v to every column of the row are formed once per row
// (shared memory, indexed by in-row slot).  Each incidence (e, a) of v needs
// only its plan word (slots of the element's other vertices): with v as the
// base vertex (any base gives the same K_e) tjac has rows f_1..f_d,
// adj(tjac) has columns h_j (cross products of the other f's), and
//   grad phi_{o_j} = h_j / det,  grad phi_a = h_a / det,  h_a = -sum_j h_j,
//   K_e[a][o_j] = (h_a . h_j) / (d! |det|),   M_e[a][o_j] = |det| / (d! (d+1)(d+2)).
// Off-diagonal entries are summed in ascending element order (the oracle's
// order); the diagonal follows from the partition of unity sum_b phi_b = 1:
//   K_vv = -sum_{w != v} K_vw,   M_vv = (2/d) sum_{w != v} M_vw.
constexpr int GATHER_BLOCK = 32;
template <int DIM>
struct GatherCfg {
    static constexpr int CTA_CAP = GATHER_BLOCK * (DIM == 2 ? 8 : 16);   // CSR entries per CTA staged in smem
    static constexpr int SLOT_CAP = GATHER_BLOCK * (DIM == 2 ? 8 : 28);  // plan words per CTA staged in smem
    static constexpr size_t SMEM = (size_t)(DIM + 2) * CTA_CAP * sizeof(double) +
                                   (size_t)(SLOT_CAP + CTA_CAP) * sizeof(uint32_t);
};

// 1/x to ~1 ulp: hardware seed + two Newton steps (x > 0, normal)
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(y, fma(-x, y, 1.0), y);
    y = fma(y, fma(-x, y, 1.0), y);
    return y;
}

// Off-diagonal contributions of incidences [i0, i1) of one row.  EV(s, f)
// yields the edge vector from the row's vertex to its column s.
template <int DIM, typename EV>
__device__ __forceinline__ void gather_row(int i0, int i1, const uint32_t* slots, EV ev, double* accK, double* accM) {
#pragma unroll 2
    for (int i = i0; i < i1; i++) {
        uint32_t sl = slots[i];
        if constexpr (DIM == 3) {
            int s1 = (sl >> 8) & 0xff, s2 = (sl >> 16) & 0xff, s3 = sl >> 24;
            double f1[3], f2[3], f3[3];
            ev(s1, f1);
            ev(s2, f2);
            ev(s3, f3);
            double h1[3] = {fma(f2[1], f3[2], -f2[2] * f3[1]), fma(f2[2], f3[0], -f2[0] * f3[2]),
                            fma(f2[0], f3[1], -f2[1] * f3[0])};
            double h2[3] = {fma(f3[1], f1[2], -f3[2] * f1[1]), fma(f3[2], f1[0], -f3[0] * f1[2]),
                            fma(f3[0], f1[1], -f3[1] * f1[0])};
            double h3[3] = {fma(f1[1], f2[2], -f1[2] * f2[1]), fma(f1[2], f2[0], -f1[0] * f2[2]),
                            fma(f1[0], f2[1], -f1[1] * f2[0])};
            double ad = fabs(fma(f1[0], h1[0], fma(f1[1], h1[1], f1[2] * h1[2])));
            double r = -rcp_nr(6.0 * ad);
            double ha[3];
#pragma unroll
            for (int c = 0; c < 3; c++) ha[c] = r * ((h1[c] + h2[c]) + h3[c]);
            double k1 = fma(ha[0], h1[0], fma(ha[1], h1[1], ha[2] * h1[2]));
            double k2 = fma(ha[0], h2[0], fma(ha[1], h2[1], ha[2] * h2[2]));
            double k3 = fma(ha[0], h3[0], fma(ha[1], h3[1], ha[2] * h3[2]));
            double m = ad * (1.0 / 120.0);
            if (accK) {
                accK[s1] += k1;
                accK[s2] += k2;
                accK[s3] += k3;
            }
            if (accM) {
                accM[s1] += m;
                accM[s2] += m;
                accM[s3] += m;
            }
        } else {
            int s1 = (sl >> 8) & 0xff, s2 = (sl >> 16) & 0xff;
            double f1[2], f2[2];
            ev(s1, f1);
            ev(s2, f2);
            // tjac rows f1, f2: adj columns h1 = (f2y, -f2x), h2 = (-f1y, f1x)
            double ad = fabs(fma(f1[0], f2[1], -f1[1] * f2[0]));
            double r = -rcp_nr(2.0 * ad);
            double hax = r * (f2[1] - f1[1]), hay = r * (f1[0] - f2[0]);
            double k1 = fma(hax, f2[1], -hay * f2[0]);
            double k2 = fma(-hax, f1[1], hay * f1[0]);
            double m = ad * (1.0 / 24.0);
            if (accK) {
                accK[s1] += k1;
                accK[s2] += k2;
            }
            if (accM) {
                accM[s1] += m;
                accM[s2] += m;
            }
        }
    }
}

// diagonal of a row (slot s0 of L) from the off-diagonal sums (partition of unity)
template <int DIM>
__device__ __forceinline__ void finish_row(int L, int s0, double* accK, double* accM) {
    double sk = 0.0, sm = 0.0;
    for (int s = 0; s < L; s++) {
        if (s == s0) continue;
        if (accK) sk += accK[s];
        if (accM) sm += accM[s];
    }
    if (accK) accK[s0] = -sk;
    if (accM) accM[s0] = DIM == 3 ? sm * (2.0 / 3.0) : sm;
}

template <int DIM>
__global__ void __launch_bounds__(GATHER_BLOCK) assemble_gather_k(int64_t nn, const double* __restrict__ coords,
                                                                  int64_t ns, int64_t cst,
                                                                  const int32_t* __restrict__ row_ptr,
                                                                  const int32_t* __restrict__ col_idx,
                                                                  const int32_t* __restrict__ nptr,
                                                                  const uint32_t* __restrict__ nslot,
                                                                  double* __restrict__ K, double* __restrict__ M) {
    using Cfg = GatherCfg<DIM>;
    constexpr int CAP = Cfg::CTA_CAP;
    extern __shared__ double smem[];
    double* F = smem;                        // [DIM][CAP]  column coordinates, then edge vectors
    double* sK = smem + DIM * CAP;           // [CAP] CTA-contiguous CSR range of K
    double* sM = sK + CAP;                   // [CAP]
    uint32_t* sSlot = reinterpret_cast<uint32_t*>(sM + CAP);     // [SLOT_CAP] plan range
    int32_t* sCol = reinterpret_cast<int32_t*>(sSlot + Cfg::SLOT_CAP);
    const int t = threadIdx.x;
    for (int64_t r0 = (int64_t)blockIdx.x * GATHER_BLOCK; r0 < nn; r0 += (int64_t)gridDim.x * GATHER_BLOCK) {
        const int64_t rend = r0 + GATHER_BLOCK < nn ? r0 + GATHER_BLOCK : nn;
        const int32_t p0 = __ldg(row_ptr + r0), p1 = __ldg(row_ptr + rend);
        const int32_t q0 = __ldg(nptr + r0), q1 = __ldg(nptr + rend);
        const int np = p1 - p0, nq = q1 - q0;
        const int64_t v = r0 + t;
        const bool own = v < rend;
        int lo = 0, L = 0, i0 = 0, i1 = 0;
        double xv[DIM];
        if (own) {
            lo = __ldg(row_ptr + v);
            L = __ldg(row_ptr + v + 1) - lo;
            i0 = __ldg(nptr + v);
            i1 = __ldg(nptr + v + 1);
#pragma unroll
            for (int c = 0; c < DIM; c++) xv[c] = __ldg(coords + c * cst + v * ns);
        }
        if (np <= CAP && nq <= Cfg::SLOT_CAP) {
            // stage the CTA's CSR columns and plan words (coalesced), zero the accumulators
#pragma unroll 4
            for (int q = t; q < np; q += GATHER_BLOCK) sCol[q] = __ldcs(col_idx + p0 + q);
#pragma unroll 4
            for (int q = t; q < nq; q += GATHER_BLOCK) sSlot[q] = __ldcs(nslot + q0 + q);
            __syncthreads();
            // gather the coordinates of every column of the CTA's range (independent loads)
#pragma unroll 4
            for (int q = t; q < np; q += GATHER_BLOCK) {
                int64_t w = sCol[q];
#pragma unroll
                for (int c = 0; c < DIM; c++) F[c * CAP + q] = __ldg(coords + c * cst + w * ns);
                sK[q] = 0.0;
                sM[q] = 0.0;
            }
            __syncthreads();
            if (own) {
                const int b = lo - p0;
                int s0 = 0;
                for (int s = 0; s < L; s++) {
                    if (sCol[b + s] == v) s0 = s;
#pragma unroll
                    for (int c = 0; c < DIM; c++) F[c * CAP + b + s] -= xv[c];
                }
                auto ev = [&](int s, double(&f)[DIM]) {
#pragma unroll
                    for (int c = 0; c < DIM; c++) f[c] = F[c * CAP + b + s];
                };
                double* aK = K ? sK + b : nullptr;
                double* aM = M ? sM + b : nullptr;
                gather_row<DIM>(i0, i1, sSlot - q0, ev, aK, aM);
                if (L > 0) finish_row<DIM>(L, s0, aK, aM);
            }
            __syncthreads();
#pragma unroll 4
            for (int q = t; q < np; q += GATHER_BLOCK) {
                if (K) stcs(K + p0 + q, sK[q]);
                if (M) stcs(M + p0 + q, sM[q]);
            }
            __syncthreads();
        } else if (own) {
            // CTA range larger than the smem budget: same ownership, everything in place in HBM
            double* aK = K ? K + lo : nullptr;
            double* aM = M ? M + lo : nullptr;
            int s0 = 0;
            for (int q = 0; q < L; q++) {
                if (aK) aK[q] = 0.0;
                if (aM) aM[q] = 0.0;
                if (__ldg(col_idx + lo + q) == v) s0 = q;
            }
            auto ev = [&](int s, double(&f)[DIM]) {
                int64_t w = __ldg(col_idx + lo + s);
#pragma unroll
                for (int c = 0; c < DIM; c++) f[c] = __ldg(coords + c * cst + w * ns) - xv[c];
            };
            gather_row<DIM>(i0, i1, nslot, ev, aK, aM);
            if (L > 0) finish_row<DIM>(L, s0, aK, aM);
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
    if (want_global && (!row_ptr || !col_idx || !node_elem_ptr || !node_elem_slot)) {
        set_error("fem_p1_assemble: gather mode needs row_ptr, col_idx, node_elem_ptr, node_elem_slot");
        return VB_ERR_ARG;
    }
    if (want_global && nn > 0) {
        static bool smem_opt_in = false;  // > 48 KB dynamic shared memory needs an opt-in per kernel
        if (!smem_opt_in) {
            cudaFuncSetAttribute(assemble_gather_k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GatherCfg<2>::SMEM);
            cudaFuncSetAttribute(assemble_gather_k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GatherCfg<3>::SMEM);
            smem_opt_in = true;
        }
        unsigned g = (unsigned)((nn + GATHER_BLOCK - 1) / GATHER_BLOCK);
        if (dim == 2) {
            assemble_gather_k<2><<<g, GATHER_BLOCK, GatherCfg<2>::SMEM, s>>>(nn, coords, node_stride, comp_stride, row_ptr,
                                                                         col_idx, node_elem_ptr, node_elem_slot, K_vals, M_vals);
        } else {
            assemble_gather_k<3><<<g, GATHER_BLOCK, GatherCfg<3>::SMEM, s>>>(nn, coords, node_stride, comp_stride, row_ptr,
                                                                         col_idx, node_elem_ptr, node_elem_slot, K_vals, M_vals);
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
