// NEXT-3: P2 stiffness and mass assembly (stiffness_matrixP2 / mass_matrixP2,
// P:1009-1049) with the coefficients of eq:K_M, c(x) = a exp(b . x), and
// intquad(gqo) rules up to degree 4.  One thread per element: the P1
// Jacobian of the (straight-edged) element gives grad lambda_b; the P2 basis
//   vertex a: lambda_a (2 lambda_a - 1),  edge (i, j): 4 lambda_i lambda_j
// (SPEC S:304 edge order) has grad phi = combinations of at most two grad lambda.
// K_e and M_e are accumulated row by row (b >= a, symmetric) over the points and
// added into the CSR values through the nv^2 element-to-nnz map of fem_pattern
// with fp64 atomics (targets zero-filled by the call).
#include "vb_internal.cuh"

namespace vb {
namespace {

struct P2Coef {
    double ka, kb[3], ma, mb[3];
    bool same;
};

// intquad(gqo, dim) barycentric points (up to 11) and weights, sum = 1/d!
struct P2Rule {
    int nip;
    double lam[11][4];
    double w[11];
};

bool p2_rule(int dim, int gqo, P2Rule& R) {
    const int nv = dim + 1;
    const double dfact = dim == 2 ? 2.0 : 6.0;
    if (gqo == 1) {
        R.nip = 1;
        for (int a = 0; a < nv; a++) R.lam[0][a] = 1.0 / nv;
        R.w[0] = 1.0 / dfact;
        return true;
    }
    if (gqo == 2) {
        const double al = dim == 2 ? 2.0 / 3.0 : 0.58541019662496845446;
        const double be = dim == 2 ? 1.0 / 6.0 : 0.13819660112501051518;
        R.nip = nv;
        for (int q = 0; q < nv; q++) {
            for (int a = 0; a < nv; a++) R.lam[q][a] = a == q ? al : be;
            R.w[q] = 1.0 / (dfact * nv);
        }
        return true;
    }
    if (gqo == 4 && dim == 2) {  // Dunavant, 6 points
        const double as[2] = {0.44594849091596488632, 0.09157621350977074346};
        const double ws[2] = {0.22338158967801146570, 0.10995174365532186764};
        int q = 0;
        for (int k = 0; k < 2; k++)
            for (int p = 0; p < 3; p++) {
                for (int a = 0; a < 3; a++) R.lam[q][a] = a == p ? 1.0 - 2.0 * as[k] : as[k];
                R.w[q++] = ws[k] / 2.0;
            }
        R.nip = 6;
        return true;
    }
    if (gqo == 4 && dim == 3) {  // Keast, 11 points
        int q = 0;
        for (int a = 0; a < 4; a++) R.lam[q][a] = 0.25;
        R.w[q++] = -74.0 / 5625.0;
        for (int p = 0; p < 4; p++) {
            for (int a = 0; a < 4; a++) R.lam[q][a] = a == p ? 11.0 / 14.0 : 1.0 / 14.0;
            R.w[q++] = 343.0 / 45000.0;
        }
        const double pa = (1.0 + sqrt(5.0 / 14.0)) / 4.0, pb = (1.0 - sqrt(5.0 / 14.0)) / 4.0;
        for (int i = 0; i < 4; i++)
            for (int j = i + 1; j < 4; j++) {
                for (int a = 0; a < 4; a++) R.lam[q][a] = (a == i || a == j) ? pa : pb;
                R.w[q++] = 56.0 / 2250.0;
            }
        R.nip = 11;
        return true;
    }
    return false;
}

template <int DIM>
struct P2Topo;
template <>
struct P2Topo<2> {
    static constexpr int NV = 3, NLB = 6;
    __device__ static constexpr int ei(int k) { return k == 0 ? 0 : (k == 1 ? 1 : 0); }
    __device__ static constexpr int ej(int k) { return k == 0 ? 1 : 2; }
};
template <>
struct P2Topo<3> {
    static constexpr int NV = 4, NLB = 10;
    // edges (0,1) (0,2) (0,3) (1,2) (1,3) (2,3)
    __device__ static constexpr int ei(int k) { return k < 3 ? 0 : (k < 5 ? 1 : 2); }
    __device__ static constexpr int ej(int k) { return k < 3 ? k + 1 : (k < 5 ? k - 1 : 3); }
};

// value and gradient of basis function k at barycentric point lam
template <int DIM>
__device__ __forceinline__ void p2_basis(int k, const double* lam, const double (&gl)[DIM + 1][DIM], double& phi,
                                         double (&g)[DIM]) {
    using T = P2Topo<DIM>;
    if (k < T::NV) {
        phi = lam[k] * (2.0 * lam[k] - 1.0);
        const double s = 4.0 * lam[k] - 1.0;
#pragma unroll
        for (int c = 0; c < DIM; c++) g[c] = s * gl[k][c];
    } else {
        const int i = T::ei(k - T::NV), j = T::ej(k - T::NV);
        phi = 4.0 * lam[i] * lam[j];
#pragma unroll
        for (int c = 0; c < DIM; c++) g[c] = 4.0 * fma(lam[j], gl[i][c], lam[i] * gl[j][c]);
    }
}

constexpr int P2_BLOCK = 64;   // 55 x 64 doubles of M staging (28 KB static smem in 3D)

template <int DIM>
__global__ void __launch_bounds__(P2_BLOCK) p2_assemble_k(int64_t ne, const double* __restrict__ coords, int64_t ns,
                                                     int64_t cst, const int32_t* __restrict__ elems, int64_t eld,
                                                     const int32_t* __restrict__ e2n, const P2Rule R, const P2Coef cp,
                                                     double* __restrict__ K, double* __restrict__ M,
                                                     double* __restrict__ Kl, double* __restrict__ Ml) {
    using T = P2Topo<DIM>;
    constexpr int NV = T::NV, NLB = T::NLB;
    __shared__ double Mst[NLB * (NLB + 1) / 2 * P2_BLOCK];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += stride) {
        double x[NV][DIM];
#pragma unroll
        for (int a = 0; a < NV; a++) {
            const int64_t v = __ldg(elems + a * eld + e);
#pragma unroll
            for (int c = 0; c < DIM; c++) x[a][c] = __ldg(coords + c * cst + v * ns);
        }
        // grad lambda_b (rows of G^T): tjac rows x_{r+1} - x_0, G = tjac^{-1} D
        double J[DIM][DIM], inv[DIM][DIM], det;
#pragma unroll
        for (int r = 0; r < DIM; r++)
#pragma unroll
            for (int c = 0; c < DIM; c++) J[r][c] = x[r + 1][c] - x[0][c];
        if constexpr (DIM == 2) {
            det = fma(J[0][0], J[1][1], -J[0][1] * J[1][0]);
            const double r = 1.0 / det;
            inv[0][0] = J[1][1] * r;
            inv[0][1] = -J[0][1] * r;
            inv[1][0] = -J[1][0] * r;
            inv[1][1] = J[0][0] * r;
        } else {
            double a00 = fma(J[1][1], J[2][2], -J[1][2] * J[2][1]);
            double a10 = fma(J[1][2], J[2][0], -J[1][0] * J[2][2]);
            double a20 = fma(J[1][0], J[2][1], -J[1][1] * J[2][0]);
            det = fma(J[0][0], a00, fma(J[0][1], a10, J[0][2] * a20));
            const double r = 1.0 / det;
            inv[0][0] = a00 * r;
            inv[1][0] = a10 * r;
            inv[2][0] = a20 * r;
            inv[0][1] = fma(J[0][2], J[2][1], -J[0][1] * J[2][2]) * r;
            inv[1][1] = fma(J[0][0], J[2][2], -J[0][2] * J[2][0]) * r;
            inv[2][1] = fma(J[0][1], J[2][0], -J[0][0] * J[2][1]) * r;
            inv[0][2] = fma(J[0][1], J[1][2], -J[0][2] * J[1][1]) * r;
            inv[1][2] = fma(J[0][2], J[1][0], -J[0][0] * J[1][2]) * r;
            inv[2][2] = fma(J[0][0], J[1][1], -J[0][1] * J[1][0]) * r;
        }
        const double ad = fabs(det);
        double gl[NV][DIM];  // grad lambda_b
#pragma unroll
        for (int c = 0; c < DIM; c++) {
            double s = 0.0;
#pragma unroll
            for (int b = 1; b < NV; b++) {
                gl[b][c] = inv[c][b - 1];
                s += inv[c][b - 1];
            }
            gl[0][c] = -s;
        }
        // coefficients at the points
        double cK[11], cM[11];
        for (int q = 0; q < R.nip; q++) {
            double ek = 0.0, em = 0.0;
#pragma unroll
            for (int c = 0; c < DIM; c++) {
                double xc = 0.0;
#pragma unroll
                for (int a = 0; a < NV; a++) xc = fma(R.lam[q][a], x[a][c], xc);
                ek = fma(cp.kb[c], xc, ek);
                em = fma(cp.mb[c], xc, em);
            }
            cK[q] = R.w[q] * ad * cp.ka * exp(ek);
            cM[q] = cp.same ? cK[q] : R.w[q] * ad * cp.ma * exp(em);
        }
        // Two passes over the points (M, then K), each with the unique entries b >= a
        // of the element matrix in registers and the basis evaluated once per point
        // (55 + 30 live doubles for K in 3D); the M entries wait in a thread-private
        // shared-memory strip so each element-to-nnz position is loaded once and its
        // K and M atomics go out together.
        constexpr int NP = NLB * (NLB + 1) / 2;
        double* mst = Mst + threadIdx.x;   // entry p at mst[p * blockDim.x]
        if (M || Ml) {
            double acc[NP];
#pragma unroll
            for (int p = 0; p < NP; p++) acc[p] = 0.0;
            for (int q = 0; q < R.nip; q++) {
                double ph[NLB];
#pragma unroll
                for (int k = 0; k < NLB; k++) {
                    double g[DIM];
                    p2_basis<DIM>(k, R.lam[q], gl, ph[k], g);
                }
                int p = 0;
#pragma unroll
                for (int a = 0; a < NLB; a++) {
                    const double ca = cM[q] * ph[a];
#pragma unroll
                    for (int b = a; b < NLB; b++, p++) acc[p] = fma(ca, ph[b], acc[p]);
                }
            }
#pragma unroll
            for (int p = 0; p < NP; p++) mst[p * P2_BLOCK] = acc[p];
        }
        double acc[NP];
#pragma unroll
        for (int p = 0; p < NP; p++) acc[p] = 0.0;
        if (K || Kl) {
            for (int q = 0; q < R.nip; q++) {
                double g[NLB][DIM];
#pragma unroll
                for (int k = 0; k < NLB; k++) {
                    double phi;
                    p2_basis<DIM>(k, R.lam[q], gl, phi, g[k]);
                }
                int p = 0;
#pragma unroll
                for (int a = 0; a < NLB; a++)
#pragma unroll
                    for (int b = a; b < NLB; b++, p++) {
                        double d = g[a][0] * g[b][0];
#pragma unroll
                        for (int c = 1; c < DIM; c++) d = fma(g[a][c], g[b][c], d);
                        acc[p] = fma(cK[q], d, acc[p]);
                    }
            }
        }
        int p = 0;
#pragma unroll
        for (int a = 0; a < NLB; a++)
#pragma unroll
            for (int b = a; b < NLB; b++, p++) {
                const double kv = acc[p];
                const double mv = (M || Ml) ? mst[p * P2_BLOCK] : 0.0;
                if (K || M) {
                    const int32_t pab = __ldcs(e2n + (int64_t)(a * NLB + b) * ne + e);
                    if (K) atomicAdd(K + pab, kv);
                    if (M) atomicAdd(M + pab, mv);
                    if (b != a) {
                        const int32_t pba = __ldcs(e2n + (int64_t)(b * NLB + a) * ne + e);
                        if (K) atomicAdd(K + pba, kv);
                        if (M) atomicAdd(M + pba, mv);
                    }
                }
                if (Kl) {
                    stcs(Kl + (int64_t)(a + b * NLB) * ne + e, kv);
                    if (b != a) stcs(Kl + (int64_t)(b + a * NLB) * ne + e, kv);
                }
                if (Ml) {
                    stcs(Ml + (int64_t)(a + b * NLB) * ne + e, mv);
                    if (b != a) stcs(Ml + (int64_t)(b + a * NLB) * ne + e, mv);
                }
            }
    }
}

__global__ void zero2_p2_k(double* __restrict__ a, double* __restrict__ b, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (a) a[i] = 0.0;
        if (b) b[i] = 0.0;
    }
}

}  // namespace
}  // namespace vb

using namespace vb;

extern "C" vb_status fem_p2_assemble(int dim, int64_t nn, int64_t ne, const double* coords, int64_t node_stride,
                                     int64_t comp_stride, const int32_t* elems, int64_t elem_ld,
                                     const int32_t* elem2nnz, int64_t nnz, int gqo, double cK_a, const double* cK_b,
                                     double cM_a, const double* cM_b, double* K_vals, double* M_vals, double* K_local,
                                     double* M_local, vb_stream_t stream) {
    clear_error();
    if (dim != 2 && dim != 3) { set_error("fem_p2_assemble: dim=%d, need 2 or 3", dim); return VB_ERR_UNSUPPORTED; }
    if (nn < 0 || ne < 0 || nnz < 0) { set_error("fem_p2_assemble: negative size"); return VB_ERR_ARG; }
    P2Rule R;
    if (!p2_rule(dim, gqo, R)) { set_error("fem_p2_assemble: gqo=%d unsupported (1, 2, 4)", gqo); return VB_ERR_UNSUPPORTED; }
    if (ne > 0 && (!coords || !elems)) { set_error("fem_p2_assemble: NULL coords or elems"); return VB_ERR_ARG; }
    if ((K_vals || M_vals) && !elem2nnz) { set_error("fem_p2_assemble: K/M need elem2nnz (fem_pattern)"); return VB_ERR_ARG; }
    if (elem_ld < ne) { set_error("fem_p2_assemble: elem_ld < ne"); return VB_ERR_ARG; }
    P2Coef cp{cK_a, {0, 0, 0}, cM_a, {0, 0, 0}, false};
    for (int c = 0; c < dim; c++) {
        cp.kb[c] = cK_b ? cK_b[c] : 0.0;
        cp.mb[c] = cM_b ? cM_b[c] : 0.0;
    }
    cp.same = cK_a == cM_a && cp.kb[0] == cp.mb[0] && cp.kb[1] == cp.mb[1] && cp.kb[2] == cp.mb[2];
    cudaStream_t s = cs(stream);
    if ((K_vals || M_vals) && nnz > 0) zero2_p2_k<<<grid_for(nnz, 256, 8), 256, 0, s>>>(K_vals, M_vals, nnz);
    if (ne > 0 && (K_vals || M_vals || K_local || M_local)) {
        unsigned g = grid_for(ne, P2_BLOCK, 8);
        if (dim == 2) p2_assemble_k<2><<<g, P2_BLOCK, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, elem2nnz, R, cp, K_vals, M_vals, K_local, M_local);
        else p2_assemble_k<3><<<g, P2_BLOCK, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, elem2nnz, R, cp, K_vals, M_vals, K_local, M_local);
    }
    return launch_check("fem_p2_assemble");
}
