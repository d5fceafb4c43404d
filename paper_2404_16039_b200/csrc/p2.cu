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

#ifndef VB_P2_KMOMENTS
#define VB_P2_KMOMENTS 1   // K entries from the moments of the weights (0: point by point)
#endif
constexpr int P2_BLOCK = 64;   // elements per block; 2 x 55 x 64 doubles of strips (56 KB in 3D)

template <int DIM>
__global__ void __launch_bounds__(P2_BLOCK) p2_assemble_k(int64_t ne, const double* __restrict__ coords, int64_t ns,
                                                     int64_t cst, const int32_t* __restrict__ elems, int64_t eld,
                                                     const int32_t* __restrict__ e2n, const P2Rule R, const P2Coef cp,
                                                     double* __restrict__ K, double* __restrict__ M,
                                                     double* __restrict__ Kl, double* __restrict__ Ml,
                                                     double* __restrict__ Kst, double* __restrict__ Mst_g) {
    using T = P2Topo<DIM>;
    constexpr int NV = T::NV, NLB = T::NLB;
    constexpr int NP = NLB * (NLB + 1) / 2;   // unique entries b >= a (odd: 21 / 55)
    extern __shared__ double p2_smem[];       // thread-private strips [tid][NP]: M, then K (staging)
    double* MS = p2_smem;
    double* KS = p2_smem + P2_BLOCK * NP;
    const int64_t stride = (int64_t)gridDim.x * P2_BLOCK;
    for (int64_t base = (int64_t)blockIdx.x * P2_BLOCK; base < ne; base += stride) {
        const int64_t e = base + threadIdx.x;
        const bool active = e < ne;
        if (active) {
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
        double* mst = MS + threadIdx.x * NP;   // entry p at mst[p] (odd stride: 2-way conflicts at most)
        if (M || Ml || Mst_g) {
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
            for (int p = 0; p < NP; p++) mst[p] = acc[p];
        }
        double acc[NP];
#pragma unroll
        for (int p = 0; p < NP; p++) acc[p] = 0.0;
        if (K || Kl || Kst) {
#if VB_P2_KMOMENTS
            // K through the moments of the weights (round 2).  grad phi is linear in lambda:
            //   vertex a: (4 lam_a - 1) grad lam_a,   edge (i, j): 4 (lam_i grad lam_j + lam_j grad lam_i),
            // so sum_q c_q grad phi_a . grad phi_b = combinations of the Gram entries G_ij = grad lam_i . grad lam_j
            // with S0 = sum c_q, S1_i = sum c_q lam_i, S2_ij = sum c_q lam_i lam_j: the same sum over the points
            // regrouped (about 460 fp64 operations per tet in 3D instead of 2400 with 11 points).
            double S0 = 0.0, S1[NV], S2[NV][NV], G[NV][NV];
#pragma unroll
            for (int i = 0; i < NV; i++) {
                S1[i] = 0.0;
#pragma unroll
                for (int j = 0; j < NV; j++) S2[i][j] = 0.0;
            }
            for (int q = 0; q < R.nip; q++) {
                S0 += cK[q];
#pragma unroll
                for (int i = 0; i < NV; i++) {
                    const double t = cK[q] * R.lam[q][i];
                    S1[i] += t;
#pragma unroll
                    for (int j = i; j < NV; j++) S2[i][j] = fma(t, R.lam[q][j], S2[i][j]);
                }
            }
#pragma unroll
            for (int i = 0; i < NV; i++)
#pragma unroll
                for (int j = i; j < NV; j++) {
                    double d = gl[i][0] * gl[j][0];
#pragma unroll
                    for (int c = 1; c < DIM; c++) d = fma(gl[i][c], gl[j][c], d);
                    G[i][j] = G[j][i] = d;
                    S2[j][i] = S2[i][j];
                }
            int p = 0;
#pragma unroll
            for (int a = 0; a < NLB; a++)
#pragma unroll
                for (int b = a; b < NLB; b++, p++) {
                    double v;
                    if (b < NV) {   // vertex, vertex
                        v = G[a][b] * (fma(16.0, S2[a][b], S0) - 4.0 * (S1[a] + S1[b]));
                    } else if (a < NV) {   // vertex a, edge (i, j)
                        const int i = T::ei(b - NV), j = T::ej(b - NV);
                        v = 4.0 * fma(G[a][j], fma(4.0, S2[a][i], -S1[i]), G[a][i] * fma(4.0, S2[a][j], -S1[j]));
                    } else {   // edge (i, j), edge (k, l)
                        const int i = T::ei(a - NV), j = T::ej(a - NV), k = T::ei(b - NV), l = T::ej(b - NV);
                        v = 16.0 * fma(S2[i][k], G[j][l], fma(S2[i][l], G[j][k], fma(S2[j][k], G[i][l], S2[j][l] * G[i][k])));
                    }
                    acc[p] = v;
                }
#else
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
#endif
        }
        int p = 0;
#pragma unroll
        for (int a = 0; a < NLB; a++)
#pragma unroll
            for (int b = a; b < NLB; b++, p++) {
                const double kv = acc[p];
                const double mv = (M || Ml || Mst_g) ? mst[p] : 0.0;
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
                if (Kst) KS[threadIdx.x * NP + p] = kv;
            }
        }
        if (Kst || Mst_g) {
            // gather staging: element-major full matrices (row a of element e contiguous),
            // written cooperatively by the block from the strips -> coalesced stores
            __syncthreads();
            const int nact = (int)(ne - base < P2_BLOCK ? ne - base : P2_BLOCK);
            constexpr int NN = NLB * NLB;
            double2* out = reinterpret_cast<double2*>(Kst);   // (K, M) pairs, [e][a][b]
            // this thread's entries r = tid, tid + P2_BLOCK of every element: their strip positions once
            constexpr int NR = (NN + P2_BLOCK - 1) / P2_BLOCK;
            int pp[NR];
#pragma unroll
            for (int k = 0; k < NR; k++) {
                const int r = threadIdx.x + k * P2_BLOCK;
                const int a = r / NLB, b = r - a * NLB;
                const int lo = a < b ? a : b, hi = a < b ? b : a;
                pp[k] = r < NN ? lo * NLB - lo * (lo - 1) / 2 + (hi - lo) : -1;
            }
            double2* o = out + base * NN + threadIdx.x;
            for (int j = 0; j < nact; j++, o += NN) {
#pragma unroll
                for (int k = 0; k < NR; k++)
                    if (pp[k] >= 0) __stcs(o + k * P2_BLOCK, make_double2(KS[j * NP + pp[k]], MS[j * NP + pp[k]]));
            }
            __syncthreads();
        }
    }
}

// Deterministic P2 assembly, phase 2: every row v sums, in ascending element order, row a of the staged
// K_e / M_e of each of its incidences (e, a) into per-slot accumulators in shared memory (rows of up to
// P2_RS entries; longer rows accumulate in place in HBM), then writes the row once.
constexpr int P2_RS = 72;

// A warp takes G = 32 / NLB consecutive rows, NLB lanes each.  Lane (g, b) loads
// entry b of the staged element row of row g's next incidence (one coalesced 16 NLB-byte piece per row) and
// its slot byte, and adds the (K, M) pair into the row's accumulators in shared memory (RS + 1 pairs per row:
// 1.2 KB instead of the 37 KB per warp of the one-thread-per-row kernel, so 40+ warps are resident instead
// of 6).  The NLB slots of one incidence are distinct columns, so the lanes of a row never collide; incidences
// are taken in ascending order, U at a time in flight: the same summation order as before, bitwise
// reproducible.  Rows longer than RS are summed in place in HBM by lane 0 of their group.
constexpr int P2C_WARPS = 4;
template <int NLB, int RS, int U>
__global__ void __launch_bounds__(32 * P2C_WARPS) p2_gather_coop_k(int64_t nn, const int32_t* __restrict__ row_ptr,
                                                                  const int32_t* __restrict__ nptr,
                                                                  const int32_t* __restrict__ nelem,
                                                                  const uint32_t* __restrict__ nslot,
                                                                  const double2* __restrict__ KMst,
                                                                  double* __restrict__ K, double* __restrict__ M) {
    constexpr int G = 32 / NLB;
    constexpr int NW = (NLB + 3) / 4;
    constexpr int ST = RS + 1;
    __shared__ double2 acc_s[P2C_WARPS][G][ST];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int g = lane / NLB, b = lane - g * NLB;
    const bool act = g < G;
    double2* acc = acc_s[wl][act ? g : 0];
    const int64_t nwarps = (int64_t)gridDim.x * P2C_WARPS;
    for (int64_t v0 = ((int64_t)blockIdx.x * P2C_WARPS + wl) * G; v0 < nn; v0 += nwarps * G) {
        const int64_t v = v0 + g;
        const bool own = act && v < nn;
        const int lo = own ? __ldg(row_ptr + v) : 0, L = own ? __ldg(row_ptr + v + 1) - lo : 0;
        const int i0 = own ? __ldg(nptr + v) : 0, i1 = own ? __ldg(nptr + v + 1) : 0;
        const bool fast = L <= RS;
        if (fast) {
            for (int sl = b; sl < L; sl += NLB) acc[sl] = make_double2(0.0, 0.0);
        } else if (b == 0) {
            for (int sl = 0; sl < L; sl++) {
                if (K) K[lo + sl] = 0.0;
                if (M) M[lo + sl] = 0.0;
            }
        }
        __syncwarp();
        const int nmax = __reduce_max_sync(0xffffffffu, i1 - i0);   // warp-uniform trip count
        for (int k = 0; k < nmax; k += U) {
            int sl[U];
            double2 km[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int i = i0 + k + u;
                sl[u] = -1;
                km[u] = make_double2(0.0, 0.0);
                if (i < i1) {
                    const int32_t ea = __ldg(nelem + i);
                    const uint32_t w = __ldg(nslot + (int64_t)i * NW + b / 4);
                    sl[u] = (w >> (8 * (b % 4))) & 0xff;
                    km[u] = __ldcs(KMst + (int64_t)(ea >> 4) * (NLB * NLB) + (ea & 15) * NLB + b);
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (sl[u] >= 0) {
                    if (fast) {
                        double2 x = acc[sl[u]];
                        x.x += km[u].x;
                        x.y += km[u].y;
                        acc[sl[u]] = x;
                    } else {
                        // a long row: its NLB lanes take turns (the order within an incidence is free: distinct slots)
                        if (K) K[lo + sl[u]] += km[u].x;
                        if (M) M[lo + sl[u]] += km[u].y;
                    }
                }
                __syncwarp();   // the next incidence may hit the same slot from another lane
            }
        }
        if (fast) {
            for (int j = b; j < L; j += NLB) {
                const double2 x = acc[j];
                if (K) stcs(K + lo + j, x.x);
                if (M) stcs(M + lo + j, x.y);
            }
        }
        __syncwarp();
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
                                     const int32_t* row_ptr, const int32_t* elem2nnz, int64_t nnz,
                                     const int32_t* node_elem_ptr, const int32_t* node_elem,
                                     const uint32_t* node_elem_slot, int gqo, double cK_a, const double* cK_b,
                                     double cM_a, const double* cM_b, double* K_vals, double* M_vals, double* K_local,
                                     double* M_local, int mode, void* work, size_t* work_bytes, vb_stream_t stream) {
    clear_error();
    const char* fn = "fem_p2_assemble";
    if (dim != 2 && dim != 3) { set_error("%s: dim=%d, need 2 or 3", fn, dim); return VB_ERR_UNSUPPORTED; }
    if (nn < 0 || ne < 0 || nnz < 0) { set_error("%s: negative size", fn); return VB_ERR_ARG; }
    if (mode != VB_ASSEMBLE_ATOMIC && mode != VB_ASSEMBLE_GATHER) { set_error("%s: unknown mode %d", fn, mode); return VB_ERR_ARG; }
    const int nlb = dim == 2 ? 6 : 10;
    const bool want_global = K_vals || M_vals;
    const size_t wbytes = (size_t)2 * nlb * nlb * (size_t)ne * 8 + 16;
    if (mode == VB_ASSEMBLE_GATHER && !work) {   // size query (CUB convention)
        if (!work_bytes) { set_error("%s: gather mode: work and work_bytes both NULL", fn); return VB_ERR_ARG; }
        *work_bytes = wbytes;
        return VB_OK;
    }
    P2Rule R;
    if (!p2_rule(dim, gqo, R)) { set_error("%s: gqo=%d unsupported (1, 2, 4)", fn, gqo); return VB_ERR_UNSUPPORTED; }
    if (ne > 0 && (!coords || !elems)) { set_error("%s: NULL coords or elems", fn); return VB_ERR_ARG; }
    if (elem_ld < ne) { set_error("%s: elem_ld < ne", fn); return VB_ERR_ARG; }
    if (mode == VB_ASSEMBLE_ATOMIC && want_global && !elem2nnz) { set_error("%s: atomic mode needs elem2nnz (fem_pattern)", fn); return VB_ERR_ARG; }
    if (mode == VB_ASSEMBLE_GATHER && want_global) {
        if (!row_ptr || !node_elem_ptr || !node_elem || !node_elem_slot) {
            set_error("%s: gather mode needs row_ptr, node_elem_ptr, node_elem, node_elem_slot", fn);
            return VB_ERR_ARG;
        }
        if (work_bytes && *work_bytes < wbytes) {
            set_error("%s: work buffer too small (%zu < %zu)", fn, *work_bytes, wbytes);
            return VB_ERR_WORKSPACE;
        }
    }
    P2Coef cp{cK_a, {0, 0, 0}, cM_a, {0, 0, 0}, false};
    for (int c = 0; c < dim; c++) {
        cp.kb[c] = cK_b ? cK_b[c] : 0.0;
        cp.mb[c] = cM_b ? cM_b[c] : 0.0;
    }
    cp.same = cK_a == cM_a && cp.kb[0] == cp.mb[0] && cp.kb[1] == cp.mb[1] && cp.kb[2] == cp.mb[2];
    cudaStream_t s = cs(stream);
    const bool gather = mode == VB_ASSEMBLE_GATHER && want_global;
    // gather staging: (K, M) pairs of the full element matrices, element-major
    double* Kst = gather ? reinterpret_cast<double*>(work) : nullptr;
    double* Mst = Kst;   // non-null: the M pass runs (its strip feeds the pairs)
    double* Ka = gather ? nullptr : K_vals;
    double* Ma = gather ? nullptr : M_vals;
    if ((Ka || Ma) && nnz > 0) zero2_p2_k<<<grid_for(nnz, 256, 8), 256, 0, s>>>(Ka, Ma, nnz);
    if (ne > 0 && (Ka || Ma || K_local || M_local || Kst || Mst)) {
        unsigned g = grid_for(ne, P2_BLOCK, 8);
        const size_t sm2 = (size_t)2 * P2_BLOCK * 21 * 8, sm3 = (size_t)2 * P2_BLOCK * 55 * 8;
        static bool attr = false;   // > 48 KB dynamic shared memory needs an opt-in
        if (!attr) {
            cudaFuncSetAttribute(p2_assemble_k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3);
            attr = true;
        }
        if (dim == 2) p2_assemble_k<2><<<g, P2_BLOCK, sm2, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, elem2nnz, R, cp, Ka, Ma, K_local, M_local, Kst, Mst);
        else p2_assemble_k<3><<<g, P2_BLOCK, sm3, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, elem2nnz, R, cp, Ka, Ma, K_local, M_local, Kst, Mst);
    }
    if (gather && nn > 0) {
        const double2* km = reinterpret_cast<const double2*>(work);
        auto runc = [&](auto kern, int G) {
            int occ = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * P2C_WARPS, 0);
            const int64_t cap = (int64_t)sm_count() * (occ > 0 ? occ : 1);
            const int64_t needc = (nn + (int64_t)G * P2C_WARPS - 1) / ((int64_t)G * P2C_WARPS);
            kern<<<(unsigned)(needc < cap ? needc : cap), 32 * P2C_WARPS, 0, s>>>(nn, row_ptr, node_elem_ptr, node_elem,
                                                                                 node_elem_slot, km, K_vals, M_vals);
        };
        if (dim == 2) runc(p2_gather_coop_k<6, P2_RS, 4>, 5);
        else runc(p2_gather_coop_k<10, P2_RS, 4>, 3);
    }
    return launch_check(fn);
}
