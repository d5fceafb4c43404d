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
#include <algorithm>
#include <atomic>
#include <type_traits>

#include "vb_internal.cuh"

namespace vb {
namespace {

template <int DIM>
struct P1 {
    static constexpr double INV_DFACT = DIM == 2 ? 0.5 : 1.0 / 6.0;
    static constexpr double MFACT = DIM == 2 ? 1.0 / 24.0 : 1.0 / 120.0;  // 1/(d! (d+1)(d+2))
};

// Coefficients c(x) = a exp(b . x) for K and M and the intquad order (NEXT-1).
struct CoefSpec {
    double ka, kb[3], ma, mb[3];
    int gqo;
    bool same;  // c_K == c_M: evaluate once
};

// intquad(2, dim): symmetric degree-2 rules, point q = (ALPHA at vertex q, BETA
// elsewhere), weight W each; WSUM = |T_ref| = 1/d! (reading: DESIGN.md §4).
template <int DIM>
struct QuadRule;
template <>
struct QuadRule<2> {
    static constexpr double ALPHA = 2.0 / 3.0, BETA = 1.0 / 6.0, W = 1.0 / 6.0, WSUM = 0.5, DFACT = 2.0;
};
template <>
struct QuadRule<3> {
    static constexpr double ALPHA = 0.58541019662496845446, BETA = 0.13819660112501051518, W = 1.0 / 24.0,
                            WSUM = 1.0 / 6.0, DFACT = 6.0;
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

// Element factors with coefficients (NEXT-1): kbar = d! sum_q w_q c_K(x_q) scales
// the c = 1 stiffness; Mloc[a][b] = |det| sum_q w_q c_M(x_q) lam_a(q) lam_b(q).
template <int DIM>
__device__ __forceinline__ double elem_coef(const double (&x)[DIM + 1][DIM], double adet, const CoefSpec& cp,
                                            double (&Mloc)[DIM + 1][DIM + 1]) {
    constexpr int NV = DIM + 1;
    const bool one = cp.gqo == 1;
    const double al = one ? 1.0 / NV : QuadRule<DIM>::ALPHA, be = one ? 1.0 / NV : QuadRule<DIM>::BETA;
    const double wq = one ? QuadRule<DIM>::WSUM : QuadRule<DIM>::W;
    const int nip = one ? 1 : NV;
    double sk = 0.0;
#pragma unroll
    for (int a = 0; a < NV; a++)
#pragma unroll
        for (int b = 0; b < NV; b++) Mloc[a][b] = 0.0;
#pragma unroll
    for (int q = 0; q < NV; q++) {
        if (q >= nip) break;
        double ek = 0.0, em = 0.0;
#pragma unroll
        for (int c = 0; c < DIM; c++) {
            double xc = 0.0;
#pragma unroll
            for (int a = 0; a < NV; a++) xc = fma(a == q ? al : be, x[a][c], xc);
            ek = fma(cp.kb[c], xc, ek);
            em = fma(cp.mb[c], xc, em);
        }
        const double ck = cp.ka * exp(ek);
        const double cm = cp.same ? ck : cp.ma * exp(em);
        sk += ck;
#pragma unroll
        for (int a = 0; a < NV; a++)
#pragma unroll
            for (int b = 0; b < NV; b++) Mloc[a][b] = fma(cm * (a == q ? al : be), b == q ? al : be, Mloc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < NV; a++)
#pragma unroll
        for (int b = 0; b < NV; b++) Mloc[a][b] *= adet * wq;
    return QuadRule<DIM>::DFACT * wq * sk;
}

// ------------------------------------------------------------ atomic variant
// Warp-aggregated scatter: lanes of one instruction that hit the same CSR entry (neighbouring elements
// share edges and vertices: 16 -> about 6 distinct targets per tet and matrix in Kuhn cell order) are found
// with match.any, every lane sums the values of its peers (one shuffle pair per round, rounds = the
// largest group of the warp) and the lowest lane of each group issues one RED for K and one for M.
// idx < 0: this lane has nothing to add.  Measured (tools/time_atomic.py): configs[4] 2.19 -> 1.85 ms (402.7 M
// -> ~153 M REDs; the match and the shuffle rounds cost most of what the L2 saves), configs[3] 0.85 -> 1.07 ms
// (6 of 9 targets per triangle are already distinct): aggregated in 3D only.
#ifndef VB_ATOMIC_AGG
#define VB_ATOMIC_AGG 1
#endif
template <bool AGG>
__device__ __forceinline__ void red_pair(double* __restrict__ K, double* __restrict__ M, int idx, double k,
                                         double m, int lane) {
  if constexpr (AGG) {
    const unsigned peers = __match_any_sync(0xffffffffu, idx < 0 ? -1 - lane : idx);
    const int rounds = __reduce_max_sync(0xffffffffu, __popc(peers));
    double ks = k, ms = m;
    unsigned rem = peers & ~(1u << lane);
    for (int r = 1; r < rounds; r++) {   // warp-uniform trip count
        const int src = rem ? __ffs(rem) - 1 : lane;
        rem &= rem - 1;
        const double kv = __shfl_sync(0xffffffffu, k, src), mv = __shfl_sync(0xffffffffu, m, src);
        if (src != lane) {
            ks += kv;
            ms += mv;
        }
    }
    if (idx >= 0 && (peers & ((1u << lane) - 1)) == 0) {
        if (K) atomicAdd(K + idx, ks);
        if (M) atomicAdd(M + idx, ms);
    }
  } else {
    if (idx >= 0) {
        if (K) atomicAdd(K + idx, k);
        if (M) atomicAdd(M + idx, m);
    }
  }
}

template <int DIM, bool COEF>
__global__ void __launch_bounds__(256) assemble_atomic_k(int64_t ne, const double* __restrict__ coords, int64_t ns,
                                                         int64_t cst, const int32_t* __restrict__ elems, int64_t eld,
                                                         const int32_t* __restrict__ e2n, double* __restrict__ K,
                                                         double* __restrict__ M, double* __restrict__ Kl,
                                                         double* __restrict__ Ml, const CoefSpec cp) {
    constexpr int NV = DIM + 1;
    constexpr bool AGG = VB_ATOMIC_AGG && DIM == 3;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    // whole warps run the loop (the aggregation is a warp collective); lanes past the end carry no element
    for (int64_t eb = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); eb < ne; eb += stride) {
        const bool valid = eb + lane < ne;
        const int64_t e = valid ? eb + lane : ne - 1;
        int32_t vid[NV];
        double x[NV][DIM], H[DIM][NV];
        load_element<DIM>(e, elems, eld, coords, ns, cst, vid, x);
        double det = element_H<DIM>(x, H);
        double adet = fabs(det);
        double s = P1<DIM>::INV_DFACT / adet;
        double m = P1<DIM>::MFACT * adet;
        double Mloc[NV][NV];
        if constexpr (COEF) s *= elem_coef<DIM>(x, adet, cp, Mloc);
#pragma unroll
        for (int a = 0; a < NV; a++)
#pragma unroll
            for (int b = a; b < NV; b++) {
                double d = H[0][a] * H[0][b];
#pragma unroll
                for (int r = 1; r < DIM; r++) d = fma(H[r][a], H[r][b], d);
                double k = s * d;
                double mm = COEF ? Mloc[a][b] : ((a == b) ? 2.0 * m : m);
                if (K || M) {
                    const int32_t pab = __ldcs(e2n + (int64_t)(a * NV + b) * ne + e);
                    red_pair<AGG>(K, M, valid ? pab : -1, k, mm, lane);
                }
                if (valid) {
                    if (Kl) stcs(Kl + (int64_t)(a + b * NV) * ne + e, k);
                    if (Ml) stcs(Ml + (int64_t)(a + b * NV) * ne + e, mm);
                }
                if (a != b) {
                    if (K || M) {
                        const int32_t pba = __ldcs(e2n + (int64_t)(b * NV + a) * ne + e);
                        red_pair<AGG>(K, M, valid ? pba : -1, k, mm, lane);
                    }
                    if (valid) {
                        if (Kl) stcs(Kl + (int64_t)(b + a * NV) * ne + e, k);
                        if (Ml) stcs(Ml + (int64_t)(b + a * NV) * ne + e, mm);
                    }
                }
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
// Persistent, software-pipelined: each CTA is one warp owning blocks of 32
// consecutive rows (lane = row).  The CSR columns and plan words of block k+1
// stream in through TMA bulk copies (cp.async.bulk + mbarrier) while block k is
// computed; each lane then gathers the coordinates of its next row's columns
// with cp.async (all requests in flight at once); that latency is covered by
// the other CTAs resident on the SM.  Per-row data (edge vectors, K and M
// accumulators) live in a lane-interleaved shared-memory layout ([slot][lane]),
// so every shared access of the inner loop is bank-conflict free; results are
// transposed to CSR order through shared memory and stored coalesced.
constexpr int GATHER_ROWS = 32;
// Shared-memory budget of one warp-CTA.  Per row of its block (averages over the
// block's 32 rows): CAP CSR entries, SLOT plan words.  Each row keeps its first
// RS columns in conflict-free [slot][lane] arrays; columns past RS go to an
// overflow area of OVF entries per block (CSR-like, rows in lane order).  A row
// that does not fit is computed by its lane in place in HBM.  The defaults keep
// 7 CTAs per SM in 3D (Kuhn rows: <= 15 columns, <= 24 incidences; Delaunay
// rows: mean ~16, ~26 incidences, ~40 % above 16 columns, <= ~60 overflow
// entries per block) and 16 in 2D.
#ifndef VB_GATHER_RS3
#define VB_GATHER_RS3 16
#endif
#ifndef VB_GATHER_CAP3
#define VB_GATHER_CAP3 17
#endif
#ifndef VB_GATHER_SLOT3
#define VB_GATHER_SLOT3 28
#endif
#ifndef VB_GATHER_OVF3
#define VB_GATHER_OVF3 56
#endif
#ifndef VB_GATHER_RS2
#define VB_GATHER_RS2 8
#endif
#ifndef VB_GATHER_CAP2
#define VB_GATHER_CAP2 8
#endif
#ifndef VB_GATHER_SLOT2
#define VB_GATHER_SLOT2 8
#endif
#ifndef VB_GATHER_OVF2
#define VB_GATHER_OVF2 32
#endif
// BUD = 1: the compact budget for meshes whose 32-row blocks all have rows of <= 15
// columns, <= 16*32 CSR entries and <= 25*32 incidences (Kuhn cubes; fem_plan_stats
// reports the plan's maxima, the caller passes VB_GATHER_HINT_COMPACT) with 16-bit
// plan words (fem_plan_pack_slots): 24.6 KB per CTA, 8 CTAs per SM in 3D (9 fit;
// see gather_ctas_per_sm).  Blocks that do not fit stay correct (in-place path).
template <int DIM, int NC = DIM, int BUD = 0>   // NC doubles staged per column slot: coordinates (+ coefficient factors)
struct GatherCfg {
    static constexpr bool CMP = BUD == 1 && DIM == 3;
    static constexpr int RS = CMP ? 15 : (DIM == 2 ? VB_GATHER_RS2 : VB_GATHER_RS3);  // columns per row in the lane arrays
    static constexpr int OVF = CMP ? 0 : (DIM == 2 ? VB_GATHER_OVF2 : VB_GATHER_OVF3);  // overflow columns per block
    static constexpr int LANE_CAP = GATHER_ROWS * RS;
    static constexpr int ACC_N = LANE_CAP + OVF;                         // accumulator / edge-vector slots
    static constexpr int CAP = GATHER_ROWS * (CMP ? 16 : (DIM == 2 ? VB_GATHER_CAP2 : VB_GATHER_CAP3));  // CSR entries of a block
    static constexpr int SLOT_CAP = GATHER_ROWS * (CMP ? 25 : (DIM == 2 ? VB_GATHER_SLOT2 : VB_GATHER_SLOT3));  // plan words
    // plan words: the packed 16-bit form (fem_plan_pack_slots) with the compact budget
    using SW = std::conditional_t<CMP, uint16_t, uint32_t>;
    static constexpr int SW_PER16 = 16 / (int)sizeof(SW);                // words per 16-byte TMA chunk
    static constexpr int COLS_PAD = CAP + 8, SLOTS_PAD = SLOT_CAP + 2 * SW_PER16;  // alignment slack of TMA copies
#ifndef VB_GATHER_RING
#define VB_GATHER_RING 2
#endif
    static constexpr int RING = VB_GATHER_RING;                          // plan-word buffers (2: double-buffered)
    static constexpr size_t COLS_BYTES = (size_t)COLS_PAD * 4;           // columns: one buffer (consumed early)
    static constexpr size_t SLOTS_BYTES = (size_t)SLOTS_PAD * sizeof(SW);
    static constexpr size_t SLOTS_OFF = COLS_BYTES;
    static constexpr size_t F_OFF = SLOTS_OFF + RING * SLOTS_BYTES;      // edge vectors / CSR staging
    static constexpr size_t ACC_OFF = F_OFF + (size_t)NC * ACC_N * 8;    // (K, M) pairs
    static constexpr size_t BAR_OFF = ACC_OFF + (size_t)2 * ACC_N * 8;
    static constexpr size_t SMEM = BAR_OFF + RING * 8;
    static_assert(2 * CAP <= NC * ACC_N, "K and M staging fit in the edge-vector buffer");
    static_assert(COLS_BYTES % 16 == 0 && SLOTS_BYTES % 16 == 0, "TMA destinations must stay 16-byte aligned");
    static_assert(DIM >= 2, "staging of K and M in CSR order reuses the edge-vector buffer");
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(smem_u32(bar)), "r"(parity)
                     : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// 1/x to ~1 ulp: hardware seed + two Newton steps (x > 0, normal)
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(y, fma(-x, y, 1.0), y);
    y = fma(y, fma(-x, y, 1.0), y);
    return y;
}

// One incidence: the element's K_e[a][o_j] (k[j]) and |det| (ad) with v = a as
// base vertex, from the edge vectors f_j = x_{o_j} - x_v (j = 1..d).  With
// coefficients (COEF) also M_e[a][o_j] (m[j]) and the row sum
// sum_b M_e[a][b] (mrow), and k scaled by the quadrature average of c_K.
template <int DIM>
struct IncOut {
    double k[DIM];
    double ad;
    int s[DIM];
    double m[DIM];
    double mrow;
};

// Coefficient-weighted evaluation (NEXT-1, Code stiff_scalar_P1 P:978-1004 with
// c(x) = a exp(b . x)): intquad(gqo) points in barycentric form, "point q near
// vertex q" (symmetric rules: lambda_q = alpha at vertex q, beta elsewhere),
// vertex 0 = the row's vertex, 1..d = the others.
// FAC (c_K = c_M): the coefficient at point q is taken from per-vertex factors
// P_i = exp(beta b.x_i), R_i = exp((alpha - beta) b.x_i) as a R_q prod_i P_i
// (= a exp(b.x_q) exactly in real arithmetic; gqo = 1: P_i = exp(b.x_i / nv),
// R = 1), so the hot loop evaluates no exponential.
template <int DIM, bool FAC>
__device__ __forceinline__ void apply_coef(IncOut<DIM>& o, const double (&xv)[DIM], const double (&f)[DIM][DIM],
                                           const CoefSpec& cp, const double (&P)[DIM + 1],
                                           const double (&R)[DIM + 1]) {
    constexpr int NV = DIM + 1;
    const bool one = cp.gqo == 1;
    const double al = one ? 1.0 / NV : QuadRule<DIM>::ALPHA, be = one ? 1.0 / NV : QuadRule<DIM>::BETA;
    const double wq = one ? QuadRule<DIM>::WSUM : QuadRule<DIM>::W;
    const int nip = one ? 1 : NV;
    double sk = 0.0, mrow = 0.0, mj[DIM];
#pragma unroll
    for (int j = 0; j < DIM; j++) mj[j] = 0.0;
    double prodP = 1.0;
    if constexpr (FAC) {
        prodP = cp.ka * P[0];
#pragma unroll
        for (int j = 1; j < NV; j++) prodP *= P[j];
    }
#pragma unroll
    for (int q = 0; q < NV; q++) {
        if (q >= nip) break;
        double ck, cm;
        if constexpr (FAC) {
            ck = one ? prodP : prodP * R[q];
            cm = ck;
        } else {
            double x[DIM];
#pragma unroll
            for (int c = 0; c < DIM; c++) {
                double s = xv[c];
#pragma unroll
                for (int j = 0; j < DIM; j++) s = fma(q == j + 1 ? al : be, f[j][c], s);
                x[c] = s;
            }
            double ek = 0.0, em = 0.0;
#pragma unroll
            for (int c = 0; c < DIM; c++) {
                ek = fma(cp.kb[c], x[c], ek);
                em = fma(cp.mb[c], x[c], em);
            }
            ck = cp.ka * exp(ek);
            cm = cp.same ? ck : cp.ma * exp(em);
        }
        sk += ck;
        const double la = q == 0 ? al : be;
        mrow = fma(cm, la, mrow);
#pragma unroll
        for (int j = 0; j < DIM; j++) mj[j] = fma(cm * la, q == j + 1 ? al : be, mj[j]);
    }
    const double kbar = QuadRule<DIM>::DFACT * wq * sk;   // d! sum_q w_q c_K(x_q): 1 for c = 1
#pragma unroll
    for (int j = 0; j < DIM; j++) {
        o.k[j] *= kbar;
        o.m[j] = o.ad * wq * mj[j];
    }
    o.mrow = o.ad * wq * mrow;
}

// fv(s, P, R): the per-vertex coefficient factors of column slot s (FAC);
// pv: those of the row's vertex
// sl: the incidence's plan word; PK: packed 16-bit form (4 bits per other vertex)
template <int DIM, bool COEF, bool FAC, bool PK, typename EV, typename FV>
__device__ __forceinline__ IncOut<DIM> incidence(uint32_t sl, EV ev, FV fv, const double (&xv)[DIM],
                                                 const double (&pv)[2], const CoefSpec& cp) {
    IncOut<DIM> o;
    double P[DIM + 1], R[DIM + 1];
    if constexpr (FAC) {
        P[0] = pv[0];
        R[0] = pv[1];
    }
    if constexpr (DIM == 3) {
        o.s[0] = PK ? (sl & 15) : ((sl >> 8) & 0xff);
        o.s[1] = PK ? ((sl >> 4) & 15) : ((sl >> 16) & 0xff);
        o.s[2] = PK ? ((sl >> 8) & 15) : (sl >> 24);
        double f1[3], f2[3], f3[3];
        ev(o.s[0], f1);
        ev(o.s[1], f2);
        ev(o.s[2], f3);
        double h1[3] = {fma(f2[1], f3[2], -f2[2] * f3[1]), fma(f2[2], f3[0], -f2[0] * f3[2]),
                        fma(f2[0], f3[1], -f2[1] * f3[0])};
        double h2[3] = {fma(f3[1], f1[2], -f3[2] * f1[1]), fma(f3[2], f1[0], -f3[0] * f1[2]),
                        fma(f3[0], f1[1], -f3[1] * f1[0])};
        double h3[3] = {fma(f1[1], f2[2], -f1[2] * f2[1]), fma(f1[2], f2[0], -f1[0] * f2[2]),
                        fma(f1[0], f2[1], -f1[1] * f2[0])};
        double ad = fabs(fma(f1[0], h1[0], fma(f1[1], h1[1], f1[2] * h1[2])));
        double r = rcp_nr(ad) * (-1.0 / 6.0);
        double ha[3];
#pragma unroll
        for (int c = 0; c < 3; c++) ha[c] = r * ((h1[c] + h2[c]) + h3[c]);
        o.k[0] = fma(ha[0], h1[0], fma(ha[1], h1[1], ha[2] * h1[2]));
        o.k[1] = fma(ha[0], h2[0], fma(ha[1], h2[1], ha[2] * h2[2]));
        o.k[2] = fma(ha[0], h3[0], fma(ha[1], h3[1], ha[2] * h3[2]));
        o.ad = ad;
        if constexpr (COEF) {
            const double f[3][3] = {{f1[0], f1[1], f1[2]}, {f2[0], f2[1], f2[2]}, {f3[0], f3[1], f3[2]}};
            if constexpr (FAC)
#pragma unroll
                for (int j = 0; j < 3; j++) fv(o.s[j], P[j + 1], R[j + 1]);
            apply_coef<3, FAC>(o, xv, f, cp, P, R);
        }
    } else {
        o.s[0] = PK ? (sl & 15) : ((sl >> 8) & 0xff);
        o.s[1] = PK ? ((sl >> 4) & 15) : ((sl >> 16) & 0xff);
        double f1[2], f2[2];
        ev(o.s[0], f1);
        ev(o.s[1], f2);
        // tjac rows f1, f2: adj columns h1 = (f2y, -f2x), h2 = (-f1y, f1x)
        double ad = fabs(fma(f1[0], f2[1], -f1[1] * f2[0]));
        double r = rcp_nr(ad) * -0.5;
        double hax = r * (f2[1] - f1[1]), hay = r * (f1[0] - f2[0]);
        o.k[0] = fma(hax, f2[1], -hay * f2[0]);
        o.k[1] = fma(-hax, f1[1], hay * f1[0]);
        o.ad = ad;
        if constexpr (COEF) {
            const double f[2][2] = {{f1[0], f1[1]}, {f2[0], f2[1]}};
            if constexpr (FAC)
#pragma unroll
                for (int j = 0; j < 2; j++) fv(o.s[j], P[j + 1], R[j + 1]);
            apply_coef<2, FAC>(o, xv, f, cp, P, R);
        }
    }
    return o;
}

// Accumulators of slot s at acc[ix(s)]: K at accK[ix(s)], M at accM[ix(s)], or
// (PACKED) the (K, M) pair at accK + ix(s), one 16-byte access for both.  An
// incidence's d slots are distinct vertices: load all, then store all.
template <int DIM, bool PACKED, bool WK, bool WM, bool COEF, typename IX>
__device__ __forceinline__ void accumulate(const IncOut<DIM>& o, double* __restrict__ accK, double* __restrict__ accM,
                                           IX ix, double& mrow) {
    int x[DIM];
#pragma unroll
    for (int j = 0; j < DIM; j++) x[j] = ix(o.s[j]);
    if constexpr (PACKED) {
        static_assert(WK && WM, "packed pairs carry both matrices");
        double2 a[DIM];
#pragma unroll
        for (int j = 0; j < DIM; j++) a[j] = *reinterpret_cast<const double2*>(accK + x[j]);
#pragma unroll
        for (int j = 0; j < DIM; j++)
            *reinterpret_cast<double2*>(accK + x[j]) = make_double2(a[j].x + o.k[j], a[j].y + (COEF ? o.m[j] : o.ad));
        if constexpr (COEF) mrow += o.mrow;
        return;
    }
    if constexpr (WK) {
        double a[DIM];
#pragma unroll
        for (int j = 0; j < DIM; j++) a[j] = accK[x[j]];
#pragma unroll
        for (int j = 0; j < DIM; j++) accK[x[j]] = a[j] + o.k[j];
    }
    if constexpr (WM) {
        double a[DIM];
#pragma unroll
        for (int j = 0; j < DIM; j++) a[j] = accM[x[j]];
#pragma unroll
        for (int j = 0; j < DIM; j++) accM[x[j]] = a[j] + (COEF ? o.m[j] : o.ad);
        if constexpr (COEF) mrow += o.mrow;
    }
}

// Off-diagonal contributions of incidences [i0, i1) of one row: K into accK,
// M into accM (c = 1: |det|, scaled by 1/(d!(d+1)(d+2)) when the row is
// finished); slot s of the row at acc[ix(s)].  EV(s, f) yields the edge vector
// from the row's vertex to its column s.  Incidences are evaluated U at a time
// (all loads and arithmetic before any accumulator store) and accumulated in
// ascending element order.  Returns the row sum of M (COEF only).
template <int DIM, bool PACKED, bool WK, bool WM, bool COEF, bool FAC, typename SW, typename EV, typename FV,
          typename IX>
__device__ __forceinline__ double gather_row_t(int i0, int i1, const SW* __restrict__ slots, EV ev, FV fv, IX ix,
                                               double* __restrict__ accK, double* __restrict__ accM,
                                               const double (&xv)[DIM], const double (&pv)[2],
                                               const CoefSpec& cp) {
#ifndef VB_GATHER_U
#define VB_GATHER_U 6   // 4: +2 % on config 5 (24 incidences per row = 4 chunks), -3 % on Delaunay
#endif
#ifndef VB_GATHER_UF
#define VB_GATHER_UF 4  // coefficient factors (FAC): 2 / 3 / 4 -> 1.29 / 1.28 / 1.25 ms (tab:KM_P1_3D L7)
#endif
    constexpr int U = COEF ? (FAC ? VB_GATHER_UF : 2) : VB_GATHER_U;
    constexpr bool PK = sizeof(SW) == 2;
    // (A lane-rotated incidence order, which makes the plan-word reads bank-conflict
    // free -- 8 -> 1 wavefronts, 13 % of the kernel's shared-memory wavefronts --
    // measured 0.530 vs 0.528 ms on config 5 and would give up the ascending order.)
    double mrow = 0.0;
    int i = i0;
    for (; i + U - 1 < i1; i += U) {
        IncOut<DIM> o[U];
#pragma unroll
        for (int u = 0; u < U; u++) o[u] = incidence<DIM, COEF, FAC, PK>(slots[i + u], ev, fv, xv, pv, cp);
#pragma unroll
        for (int u = 0; u < U; u++) accumulate<DIM, PACKED, WK, WM, COEF>(o[u], accK, accM, ix, mrow);
    }
    for (; i < i1; i++)
        accumulate<DIM, PACKED, WK, WM, COEF>(incidence<DIM, COEF, FAC, PK>(slots[i], ev, fv, xv, pv, cp), accK, accM, ix,
                                              mrow);
    return mrow;
}

// PAIRS: accM == accK + 1 (interleaved pairs), packed access when both are wanted
template <int DIM, bool PAIRS, bool COEF, bool FAC, typename SW, typename EV, typename FV, typename IX>
__device__ __forceinline__ double gather_row(int i0, int i1, const SW* __restrict__ slots, EV ev, FV fv, IX ix,
                                             double* __restrict__ accK, double* __restrict__ accM,
                                             const double (&xv)[DIM], const double (&pv)[2], const CoefSpec& cp) {
    if (accK && accM)
        return gather_row_t<DIM, PAIRS, true, true, COEF, FAC, SW>(i0, i1, slots, ev, fv, ix, accK, accM, xv, pv, cp);
    if (accK)
        return gather_row_t<DIM, false, true, false, COEF, FAC, SW>(i0, i1, slots, ev, fv, ix, accK, accM, xv, pv, cp);
    if (accM)
        return gather_row_t<DIM, false, false, true, COEF, FAC, SW>(i0, i1, slots, ev, fv, ix, accK, accM, xv, pv, cp);
    return 0.0;
}

// Diagonal of a row (slot s0 of L) from the off-diagonal sums (partition of
// unity): K_vv = -sum_{w!=v} K_vw; M_vv = (2/d) sum_{w!=v} M_vw for c = 1
// (the |det| sums are scaled here), M_vv = rowsum - sum_{w!=v} M_vw otherwise.
template <int DIM, int ST, bool COEF>
__device__ __forceinline__ void finish_row(int L, int s0, double* accK, double* accM, double mrow) {
    constexpr double MS = COEF ? 1.0 : (DIM == 2 ? 1.0 / 24.0 : 1.0 / 120.0);     // 1/(d! (d+1)(d+2))
    double sk = 0.0, sm = 0.0;
    for (int s = 0; s < L; s++) {
        if (s == s0) continue;
        if (accK) sk += accK[s * ST];
        if (accM) {
            double m = accM[s * ST] * MS;
            accM[s * ST] = m;
            sm += m;
        }
    }
    if (accK) accK[s0 * ST] = -sk;
    if (accM) accM[s0 * ST] = COEF ? mrow - sm : (DIM == 3 ? sm * (2.0 / 3.0) : sm);
}

struct BlockBounds {
    int64_t r0, r1;
    int32_t p0, p1, q0, q1;
    bool valid, fit;
};

template <int DIM, int BUD>
__device__ __forceinline__ BlockBounds block_bounds(int64_t b, int64_t nblocks, int64_t nn,
                                                    const int32_t* __restrict__ row_ptr,
                                                    const int32_t* __restrict__ nptr) {
    BlockBounds B{};
    B.valid = b < nblocks;
    if (!B.valid) return B;
    B.r0 = b * GATHER_ROWS;
    B.r1 = B.r0 + GATHER_ROWS < nn ? B.r0 + GATHER_ROWS : nn;
    B.p0 = __ldg(row_ptr + B.r0);
    B.p1 = __ldg(row_ptr + B.r1);
    B.q0 = __ldg(nptr + B.r0);
    B.q1 = __ldg(nptr + B.r1);
    using C = GatherCfg<DIM, DIM, BUD>;
    B.fit = (B.p1 - B.p0) <= C::CAP && (B.q1 - B.q0) <= C::SLOT_CAP;
    return B;
}

// per-lane view of one row of a block
struct RowInfo {
    int64_t v;
    int lo, L, i0, i1, s0;
    int ov;      // first overflow entry of the row (columns RS..L-1)
    bool own;    // the lane has a row
    bool fast;   // the row is computed in shared memory
    bool ovb;    // some row of the block uses the overflow area (warp-uniform)
};

template <int DIM, int NC, int BUD>
struct GatherSmem {
    using C = GatherCfg<DIM, NC, BUD>;
    char* base;
    __device__ int32_t* cols() { return reinterpret_cast<int32_t*>(base); }
    __device__ typename C::SW* slots(int r) {
        return reinterpret_cast<typename C::SW*>(base + C::SLOTS_OFF + r * C::SLOTS_BYTES);
    }
    __device__ double* F() { return reinterpret_cast<double*>(base + C::F_OFF); }
    __device__ double* acc() { return reinterpret_cast<double*>(base + C::ACC_OFF); }
    __device__ uint64_t* bar(int r) { return reinterpret_cast<uint64_t*>(base + C::BAR_OFF) + r; }
};

// Where slot s of lane t lives.  Edge-vector / column-coordinate buffer F:
// coordinate c of slot s < RS at [slot][coord][lane] -- every access of the
// inner loop is bank-conflict free; slot s >= RS at overflow entry ov + s - RS.
// Accumulators: (K, M) pair of slot s < RS at [slot][lane], else overflow.
// Blocks without overflow rows (all of Kuhn's) use the map without the select
// (OV = false): the select on every access cost 20 % on config 5.
// Measured and not kept: plan words read through L1 instead of TMA staging
// (0.572 vs 0.540 ms, even with 9 instead of 7 CTAs per SM); two warps per
// block sharing the staged data, each with its own accumulators over half of
// every row's incidences (10 warps per SM: 0.62 vs 0.55 ms).
// (Interleaving (x, y) pairs for 128-bit F loads measured slower: 0.549 vs 0.530 ms.)
template <int DIM, bool OV, int NC, int BUD>
struct LaneMap {
    int t, ov;
    __device__ __forceinline__ int f(int s, int c) const {   // component c of slot s
        using C = GatherCfg<DIM, NC, BUD>;
        if constexpr (!OV) return (s * NC + c) * GATHER_ROWS + t;
        return s < C::RS ? (s * NC + c) * GATHER_ROWS + t : NC * C::LANE_CAP + (ov + s - C::RS) * NC + c;
    }
    __device__ __forceinline__ int a(int s) const {   // in doubles: K at a(s), M at a(s) + 1
        using C = GatherCfg<DIM, NC, BUD>;
        if constexpr (!OV) return 2 * (s * GATHER_ROWS + t);
        return 2 * (s < C::RS ? s * GATHER_ROWS + t : C::LANE_CAP + ov + s - C::RS);
    }
};

// word offset of element x within its 16-byte aligned TMA chunk
__device__ __forceinline__ int tma_shift(int32_t x) { return x & 3; }

// lane 0 only: stream block B's columns (single buffer: the previous block's were
// consumed by its coordinate gather) and plan words (ring slot r)
template <int DIM, int NC, int BUD>
__device__ __forceinline__ void issue_tma(GatherSmem<DIM, NC, BUD>& S, int r, const BlockBounds& B,
                                          const int32_t* __restrict__ col_idx,
                                          const typename GatherCfg<DIM, NC, BUD>::SW* __restrict__ nslot) {
    using C = GatherCfg<DIM, NC, BUD>;
    constexpr uint32_t WM = C::SW_PER16 - 1;
    if (!B.valid) return;
    if (!B.fit) {  // keep the barrier's phase count in step with the ring: arrive with no bytes
        mbar_expect_tx(S.bar(r), 0);
        return;
    }
    uint32_t c0 = (uint32_t)B.p0 & ~3u, c1 = ((uint32_t)B.p1 + 3u) & ~3u;
    uint32_t s0 = (uint32_t)B.q0 & ~WM, s1 = ((uint32_t)B.q1 + WM) & ~WM;
    uint32_t bc = (c1 - c0) * 4, bs = (s1 - s0) * (uint32_t)sizeof(typename C::SW);
    // generic-proxy reads of the column buffer (previous block) before the async-proxy overwrite
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(S.bar(r), bc + bs);
    if (bc) tma_load_1d(S.cols(), col_idx + c0, bc, S.bar(r));
    if (bs) tma_load_1d(S.slots(r), nslot + s0, bs, S.bar(r));
}

// Load the lane's row of block B.  If the block is staged (its CSR and plan
// ranges fit), place the row (lane arrays + overflow), find its diagonal slot and
// gather its column coordinates into F.  Returns whether the block is staged.
template <int DIM, int NC, int BUD>
__device__ __forceinline__ bool prepare_block(GatherSmem<DIM, NC, BUD>& S, BlockBounds& B, RowInfo& R,
                                              const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ nptr,
                                              const double* __restrict__ coords, int64_t ns, int64_t cst) {
    using C = GatherCfg<DIM, NC, BUD>;
    const int t = threadIdx.x;
    R.v = B.r0 + t;
    R.own = B.valid && R.v < B.r1;
    R.lo = R.L = R.i0 = R.i1 = R.s0 = 0;
    if (R.own) {
        R.lo = __ldg(row_ptr + R.v);
        R.L = __ldg(row_ptr + R.v + 1) - R.lo;
        R.i0 = __ldg(nptr + R.v);
        R.i1 = __ldg(nptr + R.v + 1);
    }
    const bool staged = B.valid && B.fit;
    // overflow placement: exclusive warp scan of the columns past RS
    const int ex = staged && R.own && R.L > C::RS ? R.L - C::RS : 0;
    int inc = ex;
    if (__any_sync(0xffffffffu, ex > 0)) {
#pragma unroll
        for (int d = 1; d < GATHER_ROWS; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, d);
            if (t >= d) inc += y;
        }
    }
    R.ov = inc - ex;
    R.fast = staged && R.own && R.L > 0 && (ex == 0 || inc <= C::OVF);
    R.ovb = __any_sync(0xffffffffu, R.fast && ex > 0);
    if (R.fast) {
        const int32_t* cols = S.cols() + tma_shift(B.p0) + (R.lo - B.p0);
        double* F = S.F();
        auto gather = [&](auto lm) {
            for (int s = 0; s < R.L; s++) {
                int64_t w = cols[s];
                if (w == R.v) R.s0 = s;
#pragma unroll
                for (int c = 0; c < DIM; c++) cp_async8(F + lm.f(s, c), coords + c * cst + w * ns);
            }
        };
        if (R.ovb) gather(LaneMap<DIM, true, NC, BUD>{t, R.ov});
        else gather(LaneMap<DIM, false, NC, BUD>{t, R.ov});
    }
    return staged;
}

template <int DIM, bool COEF, bool FAC, int BUD>
__global__ void __launch_bounds__(GATHER_ROWS) assemble_gather_k(int64_t nn, const double* __restrict__ coords,
                                                                 int64_t ns, int64_t cst,
                                                                 const int32_t* __restrict__ row_ptr,
                                                                 const int32_t* __restrict__ col_idx,
                                                                 const int32_t* __restrict__ nptr,
                                                                 const void* __restrict__ nslot_v,
                                                                 double* __restrict__ K, double* __restrict__ M,
                                                                 const CoefSpec cp, unsigned int* __restrict__ ctr) {
    static_assert(COEF || !FAC, "factors are a coefficient mode");
    constexpr int NC = FAC ? DIM + 2 : DIM;   // staged per slot: coordinates (+ P, R factors)
    using Cfg = GatherCfg<DIM, NC, BUD>;
    constexpr int W = GATHER_ROWS;
    constexpr double MS = COEF ? 1.0 : (DIM == 2 ? 1.0 / 24.0 : 1.0 / 120.0);  // 1/(d! (d+1)(d+2))
    extern __shared__ __align__(16) char smem_raw[];
    GatherSmem<DIM, NC, BUD> S{smem_raw};
    using SW = typename Cfg::SW;
    const SW* __restrict__ nslot = static_cast<const SW*>(nslot_v);
    const int t = threadIdx.x;
    const int64_t nblocks = (nn + W - 1) / W;
    const int64_t gstep = gridDim.x;
    if (t == 0)
        for (int r = 0; r < Cfg::RING; r++) mbar_init(S.bar(r));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();

    // block schedule: the first two blocks of a CTA are static, the rest are taken
    // from a per-launch counter (ctr, zeroed by the host) as the CTA gets to them, so
    // CTAs on busier SM sub-partitions take fewer blocks; ctr == NULL: static stride
    // (the counter is read one block ahead of its use, so its latency is hidden)
    int64_t kstat = 2;
    unsigned int pending = 0;
    if (ctr && t == 0) pending = atomicAdd(ctr, 1u);
    auto next_block = [&]() -> int64_t {
        if (!ctr) return blockIdx.x + (kstat++) * gstep;
        const unsigned int v = __shfl_sync(0xffffffffu, pending, 0);
        if (t == 0) pending = atomicAdd(ctr, 1u);
        return 2 * gstep + v;
    };
    // prologue: TMA for this CTA's first block, then its coordinate gather
    BlockBounds B0 = block_bounds<DIM, BUD>(blockIdx.x, nblocks, nn, row_ptr, nptr);
    BlockBounds B1 = block_bounds<DIM, BUD>(blockIdx.x + gstep, nblocks, nn, row_ptr, nptr);
    if (t == 0) issue_tma<DIM, NC, BUD>(S, 0, B0, col_idx, nslot);
    if (B0.valid) mbar_wait(S.bar(0), 0);
    RowInfo R;
    bool staged = prepare_block<DIM, NC, BUD>(S, B0, R, row_ptr, nptr, coords, ns, cst);
    cp_async_commit();

    double* F = S.F();
    double* acc = S.acc();
    for (int64_t k = 0;; k++) {
        if (!B0.valid) break;
        constexpr bool DB = Cfg::RING == 2;
        const int rc = DB ? (int)(k & 1) : 0, rn = DB ? rc ^ 1 : 0;
        // stage k+1: stream its columns and plan words (every lane is past its column
        // reads); with a single plan buffer only once block k's incidences are done
        auto issue_next = [&]() {
            __syncwarp();
            if (t == 0) issue_tma<DIM, NC, BUD>(S, rn, B1, col_idx, nslot);
        };
        if (DB || !staged) issue_next();
        BlockBounds B2 = block_bounds<DIM, BUD>(B1.valid ? next_block() : nblocks, nblocks, nn, row_ptr, nptr);
        // stage k: its coordinates have landed
        cp_async_wait<0>();
        __syncwarp();
        if (staged) {
            const SW* slots = S.slots(rc) + (B0.q0 & (Cfg::SW_PER16 - 1)) - B0.q0;
            const int np = B0.p1 - B0.p0;
            auto run = [&](auto lm) {
                double mrow = 0.0;
                if (R.fast) {
                    for (int s = 0; s < R.L; s++) *reinterpret_cast<double2*>(acc + lm.a(s)) = make_double2(0.0, 0.0);
                    if constexpr (FAC) {
                        // per-slot coefficient factors from the staged coordinates (apply_coef)
                        constexpr int NV = DIM + 1;
                        const bool one = cp.gqo == 1;
                        const double be = one ? 1.0 / NV : QuadRule<DIM>::BETA;
                        const double amb = QuadRule<DIM>::ALPHA - QuadRule<DIM>::BETA;
                        for (int s = 0; s < R.L; s++) {
                            double bx = 0.0;
#pragma unroll
                            for (int c = 0; c < DIM; c++) bx = fma(cp.kb[c], F[lm.f(s, c)], bx);
                            F[lm.f(s, DIM)] = exp(be * bx);
                            F[lm.f(s, DIM + 1)] = one ? 1.0 : exp(amb * bx);
                        }
                    }
                    double xv[DIM], pv[2] = {1.0, 1.0};
#pragma unroll
                    for (int c = 0; c < DIM; c++) xv[c] = F[lm.f(R.s0, c)];
                    if constexpr (FAC) {
                        pv[0] = F[lm.f(R.s0, DIM)];
                        pv[1] = F[lm.f(R.s0, DIM + 1)];
                    }
                    auto ev = [&](int s, double(&f)[DIM]) {
                        VB_CHECK(s < R.L && s != R.s0);
#pragma unroll
                        for (int c = 0; c < DIM; c++) f[c] = F[lm.f(s, c)] - xv[c];
                    };
                    auto fv = [&](int s, double& P, double& Rq) {
                        P = F[lm.f(s, DIM)];
                        Rq = F[lm.f(s, DIM + 1)];
                    };
                    auto ix = [&](int s) { return lm.a(s); };
                    VB_CHECK(R.i0 >= B0.q0 && R.i1 <= B0.q1 && R.lo >= B0.p0 && R.lo + R.L <= B0.p1);
                    mrow = gather_row<DIM, true, COEF, FAC>(R.i0, R.i1, slots, ev, fv, ix, K ? acc : nullptr,
                                                            M ? acc + 1 : nullptr, xv, pv, cp);
                }
                if constexpr (!DB) issue_next();
                __syncwarp();
                // finish the row (diagonal from the partition of unity, M scale) while
                // transposing it to CSR order through the (now dead) edge-vector buffer
                double* stK = F;
                double* stM = F + Cfg::CAP;
                if (R.fast) {
                    double sk = 0.0, sm = 0.0;
                    const int b = R.lo - B0.p0;
                    for (int s = 0; s < R.L; s++) {
                        if (s == R.s0) continue;
                        const double2 km = *reinterpret_cast<const double2*>(acc + lm.a(s));
                        const double mm = km.y * MS;
                        sk += km.x;
                        sm += mm;
                        stK[b + s] = km.x;
                        stM[b + s] = mm;
                    }
                    stK[b + R.s0] = -sk;
                    stM[b + R.s0] = COEF ? mrow - sm : (DIM == 3 ? sm * (2.0 / 3.0) : sm);
                }
                __syncwarp();
                for (int q = t; q < np; q += W) {
                    if (K) stcs(K + B0.p0 + q, stK[q]);
                    if (M) stcs(M + B0.p0 + q, stM[q]);
                }
            };
            if (R.ovb) run(LaneMap<DIM, true, NC, BUD>{t, R.ov});
            else run(LaneMap<DIM, false, NC, BUD>{t, R.ov});
        }
        __syncwarp();   // orders the staged stores above before the in-place rows below
        if (R.own && R.L > 0 && !R.fast) {
            // rows that did not fit, or blocks outside the smem budget: same ownership,
            // everything in place in HBM (overwrites what the staged store left there)
            double* aK = K ? K + R.lo : nullptr;
            double* aM = M ? M + R.lo : nullptr;
            int s0 = 0;
            for (int q = 0; q < R.L; q++) {
                if (aK) aK[q] = 0.0;
                if (aM) aM[q] = 0.0;
                if (__ldg(col_idx + R.lo + q) == R.v) s0 = q;
            }
            double xv[DIM];
#pragma unroll
            for (int c = 0; c < DIM; c++) xv[c] = __ldg(coords + c * cst + R.v * ns);
            auto ev = [&](int s, double(&f)[DIM]) {
                VB_CHECK(s < R.L && s != s0);
                int64_t w = __ldg(col_idx + R.lo + s);
#pragma unroll
                for (int c = 0; c < DIM; c++) f[c] = __ldg(coords + c * cst + w * ns) - xv[c];
            };
            auto ix = [](int s) { return s; };
            const double pv[2] = {1.0, 1.0};
            auto nofac = [](int, double&, double&) {};   // no per-vertex factors on this path
            double mrow = gather_row<DIM, false, COEF, false, SW>(R.i0, R.i1, nslot, ev, nofac, ix, aK, aM, xv, pv, cp);
            finish_row<DIM, 1, COEF>(R.L, s0, aK, aM, mrow);
        }
        __syncwarp();
        // stage k+1: its columns have landed -> gather its coordinates into F (free now)
        if (B1.valid) mbar_wait(S.bar(rn), DB ? (uint32_t)(((k + 1) >> 1) & 1) : (uint32_t)((k + 1) & 1));
        staged = prepare_block<DIM, NC, BUD>(S, B1, R, row_ptr, nptr, coords, ns, cst);
        cp_async_commit();
        B0 = B1;
        B1 = B2;
    }
    cp_async_wait<0>();
}


// ------------------------------------------------------------ class variant (row classes)
// Same ownership, arithmetic and summation order as assemble_gather_k (one lane
// per row, incidences in ascending element order, diagonal from the partition
// of unity), but a warp takes up to 32 rows of one row class (fem_plan_classes:
// rows with identical signature -- row length, incidence count and plan words).
// The incidence loop is then warp-uniform: the class's plan words are decoded
// once per warp into a shared-memory table (the edge-vector offsets of each
// incidence, read with one broadcast load), the slots of an incidence are the
// same on every lane, and each lane keeps its row's K and M sums in registers:
// a uniform slot picks the register through an indexed branch (brx.idx, one
// jump-table load + branch per update) instead of a shared-memory
// read-modify-write.  Column coordinates stay in shared memory ([slot][coord][lane],
// conflict free); the edge vectors f_s = x_col(s) - x_v are formed as they are
// loaded (converting the buffer once per group measured 1.5 % slower: its shared
// traffic costs more than 9 subtractions per incidence).  Loads are pipelined one group ahead:
// the next group's rows and columns (cp.async) are requested before the
// current group's incidence loop.  Rows of the mixed class are assembled by
// their lane in place in HBM (as assemble_gather_k's fallback).
#ifndef VB_CLASS_PAIRS
#define VB_CLASS_PAIRS 1   // 3D: incidences paired over shared link edges (build_pairs)
#endif
#ifndef VB_CLASS_SKIP_DIAG
#define VB_CLASS_SKIP_DIAG 1
#endif
#ifndef VB_CLASS_SKIP_DIAG_C2
#define VB_CLASS_SKIP_DIAG_C2 1   // the 2D coefficient kernel too: 16 instead of 15 CTAs/SM (0.629 -> 0.614 ms, tab:KM_P1_2D L11)
#endif
template <int DIM, int NC = DIM>   // NC doubles staged per column slot: coordinates (+ P, R coefficient factors)
struct ClassCfg {
    // 2D: 8 columns for c = 1 (square meshes: rows of <= 7), 12 with coefficients (the
    // crossed-diagonal mesh of the paper's 2D tables: rows of 9); rows of a class longer
    // than FSLOTS are assembled in place like the mixed rows
    static constexpr int MAXL = DIM == 3 ? 16 : (NC > DIM ? 12 : 8);   // register accumulators per row
    static constexpr int FSLOTS = DIM == 3 ? 15 : (NC > DIM ? 12 : 8); // columns per row (<= the plan's maxl)
    static constexpr int MAXN = DIM == 3 ? 32 : 16;  // incidences per row (fem_plan_classes' maxn)
    // the diagonal column is the row's own vertex: its coordinates are never read from the
    // buffer (VB_CLASS_SKIP_DIAG: the buffer holds FSLOTS - 1 slots, slot s > s0 at s - 1)
    static constexpr bool SKIPD =
        VB_CLASS_SKIP_DIAG && ((DIM == 3 && NC == DIM) || (VB_CLASS_SKIP_DIAG_C2 && DIM == 2 && NC > DIM));
    static constexpr int FSTAGED = SKIPD ? FSLOTS - 1 : FSLOTS;
    static constexpr int MOFF = 32 * FSLOTS + 2;     // staging: K at [1, ..), M at [MOFF + 1, ..) (16-byte phase)
    static constexpr int FN = FSTAGED * NC * 32 > 2 * MOFF ? FSTAGED * NC * 32 : 2 * MOFF;   // doubles of the buffer
    static constexpr int SLOT_BYTES = NC * 32 * 8;   // stride of one slot in the edge-vector buffer
};

// aK[s] += k, aM[s] += m for a warp-uniform slot s (0 <= s < N): one indexed branch
#define VB_ACC_IN(i) "+d"(aK[i])
#define VB_ACC_IM(i) "+d"(aM[i])
__device__ __forceinline__ void acc_slot(double (&aK)[16], double (&aM)[16], int s, double k, double m) {
    asm(
        "{\n\t"
        "BT: .branchtargets L0, L1, L2, L3, L4, L5, L6, L7, L8, L9, L10, L11, L12, L13, L14, L15;\n\t"
        "brx.idx.uni %32, BT;\n\t"
        "L0: add.f64 %0, %0, %33; add.f64 %16, %16, %34; bra.uni END;\n\t"
        "L1: add.f64 %1, %1, %33; add.f64 %17, %17, %34; bra.uni END;\n\t"
        "L2: add.f64 %2, %2, %33; add.f64 %18, %18, %34; bra.uni END;\n\t"
        "L3: add.f64 %3, %3, %33; add.f64 %19, %19, %34; bra.uni END;\n\t"
        "L4: add.f64 %4, %4, %33; add.f64 %20, %20, %34; bra.uni END;\n\t"
        "L5: add.f64 %5, %5, %33; add.f64 %21, %21, %34; bra.uni END;\n\t"
        "L6: add.f64 %6, %6, %33; add.f64 %22, %22, %34; bra.uni END;\n\t"
        "L7: add.f64 %7, %7, %33; add.f64 %23, %23, %34; bra.uni END;\n\t"
        "L8: add.f64 %8, %8, %33; add.f64 %24, %24, %34; bra.uni END;\n\t"
        "L9: add.f64 %9, %9, %33; add.f64 %25, %25, %34; bra.uni END;\n\t"
        "L10: add.f64 %10, %10, %33; add.f64 %26, %26, %34; bra.uni END;\n\t"
        "L11: add.f64 %11, %11, %33; add.f64 %27, %27, %34; bra.uni END;\n\t"
        "L12: add.f64 %12, %12, %33; add.f64 %28, %28, %34; bra.uni END;\n\t"
        "L13: add.f64 %13, %13, %33; add.f64 %29, %29, %34; bra.uni END;\n\t"
        "L14: add.f64 %14, %14, %33; add.f64 %30, %30, %34; bra.uni END;\n\t"
        "L15: add.f64 %15, %15, %33; add.f64 %31, %31, %34;\n\t"
        "END: }\n"
        : VB_ACC_IN(0), VB_ACC_IN(1), VB_ACC_IN(2), VB_ACC_IN(3), VB_ACC_IN(4), VB_ACC_IN(5), VB_ACC_IN(6),
          VB_ACC_IN(7), VB_ACC_IN(8), VB_ACC_IN(9), VB_ACC_IN(10), VB_ACC_IN(11), VB_ACC_IN(12), VB_ACC_IN(13),
          VB_ACC_IN(14), VB_ACC_IN(15), VB_ACC_IM(0), VB_ACC_IM(1), VB_ACC_IM(2), VB_ACC_IM(3), VB_ACC_IM(4),
          VB_ACC_IM(5), VB_ACC_IM(6), VB_ACC_IM(7), VB_ACC_IM(8), VB_ACC_IM(9), VB_ACC_IM(10), VB_ACC_IM(11),
          VB_ACC_IM(12), VB_ACC_IM(13), VB_ACC_IM(14), VB_ACC_IM(15)
        : "r"(s), "d"(k), "d"(m));
}
__device__ __forceinline__ void acc_slot(double (&aK)[12], double (&aM)[12], int s, double k, double m) {
    asm(
        "{\n\t"
        "BT: .branchtargets L0, L1, L2, L3, L4, L5, L6, L7, L8, L9, L10, L11;\n\t"
        "brx.idx.uni %24, BT;\n\t"
        "L0: add.f64 %0, %0, %25; add.f64 %12, %12, %26; bra.uni END;\n\t"
        "L1: add.f64 %1, %1, %25; add.f64 %13, %13, %26; bra.uni END;\n\t"
        "L2: add.f64 %2, %2, %25; add.f64 %14, %14, %26; bra.uni END;\n\t"
        "L3: add.f64 %3, %3, %25; add.f64 %15, %15, %26; bra.uni END;\n\t"
        "L4: add.f64 %4, %4, %25; add.f64 %16, %16, %26; bra.uni END;\n\t"
        "L5: add.f64 %5, %5, %25; add.f64 %17, %17, %26; bra.uni END;\n\t"
        "L6: add.f64 %6, %6, %25; add.f64 %18, %18, %26; bra.uni END;\n\t"
        "L7: add.f64 %7, %7, %25; add.f64 %19, %19, %26; bra.uni END;\n\t"
        "L8: add.f64 %8, %8, %25; add.f64 %20, %20, %26; bra.uni END;\n\t"
        "L9: add.f64 %9, %9, %25; add.f64 %21, %21, %26; bra.uni END;\n\t"
        "L10: add.f64 %10, %10, %25; add.f64 %22, %22, %26; bra.uni END;\n\t"
        "L11: add.f64 %11, %11, %25; add.f64 %23, %23, %26;\n\t"
        "END: }\n"
        : VB_ACC_IN(0), VB_ACC_IN(1), VB_ACC_IN(2), VB_ACC_IN(3), VB_ACC_IN(4), VB_ACC_IN(5), VB_ACC_IN(6),
          VB_ACC_IN(7), VB_ACC_IN(8), VB_ACC_IN(9), VB_ACC_IN(10), VB_ACC_IN(11), VB_ACC_IM(0), VB_ACC_IM(1),
          VB_ACC_IM(2), VB_ACC_IM(3), VB_ACC_IM(4), VB_ACC_IM(5), VB_ACC_IM(6), VB_ACC_IM(7), VB_ACC_IM(8),
          VB_ACC_IM(9), VB_ACC_IM(10), VB_ACC_IM(11)
        : "r"(s), "d"(k), "d"(m));
}
__device__ __forceinline__ void acc_slot(double (&aK)[8], double (&aM)[8], int s, double k, double m) {
    asm(
        "{\n\t"
        "BT: .branchtargets L0, L1, L2, L3, L4, L5, L6, L7;\n\t"
        "brx.idx.uni %16, BT;\n\t"
        "L0: add.f64 %0, %0, %17; add.f64 %8, %8, %18; bra.uni END;\n\t"
        "L1: add.f64 %1, %1, %17; add.f64 %9, %9, %18; bra.uni END;\n\t"
        "L2: add.f64 %2, %2, %17; add.f64 %10, %10, %18; bra.uni END;\n\t"
        "L3: add.f64 %3, %3, %17; add.f64 %11, %11, %18; bra.uni END;\n\t"
        "L4: add.f64 %4, %4, %17; add.f64 %12, %12, %18; bra.uni END;\n\t"
        "L5: add.f64 %5, %5, %17; add.f64 %13, %13, %18; bra.uni END;\n\t"
        "L6: add.f64 %6, %6, %17; add.f64 %14, %14, %18; bra.uni END;\n\t"
        "L7: add.f64 %7, %7, %17; add.f64 %15, %15, %18;\n\t"
        "END: }\n"
        : VB_ACC_IN(0), VB_ACC_IN(1), VB_ACC_IN(2), VB_ACC_IN(3), VB_ACC_IN(4), VB_ACC_IN(5), VB_ACC_IN(6),
          VB_ACC_IN(7), VB_ACC_IM(0), VB_ACC_IM(1), VB_ACC_IM(2), VB_ACC_IM(3), VB_ACC_IM(4), VB_ACC_IM(5),
          VB_ACC_IM(6), VB_ACC_IM(7)
        : "r"(s), "d"(k), "d"(m));
}
#undef VB_ACC_IN
#undef VB_ACC_IM

// shared -> global bulk copy (TMA engine), bytes a multiple of 16, both ends 16-byte aligned
__device__ __forceinline__ void bulk_store(double* dst, const double* src, int bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// 3D: pair up a class's incidences whose link triangles share an edge (a, b):
// triangles (a, b, c) and (a, b, d) share fa x fb (the h of c and of d), so a
// pair loads 4 edge vectors instead of 6, forms 5 cross products instead of 6
// and makes 4 slot updates instead of 6.  Greedy in incidence order; a step is
// (x, y, z) = edge-vector offsets of a, b, c and w = a | b << 4 | c << 8 |
// d << 12 | CLASS_PAIR (slots < 16).  Reads and rewrites pat in place (step k
// is written after incidence k has been read; pairs only look ahead).
constexpr int CLASS_PAIR = 1 << 16;
__device__ __forceinline__ int staged_slot(int s, int s0, bool skip) { return skip ? s - (s > s0) : s; }
__device__ int build_pairs(int4* pat, int n, int slot_bytes, int s0, bool skip) {
    uint32_t used = 0;
    int k = 0;
    for (int i = 0; i < n; i++) {
        if ((used >> i) & 1) continue;
        used |= 1u << i;
        const int wi = pat[i].w;
        const int x = wi & 0xff, y = (wi >> 8) & 0xff, z = (wi >> 16) & 0xff;
        int step = x | y << 4 | z << 8, a = x, b = y, c = z;
        for (int j = i + 1; j < n; j++) {
            if ((used >> j) & 1) continue;
            const int wj = pat[j].w;
            const int u[3] = {wj & 0xff, (wj >> 8) & 0xff, (wj >> 16) & 0xff};
            int shared = 0, d = -1;
            for (int q = 0; q < 3; q++) {
                if (u[q] == x || u[q] == y || u[q] == z) shared++;
                else d = u[q];
            }
            if (shared != 2) continue;
            // the shared edge (a, b) and the third vertices c (of i) and d (of j)
            if (d == -1) break;
            if (x != u[0] && x != u[1] && x != u[2]) { a = y; b = z; c = x; }
            else if (y != u[0] && y != u[1] && y != u[2]) { a = z; b = x; c = y; }
            else { a = x; b = y; c = z; }
            used |= 1u << j;
            step = a | b << 4 | c << 8 | d << 12 | CLASS_PAIR;
            break;
        }
        pat[k++] = make_int4(staged_slot(a, s0, skip) * slot_bytes, staged_slot(b, s0, skip) * slot_bytes,
                             staged_slot(c, s0, skip) * slot_bytes, step);
    }
    return k;
}

// one group of the class plan as seen by lane t
struct ClassGroup {
    int pos, cnt, head;   // head < 0: mixed rows (or no group)
    int32_t v;            // the lane's row (t < cnt)
    int lo;               // row_ptr[v]
};

#ifndef VB_CLASS_SKIP_DIAG
#define VB_CLASS_SKIP_DIAG 1
#endif
#ifndef VB_CLASS_WIDTH_CHECK
#define VB_CLASS_WIDTH_CHECK 1   // 0: A/B timing only (unsafe for plans with 2D class rows of 9-12 entries)
#endif
#ifndef VB_CLASS_MINB2
#define VB_CLASS_MINB2 32   // 2D c = 1 kernel: 64 registers, 32 warps/SM (16 / 24 / 32: 0.204 / 0.184 / 0.165 ms, config 4)
#endif
#ifndef VB_CLASS_MINBC2
#define VB_CLASS_MINBC2 16  // 2D coefficient kernel (10 / 16 / 20: 0.704 / 0.637 / 0.723 ms, tab:KM_P1_2D L11)
#endif
#ifndef VB_CLASS_MINB
#define VB_CLASS_MINB 16
#endif
// COEF (3D): c_K = c_M = a exp(b . x) with the gqo = 2 rule (NEXT-1, Code
// stiff_scalar_P1 P:978-1004): per-node factors P_i = exp(beta b.x_i), R_i =
// exp((alpha - beta) b.x_i) (facP, facR) are staged next to the coordinates,
// so c at point q of an element is a R_q prod_i P_i (apply_coef); K_e is the
// c = 1 K_e times kbar = d! w sum_q c_q, M_e[v][x] = |det| w sum_q c_q
// lam_v(q) lam_x(q), and M_vv = row sum - off-diagonals.
template <int DIM, bool NS1, bool COEF = false>   // NS1: node_stride == 1 (SoA coordinate planes)
__global__ void __launch_bounds__(32, COEF ? (DIM == 2 ? VB_CLASS_MINBC2 : 10) : (DIM == 2 ? VB_CLASS_MINB2 : VB_CLASS_MINB))
    assemble_class_k(int64_t ngroups, const int4* __restrict__ groups,
                                                       const int32_t* __restrict__ class_rows,
                                                       const double* __restrict__ coords, int64_t ns, int64_t cst,
                                                       const int32_t* __restrict__ row_ptr,
                                                       const int32_t* __restrict__ col_idx,
                                                       const int32_t* __restrict__ nptr,
                                                       const uint32_t* __restrict__ nslot, double* __restrict__ K,
                                                       double* __restrict__ M, unsigned int* __restrict__ ctr,
                                                       bool bulk, int rounds, const double* __restrict__ facP,
                                                       const double* __restrict__ facR, CoefSpec cp) {
    constexpr int NC = COEF ? DIM + 2 : DIM;
    using C = ClassCfg<DIM, NC>;
    constexpr int MAXL = C::MAXL;
    constexpr unsigned FULL = 0xffffffffu;
    constexpr double MS = COEF ? 1.0 : (DIM == 2 ? 1.0 / 24.0 : 1.0 / 120.0);   // 1/(d! (d+1)(d+2))
    constexpr double KS = DIM == 2 ? -0.5 : -1.0 / 6.0;          // -1/d!
    __shared__ __align__(16) double F[C::FN];                    // edge vectors; then the CSR staging of K, M
    __shared__ __align__(16) int32_t colbuf[C::FSLOTS * 32];     // columns of the next group ([slot][lane])
    __shared__ __align__(16) int4 pat[C::MAXN];                  // decoded plan words of the current class
    const int t = threadIdx.x;
    const double* __restrict__ X[DIM];
#pragma unroll
    for (int c = 0; c < DIM; c++) X[c] = coords + c * cst;
    if constexpr (NS1) ns = 1;

    // schedule: the first `rounds` groups of a CTA are static (blockIdx.x + i * gridDim.x),
    // the rest come from a per-launch counter, fetched one group ahead (a counter fetch
    // per group made the counter's atomics a hot spot)
    unsigned int pending = 0;
    int64_t stat = 0;
    if (t == 0 && rounds <= 1 && ctr) pending = atomicAdd(ctr, 1u);
    auto next_id = [&]() -> int64_t {
        if (++stat < rounds || !ctr) {   // ctr == NULL: static schedule throughout
            if (stat == rounds - 1 && t == 0 && ctr) pending = atomicAdd(ctr, 1u);
            return (int64_t)blockIdx.x + stat * gridDim.x;
        }
        const unsigned int nx = __shfl_sync(FULL, pending, 0);
        if (t == 0) pending = atomicAdd(ctr, 1u);
        return (int64_t)rounds * gridDim.x + nx;
    };
    auto load_group = [&](int64_t g) -> int4 { return g < ngroups ? groups[g] : make_int4(0, 0, -1, 1); };
    auto rows_of = [&](const int4& G, ClassGroup& R) {   // R.v, R.lo for lane t
        R.pos = G.x;
        R.cnt = G.w ? 0 : G.y;   // w = 1 marks "no group"
        R.head = G.w ? -2 : G.z;
        R.v = 0;
        R.lo = 0;
        if (t < R.cnt) {
            R.v = __ldg(class_rows + R.pos + t);
            R.lo = __ldg(row_ptr + R.v);
        }
    };
    // columns to prefetch for a group: its row length, capped at the buffer (longer classes
    // are assembled in place and do not use the prefetched columns)
    auto clampL = [](int l) { return (DIM == 2 && !COEF && l > C::FSLOTS) ? C::FSLOTS : l; };
    auto issue_cols = [&](const ClassGroup& R, int L) {   // columns of a class group -> colbuf
        if (t < R.cnt)
            for (int s = 0; s < L; s++) cp_async4(colbuf + s * 32 + t, col_idx + R.lo + s);
        cp_async_commit();
    };

    ClassGroup cur, nxt;
    int4 G1, G2;
    {
        const int4 G0 = load_group(blockIdx.x);
        G1 = load_group(next_id());
        rows_of(G0, cur);
        if (cur.head >= 0) issue_cols(cur, clampL(__ldg(row_ptr + cur.head + 1) - __ldg(row_ptr + cur.head)));
    }
    int pat_head = -1, L = 0, n = 0, s0 = 0, nst = 0;   // nst: steps of the class's loop
    while (cur.head != -2) {
        bool fast = cur.head >= 0;
        // a class whose rows do not fit this kernel's column buffer (2D c = 1: the plan admits
        // 12 columns, the buffer holds 8) is assembled in place like the mixed rows
        if (VB_CLASS_WIDTH_CHECK && DIM == 2 && !COEF && fast && cur.head != pat_head &&
            __ldg(row_ptr + cur.head + 1) - __ldg(row_ptr + cur.head) > C::FSLOTS)
            fast = false;
        double xv[DIM], pvP = 0.0, pvR = 0.0;
        if (fast) {
            if (cur.head != pat_head) {   // class of this group: row length, incidences, decoded plan words
                pat_head = cur.head;
                L = __ldg(row_ptr + pat_head + 1) - __ldg(row_ptr + pat_head);
                const int ih = __ldg(nptr + pat_head);
                n = __ldg(nptr + pat_head + 1) - ih;
                s0 = (int)(__ldg(nslot + ih) & 0xffu);
                __syncwarp();
                for (int j = t; j < n; j += 32) {
                    const uint32_t w = __ldg(nslot + ih + j);
                    const int a = (w >> 8) & 0xff, b = (w >> 16) & 0xff, c = w >> 24;
                    pat[j] = make_int4(staged_slot(a, s0, C::SKIPD) * C::SLOT_BYTES,
                                       staged_slot(b, s0, C::SKIPD) * C::SLOT_BYTES,
                                       DIM == 3 ? staged_slot(c, s0, C::SKIPD) * C::SLOT_BYTES : 0,
                                       a | b << 8 | (DIM == 3 ? c : 0) << 16);
                }
                if constexpr (DIM == 3 && VB_CLASS_PAIRS) {
                    __syncwarp();
                    int k = 0;
                    if (t == 0) k = build_pairs(pat, n, C::SLOT_BYTES, s0, C::SKIPD);
                    nst = __shfl_sync(FULL, k, 0);
                    __syncwarp();
                } else {
                    nst = n;
                }
            }
            // this group's columns have landed: request their coordinates (into F, once the
            // previous group's bulk stores have read their staging from it)
            cp_async_wait<0>();
            if (t == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
            if (t < cur.cnt) {
                for (int s = 0; s < L; s++) {
                    if (C::SKIPD && s == s0) continue;   // the row's own vertex (xv)
                    const int w = colbuf[s * 32 + t];
                    const int sf = staged_slot(s, s0, C::SKIPD);
#pragma unroll
                    for (int c = 0; c < DIM; c++)
                        cp_async8(F + (sf * NC + c) * 32 + t, NS1 ? X[c] + w : X[c] + (int64_t)w * ns);
                    if constexpr (COEF) {
                        cp_async8(F + (sf * NC + DIM) * 32 + t, facP + w);
                        cp_async8(F + (sf * NC + DIM + 1) * 32 + t, facR + w);
                    }
                }
#pragma unroll
                for (int c = 0; c < DIM; c++) xv[c] = __ldg(X[c] + (int64_t)cur.v * ns);
                if constexpr (COEF) {
                    pvP = __ldg(facP + cur.v);
                    pvR = __ldg(facR + cur.v);
                }
            } else {
#pragma unroll
                for (int c = 0; c < DIM; c++) xv[c] = 0.0;
            }
            cp_async_commit();
        }
        // next group: its rows now, its columns once this group's coordinates have landed
        rows_of(G1, nxt);
        G2 = load_group(next_id());
        const int Ln = clampL(
            nxt.head >= 0 ? (nxt.head == pat_head ? L : __ldg(row_ptr + nxt.head + 1) - __ldg(row_ptr + nxt.head)) : 0);
        if (fast) {
            cp_async_wait<0>();
            __syncwarp();
            if (nxt.head >= 0) issue_cols(nxt, Ln);
            double aK[MAXL], aM[MAXL], mrow = 0.0;   // mrow: row sum of M (COEF)
#pragma unroll
            for (int s = 0; s < MAXL; s++) aK[s] = aM[s] = 0.0;
            const char* Fb = reinterpret_cast<const char*>(F) + t * 8;
            auto ld = [&](int off, double(&f)[DIM]) {
#pragma unroll
                for (int c = 0; c < DIM; c++)   // edge vector from the row's vertex
                    f[c] = *reinterpret_cast<const double*>(Fb + off + c * 256) - xv[c];
            };
            // incidence values: K_e[a][o_j] * (-d!) for the d other vertices, and |det|
            struct Inc {
                double k[DIM], ad;
                int w;
            };
            auto inc = [&](const int4& P) {
                Inc o;
                o.w = P.w;
                if constexpr (DIM == 3) {
                    double f1[3], f2[3], f3[3];
                    ld(P.x, f1);
                    ld(P.y, f2);
                    ld(P.z, f3);
                    const double h1[3] = {fma(f2[1], f3[2], -f2[2] * f3[1]), fma(f2[2], f3[0], -f2[0] * f3[2]),
                                          fma(f2[0], f3[1], -f2[1] * f3[0])};
                    const double h2[3] = {fma(f3[1], f1[2], -f3[2] * f1[1]), fma(f3[2], f1[0], -f3[0] * f1[2]),
                                          fma(f3[0], f1[1], -f3[1] * f1[0])};
                    const double h3[3] = {fma(f1[1], f2[2], -f1[2] * f2[1]), fma(f1[2], f2[0], -f1[0] * f2[2]),
                                          fma(f1[0], f2[1], -f1[1] * f2[0])};
                    o.ad = fabs(fma(f1[0], h1[0], fma(f1[1], h1[1], f1[2] * h1[2])));
                    const double r = rcp_nr(o.ad);
                    double S[3];
#pragma unroll
                    for (int c = 0; c < 3; c++) S[c] = r * ((h1[c] + h2[c]) + h3[c]);
                    o.k[0] = fma(S[0], h1[0], fma(S[1], h1[1], S[2] * h1[2]));
                    o.k[1] = fma(S[0], h2[0], fma(S[1], h2[1], S[2] * h2[2]));
                    o.k[2] = fma(S[0], h3[0], fma(S[1], h3[1], S[2] * h3[2]));
                } else {
                    double f1[2], f2[2];
                    ld(P.x, f1);
                    ld(P.y, f2);
                    // tjac rows f1, f2: adj columns h1 = (f2y, -f2x), h2 = (-f1y, f1x)
                    o.ad = fabs(fma(f1[0], f2[1], -f1[1] * f2[0]));
                    const double r = rcp_nr(o.ad);
                    const double hax = r * (f2[1] - f1[1]), hay = r * (f1[0] - f2[0]);
                    o.k[0] = fma(hax, f2[1], -hay * f2[0]);
                    o.k[1] = fma(-hax, f1[1], hay * f1[0]);
                }
                return o;
            };
            auto acc = [&](const Inc& o) {
#pragma unroll
                for (int q = 0; q < DIM; q++) acc_slot(aK, aM, (o.w >> (8 * q)) & 0xff, o.k[q], o.ad);
            };
            // one incidence at a time in ascending element order (two in flight, or the next
            // incidence's edge vectors loaded a step ahead, need registers the accumulators
            // hold: both measured slower)
            if constexpr (DIM == 3 && VB_CLASS_PAIRS) {
                auto cross = [](const double(&u)[3], const double(&v)[3], double(&o)[3]) {
                    o[0] = fma(u[1], v[2], -u[2] * v[1]);
                    o[1] = fma(u[2], v[0], -u[0] * v[2]);
                    o[2] = fma(u[0], v[1], -u[1] * v[0]);
                };
                auto dot = [](const double(&u)[3], const double(&v)[3]) {
                    return fma(u[0], v[0], fma(u[1], v[1], u[2] * v[2]));
                };
                int4 Pn = pat[0];
                if constexpr (COEF) {
                    constexpr double AL = QuadRule<3>::ALPHA, BE = QuadRule<3>::BETA, WQ = QuadRule<3>::W;
                    constexpr double B2 = BE * BE, GA = AL * BE - BE * BE, KW = QuadRule<3>::DFACT * WQ;
                    // per-row constants: a P_v, gamma R_v, (alpha - beta) R_v
                    const double aPv = cp.ka * pvP, gRv = GA * pvR, dRv = (AL - BE) * pvR;
                    auto lf = [&](int off, double& Pf, double& Rf) {   // the slot's staged P, R factors
                        Pf = *reinterpret_cast<const double*>(Fb + off + DIM * 256);
                        Rf = *reinterpret_cast<const double*>(Fb + off + (DIM + 1) * 256);
                    };
                    for (int j = 0; j < nst; j++) {
                        const int4 St = Pn;
                        Pn = pat[j + 1 < nst ? j + 1 : 0];
                        const int w = St.w;
                        double fa[3], fb[3], fc[3], P[3], ha[3], hb[3], Sv[3];
                        double Pa, Ra, Pb, Rb, Pc, Rc;
                        ld(St.x, fa);
                        ld(St.y, fb);
                        ld(St.z, fc);
                        lf(St.x, Pa, Ra);
                        lf(St.y, Pb, Rb);
                        lf(St.z, Pc, Rc);
                        cross(fa, fb, P);
                        cross(fb, fc, ha);
                        cross(fc, fa, hb);
                        const double ad = fabs(dot(fc, P));
                        const double r = rcp_nr(ad);
#pragma unroll
                        for (int c = 0; c < 3; c++) Sv[c] = r * ((P[c] + ha[c]) + hb[c]);
                        // element (v, a, b, c): c_q = a R_q P_v P_a P_b P_c
                        const double base = aPv * Pa * Pb, sRab = (pvR + Ra) + Rb;
                        const double p1 = base * Pc, sR1 = sRab + Rc;
                        const double kb1 = KW * p1 * sR1, mw1 = ad * WQ * p1, t1 = fma(B2, sR1, gRv);
                        double ka = kb1 * dot(Sv, ha), kb = kb1 * dot(Sv, hb);
                        const double kc = kb1 * dot(Sv, P);
                        double ma = mw1 * fma(GA, Ra, t1), mb = mw1 * fma(GA, Rb, t1);
                        const double mc = mw1 * fma(GA, Rc, t1);
                        double mr = mw1 * fma(BE, sR1, dRv);
                        if (w & CLASS_PAIR) {
                            // element (v, a, b, d)
                            double fd[3], Pd, Rd;
                            const int od = staged_slot((w >> 12) & 15, s0, C::SKIPD) * C::SLOT_BYTES;
                            ld(od, fd);
                            lf(od, Pd, Rd);
                            cross(fb, fd, ha);
                            cross(fd, fa, hb);
                            const double ad2 = fabs(dot(fd, P));
                            const double r2 = rcp_nr(ad2);
#pragma unroll
                            for (int c = 0; c < 3; c++) Sv[c] = r2 * ((P[c] + ha[c]) + hb[c]);
                            const double p2 = base * Pd, sR2 = sRab + Rd;
                            const double kb2 = KW * p2 * sR2, mw2 = ad2 * WQ * p2, t2 = fma(B2, sR2, gRv);
                            ka = fma(kb2, dot(Sv, ha), ka);
                            kb = fma(kb2, dot(Sv, hb), kb);
                            const double kd = kb2 * dot(Sv, P);
                            ma = fma(mw2, fma(GA, Ra, t2), ma);
                            mb = fma(mw2, fma(GA, Rb, t2), mb);
                            const double md = mw2 * fma(GA, Rd, t2);
                            mr = fma(mw2, fma(BE, sR2, dRv), mr);
                            acc_slot(aK, aM, w & 15, ka, ma);
                            acc_slot(aK, aM, (w >> 4) & 15, kb, mb);
                            acc_slot(aK, aM, (w >> 8) & 15, kc, mc);
                            acc_slot(aK, aM, (w >> 12) & 15, kd, md);
                        } else {
                            acc_slot(aK, aM, w & 15, ka, ma);
                            acc_slot(aK, aM, (w >> 4) & 15, kb, mb);
                            acc_slot(aK, aM, (w >> 8) & 15, kc, mc);
                        }
                        mrow += mr;
                    }
                } else
                for (int j = 0; j < nst; j++) {
                    const int4 St = Pn;
                    Pn = pat[j + 1 < nst ? j + 1 : 0];
                    const int w = St.w;
                    double fa[3], fb[3], fc[3], P[3], ha[3], hb[3], Sv[3];
                    ld(St.x, fa);
                    ld(St.y, fb);
                    ld(St.z, fc);
                    // triangle (a, b, c): h_a = fb x fc, h_b = fc x fa, h_c = fa x fb = P
                    cross(fa, fb, P);
                    cross(fb, fc, ha);
                    cross(fc, fa, hb);
                    const double ad = fabs(dot(fc, P));
                    const double r = rcp_nr(ad);
#pragma unroll
                    for (int c = 0; c < 3; c++) Sv[c] = r * ((P[c] + ha[c]) + hb[c]);
                    double ka = dot(Sv, ha), kb = dot(Sv, hb);
                    const double kc = dot(Sv, P);
                    if (w & CLASS_PAIR) {
                        // triangle (a, b, d): h_a = fb x fd, h_b = fd x fa, h_d = P
                        double fd[3];
                        ld(staged_slot((w >> 12) & 15, s0, C::SKIPD) * C::SLOT_BYTES, fd);
                        cross(fb, fd, ha);
                        cross(fd, fa, hb);
                        const double ad2 = fabs(dot(fd, P));
                        const double r2 = rcp_nr(ad2);
#pragma unroll
                        for (int c = 0; c < 3; c++) Sv[c] = r2 * ((P[c] + ha[c]) + hb[c]);
                        ka += dot(Sv, ha);
                        kb += dot(Sv, hb);
                        const double kd = dot(Sv, P);
                        const double ab = ad + ad2;
                        acc_slot(aK, aM, w & 15, ka, ab);
                        acc_slot(aK, aM, (w >> 4) & 15, kb, ab);
                        acc_slot(aK, aM, (w >> 8) & 15, kc, ad);
                        acc_slot(aK, aM, (w >> 12) & 15, kd, ad2);
                    } else {
                        acc_slot(aK, aM, w & 15, ka, ad);
                        acc_slot(aK, aM, (w >> 4) & 15, kb, ad);
                        acc_slot(aK, aM, (w >> 8) & 15, kc, ad);
                    }
                }
            } else {
                int4 Pa = pat[0];
                if constexpr (COEF && DIM == 2) {
                    // 2D coefficient path, one triangle (v, a, b) per step (as the 3D pairs)
                    constexpr double AL = QuadRule<2>::ALPHA, BE = QuadRule<2>::BETA, WQ = QuadRule<2>::W;
                    constexpr double B2 = BE * BE, GA = AL * BE - BE * BE, KW = QuadRule<2>::DFACT * WQ;
                    const double aPv = cp.ka * pvP, gRv = GA * pvR, dRv = (AL - BE) * pvR;
                    for (int j = 0; j < n; j++) {
                        const Inc o0 = inc(Pa);
                        const double Pa1 = *reinterpret_cast<const double*>(Fb + Pa.x + DIM * 256);
                        const double Ra1 = *reinterpret_cast<const double*>(Fb + Pa.x + (DIM + 1) * 256);
                        const double Pb1 = *reinterpret_cast<const double*>(Fb + Pa.y + DIM * 256);
                        const double Rb1 = *reinterpret_cast<const double*>(Fb + Pa.y + (DIM + 1) * 256);
                        Pa = pat[j + 1 < n ? j + 1 : 0];
                        const double p1 = aPv * Pa1 * Pb1, sR = (pvR + Ra1) + Rb1;
                        const double kb1 = KW * p1 * sR, mw = o0.ad * WQ * p1, t1 = fma(B2, sR, gRv);
                        acc_slot(aK, aM, o0.w & 0xff, kb1 * o0.k[0], mw * fma(GA, Ra1, t1));
                        acc_slot(aK, aM, (o0.w >> 8) & 0xff, kb1 * o0.k[1], mw * fma(GA, Rb1, t1));
                        mrow = fma(mw, fma(BE, sR, dRv), mrow);
                    }
                } else
                for (int j = 0; j < n; j++) {
                    const Inc o0 = inc(Pa);
                    Pa = pat[j + 1 < n ? j + 1 : 0];
                    acc(o0);
                }
            }
            __syncwarp();   // every lane is done with the edge vectors
            // finish the rows (diagonal from the partition of unity) and stage them in
            // CSR order: row t of the group at [t*L, t*L + L)
            const int lo0 = __shfl_sync(FULL, cur.lo, 0);
            const int sh = lo0 & 1;   // staging phase: entry q of the group at [sh + q] (16-byte aligned pairs)
            double* stK = F + sh;
            double* stM = F + C::MOFF + sh;
            if (t < cur.cnt) {
                double sk = 0.0, sm = 0.0;
#pragma unroll
                for (int s = 0; s < MAXL; s++)
                    if (s < L && s != s0) {
                        const double kk = aK[s] * KS, mm = aM[s] * MS;
                        sk += kk;
                        sm += mm;
                        stK[t * L + s] = kk;
                        stM[t * L + s] = mm;
                    }
                stK[t * L + s0] = -sk;
                stM[t * L + s0] = COEF ? mrow - sm : (DIM == 3 ? sm * (2.0 / 3.0) : sm);
            }
            __syncwarp();
            const int tot = cur.cnt * L;
            const bool contiguous = __shfl_sync(FULL, cur.lo, cur.cnt - 1) == lo0 + (cur.cnt - 1) * L;
            if (contiguous && bulk) {
                // consecutive rows: one CSR range [lo0, lo0 + tot).  Its 16-byte aligned body
                // goes out as bulk copies (cp.async.bulk, issued by lane 0); the odd first /
                // last entries as plain stores
                const int body = (tot - sh) & ~1;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (t == 0 && body > 0) {
                    if (K) bulk_store(K + lo0 + sh, stK + sh, body * 8);
                    if (M) bulk_store(M + lo0 + sh, stM + sh, body * 8);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                const int q = t == 1 ? 0 : tot - 1;   // lane 1: a leading odd entry, lane 2: a trailing one
                if ((t == 1 && sh) || (t == 2 && sh + body < tot && !(sh && tot == 1))) {
                    if (K) stcs(K + lo0 + q, stK[q]);
                    if (M) stcs(M + lo0 + q, stM[q]);
                }
            } else {
                // runs of consecutive rows, each one contiguous CSR range
                for (int k = 0; k < cur.cnt;) {
                    const int lok = __shfl_sync(FULL, cur.lo, k);
                    const unsigned brk =
                        __ballot_sync(FULL, t > k && t < cur.cnt && cur.lo != lok + (t - k) * L);
                    const int e = brk ? __ffs(brk) - 1 : cur.cnt;
                    for (int q = k * L + t; q < e * L; q += 32) {
                        if (K) stcs(K + lok + (q - k * L), stK[q]);
                        if (M) stcs(M + lok + (q - k * L), stM[q]);
                    }
                    k = e;
                }
            }
            __syncwarp();   // the staging area is the next group's edge-vector buffer
        } else {
            // (a too-wide class's prefetched columns may still be landing in colbuf)
            cp_async_wait<0>();
            __syncwarp();
            if (nxt.head >= 0) issue_cols(nxt, Ln);
            if (t < cur.cnt) {
                // mixed class: the lane's row in place in HBM
                const int32_t v = cur.v;
                const int lo = cur.lo;
                const int Lr = __ldg(row_ptr + v + 1) - lo;
                const int i0 = __ldg(nptr + v), i1 = __ldg(nptr + v + 1);
                if (Lr > 0) {
                    double* aK = K ? K + lo : nullptr;
                    double* aM = M ? M + lo : nullptr;
                    int z0 = 0;
                    for (int q = 0; q < Lr; q++) {
                        if (aK) aK[q] = 0.0;
                        if (aM) aM[q] = 0.0;
                        if (__ldg(col_idx + lo + q) == v) z0 = q;
                    }
                    double xr[DIM];
#pragma unroll
                    for (int c = 0; c < DIM; c++) xr[c] = __ldg(X[c] + (int64_t)v * ns);
                    auto ev = [&](int s, double(&f)[DIM]) {
                        int64_t w = __ldg(col_idx + lo + s);
#pragma unroll
                        for (int c = 0; c < DIM; c++) f[c] = __ldg(X[c] + w * ns) - xr[c];
                    };
                    auto ix = [](int s) { return s; };
                    if constexpr (COEF) {
                        const double pv[2] = {__ldg(facP + v), __ldg(facR + v)};
                        auto fv = [&](int s, double& Pf, double& Rf) {
                            const int64_t w = __ldg(col_idx + lo + s);
                            Pf = __ldg(facP + w);
                            Rf = __ldg(facR + w);
                        };
                        const double mr =
                            gather_row<DIM, false, true, true, uint32_t>(i0, i1, nslot, ev, fv, ix, aK, aM, xr, pv, cp);
                        finish_row<DIM, 1, true>(Lr, z0, aK, aM, mr);
                    } else {
                        const double pv[2] = {1.0, 1.0};
                        auto nofac = [](int, double&, double&) {};
                        const CoefSpec c1{1.0, {0, 0, 0}, 1.0, {0, 0, 0}, 2, true};
                        gather_row<DIM, false, false, false, uint32_t>(i0, i1, nslot, ev, nofac, ix, aK, aM, xr, pv,
                                                                       c1);
                        finish_row<DIM, 1, false>(Lr, z0, aK, aM, 0.0);
                    }
                }
            }
            __syncwarp();
        }
        cur = nxt;
        G1 = G2;
    }
    cp_async_wait<0>();
    if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Elements outside the domain of inverse_W (det tjac = 0, layeredInverse P:343-352): tjac rows
// x_{r+1} - x_0, det by cofactor expansion along row 0; warp-aggregated count into *out.
template <int DIM>
__global__ void count_degenerate_k(int64_t ne, const double* __restrict__ coords, int64_t ns, int64_t cst,
                                   const int32_t* __restrict__ elems, int64_t eld, int64_t* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t mine = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += stride) {
        double x[DIM + 1][DIM];
#pragma unroll
        for (int a = 0; a <= DIM; a++) {
            const int64_t v = elems[a * eld + e];
#pragma unroll
            for (int c = 0; c < DIM; c++) x[a][c] = coords[c * cst + v * ns];
        }
        double J[DIM][DIM];
#pragma unroll
        for (int r = 0; r < DIM; r++)
#pragma unroll
            for (int c = 0; c < DIM; c++) J[r][c] = x[r + 1][c] - x[0][c];
        double det;
        if (DIM == 2) det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        else det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                   J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
        // ... or two vertices with identical coordinates (with contracted cofactors a determinant that is 0 in
        // exact arithmetic may come out as a rounding residual): the same rule in every kernel that counts
        bool same = false;
#pragma unroll
        for (int a = 0; a <= DIM; a++)
#pragma unroll
            for (int b = a + 1; b <= DIM; b++) {
                bool eq = true;
#pragma unroll
                for (int c = 0; c < DIM; c++) eq = eq && x[a][c] == x[b][c];
                same = same || eq;
            }
        mine += det == 0.0 || same;
    }
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(reinterpret_cast<unsigned long long*>(out), (unsigned long long)mine);
}

}  // namespace
}  // namespace vb

using namespace vb;

namespace {

template <int DIM, bool COEF, bool FAC, int BUD>
void launch_gather(unsigned g, cudaStream_t s, int64_t nn, const double* coords, int64_t ns, int64_t cst,
                   const int32_t* row_ptr, const int32_t* col_idx, const int32_t* nptr, const void* nslot,
                   double* K, double* M, const CoefSpec& cp, unsigned int* ctr) {
    constexpr size_t SMEM = GatherCfg<DIM, FAC ? DIM + 2 : DIM, BUD>::SMEM;
    assemble_gather_k<DIM, COEF, FAC, BUD><<<g, GATHER_ROWS, SMEM, s>>>(nn, coords, ns, cst, row_ptr, col_idx, nptr,
                                                                        nslot, K, M, cp, ctr);
}

template <int DIM, bool COEF, bool FAC, int BUD>
int gather_ctas_per_sm() {
    static int n = 0;  // > 48 KB dynamic smem needs an opt-in; persistent grid size
    if (!n) {
        constexpr size_t SMEM = GatherCfg<DIM, FAC ? DIM + 2 : DIM, BUD>::SMEM;
        cudaFuncSetAttribute(assemble_gather_k<DIM, COEF, FAC, BUD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SMEM);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, assemble_gather_k<DIM, COEF, FAC, BUD>, GATHER_ROWS, SMEM);
        // (With a static block schedule, 4k+1 resident one-warp CTAs put 3 warps on one
        // SM sub-partition and every CTA waited for it: compact budget 9 CTAs 0.521 ms vs
        // 8 CTAs 0.476 ms.  The dynamic schedule lets those CTAs take fewer blocks:
        // 9 CTAs 0.467 ms; Delaunay 0.230 -> 0.200 ms.)
        if (n < 1) n = 1;
    }
    return n;
}

template <int DIM, bool COEF, bool FAC, int BUD>
vb_status run_gather(const char* fn, cudaStream_t s, int64_t nn, const double* coords, int64_t ns, int64_t cst,
                     const int32_t* row_ptr, const int32_t* col_idx, const int32_t* nptr, const void* nslot,
                     double* K, double* M, const CoefSpec& cp, unsigned int* ctr) {
    const int64_t nblocks = (nn + GATHER_ROWS - 1) / GATHER_ROWS;
    const int64_t cap = (int64_t)sm_count() * gather_ctas_per_sm<DIM, COEF, FAC, BUD>();
    const unsigned g = (unsigned)(nblocks < cap ? nblocks : cap);
    launch_gather<DIM, COEF, FAC, BUD>(g, s, nn, coords, ns, cst, row_ptr, col_idx, nptr, nslot, K, M, cp, ctr);
    return launch_check(fn);
}

template <int DIM, bool COEF>
void launch_element(unsigned g, cudaStream_t s, int64_t ne, const double* coords, int64_t ns, int64_t cst,
                    const int32_t* elems, int64_t eld, const int32_t* e2n, double* K, double* M, double* Kl, double* Ml,
                    const CoefSpec& cp) {
    assemble_atomic_k<DIM, COEF><<<g, 256, 0, s>>>(ne, coords, ns, cst, elems, eld, e2n, K, M, Kl, Ml, cp);
}

constexpr int ASSEMBLE_WORK_BYTES = 16;   // the launch's block counter (gather / class kernels)

template <int DIM>
vb_status assemble_impl(const char* fn, int64_t nn, int64_t ne, const double* coords, int64_t node_stride,
                        int64_t comp_stride, const int32_t* elems, int64_t elem_ld, const int32_t* row_ptr,
                        const int32_t* col_idx, int64_t nnz, const int32_t* elem2nnz, const int32_t* node_elem_ptr,
                        const uint32_t* node_elem_slot, double* K_vals, double* M_vals, double* K_local,
                        double* M_local, int mode, const CoefSpec* coef, unsigned int* ctr, int64_t* degenerate,
                        cudaStream_t s) {
    const bool compact = (mode & VB_GATHER_HINT_COMPACT) != 0;
    mode &= ~VB_GATHER_HINT_COMPACT;
    const bool want_global = K_vals || M_vals;
    const CoefSpec cp = coef ? *coef : CoefSpec{1.0, {0, 0, 0}, 1.0, {0, 0, 0}, 2, true};
    const bool C = coef != nullptr;
    vb_status st = VB_OK;
    if (degenerate) {   // elements outside the domain of inverse_W (det = 0), counted first
        cudaError_t e = cudaMemsetAsync(degenerate, 0, sizeof(int64_t), s);
        if (e != cudaSuccess) { set_error("%s: %s", fn, cudaGetErrorString(e)); return VB_ERR_CUDA; }
        if (ne > 0) {
            count_degenerate_k<DIM><<<grid_for(ne, 256, 8), 256, 0, s>>>(ne, coords, node_stride, comp_stride, elems,
                                                                         elem_ld, degenerate);
            if ((st = launch_check(fn)) != VB_OK) return st;
        }
    }
    if (mode == VB_ASSEMBLE_ATOMIC) {
        if (want_global && (!elem2nnz || !row_ptr)) { set_error("%s: atomic mode needs elem2nnz and row_ptr", fn); return VB_ERR_ARG; }
        if (want_global && nnz > 0) {
            zero2_k<<<grid_for(nnz, 256, 8), 256, 0, s>>>(K_vals, M_vals, nnz);
            if ((st = launch_check(fn)) != VB_OK) return st;
        }
        if (ne == 0 || (!want_global && !K_local && !M_local)) return VB_OK;
        unsigned g = grid_for(ne, 256, 8);
        if (C) launch_element<DIM, true>(g, s, ne, coords, node_stride, comp_stride, elems, elem_ld, elem2nnz, K_vals, M_vals, K_local, M_local, cp);
        else launch_element<DIM, false>(g, s, ne, coords, node_stride, comp_stride, elems, elem_ld, elem2nnz, K_vals, M_vals, K_local, M_local, cp);
        return launch_check(fn);
    }
    // gather mode
    if (want_global && (!row_ptr || !col_idx || !node_elem_ptr || !node_elem_slot)) {
        set_error("%s: gather mode needs row_ptr, col_idx, node_elem_ptr, node_elem_slot", fn);
        return VB_ERR_ARG;
    }
    if (want_global && nn > 0) {
        // c_K = c_M with gqo = 2 (the paper's benchmarks): per-vertex factors instead of
        // 4 exponentials per incidence (1.43 -> 1.25 ms on tab:KM_P1_3D level 7).  Not for
        // gqo = 1: one exponential per incidence is cheaper than staging the factors
        // (their smem costs 2 of 7 CTAs per SM; 0.81 -> 1.06 ms measured)
        const bool fac = C && cp.same && cp.gqo == 2;
        const bool cmp = compact && DIM == 3;
#define VB_RUN_GATHER(CO, FA, BU) \
    run_gather<DIM, CO, FA, BU>(fn, s, nn, coords, node_stride, comp_stride, row_ptr, col_idx, node_elem_ptr, \
                                node_elem_slot, K_vals, M_vals, cp, ctr)
        if (fac) st = cmp ? VB_RUN_GATHER(true, true, 1) : VB_RUN_GATHER(true, true, 0);
        else if (C) st = cmp ? VB_RUN_GATHER(true, false, 1) : VB_RUN_GATHER(true, false, 0);
        else st = cmp ? VB_RUN_GATHER(false, false, 1) : VB_RUN_GATHER(false, false, 0);
#undef VB_RUN_GATHER
        if (st != VB_OK) return st;
    }
    if ((K_local || M_local) && ne > 0) {
        unsigned g = grid_for(ne, 256, 8);
        if (C) launch_element<DIM, true>(g, s, ne, coords, node_stride, comp_stride, elems, elem_ld, nullptr, nullptr, nullptr, K_local, M_local, cp);
        else launch_element<DIM, false>(g, s, ne, coords, node_stride, comp_stride, elems, elem_ld, nullptr, nullptr, nullptr, K_local, M_local, cp);
        if ((st = launch_check(fn)) != VB_OK) return st;
    }
    return VB_OK;
}

vb_status assemble_entry(const char* fn, int dim, int64_t nn, int64_t ne, const double* coords, int64_t node_stride,
                         int64_t comp_stride, const int32_t* elems, int64_t elem_ld, const int32_t* row_ptr,
                         const int32_t* col_idx, int64_t nnz, const int32_t* elem2nnz, const int32_t* node_elem_ptr,
                         const uint32_t* node_elem_slot, double* K_vals, double* M_vals, double* K_local,
                         double* M_local, int mode, const CoefSpec* coef, void* work, size_t* work_bytes,
                         int64_t* degenerate, vb_stream_t stream) {
    clear_error();
    if (!work && work_bytes) {   // size query (CUB convention): the launch's block counter
        *work_bytes = ASSEMBLE_WORK_BYTES;
        return VB_OK;
    }
    if (work && work_bytes && *work_bytes < ASSEMBLE_WORK_BYTES) {
        set_error("%s: work_bytes %zu < %d", fn, *work_bytes, ASSEMBLE_WORK_BYTES);
        return VB_ERR_WORKSPACE;
    }
    if (dim != 2 && dim != 3) { set_error("%s: dim=%d, need 2 or 3", fn, dim); return VB_ERR_UNSUPPORTED; }
    if (nn < 0 || ne < 0 || nnz < 0) { set_error("%s: negative size", fn); return VB_ERR_ARG; }
    const int base_mode = mode & ~VB_GATHER_HINT_COMPACT;
    if (base_mode != VB_ASSEMBLE_ATOMIC && base_mode != VB_ASSEMBLE_GATHER) { set_error("%s: unknown mode %d", fn, mode); return VB_ERR_ARG; }
    if (ne > 0 && (!coords || !elems)) { set_error("%s: NULL %s", fn, !coords ? "coords" : "elems"); return VB_ERR_ARG; }
    if (elem_ld < ne) { set_error("%s: elem_ld < ne", fn); return VB_ERR_ARG; }
    if (base_mode == VB_ASSEMBLE_GATHER && (K_vals || M_vals) && nn > 0 &&
        ((col_idx && !aligned16(col_idx)) || (node_elem_slot && !aligned16(node_elem_slot)))) {
        // the gather kernels stream these two arrays with bulk copies (cp.async.bulk: 16-byte aligned sources)
        set_error("%s: col_idx and node_elem_slot must be 16-byte aligned in gather mode", fn);
        return VB_ERR_ARG;
    }
    unsigned int* ctr = nullptr;   // NULL work: static block schedule
    if (work) {
        if (!aligned16(work)) { set_error("%s: work must be 16-byte aligned", fn); return VB_ERR_ARG; }
        ctr = static_cast<unsigned int*>(work);
        cudaError_t e = cudaMemsetAsync(ctr, 0, sizeof(unsigned int), cs(stream));
        if (e != cudaSuccess) { set_error("%s: %s", fn, cudaGetErrorString(e)); return VB_ERR_CUDA; }
    }
    auto f = dim == 2 ? assemble_impl<2> : assemble_impl<3>;
    return f(fn, nn, ne, coords, node_stride, comp_stride, elems, elem_ld, row_ptr, col_idx, nnz, elem2nnz,
             node_elem_ptr, node_elem_slot, K_vals, M_vals, K_local, M_local, mode, coef, ctr, degenerate,
             cs(stream));
}

}  // namespace

extern "C" vb_status fem_p1_assemble(int dim, int64_t nn, int64_t ne, const double* coords, int64_t node_stride,
                                     int64_t comp_stride, const int32_t* elems, int64_t elem_ld,
                                     const int32_t* row_ptr, const int32_t* col_idx, int64_t nnz,
                                     const int32_t* elem2nnz, const int32_t* node_elem_ptr, const int32_t* node_elem,
                                     const uint32_t* node_elem_slot, double* K_vals, double* M_vals, double* K_local,
                                     double* M_local, int mode, void* work, size_t* work_bytes,
                                     int64_t* degenerate, vb_stream_t stream) {
    (void)node_elem;
    return assemble_entry("fem_p1_assemble", dim, nn, ne, coords, node_stride, comp_stride, elems, elem_ld, row_ptr,
                          col_idx, nnz, elem2nnz, node_elem_ptr, node_elem_slot, K_vals, M_vals, K_local, M_local,
                          mode, nullptr, work, work_bytes, degenerate, stream);
}

extern "C" vb_status fem_p1_assemble_coef(int dim, int64_t nn, int64_t ne, const double* coords, int64_t node_stride,
                                          int64_t comp_stride, const int32_t* elems, int64_t elem_ld,
                                          const int32_t* row_ptr, const int32_t* col_idx, int64_t nnz,
                                          const int32_t* elem2nnz, const int32_t* node_elem_ptr,
                                          const int32_t* node_elem, const uint32_t* node_elem_slot, int gqo,
                                          double cK_a, const double* cK_b, double cM_a, const double* cM_b,
                                          double* K_vals, double* M_vals, double* K_local, double* M_local, int mode,
                                          void* work, size_t* work_bytes, int64_t* degenerate, vb_stream_t stream) {
    (void)node_elem;
    clear_error();
    if (gqo != 1 && gqo != 2) { set_error("fem_p1_assemble_coef: gqo=%d, supported 1 and 2", gqo); return VB_ERR_UNSUPPORTED; }
    if (dim != 2 && dim != 3) { set_error("fem_p1_assemble_coef: dim=%d, need 2 or 3", dim); return VB_ERR_UNSUPPORTED; }
    CoefSpec cp{cK_a, {0, 0, 0}, cM_a, {0, 0, 0}, gqo, false};
    for (int c = 0; c < dim; c++) {
        cp.kb[c] = cK_b ? cK_b[c] : 0.0;
        cp.mb[c] = cM_b ? cM_b[c] : 0.0;
    }
    cp.same = cK_a == cM_a && cp.kb[0] == cp.mb[0] && cp.kb[1] == cp.mb[1] && cp.kb[2] == cp.mb[2];
    return assemble_entry("fem_p1_assemble_coef", dim, nn, ne, coords, node_stride, comp_stride, elems, elem_ld,
                          row_ptr, col_idx, nnz, elem2nnz, node_elem_ptr, node_elem_slot, K_vals, M_vals, K_local,
                          M_local, mode, &cp, work, work_bytes, degenerate, stream);
}

namespace vb {
namespace {

// per-node coefficient factors of the class coefficient path: P = exp(beta b.x), R = exp((alpha - beta) b.x)
template <int DIM>
__global__ void class_factors_k(int64_t nn, const double* __restrict__ coords, int64_t ns, int64_t cst, double b0,
                                double b1, double b2, double* __restrict__ P, double* __restrict__ R) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += stride) {
        double bx = fma(b0, coords[v * ns], b1 * coords[cst + v * ns]);
        if (DIM == 3) bx = fma(b0, coords[v * ns], fma(b1, coords[cst + v * ns], b2 * coords[2 * cst + v * ns]));
        P[v] = exp(QuadRule<DIM>::BETA * bx);
        R[v] = exp((QuadRule<DIM>::ALPHA - QuadRule<DIM>::BETA) * bx);
    }
}

template <typename Kern>
void class_launch(Kern kern, cudaStream_t s, int64_t ngroups, const int32_t* groups, const int32_t* class_rows,
                  const double* coords, int64_t node_stride, int64_t comp_stride, const int32_t* row_ptr,
                  const int32_t* col_idx, const int32_t* node_elem_ptr, const uint32_t* node_elem_slot, double* K,
                  double* M, unsigned int* ctr, bool bulk, const double* facP, const double* facR,
                  const CoefSpec& cp) {
    // resident CTAs per SM, cached per kernel (all instantiations share Kern's type)
    static const void* keys[16] = {};
    static int vals[16] = {};
    int n = 0, slot = -1;
    for (int i = 0; i < 16; i++) {
        if (keys[i] == reinterpret_cast<const void*>(kern)) { n = vals[i]; break; }
        if (!keys[i] && slot < 0) slot = i;
    }
    if (!n) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, 32, 0);
        if (n < 1) n = 1;
        if (slot >= 0) {
            vals[slot] = n;
            keys[slot] = reinterpret_cast<const void*>(kern);
        }
    }
    const int64_t cap = (int64_t)sm_count() * n;
    const unsigned g = (unsigned)(ngroups < cap ? ngroups : cap);
    // static rounds: about 3/4 of the groups, at least 1 (the first group)
#ifndef VB_CLASS_STATIC_Q
#define VB_CLASS_STATIC_Q 3
#endif
    const int rounds = (int)std::max<int64_t>(1, (ngroups / g) * VB_CLASS_STATIC_Q / 4);
    kern<<<g, 32, 0, s>>>(ngroups, reinterpret_cast<const int4*>(groups), class_rows, coords, node_stride,
                          comp_stride, row_ptr, col_idx, node_elem_ptr, node_elem_slot, K, M, ctr, bulk, rounds, facP,
                          facR, cp);
}

vb_status class_entry(const char* fn, int dim, int64_t nn, const double* coords, int64_t node_stride,
                      int64_t comp_stride, const int32_t* row_ptr, const int32_t* col_idx, int64_t nnz,
                      const int32_t* node_elem_ptr, const uint32_t* node_elem_slot, const int32_t* class_rows,
                      const int32_t* groups, int64_t ngroups, double* K_vals, double* M_vals, const CoefSpec* coef,
                      double* fac, unsigned int* ctr, vb_stream_t stream) {
    if (dim != 2 && dim != 3) { set_error("%s: dim=%d, need 2 or 3", fn, dim); return VB_ERR_UNSUPPORTED; }
    if (nn < 0 || nnz < 0 || ngroups < 0) { set_error("%s: negative size", fn); return VB_ERR_ARG; }
    if (!K_vals && !M_vals) return VB_OK;
    if (nn > 0 && (!coords || !row_ptr || !col_idx || !node_elem_ptr || !node_elem_slot || !class_rows || !groups)) {
        set_error("%s: NULL argument", fn);
        return VB_ERR_ARG;
    }
    if (ngroups == 0) return VB_OK;
    cudaStream_t s = cs(stream);
    if (ctr) {   // the caller's counter (work): zeroed in-stream, owned by this launch
        cudaError_t e = cudaMemsetAsync(ctr, 0, sizeof(unsigned int), s);
        if (e != cudaSuccess) { set_error("%s: %s", fn, cudaGetErrorString(e)); return VB_ERR_CUDA; }
    }
    // bulk (TMA) stores of contiguous groups need 16-byte aligned value arrays
    const bool bulk = (!K_vals || aligned16(K_vals)) && (!M_vals || aligned16(M_vals));
    const CoefSpec c1{1.0, {0, 0, 0}, 1.0, {0, 0, 0}, 2, true};
    const double* fP = nullptr;
    const double* fR = nullptr;
    if (coef) {
        fP = fac;
        fR = fac + nn;
        auto fk = dim == 3 ? class_factors_k<3> : class_factors_k<2>;
        fk<<<grid_for(nn, 256, 8), 256, 0, s>>>(nn, coords, node_stride, comp_stride, coef->kb[0], coef->kb[1],
                                                coef->kb[2], fac, fac + nn);
        vb_status st = launch_check(fn);
        if (st != VB_OK) return st;
    }
    const CoefSpec& cp = coef ? *coef : c1;
#define VB_CLASS_LAUNCH(KERN)                                                                                      \
    class_launch(KERN, s, ngroups, groups, class_rows, coords, node_stride, comp_stride, row_ptr, col_idx,          \
                 node_elem_ptr, node_elem_slot, K_vals, M_vals, ctr, bulk, fP, fR, cp)
    if (coef) {
        if (node_stride == 1) {
            if (dim == 3) VB_CLASS_LAUNCH((assemble_class_k<3, true, true>));
            else VB_CLASS_LAUNCH((assemble_class_k<2, true, true>));
        } else {
            if (dim == 3) VB_CLASS_LAUNCH((assemble_class_k<3, false, true>));
            else VB_CLASS_LAUNCH((assemble_class_k<2, false, true>));
        }
    } else if (node_stride == 1) {
        if (dim == 3) VB_CLASS_LAUNCH((assemble_class_k<3, true>));
        else VB_CLASS_LAUNCH((assemble_class_k<2, true>));
    } else {
        if (dim == 3) VB_CLASS_LAUNCH((assemble_class_k<3, false>));
        else VB_CLASS_LAUNCH((assemble_class_k<2, false>));
    }
#undef VB_CLASS_LAUNCH
    return launch_check(fn);
}

}  // namespace
}  // namespace vb

extern "C" vb_status fem_p1_assemble_classes(int dim, int64_t nn, const double* coords, int64_t node_stride,
                                             int64_t comp_stride, const int32_t* row_ptr, const int32_t* col_idx,
                                             int64_t nnz, const int32_t* node_elem_ptr,
                                             const uint32_t* node_elem_slot, const int32_t* class_rows,
                                             const int32_t* groups, int64_t ngroups, double* K_vals,
                                             double* M_vals, void* work, size_t* work_bytes, vb_stream_t stream) {
    const char* fn = "fem_p1_assemble_classes";
    clear_error();
    if (!work && work_bytes) {
        *work_bytes = ASSEMBLE_WORK_BYTES;
        return VB_OK;
    }
    if (work && ((work_bytes && *work_bytes < ASSEMBLE_WORK_BYTES) || !aligned16(work))) {
        set_error("%s: work needs %d bytes, 16-byte aligned", fn, ASSEMBLE_WORK_BYTES);
        return VB_ERR_WORKSPACE;
    }
    return class_entry(fn, dim, nn, coords, node_stride, comp_stride, row_ptr, col_idx, nnz, node_elem_ptr,
                       node_elem_slot, class_rows, groups, ngroups, K_vals, M_vals, nullptr, nullptr,
                       static_cast<unsigned int*>(work), stream);
}

extern "C" vb_status fem_p1_assemble_classes_coef(int dim, int64_t nn, const double* coords, int64_t node_stride,
                                                  int64_t comp_stride, const int32_t* row_ptr,
                                                  const int32_t* col_idx, int64_t nnz,
                                                  const int32_t* node_elem_ptr, const uint32_t* node_elem_slot,
                                                  const int32_t* class_rows, const int32_t* groups, int64_t ngroups,
                                                  int gqo, double c_a, const double* c_b, double* work,
                                                  double* K_vals, double* M_vals, vb_stream_t stream) {
    const char* fn = "fem_p1_assemble_classes_coef";
    clear_error();
    if ((dim != 2 && dim != 3) || gqo != 2) {
        set_error("%s: dim=%d gqo=%d: the class coefficient path needs gqo = 2", fn, dim, gqo);
        return VB_ERR_UNSUPPORTED;
    }
    if (nn > 0 && (K_vals || M_vals) && !work) { set_error("%s: NULL work (2 nn doubles)", fn); return VB_ERR_ARG; }
    CoefSpec cp{c_a, {0, 0, 0}, c_a, {0, 0, 0}, 2, true};
    for (int c = 0; c < dim; c++) cp.kb[c] = cp.mb[c] = c_b ? c_b[c] : 0.0;   // c_b holds dim doubles
    // work: 2 nn factors, then the launch's block counter
    return class_entry(fn, dim, nn, coords, node_stride, comp_stride, row_ptr, col_idx, nnz, node_elem_ptr,
                       node_elem_slot, class_rows, groups, ngroups, K_vals, M_vals, &cp, work,
                       work ? reinterpret_cast<unsigned int*>(work + 2 * nn) : nullptr, stream);
}
