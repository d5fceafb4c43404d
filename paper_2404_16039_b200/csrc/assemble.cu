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
template <int DIM>
struct GatherCfg {
    static constexpr int RS = DIM == 2 ? 8 : 16;                        // max columns per row (fast path)
    static constexpr int CAP = GATHER_ROWS * RS;                         // CSR entries per block
    static constexpr int SLOT_CAP = GATHER_ROWS * (DIM == 2 ? 8 : 28);   // plan words per block
    static constexpr int COLS_PAD = CAP + 8, SLOTS_PAD = SLOT_CAP + 8;  // 16-byte alignment slack of TMA copies
    static constexpr int RING = 2;
    static constexpr size_t RING_BYTES = (size_t)(COLS_PAD + SLOTS_PAD) * 4;
    static constexpr size_t F_OFF = RING * RING_BYTES;                   // [RS*DIM][32] edge vectors / CSR staging
    static constexpr size_t ACC_OFF = F_OFF + (size_t)DIM * CAP * 8;     // [RS][32] K, then [RS][32] M
    static constexpr size_t BAR_OFF = ACC_OFF + (size_t)2 * CAP * 8;
    static constexpr size_t SMEM = BAR_OFF + RING * 8;
    static_assert(RING_BYTES % 16 == 0, "TMA destinations must stay 16-byte aligned");
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
// base vertex, from the edge vectors f_j = x_{o_j} - x_v (j = 1..d).
template <int DIM>
struct IncOut {
    double k[DIM];
    double ad;
    int s[DIM];
};

template <int DIM, typename EV>
__device__ __forceinline__ IncOut<DIM> incidence(uint32_t sl, EV ev) {
    IncOut<DIM> o;
    if constexpr (DIM == 3) {
        o.s[0] = (sl >> 8) & 0xff;
        o.s[1] = (sl >> 16) & 0xff;
        o.s[2] = sl >> 24;
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
    } else {
        o.s[0] = (sl >> 8) & 0xff;
        o.s[1] = (sl >> 16) & 0xff;
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
    }
    return o;
}

// acc[s*ST] += contributions of one incidence (its d slots are distinct
// vertices: load all, then store all)
template <int DIM, int ST, bool WK, bool WM>
__device__ __forceinline__ void accumulate(const IncOut<DIM>& o, double* __restrict__ accK, double* __restrict__ accM) {
    if constexpr (WK) {
        double a[DIM];
#pragma unroll
        for (int j = 0; j < DIM; j++) a[j] = accK[o.s[j] * ST];
#pragma unroll
        for (int j = 0; j < DIM; j++) accK[o.s[j] * ST] = a[j] + o.k[j];
    }
    if constexpr (WM) {
        double a[DIM];
#pragma unroll
        for (int j = 0; j < DIM; j++) a[j] = accM[o.s[j] * ST];
#pragma unroll
        for (int j = 0; j < DIM; j++) accM[o.s[j] * ST] = a[j] + o.ad;
    }
}

// Off-diagonal contributions of incidences [i0, i1) of one row: K into accK,
// |det| into accM (scaled by 1/(d!(d+1)(d+2)) in finish_row); slot s of the
// row lives at acc[s * ST].  EV(s, f) yields the edge vector from the row's
// vertex to its column s.  Incidences are evaluated four at a time (all loads
// and arithmetic of all before any accumulator store) and accumulated in
// ascending element order.
template <int DIM, int ST, bool WK, bool WM, typename EV>
__device__ __forceinline__ void gather_row_t(int i0, int i1, const uint32_t* __restrict__ slots, EV ev,
                                             double* __restrict__ accK, double* __restrict__ accM) {
    constexpr int U = 4;
    int i = i0;
    for (; i + U - 1 < i1; i += U) {
        IncOut<DIM> o[U];
#pragma unroll
        for (int u = 0; u < U; u++) o[u] = incidence<DIM>(slots[i + u], ev);
#pragma unroll
        for (int u = 0; u < U; u++) accumulate<DIM, ST, WK, WM>(o[u], accK, accM);
    }
    for (; i < i1; i++) accumulate<DIM, ST, WK, WM>(incidence<DIM>(slots[i], ev), accK, accM);
}

template <int DIM, int ST, typename EV>
__device__ __forceinline__ void gather_row(int i0, int i1, const uint32_t* __restrict__ slots, EV ev,
                                           double* __restrict__ accK, double* __restrict__ accM) {
    if (accK && accM) gather_row_t<DIM, ST, true, true>(i0, i1, slots, ev, accK, accM);
    else if (accK) gather_row_t<DIM, ST, true, false>(i0, i1, slots, ev, accK, accM);
    else if (accM) gather_row_t<DIM, ST, false, true>(i0, i1, slots, ev, accK, accM);
}

// Diagonal of a row (slot s0 of L) from the off-diagonal sums (partition of
// unity), and the |det| sums of M scaled to M entries.
template <int DIM, int ST>
__device__ __forceinline__ void finish_row(int L, int s0, double* accK, double* accM) {
    constexpr double MS = DIM == 2 ? 1.0 / 24.0 : 1.0 / 120.0;     // 1/(d! (d+1)(d+2))
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
    if (accM) accM[s0 * ST] = DIM == 3 ? sm * (2.0 / 3.0) : sm;
}

struct BlockBounds {
    int64_t r0, r1;
    int32_t p0, p1, q0, q1;
    bool valid, fit;
};

template <int DIM>
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
    B.fit = (B.p1 - B.p0) <= GatherCfg<DIM>::CAP && (B.q1 - B.q0) <= GatherCfg<DIM>::SLOT_CAP;
    return B;
}

// per-lane view of one row of a block
struct RowInfo {
    int64_t v;
    int lo, L, i0, i1, s0;
    bool own;
};

template <int DIM>
struct GatherSmem {
    char* base;
    __device__ int32_t* cols(int r) { return reinterpret_cast<int32_t*>(base + r * GatherCfg<DIM>::RING_BYTES); }
    __device__ uint32_t* slots(int r) {
        return reinterpret_cast<uint32_t*>(base + r * GatherCfg<DIM>::RING_BYTES + GatherCfg<DIM>::COLS_PAD * 4);
    }
    __device__ double* F() { return reinterpret_cast<double*>(base + GatherCfg<DIM>::F_OFF); }
    __device__ double* accK() { return reinterpret_cast<double*>(base + GatherCfg<DIM>::ACC_OFF); }
    __device__ double* accM() { return accK() + GatherCfg<DIM>::CAP; }
    __device__ uint64_t* bar(int r) { return reinterpret_cast<uint64_t*>(base + GatherCfg<DIM>::BAR_OFF) + r; }
};

// word offset of element x within its 16-byte aligned TMA chunk
__device__ __forceinline__ int tma_shift(int32_t x) { return x & 3; }

template <int DIM>
__device__ __forceinline__ void issue_tma(GatherSmem<DIM>& S, int r, const BlockBounds& B,
                                          const int32_t* __restrict__ col_idx, const uint32_t* __restrict__ nslot) {
    if (!B.valid) return;
    if (!B.fit) {  // keep the barrier's phase count in step with the ring: arrive with no bytes
        mbar_expect_tx(S.bar(r), 0);
        return;
    }
    uint32_t c0 = (uint32_t)B.p0 & ~3u, c1 = ((uint32_t)B.p1 + 3u) & ~3u;
    uint32_t s0 = (uint32_t)B.q0 & ~3u, s1 = ((uint32_t)B.q1 + 3u) & ~3u;
    uint32_t bc = (c1 - c0) * 4, bs = (s1 - s0) * 4;
    mbar_expect_tx(S.bar(r), bc + bs);
    if (bc) tma_load_1d(S.cols(r), col_idx + c0, bc, S.bar(r));
    if (bs) tma_load_1d(S.slots(r), nslot + s0, bs, S.bar(r));
}

// Load the lane's row of block B; if the whole block fits the fast path, find the
// diagonal slot and gather the row's column coordinates into F[slot][c][lane].
template <int DIM>
__device__ __forceinline__ bool prepare_block(GatherSmem<DIM>& S, int r, BlockBounds& B, RowInfo& R,
                                              const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ nptr,
                                              const double* __restrict__ coords, int64_t ns, int64_t cst) {
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
    const bool fast = __all_sync(0xffffffffu, R.L <= GatherCfg<DIM>::RS) && B.valid && B.fit;
    if (fast && R.own) {
        const int32_t* cols = S.cols(r) + tma_shift(B.p0) + (R.lo - B.p0);
        double* F = S.F();
        for (int s = 0; s < R.L; s++) {
            int64_t w = cols[s];
            if (w == R.v) R.s0 = s;
#pragma unroll
            for (int c = 0; c < DIM; c++) cp_async8(F + (s * DIM + c) * GATHER_ROWS + t, coords + c * cst + w * ns);
        }
    }
    return fast;
}

template <int DIM>
__global__ void __launch_bounds__(GATHER_ROWS) assemble_gather_k(int64_t nn, const double* __restrict__ coords,
                                                                 int64_t ns, int64_t cst,
                                                                 const int32_t* __restrict__ row_ptr,
                                                                 const int32_t* __restrict__ col_idx,
                                                                 const int32_t* __restrict__ nptr,
                                                                 const uint32_t* __restrict__ nslot,
                                                                 double* __restrict__ K, double* __restrict__ M) {
    using Cfg = GatherCfg<DIM>;
    constexpr int W = GATHER_ROWS;
    extern __shared__ __align__(16) char smem_raw[];
    GatherSmem<DIM> S{smem_raw};
    const int t = threadIdx.x;
    const int64_t nblocks = (nn + W - 1) / W;
    const int64_t gstep = gridDim.x;
    if (t == 0)
        for (int r = 0; r < Cfg::RING; r++) mbar_init(S.bar(r));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();

    // prologue: TMA for this CTA's first block, then its coordinate gather
    BlockBounds B0 = block_bounds<DIM>(blockIdx.x, nblocks, nn, row_ptr, nptr);
    BlockBounds B1 = block_bounds<DIM>(blockIdx.x + gstep, nblocks, nn, row_ptr, nptr);
    if (t == 0) issue_tma<DIM>(S, 0, B0, col_idx, nslot);
    if (B0.valid) mbar_wait(S.bar(0), 0);
    RowInfo R0;
    bool fast0 = prepare_block<DIM>(S, 0, B0, R0, row_ptr, nptr, coords, ns, cst);
    cp_async_commit();

    double* F = S.F();
    double* aKs = S.accK() + t;
    double* aMs = S.accM() + t;
    for (int64_t k = 0;; k++) {
        const int64_t b = blockIdx.x + k * gstep;
        if (b >= nblocks) break;
        const int rc = (int)(k & 1), rn = rc ^ 1;
        // stage k+1: stream its columns and plan words (ring slot of block k-1 is free)
        if (t == 0) issue_tma<DIM>(S, rn, B1, col_idx, nslot);
        BlockBounds B2 = block_bounds<DIM>(blockIdx.x + (k + 2) * gstep, nblocks, nn, row_ptr, nptr);
        // stage k: its coordinates have landed
        cp_async_wait<0>();
        __syncwarp();
        const RowInfo& R = R0;
        if (fast0) {
            const uint32_t* slots = S.slots(rc) + tma_shift(B0.q0) - B0.q0;
            double* aK = K ? aKs : nullptr;
            double* aM = M ? aMs : nullptr;
            if (R.own) {
                for (int s = 0; s < R.L; s++) {
                    aKs[s * W] = 0.0;
                    aMs[s * W] = 0.0;
                }
                double xv[DIM];
#pragma unroll
                for (int c = 0; c < DIM; c++) xv[c] = F[(R.s0 * DIM + c) * W + t];
                auto ev = [&](int s, double(&f)[DIM]) {
#pragma unroll
                    for (int c = 0; c < DIM; c++) f[c] = F[(s * DIM + c) * W + t] - xv[c];
                };
                gather_row<DIM, W>(R.i0, R.i1, slots, ev, aK, aM);
            }
            __syncwarp();
            // finish the row (diagonal from the partition of unity, M scale) while
            // transposing it to CSR order through the (now dead) edge-vector buffer
            const int np = B0.p1 - B0.p0;
            double* stK = F;
            double* stM = F + Cfg::CAP;
            if (R.own && R.L > 0) {
                constexpr double MS = DIM == 2 ? 1.0 / 24.0 : 1.0 / 120.0;     // 1/(d! (d+1)(d+2))
                double sk = 0.0, sm = 0.0;
                const int b = R.lo - B0.p0;
                for (int s = 0; s < R.L; s++) {
                    if (s == R.s0) continue;
                    double kk = aKs[s * W], mm = aMs[s * W] * MS;
                    sk += kk;
                    sm += mm;
                    stK[b + s] = kk;
                    stM[b + s] = mm;
                }
                stK[b + R.s0] = -sk;
                stM[b + R.s0] = DIM == 3 ? sm * (2.0 / 3.0) : sm;
            }
            __syncwarp();
            for (int q = t; q < np; q += W) {
                if (K) stcs(K + B0.p0 + q, stK[q]);
                if (M) stcs(M + B0.p0 + q, stM[q]);
            }
        } else if (R.own && R.L > 0) {
            // block outside the smem budget: same ownership, everything in place in HBM
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
                int64_t w = __ldg(col_idx + R.lo + s);
#pragma unroll
                for (int c = 0; c < DIM; c++) f[c] = __ldg(coords + c * cst + w * ns) - xv[c];
            };
            gather_row<DIM, 1>(R.i0, R.i1, nslot, ev, aK, aM);
            finish_row<DIM, 1>(R.L, s0, aK, aM);
        }
        __syncwarp();
        // stage k+1: its columns have landed -> gather its coordinates into F (free now)
        if (B1.valid) mbar_wait(S.bar(rn), (uint32_t)(((k + 1) >> 1) & 1));
        fast0 = prepare_block<DIM>(S, rn, B1, R0, row_ptr, nptr, coords, ns, cst);
        cp_async_commit();
        B0 = B1;
        B1 = B2;
    }
    cp_async_wait<0>();
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
        static int ctas_per_sm[2] = {0, 0};  // > 48 KB dynamic smem needs an opt-in; persistent grid size
        if (!ctas_per_sm[0]) {
            cudaFuncSetAttribute(assemble_gather_k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GatherCfg<2>::SMEM);
            cudaFuncSetAttribute(assemble_gather_k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GatherCfg<3>::SMEM);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm[0], assemble_gather_k<2>, GATHER_ROWS, GatherCfg<2>::SMEM);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm[1], assemble_gather_k<3>, GATHER_ROWS, GatherCfg<3>::SMEM);
            for (int& c : ctas_per_sm) c = c > 0 ? c : 1;
        }
        int64_t nblocks = (nn + GATHER_ROWS - 1) / GATHER_ROWS;
        int64_t cap = (int64_t)sm_count() * ctas_per_sm[dim == 3];
        unsigned g = (unsigned)(nblocks < cap ? nblocks : cap);
        if (dim == 2) {
            assemble_gather_k<2><<<g, GATHER_ROWS, GatherCfg<2>::SMEM, s>>>(nn, coords, node_stride, comp_stride, row_ptr,
                                                                        col_idx, node_elem_ptr, node_elem_slot, K_vals, M_vals);
        } else {
            assemble_gather_k<3><<<g, GATHER_ROWS, GatherCfg<3>::SMEM, s>>>(nn, coords, node_stride, comp_stride, row_ptr,
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
