// Tile plan and tile-variant P1 assembly (fem_plan_tiles, fem_p1_assemble_tiles):
// every element's K_e / M_e evaluated ONCE per tile of rows it touches, instead
// of once per vertex as in the row-gather variants (assemble.cu).
//
// What is computed is eq:K_M with c = 1 assembled as
// sparse(X3D(:),Y3D(:),K3D(:)): per element tjac = D X^T
// (P:941), |T| = |det tjac| / d!, G = tjac^{-1} D,
// K_e = |T| G^T G, M_e = |T| / ((d+1)(d+2)) (1 + delta_ab) (P:1007,
// P:1020-1021); K_e[a][b] = (h_a . h_b) / (d! |det|) with h = adj(tjac) D.
//
// Tiles.  The rows are ordered along a Morton curve of the node coordinates and
// cut into tiles of TR = 128 consecutive rows, so a tile is a compact patch of
// the mesh (8x4x4 nodes of a structured cube).  The elements of a tile are those
// with at least one vertex in it; an element is evaluated once by every tile it
// touches (on the 128^3 Kuhn cube about 1.5 times, against 4 times in the row
// gather).  A tile's K and M rows live in shared memory ([slot][row] pairs,
// 32 KB) while its elements add their off-diagonal entries into them; two
// elements that update the same (row, slot) never run together: the plan colors
// the tile's elements greedily (first fit, ascending element id) so that the
// elements of one color have disjoint targets, and the kernel runs the colors
// one after another between barriers.  No atomics; the summation order is fixed
// by the plan, so the result is bitwise reproducible.  Diagonals follow from the
// partition of unity (K_vv = -sum_{w!=v} K_vw, M_vv = (2/d) sum_{w!=v} M_vw), as
// in the other deterministic variants.  Finished rows leave as coalesced runs of
// their CSR ranges; every CSR entry is written exactly once.
//
// Plan (built on the GPU, deterministic): Morton keys -> radix sort -> rank of
// each node -> (tile, element) pairs -> radix sort -> per tile one CTA builds
// the local node table (owned rows first, then the halo in ascending id), the
// per-element entry (local vertex ids, in-row slots of the other vertices for
// every owned vertex) and the coloring.
#include <cub/device/device_radix_sort.cuh>

#include "vb_internal.cuh"

namespace vb {
namespace {

constexpr int TR = VB_TILE_ROWS;     // rows per tile = threads per CTA
constexpr int TS = 16;               // slots per row (row length cap; 4-bit slots)
constexpr int NLOC = VB_TILE_NLOC;   // local nodes per tile (node table stride)
constexpr int MAXC = VB_TILE_MAXC;   // colors per tile
constexpr int MAXE = 3072;           // elements per tile (plan build staging)
constexpr int HS = 2048;             // halo hash table (power of two, >= 2 * (NLOC - 0))

enum TileErr { TE_OK = 0, TE_ROW = 1, TE_ELEMS = 2, TE_NODES = 3, TE_COLORS = 4 };

__device__ __forceinline__ unsigned long long ord_key(double x) {   // order-preserving double -> u64
    const unsigned long long u = (unsigned long long)__double_as_longlong(x);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

__global__ void tl_init_k(unsigned long long* __restrict__ bbox, unsigned long long* __restrict__ stats) {
    const int i = threadIdx.x;
    if (i < 3) bbox[i] = ~0ull;
    else if (i < 6) bbox[i] = 0ull;
    if (i < 8) stats[i] = 0ull;
}

template <int DIM>
__global__ void tl_bbox_k(int64_t nn, const double* __restrict__ coords, int64_t ns, int64_t cst,
                          unsigned long long* __restrict__ bbox) {
    unsigned long long lo[DIM], hi[DIM];
#pragma unroll
    for (int c = 0; c < DIM; c++) lo[c] = ~0ull, hi[c] = 0ull;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int c = 0; c < DIM; c++) {
            const unsigned long long k = ord_key(coords[c * cst + v * ns]);
            lo[c] = k < lo[c] ? k : lo[c];
            hi[c] = k > hi[c] ? k : hi[c];
        }
#pragma unroll
    for (int c = 0; c < DIM; c++) {
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo[c], o);
            const unsigned long long b = __shfl_xor_sync(0xffffffffu, hi[c], o);
            lo[c] = a < lo[c] ? a : lo[c];
            hi[c] = b > hi[c] ? b : hi[c];
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(bbox + c, lo[c]);
            atomicMax(bbox + 3 + c, hi[c]);
        }
    }
}

__device__ __forceinline__ uint64_t spread3(uint64_t x) {   // 21 bits -> every third bit
    x &= 0x1fffffull;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}
__device__ __forceinline__ uint64_t spread2(uint64_t x) {   // 31 bits -> every second bit
    x &= 0x7fffffffull;
    x = (x | x << 16) & 0x0000ffff0000ffffull;
    x = (x | x << 8) & 0x00ff00ff00ff00ffull;
    x = (x | x << 4) & 0x0f0f0f0f0f0f0f0full;
    x = (x | x << 2) & 0x3333333333333333ull;
    x = (x | x << 1) & 0x5555555555555555ull;
    return x;
}

template <int DIM>
__global__ void tl_morton_k(int64_t nn, const double* __restrict__ coords, int64_t ns, int64_t cst,
                            const unsigned long long* __restrict__ bbox, uint64_t* __restrict__ keys,
                            int32_t* __restrict__ nodes) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nn) return;
    constexpr double Q = DIM == 3 ? 2097151.0 : 2147483647.0;
    uint64_t key = 0;
#pragma unroll
    for (int c = 0; c < DIM; c++) {
        const double lo = ord_val(bbox[c]), hi = ord_val(bbox[3 + c]);
        const double span = hi - lo;
        double q = span > 0.0 ? (coords[c * cst + v * ns] - lo) / span * Q : 0.0;
        q = q < 0.0 ? 0.0 : (q > Q ? Q : q);
        const uint64_t u = (uint64_t)q;
        key |= (DIM == 3 ? spread3(u) : spread2(u)) << c;
    }
    keys[v] = key;
    nodes[v] = (int32_t)v;
}

__global__ void tl_rank_k(int64_t nn, const int32_t* __restrict__ perm, int32_t* __restrict__ rank_of) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nn) rank_of[perm[i]] = (int32_t)i;
}

// distinct tiles of element e's vertices, ascending
template <int NV>
__device__ __forceinline__ int elem_tiles(int64_t e, const int32_t* __restrict__ elems, int64_t eld,
                                          const int32_t* __restrict__ rank_of, int (&tl)[NV]) {
    int n = 0;
#pragma unroll
    for (int a = 0; a < NV; a++) {
        const int t = rank_of[elems[a * eld + e]] / TR;
        bool seen = false;
        for (int q = 0; q < n; q++) seen |= tl[q] == t;
        if (!seen) tl[n++] = t;
    }
    return n;
}

template <int NV>
__global__ void tl_count_k(int64_t ne, const int32_t* __restrict__ elems, int64_t eld,
                           const int32_t* __restrict__ rank_of, int32_t* __restrict__ cnt) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne) return;
    int tl[NV];
    cnt[e] = elem_tiles<NV>(e, elems, eld, rank_of, tl);
}

template <int NV>
__global__ void tl_fill_k(int64_t ne, const int32_t* __restrict__ elems, int64_t eld,
                          const int32_t* __restrict__ rank_of, const int32_t* __restrict__ off,
                          uint64_t* __restrict__ keys) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne) return;
    int tl[NV];
    const int n = elem_tiles<NV>(e, elems, eld, rank_of, tl);
    for (int q = 0; q < n; q++) keys[off[e] + q] = (uint64_t)tl[q] << 32 | (uint64_t)e;
}

// first sorted pair of each tile (tile T: the pair count)
__global__ void tl_start_k(int64_t T, int64_t P, const uint64_t* __restrict__ keys, int32_t* __restrict__ tstart) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t > T) return;
    const uint64_t k = (uint64_t)t << 32;
    int64_t lo = 0, hi = P;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    tstart[t] = (int32_t)lo;
}

__device__ __forceinline__ uint32_t hslot(int32_t v) { return ((uint32_t)v * 2654435761u) >> (32 - 11); }
static_assert(HS == 2048, "hslot assumes 11 bits");

__device__ __forceinline__ bool h_insert(int32_t* hkey, int32_t v) {   // false: table full
    uint32_t h = hslot(v);
    for (int p = 0; p < HS; p++) {
        const int32_t old = atomicCAS(hkey + h, -1, v);
        if (old == -1 || old == v) return true;
        h = (h + 1) & (HS - 1);
    }
    return false;
}
__device__ __forceinline__ int h_find(const int32_t* hkey, int32_t v) {
    uint32_t h = hslot(v);
    while (hkey[h] != v) h = (h + 1) & (HS - 1);
    return (int)h;
}

struct BuildSmem {
    uint4 ent[MAXE];
    int32_t E[MAXE];   // element ids; later the output position of each entry
    int32_t hkey[HS], hval[HS];
    int32_t halo[NLOC];
    uint32_t mask[TS * TR];
    int32_t rcol[TR * TS];   // owned rows' columns
    int32_t rL[TR];
    int32_t ccnt[MAXC + 1];
    uint8_t col[MAXE];
    int nh, err;
};

template <int DIM>
__global__ void __launch_bounds__(TR) tl_build_k(int64_t nn, const int32_t* __restrict__ elems, int64_t eld,
                                                 const int32_t* __restrict__ perm,
                                                 const int32_t* __restrict__ rank_of,
                                                 const uint64_t* __restrict__ skeys,
                                                 const int32_t* __restrict__ tstart,
                                                 const int32_t* __restrict__ row_ptr,
                                                 const int32_t* __restrict__ col_idx, int4* __restrict__ meta,
                                                 int32_t* __restrict__ tnodes, int2* __restrict__ trows,
                                                 int32_t* __restrict__ tcolors, uint4* __restrict__ telems,
                                                 unsigned long long* __restrict__ stats) {
    constexpr int NV = DIM + 1;
    constexpr int SB = 4 * (NV - 1);   // slot bits per owned vertex
    extern __shared__ __align__(16) unsigned char smraw[];
    BuildSmem& S = *reinterpret_cast<BuildSmem*>(smraw);
    const int64_t t = blockIdx.x;
    const int tid = threadIdx.x;
    const int nown = (int)(nn - t * TR < TR ? nn - t * TR : TR);
    const int e0 = tstart[t], net = tstart[t + 1] - e0;
    if (tid == 0) S.nh = 0, S.err = TE_OK;
    for (int i = tid; i < HS; i += TR) S.hkey[i] = -1;
    for (int i = tid; i < TS * TR; i += TR) S.mask[i] = 0u;
    for (int i = tid; i <= MAXC; i += TR) S.ccnt[i] = 0;
    if (tid == 0) atomicMax(stats + 1, (unsigned long long)net);
    if (net > MAXE) {
        if (tid == 0) atomicMax(stats + 4, (unsigned long long)TE_ELEMS);
        return;
    }
    __syncthreads();
    // owned rows: columns, length, diagonal slot
    if (tid < nown) {
        const int32_t g = perm[t * TR + tid];
        const int lo = row_ptr[g], L = row_ptr[g + 1] - lo;
        int s0 = -1;
        for (int q = 0; q < L && q < TS; q++) {
            const int32_t c = col_idx[lo + q];
            S.rcol[tid * TS + q] = c;
            if (c == g) s0 = q;
        }
        if (L > TS || (L > 0 && s0 < 0)) atomicExch(&S.err, TE_ROW);   // L = 0: an isolated node
        S.rL[tid] = L;
        trows[t * TR + tid] = make_int2(lo, L | (s0 & 0xff) << 8);
        tnodes[t * NLOC + tid] = g;
    }
    // elements and their halo vertices
    for (int i = tid; i < net; i += TR) {
        const int64_t e = (int64_t)(skeys[e0 + i] & 0xffffffffull);
        S.E[i] = (int32_t)e;
#pragma unroll
        for (int a = 0; a < NV; a++) {
            const int32_t v = elems[a * eld + e];
            if (rank_of[v] / TR != t && !h_insert(S.hkey, v)) atomicExch(&S.err, TE_NODES);
        }
    }
    __syncthreads();
    for (int h = tid; h < HS; h += TR)
        if (S.hkey[h] >= 0) {
            const int p = atomicAdd(&S.nh, 1);
            if (p < NLOC) S.halo[p] = S.hkey[h];
        }
    __syncthreads();
    const int nh = S.nh, nloc = nown + nh;
    if (tid == 0) atomicMax(stats + 2, (unsigned long long)nloc);
    if (nloc > NLOC || S.err != TE_OK) {
        if (tid == 0) atomicMax(stats + 4, (unsigned long long)(S.err != TE_OK ? S.err : TE_NODES));
        return;
    }
    // halo in ascending node id: local index nown + rank
    for (int j = tid; j < nh; j += TR) {
        const int32_t v = S.halo[j];
        int c = 0;
        for (int k = 0; k < nh; k++) c += S.halo[k] < v;
        S.hval[h_find(S.hkey, v)] = nown + c;
        tnodes[t * NLOC + nown + c] = v;
    }
    __syncthreads();
    // entries: local vertex ids (16 bits each), in-row slots of the other vertices per owned vertex
    for (int i = tid; i < net; i += TR) {
        const int64_t e = S.E[i];
        int32_t v[NV];
        int l[NV];
#pragma unroll
        for (int a = 0; a < NV; a++) {
            v[a] = elems[a * eld + e];
            const int r = rank_of[v[a]];
            l[a] = r / TR == t ? r - (int)(t * TR) : S.hval[h_find(S.hkey, v[a])];
        }
        uint64_t sb = 0;
#pragma unroll
        for (int a = 0; a < NV; a++) {
            if (l[a] >= nown) continue;
            int j = 0;
#pragma unroll
            for (int b = 0; b < NV; b++) {
                if (b == a) continue;
                const int L = S.rL[l[a]];
                int s = 0;
                while (s < L && S.rcol[l[a] * TS + s] != v[b]) s++;
                sb |= (uint64_t)(s & 15) << (SB * a + 4 * j);
                j++;
            }
        }
        S.ent[i] = make_uint4((uint32_t)l[0] | (uint32_t)l[1] << 16, (uint32_t)l[2] | (uint32_t)(DIM == 3 ? l[3] : 0) << 16,
                              (uint32_t)sb, (uint32_t)(sb >> 32));
    }
    __syncthreads();
    // first-fit coloring in ascending element id: the elements of a color update disjoint (row, slot)
    if (tid == 0) {
        int ncol = 0;
        for (int i = 0; i < net; i++) {
            const uint4 q = S.ent[i];
            const int l[4] = {(int)(q.x & 0xffff), (int)(q.x >> 16), (int)(q.y & 0xffff), (int)(q.y >> 16)};
            const uint64_t sb = (uint64_t)q.z | (uint64_t)q.w << 32;
            uint32_t forb = 0;
            for (int a = 0; a < NV; a++)
                if (l[a] < nown)
                    for (int j = 0; j < NV - 1; j++) forb |= S.mask[((sb >> (SB * a + 4 * j)) & 15) * TR + l[a]];
            if (forb == 0xffffffffu) {
                S.err = TE_COLORS;
                break;
            }
            const int c = __ffs(~forb) - 1;
            for (int a = 0; a < NV; a++)
                if (l[a] < nown)
                    for (int j = 0; j < NV - 1; j++) S.mask[((sb >> (SB * a + 4 * j)) & 15) * TR + l[a]] |= 1u << c;
            S.col[i] = (uint8_t)c;
            S.ccnt[c]++;
            ncol = c + 1 > ncol ? c + 1 : ncol;
        }
        if (S.err == TE_OK) {
            // color offsets and each entry's position in (color, element) order
            int run = 0;
            for (int c = 0; c <= ncol; c++) {
                const int k = c < ncol ? S.ccnt[c] : 0;
                tcolors[t * (MAXC + 1) + c] = e0 + run;
                S.ccnt[c] = run;
                run += k;
            }
            for (int i = 0; i < net; i++) S.E[i] = S.ccnt[S.col[i]]++;
            meta[t] = make_int4(nown, nloc, ncol, e0);
            atomicMax(stats + 3, (unsigned long long)ncol);
        } else {
            atomicMax(stats + 4, (unsigned long long)S.err);
        }
    }
    __syncthreads();
    if (S.err != TE_OK) return;
    for (int i = tid; i < net; i += TR) telems[e0 + S.E[i]] = S.ent[i];
}

// ------------------------------------------------------------------ assembly
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}

// Persistent CTAs of TR threads, one tile at a time: the tile's entries arrive
// in shared memory with one bulk (TMA) copy and its node coordinates with
// cp.async; then the colors run one after another (barrier between colors),
// each thread taking the color's entries by stride; then the diagonals and the
// coalesced write-out of the tile's rows.
template <int DIM>
__global__ void __launch_bounds__(TR, 3) assemble_tile_k(int64_t T, const int4* __restrict__ meta,
                                                         const int32_t* __restrict__ tnodes,
                                                         const int2* __restrict__ trows,
                                                         const int32_t* __restrict__ tcolors,
                                                         const uint4* __restrict__ telems,
                                                         const double* __restrict__ coords, int64_t ns, int64_t cst,
                                                         int ek, int xstride, double* __restrict__ K,
                                                         double* __restrict__ M) {
    constexpr int NV = DIM + 1;
    constexpr int SB = 4 * (NV - 1);
    constexpr double KF = DIM == 3 ? 1.0 / 6.0 : 0.5;            // 1/d!
    constexpr double MF = DIM == 3 ? 1.0 / 120.0 : 1.0 / 24.0;   // |det| / (d! (d+1)(d+2))
    constexpr double MD = 2.0 / DIM;                             // M_vv / sum_{w!=v} M_vw
    extern __shared__ __align__(16) double2 acc[];               // [slot][row] (K, M) pairs
    uint4* ent = reinterpret_cast<uint4*>(acc + TS * TR);        // the tile's entries
    double* xs = reinterpret_cast<double*>(ent + ek);            // [coord][local node]
    __shared__ int2 rinfo[TR];
    __shared__ int cptr[MAXC + 1];
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t parity = 0;
    for (int64_t t = blockIdx.x; t < T; t += gridDim.x) {
        const int4 mt = meta[t];
        const int nown = mt.x, nloc = mt.y, ncol = mt.z;
        const int32_t* tc = tcolors + t * (MAXC + 1);
        const int e0 = tc[0], ne_t = tc[ncol] - e0;
        if (tid == 0 && ne_t > 0) {
            const uint32_t bytes = (uint32_t)ne_t * 16u;
            // the generic-proxy reads of the previous tile's entries (ordered by the __syncthreads that ended
            // it) before this async-proxy overwrite of the same buffer
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar)), "r"(bytes)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(ent)),
                "l"(telems + e0), "r"(bytes), "r"(smem_addr(&bar))
                : "memory");
        }
        for (int i = tid; i < nloc; i += TR) {
            const int64_t g = tnodes[t * NLOC + i];
#pragma unroll
            for (int c = 0; c < DIM; c++) cp_async8(xs + c * xstride + i, coords + c * cst + g * ns);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (tid < nown) rinfo[tid] = trows[t * TR + tid];
        if (tid <= ncol) cptr[tid] = tc[tid] - e0;
#pragma unroll 4
        for (int i = tid; i < TS * TR; i += TR) acc[i] = make_double2(0.0, 0.0);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        if (ne_t > 0) {
            uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                    : "=r"(done)
                    : "r"(smem_addr(&bar)), "r"(parity)
                    : "memory");
            parity ^= 1u;
        }
        __syncthreads();
        VB_CHECK(ne_t <= ek && nloc <= xstride && ncol <= MAXC);
        for (int c = 0; c < ncol; c++) {
            const int i1 = cptr[c + 1];
            for (int i = cptr[c] + tid; i < i1; i += TR) {
                const uint4 q = ent[i];
                const int l4[4] = {(int)(q.x & 0xffff), (int)(q.x >> 16), (int)(q.y & 0xffff), (int)(q.y >> 16)};
                int l[NV];
#pragma unroll
                for (int a = 0; a < NV; a++) l[a] = l4[a];
                const uint64_t sb = (uint64_t)q.z | (uint64_t)q.w << 32;
#pragma unroll
                for (int a = 0; a < NV; a++) VB_CHECK(l[a] < nloc);
                double k[NV][NV], ad;
                if constexpr (DIM == 3) {
                    double f[3][3];
#pragma unroll
                    for (int r = 0; r < 3; r++)
#pragma unroll
                        for (int c2 = 0; c2 < 3; c2++) f[r][c2] = xs[c2 * xstride + l[r + 1]] - xs[c2 * xstride + l[0]];
                    double h[4][3];
                    auto cross = [](const double(&u)[3], const double(&v)[3], double(&o)[3]) {
                        o[0] = fma(u[1], v[2], -u[2] * v[1]);
                        o[1] = fma(u[2], v[0], -u[0] * v[2]);
                        o[2] = fma(u[0], v[1], -u[1] * v[0]);
                    };
                    cross(f[1], f[2], h[1]);
                    cross(f[2], f[0], h[2]);
                    cross(f[0], f[1], h[3]);
                    const double det = fma(f[0][0], h[1][0], fma(f[0][1], h[1][1], f[0][2] * h[1][2]));
                    ad = fabs(det);
                    const double s = KF / ad;
#pragma unroll
                    for (int c2 = 0; c2 < 3; c2++) h[0][c2] = -((h[1][c2] + h[2][c2]) + h[3][c2]);
#pragma unroll
                    for (int a = 0; a < 4; a++)
#pragma unroll
                        for (int b = a + 1; b < 4; b++)
                            k[a][b] = k[b][a] = s * fma(h[a][0], h[b][0], fma(h[a][1], h[b][1], h[a][2] * h[b][2]));
                } else {
                    double f[2][2];
#pragma unroll
                    for (int r = 0; r < 2; r++)
#pragma unroll
                        for (int c2 = 0; c2 < 2; c2++) f[r][c2] = xs[c2 * xstride + l[r + 1]] - xs[c2 * xstride + l[0]];
                    // adj(tjac) D: h1 = (f2y, -f2x), h2 = (-f1y, f1x), h0 = -(h1 + h2)
                    double h[3][2] = {{0, 0}, {f[1][1], -f[1][0]}, {-f[0][1], f[0][0]}};
                    h[0][0] = -(h[1][0] + h[2][0]);
                    h[0][1] = -(h[1][1] + h[2][1]);
                    const double det = fma(f[0][0], f[1][1], -f[0][1] * f[1][0]);
                    ad = fabs(det);
                    const double s = KF / ad;
#pragma unroll
                    for (int a = 0; a < 3; a++)
#pragma unroll
                        for (int b = a + 1; b < 3; b++) k[a][b] = k[b][a] = s * fma(h[a][0], h[b][0], h[a][1] * h[b][1]);
                }
                const double m = ad * MF;
                // the element's targets are distinct (row, slot) pairs: all loads, then all stores
                double2 v[NV][NV - 1];
                int adr[NV][NV - 1];
#pragma unroll
                for (int a = 0; a < NV; a++) {
                    int j = 0;
#pragma unroll
                    for (int b = 0; b < NV; b++) {
                        if (b == a) continue;
                        adr[a][j] = (int)((sb >> (SB * a + 4 * j)) & 15) * TR + l[a];
                        VB_CHECK(l[a] >= nown || (int)((sb >> (SB * a + 4 * j)) & 15) < (rinfo[l[a]].y & 0xff));
                        if (l[a] < nown) v[a][j] = acc[adr[a][j]];
                        j++;
                    }
                }
#pragma unroll
                for (int a = 0; a < NV; a++) {
                    int j = 0;
#pragma unroll
                    for (int b = 0; b < NV; b++) {
                        if (b == a) continue;
                        if (l[a] < nown) acc[adr[a][j]] = make_double2(v[a][j].x + k[a][b], v[a][j].y + m);
                        j++;
                    }
                }
            }
            __syncthreads();
        }
        // diagonals from the partition of unity
        if (tid < nown && (rinfo[tid].y & 0xff) > 0) {
            const int L = rinfo[tid].y & 0xff, s0 = rinfo[tid].y >> 8;
            double sk = 0.0, sm = 0.0;
#pragma unroll
            for (int s = 0; s < TS; s++)
                if (s < L && s != s0) {
                    const double2 x = acc[s * TR + tid];
                    sk += x.x;
                    sm += x.y;
                }
            acc[s0 * TR + tid] = make_double2(-sk, MD * sm);
        }
        __syncthreads();
        // write-out: a half warp per row, lane s -> CSR entry lo + s
        const int lane = tid & 31, w = tid >> 5, hw = lane >> 4, s = lane & 15;
        for (int i = w * 2 + hw; i < nown; i += TR / 16) {
            const int2 ri = rinfo[i];
            if (s < (ri.y & 0xff)) {
                const double2 x = acc[s * TR + i];
                if (K) stcs(K + ri.x + s, x.x);
                if (M) stcs(M + ri.x + s, x.y);
            }
        }
        __syncthreads();   // shared memory is the next tile's
    }
}

// ------------------------------------------------------------------ plan workspace
struct TileWork {
    unsigned long long *bbox, *stats;
    uint64_t *mk1, *mk2, *pk1, *pk2;
    int32_t *n1, *perm, *rank_of, *cnt, *off, *tstart;
    void* cub;
    size_t cub_bytes;
    void* scan;
};

size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t tile_layout(int64_t nn, int64_t ne, int nv, char* base, TileWork* w) {
    const int64_t pmax = (int64_t)nv * ne > 0 ? (int64_t)nv * ne : 1;
    const int64_t T = (nn + TR - 1) / TR;
    size_t c1 = 0, c2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, c1, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, (int)nn);
    cub::DeviceRadixSort::SortKeys(nullptr, c2, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int)pmax);
    const size_t cubb = c1 > c2 ? c1 : c2;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* p = base ? base + off : nullptr;
        off += al256(bytes);
        return p;
    };
    TileWork W{};
    W.bbox = (unsigned long long*)take(8 * 8);
    W.stats = (unsigned long long*)take(8 * 8);
    W.mk1 = (uint64_t*)take(8 * nn);
    W.mk2 = (uint64_t*)take(8 * nn);
    W.n1 = (int32_t*)take(4 * nn);
    W.perm = (int32_t*)take(4 * nn);
    W.rank_of = (int32_t*)take(4 * nn);
    W.cnt = (int32_t*)take(4 * ne);
    W.off = (int32_t*)take(4 * (ne + 1));
    W.pk1 = (uint64_t*)take(8 * pmax);
    W.pk2 = (uint64_t*)take(8 * pmax);
    W.tstart = (int32_t*)take(4 * (T + 1));
    W.cub = take(cubb);
    W.cub_bytes = cubb;
    W.scan = take(scan_tmp_bytes(ne > nn ? ne : nn));
    if (w) *w = W;
    return off;
}

int bits_for(int64_t x) {
    int b = 0;
    while (b < 63 && ((int64_t)1 << b) <= x) b++;
    return b;
}

}  // namespace
}  // namespace vb

using namespace vb;

extern "C" vb_status fem_plan_tiles(int dim, int64_t nn, int64_t ne, const double* coords, int64_t node_stride,
                                    int64_t comp_stride, const int32_t* elems, int64_t elem_ld,
                                    const int32_t* row_ptr, const int32_t* col_idx, void* work, size_t* work_bytes,
                                    int32_t* tile_meta, int32_t* tile_nodes, int32_t* tile_rows,
                                    int32_t* tile_colors, uint32_t* tile_elems, int64_t elems_cap,
                                    int64_t* stats_out, vb_stream_t stream) {
    const char* fn = "fem_plan_tiles";
    clear_error();
    if (dim != 2 && dim != 3) { set_error("%s: dim=%d, need 2 or 3", fn, dim); return VB_ERR_UNSUPPORTED; }
    if (nn < 0 || ne < 0 || !work_bytes) { set_error("%s: bad size or NULL work_bytes", fn); return VB_ERR_ARG; }
    const int nv = dim + 1;
    if (nn >= (int64_t)1 << 30 || (int64_t)nv * ne >= (int64_t)1 << 31) {
        set_error("%s: nn=%lld ne=%lld too large", fn, (long long)nn, (long long)ne);
        return VB_ERR_OVERFLOW;
    }
    const int64_t n1 = nn > 0 ? nn : 1, e1 = ne > 0 ? ne : 1;
    const size_t need = tile_layout(n1, e1, nv, nullptr, nullptr);
    if (!work) { *work_bytes = need; return VB_OK; }
    if (*work_bytes < need) { set_error("%s: work %zu < %zu bytes", fn, *work_bytes, need); return VB_ERR_WORKSPACE; }
    if (!stats_out) { set_error("%s: NULL stats_out", fn); return VB_ERR_ARG; }
    for (int i = 0; i < 6; i++) stats_out[i] = 0;
    const int64_t T = (nn + TR - 1) / TR;
    stats_out[5] = T;
    if (nn == 0) return VB_OK;
    if (!coords || !row_ptr || !tile_meta || !tile_nodes || !tile_rows || !tile_colors ||
        (ne > 0 && (!elems || !col_idx || !tile_elems))) {
        set_error("%s: NULL argument", fn);
        return VB_ERR_ARG;
    }
    if (elem_ld < ne) { set_error("%s: elem_ld %lld < ne %lld", fn, (long long)elem_ld, (long long)ne); return VB_ERR_ARG; }
    cudaStream_t s = cs(stream);
    TileWork W;
    tile_layout(n1, e1, nv, static_cast<char*>(work), &W);
    vb_status st;
    tl_init_k<<<1, 32, 0, s>>>(W.bbox, W.stats);
    const unsigned gn = (unsigned)((nn + 255) / 256), ge = (unsigned)((e1 + 255) / 256);
    if (dim == 3) {
        tl_bbox_k<3><<<grid_for(nn, 256, 8), 256, 0, s>>>(nn, coords, node_stride, comp_stride, W.bbox);
        tl_morton_k<3><<<gn, 256, 0, s>>>(nn, coords, node_stride, comp_stride, W.bbox, W.mk1, W.n1);
    } else {
        tl_bbox_k<2><<<grid_for(nn, 256, 8), 256, 0, s>>>(nn, coords, node_stride, comp_stride, W.bbox);
        tl_morton_k<2><<<gn, 256, 0, s>>>(nn, coords, node_stride, comp_stride, W.bbox, W.mk1, W.n1);
    }
    if ((st = launch_check(fn)) != VB_OK) return st;
    size_t b = W.cub_bytes;
    if (cub::DeviceRadixSort::SortPairs(W.cub, b, W.mk1, W.mk2, W.n1, W.perm, (int)nn, 0, 64, s) != cudaSuccess) {
        set_error("%s: radix sort failed", fn);
        return VB_ERR_CUDA;
    }
    tl_rank_k<<<gn, 256, 0, s>>>(nn, W.perm, W.rank_of);
    if ((st = launch_check(fn)) != VB_OK) return st;
    int64_t P = 0;
    if (ne > 0) {
        if (dim == 3) tl_count_k<4><<<ge, 256, 0, s>>>(ne, elems, elem_ld, W.rank_of, W.cnt);
        else tl_count_k<3><<<ge, 256, 0, s>>>(ne, elems, elem_ld, W.rank_of, W.cnt);
        if ((st = launch_check(fn)) != VB_OK) return st;
        if ((st = exclusive_scan_i32(W.cnt, W.off, ne, W.scan, s, nullptr)) != VB_OK) return st;
        int32_t p32 = 0;
        if ((st = read_small(s, W.off + ne, sizeof(int32_t), &p32, fn)) != VB_OK) return st;
        P = p32;
    }
    stats_out[0] = P;
    if (P > elems_cap) {
        set_error("%s: %lld tile entries, elems_cap %lld", fn, (long long)P, (long long)elems_cap);
        return VB_ERR_WORKSPACE;
    }
    const uint64_t* sk = W.pk1;
    if (P > 0) {
        if (dim == 3) tl_fill_k<4><<<ge, 256, 0, s>>>(ne, elems, elem_ld, W.rank_of, W.off, W.pk1);
        else tl_fill_k<3><<<ge, 256, 0, s>>>(ne, elems, elem_ld, W.rank_of, W.off, W.pk1);
        if ((st = launch_check(fn)) != VB_OK) return st;
        b = W.cub_bytes;
        if (cub::DeviceRadixSort::SortKeys(W.cub, b, W.pk1, W.pk2, (int)P, 0, 32 + bits_for(T), s) != cudaSuccess) {
            set_error("%s: radix sort failed", fn);
            return VB_ERR_CUDA;
        }
        sk = W.pk2;
    }
    tl_start_k<<<(unsigned)((T + 1 + 255) / 256), 256, 0, s>>>(T, P, sk, W.tstart);
    if ((st = launch_check(fn)) != VB_OK) return st;
    const size_t smem = sizeof(BuildSmem);
    auto build = dim == 3 ? tl_build_k<3> : tl_build_k<2>;
    cudaFuncSetAttribute(build, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    build<<<(unsigned)T, TR, smem, s>>>(nn, elems, elem_ld, W.perm, W.rank_of, sk, W.tstart, row_ptr, col_idx,
                                        reinterpret_cast<int4*>(tile_meta), tile_nodes,
                                        reinterpret_cast<int2*>(tile_rows), tile_colors,
                                        reinterpret_cast<uint4*>(tile_elems), W.stats);
    if ((st = launch_check(fn)) != VB_OK) return st;
    unsigned long long hs[5];
    if ((st = read_small(s, W.stats, sizeof(hs), hs, fn)) != VB_OK) return st;
    stats_out[1] = (int64_t)hs[1];
    stats_out[2] = (int64_t)hs[2];
    stats_out[3] = (int64_t)hs[3];
    stats_out[4] = (int64_t)hs[4];
    if (hs[4] != TE_OK) {
        static const char* why[] = {"", "a row longer than 16 entries", "a tile with more than 3072 elements",
                                    "a tile with more than VB_TILE_NLOC local nodes",
                                    "a tile needing more than VB_TILE_MAXC colors"};
        set_error("%s: mesh not supported by the tile variant: %s", fn, why[hs[4] < 5 ? hs[4] : 0]);
        return VB_ERR_UNSUPPORTED;
    }
    return VB_OK;
}

extern "C" vb_status fem_p1_assemble_tiles(int dim, int64_t nn, const double* coords, int64_t node_stride,
                                           int64_t comp_stride, int64_t nnz, const int32_t* tile_meta,
                                           const int32_t* tile_nodes, const int32_t* tile_rows,
                                           const int32_t* tile_colors, const uint32_t* tile_elems, int nloc_max,
                                           int elems_max, double* K_vals, double* M_vals, vb_stream_t stream) {
    const char* fn = "fem_p1_assemble_tiles";
    clear_error();
    if (dim != 2 && dim != 3) { set_error("%s: dim=%d, need 2 or 3", fn, dim); return VB_ERR_UNSUPPORTED; }
    if (nn < 0 || nnz < 0) { set_error("%s: negative size", fn); return VB_ERR_ARG; }
    if (nloc_max < 0 || nloc_max > NLOC) { set_error("%s: nloc_max=%d outside [0, %d]", fn, nloc_max, NLOC); return VB_ERR_ARG; }
    if (nn == 0 || (!K_vals && !M_vals)) return VB_OK;
    if (!coords || !tile_meta || !tile_nodes || !tile_rows || !tile_colors || !tile_elems) {
        set_error("%s: NULL argument", fn);
        return VB_ERR_ARG;
    }
    if (!aligned16(tile_elems) || !aligned16(tile_meta)) {   // streamed with bulk copies / read as int4
        set_error("%s: tile_elems and tile_meta must be 16-byte aligned", fn);
        return VB_ERR_ARG;
    }
    const int64_t T = (nn + TR - 1) / TR;
    if (elems_max < 0 || elems_max > (1 << 20)) { set_error("%s: elems_max=%d out of range", fn, elems_max); return VB_ERR_ARG; }
    const int xstride = (nloc_max + 1) & ~1;
    const int ek = elems_max > 0 ? elems_max : 1;
    const size_t smem = sizeof(double2) * TS * TR + 16 * (size_t)ek + sizeof(double) * dim * xstride;
    if (smem > 227 * 1024) { set_error("%s: tile needs %zu bytes of shared memory", fn, smem); return VB_ERR_UNSUPPORTED; }
    cudaStream_t s = cs(stream);
    auto k = dim == 3 ? assemble_tile_k<3> : assemble_tile_k<2>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, TR, smem);
    const int64_t cap = (int64_t)sm_count() * (occ > 0 ? occ : 1);
    const unsigned grid = (unsigned)(T < cap ? T : cap);
    k<<<grid, TR, smem, s>>>(T, reinterpret_cast<const int4*>(tile_meta), tile_nodes,
                             reinterpret_cast<const int2*>(tile_rows), tile_colors,
                             reinterpret_cast<const uint4*>(tile_elems), coords, node_stride, comp_stride, ek,
                             xstride, K_vals, M_vals);
    return launch_check(fn);
}
