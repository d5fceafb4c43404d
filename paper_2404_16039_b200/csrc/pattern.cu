// a14/a15: topological CSR pattern of sparse(X3D(:),Y3D(:),...)
// and the two scatter plans, built on the GPU without a global sort:
//   1. node degree histogram, exclusive scan, bucket fill -> node->element
//      incidence lists (packed e << SH | a), each list sorted ascending (determinism);
//   2. one thread per row builds the sorted unique column set of its row from
//      the vertices of its incident elements in a per-thread shared-memory list
//      (rows longer than CAP go to a single-thread fallback with a 4096-entry
//      list); row lengths -> scan -> row_ptr;
//   3. fill: the same per-row sets are written to col_idx, and every incidence
//      (e, a) of row v records the in-row position of each of its element's
//      vertices: elem2nnz (atomic scatter plan) and node_elem_slot (gather plan).
// fem_p1_pattern: P1 (nv = dim+1 <= 4, packing e*4+a, 64-entry rows);
// fem_pattern: any element with nv <= 16 nodes (P2: 6 / 10; packing e*16+a,
// 128-entry rows), no gather plan.
#include "vb_internal.cuh"

namespace vb {
namespace {

constexpr int ROW_CAP_BIG = 4096;      // single-thread fallback list
constexpr int FLAG_OVERFLOW_ROWS = 0;  // number of rows that took the fallback
constexpr int FLAG_TOO_LONG = 1;       // a row exceeded ROW_CAP_BIG
constexpr int FLAG_SLOT_RANGE = 2;     // a row had > 255 entries while slots requested

__global__ void degree_k(int64_t ne, int nv, const int32_t* __restrict__ elems, int64_t eld, int32_t* __restrict__ deg) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += stride)
        for (int a = 0; a < nv; a++) atomicAdd(deg + elems[a * eld + e], 1);
}

template <int SH>
__global__ void bucket_fill_k(int64_t ne, int nv, const int32_t* __restrict__ elems, int64_t eld,
                              int32_t* __restrict__ cursor, int32_t* __restrict__ node_elem) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += stride)
        for (int a = 0; a < nv; a++) {
            int pos = atomicAdd(cursor + elems[a * eld + e], 1);
            node_elem[pos] = (int32_t)((e << SH) + a);
        }
}

// insertion sort of each node's incidence list (ascending e, hence ascending e << SH | a).
// Lists of up to SORT_CAP entries are loaded into a per-thread shared-memory
// strip (stride SORT_BLOCK, bank-conflict free), sorted there and written back;
// longer lists are sorted in place in global memory.
// Lists of up to 32 entries (every list of the Kuhn and square meshes: 24 / 6 incidences per interior node) are
// sorted in registers by a bitonic network padded with INT_MAX (240 compare-exchanges for 32 values, all indices
// compile-time): the bucket fill's atomics leave a list in arrival order, which is random within a wave of the
// grid, so the insertion sort paid n^2/4 shared-memory moves per list (ncu r02g: 214 M warp instructions, 0.43 ms).
#ifndef VB_SORT_NET
#define VB_SORT_NET 1   // 0: insertion sort only; 2: networks with word accesses (A/B timing)
#endif
template <int N>
__device__ __forceinline__ void sort_net(int32_t* __restrict__ p, int n) {
    int32_t r[N];
#pragma unroll
    for (int i = 0; i < N; i++) r[i] = i < n ? p[i] : 0x7fffffff;
#pragma unroll
    for (int k = 2; k <= N; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < N; i++) {
                const int l = i ^ j;
                if (l > i) {
                    const int32_t lo = min(r[i], r[l]), hi = max(r[i], r[l]);
                    const bool asc = (i & k) == 0;
                    r[i] = asc ? lo : hi;
                    r[l] = asc ? hi : lo;
                }
            }
#pragma unroll
    for (int i = 0; i < N; i++)
        if (i < n) p[i] = r[i];
}

// The same through 128-bit accesses: the list [lo, lo + n) sits at offset h = lo & 3 of the aligned quads that cover
// it (h + n <= N); values of the neighbouring lists in the first and last quad are replaced by -inf / +inf
// sentinels, so after the network position j holds the sorted entry j - h, and only positions [h, h + n) are
// written back (whole quads where they lie inside the list).  A per-thread list is 96 bytes apart from its
// neighbour's: 6-8 quad loads instead of 24 word loads per list.
template <int N>
__device__ __forceinline__ void sort_net_quads(int32_t* __restrict__ pa, int h, int n) {
    int32_t r[N];
    const int4* q = reinterpret_cast<const int4*>(pa);
#pragma unroll
    for (int qi = 0; qi < N / 4; qi++) {
        int4 t = make_int4(0, 0, 0, 0);
        if (qi * 4 < h + n) t = q[qi];
        r[4 * qi] = t.x;
        r[4 * qi + 1] = t.y;
        r[4 * qi + 2] = t.z;
        r[4 * qi + 3] = t.w;
    }
#pragma unroll
    for (int j = 0; j < N; j++) r[j] = j < h ? (int32_t)0x80000000 : (j < h + n ? r[j] : 0x7fffffff);
#pragma unroll
    for (int k = 2; k <= N; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < N; i++) {
                const int l = i ^ j;
                if (l > i) {
                    const int32_t lo = min(r[i], r[l]), hi = max(r[i], r[l]);
                    const bool asc = (i & k) == 0;
                    r[i] = asc ? lo : hi;
                    r[l] = asc ? hi : lo;
                }
            }
#pragma unroll
    for (int qi = 0; qi < N / 4; qi++) {
        if (4 * qi >= h && 4 * qi + 4 <= h + n) {
            reinterpret_cast<int4*>(pa)[qi] = make_int4(r[4 * qi], r[4 * qi + 1], r[4 * qi + 2], r[4 * qi + 3]);
        } else {
#pragma unroll
            for (int c = 0; c < 4; c++)
                if (4 * qi + c >= h && 4 * qi + c < h + n) pa[4 * qi + c] = r[4 * qi + c];
        }
    }
}

constexpr int SORT_BLOCK = 128;
constexpr int SORT_CAP = 48;
__global__ void __launch_bounds__(SORT_BLOCK) sort_incidences_k(int64_t nn, const int32_t* __restrict__ nptr,
                                                                int32_t* __restrict__ node_elem) {
    __shared__ int32_t strip[SORT_CAP * SORT_BLOCK];
    int32_t* L = strip + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += stride) {
        int lo = nptr[v], hi = nptr[v + 1];
        const int n = hi - lo;
        if (VB_SORT_NET && n <= 32) {
            if (n <= 1) continue;
            const int h = lo & 3;   // node_elem is 256-byte aligned in the work buffer (carve)
            int32_t* pa = node_elem + (lo - h);
            if (VB_SORT_NET == 2 || h + n > 32) {
                if (n <= 8) sort_net<8>(node_elem + lo, n);
                else if (n <= 16) sort_net<16>(node_elem + lo, n);
                else sort_net<32>(node_elem + lo, n);
            } else if (h + n <= 8) sort_net_quads<8>(pa, h, n);
            else if (h + n <= 16) sort_net_quads<16>(pa, h, n);
            else sort_net_quads<32>(pa, h, n);
            continue;
        }
        if (n <= SORT_CAP) {
            for (int i = 0; i < n; i++) {
                int32_t x = node_elem[lo + i];
                int j = i - 1;
                while (j >= 0 && L[j * SORT_BLOCK] > x) {
                    L[(j + 1) * SORT_BLOCK] = L[j * SORT_BLOCK];
                    j--;
                }
                L[(j + 1) * SORT_BLOCK] = x;
            }
            for (int i = 0; i < n; i++) node_elem[lo + i] = L[i * SORT_BLOCK];
            continue;
        }
        for (int i = lo + 1; i < hi; i++) {
            int32_t x = node_elem[i];
            int j = i - 1;
            while (j >= lo && node_elem[j] > x) {
                node_elem[j + 1] = node_elem[j];
                j--;
            }
            node_elem[j + 1] = x;
        }
    }
}

// sorted-unique insertion into a list with element stride `st`; returns false on overflow
__device__ __forceinline__ int lower_bound_s(const int32_t* L, int st, int cnt, int32_t w) {
    int lo = 0, hi = cnt;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (L[mid * st] < w) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ bool insert_unique(int32_t* L, int st, int& cnt, int cap, int32_t w) {
    int pos = lower_bound_s(L, st, cnt, w);
    if (pos < cnt && L[pos * st] == w) return true;
    if (cnt == cap) return false;
    for (int i = cnt; i > pos; i--) L[i * st] = L[(i - 1) * st];
    L[pos * st] = w;
    cnt++;
    return true;
}

// Incidences are processed in chunks of CH: all their element ids, then all
// their vertex ids, are loaded before any list work, so a thread keeps CH (x nv)
// independent global loads in flight instead of one dependent pair at a time.
template <int SH>
struct Chunk {
    static constexpr int NVM = 1 << SH;       // max vertices per element of this packing
    static constexpr int CH = SH == 2 ? 8 : 2;
};

// vertices of the incidences [i0, i0 + CH) of a row (-1 past hi / past nv)
template <int SH>
__device__ __forceinline__ void load_chunk(int i0, int hi, int nv, const int32_t* __restrict__ elems, int64_t eld,
                                           const int32_t* __restrict__ node_elem, int32_t (&ea)[Chunk<SH>::CH],
                                           int32_t (&w)[Chunk<SH>::CH][Chunk<SH>::NVM]) {
    constexpr int CH = Chunk<SH>::CH, NVM = Chunk<SH>::NVM;
#pragma unroll
    for (int k = 0; k < CH; k++) ea[k] = i0 + k < hi ? __ldg(node_elem + i0 + k) : -1;
#pragma unroll
    for (int k = 0; k < CH; k++)
#pragma unroll
        for (int b = 0; b < NVM; b++)
            w[k][b] = (ea[k] >= 0 && b < nv) ? __ldg(elems + b * eld + (ea[k] >> SH)) : -1;
}

// Build row v's sorted unique column list into L (stride st, capacity cap):
// v itself, then the other vertices of every incident element.
// Returns the count, or -1 on overflow.
template <int SH>
__device__ int build_row(int64_t v, int nv, const int32_t* __restrict__ elems, int64_t eld,
                         const int32_t* __restrict__ nptr, const int32_t* __restrict__ node_elem,
                         int32_t* L, int st, int cap) {
    constexpr int CH = Chunk<SH>::CH, NVM = Chunk<SH>::NVM;
    int lo = nptr[v], hi = nptr[v + 1];
    if (lo == hi) return 0;
    int cnt = 1;
    L[0] = (int32_t)v;
    for (int i0 = lo; i0 < hi; i0 += CH) {
        int32_t ea[CH], w[CH][NVM];
        load_chunk<SH>(i0, hi, nv, elems, eld, node_elem, ea, w);
#pragma unroll
        for (int k = 0; k < CH; k++)
#pragma unroll
            for (int b = 0; b < NVM; b++)
                if (w[k][b] >= 0 && b != (ea[k] & (NVM - 1)))
                    if (!insert_unique(L, st, cnt, cap, w[k][b])) return -1;
    }
    return cnt;
}

// write col_idx and the plans for row v whose list L (stride st) has cnt entries
template <int SH>
__device__ void emit_row(int64_t v, int cnt, int nv, int64_t ne, const int32_t* __restrict__ elems, int64_t eld,
                         const int32_t* __restrict__ nptr, const int32_t* __restrict__ node_elem,
                         const int32_t* L, int st, const int32_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx,
                         int32_t* __restrict__ elem2nnz, uint32_t* __restrict__ slots, int* flags) {
    constexpr int CH = Chunk<SH>::CH, NVM = Chunk<SH>::NVM;
    int32_t base = row_ptr[v];
    for (int i = 0; i < cnt; i++) col_idx[base + i] = L[i * st];
    if (!elem2nnz && !slots) return;
    if (slots && cnt > 255) atomicExch(flags + FLAG_SLOT_RANGE, 1);
    int lo = nptr[v], hi = nptr[v + 1];
    // the row's own vertex (local vertex a of every incidence) has one position: searched once per row
    const int pos_self = lower_bound_s(L, st, cnt, (int32_t)v);
    for (int i0 = lo; i0 < hi; i0 += CH) {
        int32_t ea[CH], w[CH][NVM];
        load_chunk<SH>(i0, hi, nv, elems, eld, node_elem, ea, w);
#pragma unroll
        for (int k = 0; k < CH; k++) {
            if (ea[k] < 0) break;
            int64_t e = ea[k] >> SH;
            int a = ea[k] & (NVM - 1);
            if constexpr (SH == 2) {
                // P1: byte 0: in-row offset of the row's own vertex (the diagonal);
                // bytes 1..nv-1: offsets of the element's other vertices, ascending b
                uint32_t packed = 0;
                int byte = 1;
#pragma unroll
                for (int b = 0; b < NVM; b++) {
                    if (b >= nv) break;
                    int pos = (b == a) ? pos_self : lower_bound_s(L, st, cnt, w[k][b]);
                    VB_CHECK(pos < cnt && L[pos * st] == w[k][b]);   // every vertex is in the row
                    if (elem2nnz) elem2nnz[(int64_t)(a * nv + b) * ne + e] = base + pos;
                    int sh = (b == a) ? 0 : 8 * byte++;
                    if (sh < 32) packed |= (uint32_t)(pos & 0xff) << sh;
                }
                if (slots) slots[i0 + k] = packed;
            } else {
                // generic: byte b (word b / 4) = in-row offset of node b, natural order
                constexpr int NW = NVM / 4;
                uint32_t packed[NW];
#pragma unroll
                for (int j = 0; j < NW; j++) packed[j] = 0;
#pragma unroll
                for (int b = 0; b < NVM; b++) {
                    if (b >= nv) break;
                    int pos = (b == a) ? pos_self : lower_bound_s(L, st, cnt, w[k][b]);
                    VB_CHECK(pos < cnt && L[pos * st] == w[k][b]);
                    if (elem2nnz) elem2nnz[(int64_t)(a * nv + b) * ne + e] = base + pos;
                    packed[b / 4] |= (uint32_t)(pos & 0xff) << (8 * (b % 4));
                }
                if (slots) {
                    const int nw = (nv + 3) / 4;
#pragma unroll
                    for (int j = 0; j < NW; j++)
                        if (j < nw) slots[(int64_t)(i0 + k) * nw + j] = packed[j];
                }
            }
        }
    }
}

// Row lists of up to RL entries are kept in the work buffer (stride RL) by the
// count phase, so the fill phase need not rebuild them.
constexpr int RL = 32;

template <int SH, int CAP, int BLOCK>
__global__ void __launch_bounds__(BLOCK) row_count_k(int64_t nn, int nv, const int32_t* __restrict__ elems,
                                                     int64_t eld, const int32_t* __restrict__ nptr,
                                                     const int32_t* __restrict__ node_elem,
                                                     int32_t* __restrict__ row_len, int32_t* __restrict__ ovf_list,
                                                     int32_t* __restrict__ rowlist, int* flags) {
    __shared__ int32_t Ls[CAP * BLOCK];
    int32_t* L = Ls + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += stride) {
        int cnt = build_row<SH>(v, nv, elems, eld, nptr, node_elem, L, BLOCK, CAP);
        if (cnt < 0) {
            int k = atomicAdd(flags + FLAG_OVERFLOW_ROWS, 1);
            ovf_list[k] = (int32_t)v;
            cnt = 0;  // fixed by the fallback
        } else if (cnt <= RL) {
            int32_t* out = rowlist + v * RL;
            for (int i = 0; i < cnt; i++) out[i] = L[i * BLOCK];
        }
        row_len[v] = cnt;
    }
}

// fallback for rows with more than CAP columns: one thread per row, big list
template <int SH>
__global__ void row_count_big_k(int nv, const int32_t* __restrict__ elems, int64_t eld, const int32_t* __restrict__ nptr,
                                const int32_t* __restrict__ node_elem, int32_t* __restrict__ row_len,
                                const int32_t* __restrict__ ovf_list, int* flags) {
    __shared__ int32_t L[ROW_CAP_BIG];
    int n_ovf = flags[FLAG_OVERFLOW_ROWS];
    for (int k = blockIdx.x; k < n_ovf; k += gridDim.x) {
        if (threadIdx.x == 0) {
            int64_t v = ovf_list[k];
            int cnt = build_row<SH>(v, nv, elems, eld, nptr, node_elem, L, 1, ROW_CAP_BIG);
            if (cnt < 0) { atomicExch(flags + FLAG_TOO_LONG, 1); cnt = 0; }
            row_len[v] = cnt;
        }
        __syncthreads();
    }
}

// rowlist != NULL: rows of <= RL entries take their list from the count phase
// (row_ptr gives the length); longer rows are rebuilt.
template <int SH, int CAP, int BLOCK>
__global__ void __launch_bounds__(BLOCK) row_fill_k(int64_t nn, int64_t ne, int nv, const int32_t* __restrict__ elems,
                                                    int64_t eld, const int32_t* __restrict__ nptr,
                                                    const int32_t* __restrict__ node_elem,
                                                    const int32_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx,
                                                    int32_t* __restrict__ elem2nnz, uint32_t* __restrict__ slots,
                                                    const int32_t* __restrict__ rowlist,
                                                    int32_t* __restrict__ ovf_list, int* flags) {
    __shared__ int32_t Ls[CAP * BLOCK];
    int32_t* L = Ls + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += stride) {
        int cnt = row_ptr[v + 1] - row_ptr[v];
        if (rowlist && cnt <= RL) {
            const int32_t* in = rowlist + v * RL;
            for (int i = 0; i < cnt; i++) L[i * BLOCK] = in[i];
        } else {
            cnt = build_row<SH>(v, nv, elems, eld, nptr, node_elem, L, BLOCK, CAP);
        }
        if (cnt < 0) {  // long row: the single-thread fallback fills it
            ovf_list[atomicAdd(flags + FLAG_OVERFLOW_ROWS, 1)] = (int32_t)v;
            continue;
        }
        emit_row<SH>(v, cnt, nv, ne, elems, eld, nptr, node_elem, L, BLOCK, row_ptr, col_idx, elem2nnz, slots, flags);
    }
}

template <int SH>
__global__ void row_fill_big_k(int64_t ne, int nv, const int32_t* __restrict__ elems, int64_t eld,
                               const int32_t* __restrict__ nptr, const int32_t* __restrict__ node_elem,
                               const int32_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx,
                               int32_t* __restrict__ elem2nnz, uint32_t* __restrict__ slots,
                               const int32_t* __restrict__ ovf_list, int* flags) {
    __shared__ int32_t L[ROW_CAP_BIG];
    int n_ovf = flags[FLAG_OVERFLOW_ROWS];
    for (int k = blockIdx.x; k < n_ovf; k += gridDim.x) {
        if (threadIdx.x == 0) {
            int64_t v = ovf_list[k];
            int cnt = build_row<SH>(v, nv, elems, eld, nptr, node_elem, L, 1, ROW_CAP_BIG);
            if (cnt >= 0)
                emit_row<SH>(v, cnt, nv, ne, elems, eld, nptr, node_elem, L, 1, row_ptr, col_idx, elem2nnz, slots, flags);
        }
        __syncthreads();
    }
}

// State the count phase leaves in the work buffer for the fill phase.
struct Stamp {
    int64_t magic, nn, ne, nv, elem_ld;
    const void* elems;
    int64_t pad[2];
};
constexpr int64_t STAMP_MAGIC = 0x5642504154543031ll;   // "VBPATT01"

struct Work {
    Stamp* stamp;       // 64 bytes
    int32_t* cursor;    // nn+1
    int32_t* nptr;      // nn+1
    int32_t* node_elem; // nv*ne
    int32_t* row_len;   // nn+1
    int32_t* ovf;       // nn
    int32_t* rowlist;   // nn*RL
    int* flags;         // 4 ints
    int64_t* total;     // 2 int64
    void* scan_tmp;
    size_t bytes;
};

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

Work carve(void* base, int64_t nn, int64_t ne, int nv) {
    Work w{};
    char* p = reinterpret_cast<char*>(base);
    size_t off = 0;
    auto take = [&](size_t b) { char* r = p ? p + off : nullptr; off += al(b); return r; };
    w.stamp = (Stamp*)take(sizeof(Stamp));
    w.cursor = (int32_t*)take(4 * (nn + 1));
    w.nptr = (int32_t*)take(4 * (nn + 1));
    w.node_elem = (int32_t*)take(4 * (size_t)nv * ne + 4);
    w.row_len = (int32_t*)take(4 * (nn + 1));
    w.ovf = (int32_t*)take(4 * (nn + 1));
    w.rowlist = (int32_t*)take(4 * (size_t)nn * RL + 4);
    w.flags = (int*)take(64);
    w.total = (int64_t*)take(64);
    int64_t smax = nn > nv * ne ? nn : nv * ne;
    w.scan_tmp = take(scan_tmp_bytes(smax + 1));
    w.bytes = off;
    return w;
}

__global__ void write_stamp_k(Stamp* st, Stamp v) { *st = v; }

// optional validation (VB_PATTERN_VALIDATE): the first (element, vertex) slot, as e * nv + a, whose id is
// outside [0, nn) -> *first (initialised to INT64_MAX)
__global__ void init_first_k(long long* first) { *first = 0x7fffffffffffffffll; }
__global__ void validate_k(int64_t ne, int nv, int64_t nn, const int32_t* __restrict__ elems, int64_t eld,
                           long long* __restrict__ first) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x)
        for (int a = 0; a < nv; a++) {
            const int32_t v = elems[a * eld + e];
            if (v < 0 || v >= nn) {
                atomicMin(first, (long long)(e * nv + a));
                break;
            }
        }
}

template <int SH, int CAP, int BLOCK>
vb_status pattern_impl(const char* fn, int nv, int64_t nn, int64_t ne, const int32_t* elems, int64_t elem_ld,
                       void* work, size_t* work_bytes, int32_t* row_ptr, int32_t* col_idx, int64_t col_cap,
                       int32_t* elem2nnz, int32_t* node_elem_ptr, int32_t* node_elem, uint32_t* node_elem_slot,
                       int64_t* nnz_out, vb_stream_t stream, bool validate) {
    if (nn < 0 || ne < 0) { set_error("%s: negative nn or ne", fn); return VB_ERR_ARG; }
    if (ne >= (1ll << (31 - SH)) || (int64_t)nv * nv * ne >= (1ll << 31) || nn >= (1ll << 31) - 1) {
        set_error("%s: ne=%lld / nn=%lld too large for int32 plans", fn, (long long)ne, (long long)nn);
        return VB_ERR_OVERFLOW;
    }
    Work w = carve(nullptr, nn, ne, nv);
    if (!work) {
        if (!work_bytes) { set_error("%s: work and work_bytes both NULL", fn); return VB_ERR_ARG; }
        *work_bytes = w.bytes;
        return VB_OK;
    }
    if (work_bytes && *work_bytes < w.bytes) { set_error("%s: work buffer too small (%zu < %zu)", fn, *work_bytes, w.bytes); return VB_ERR_WORKSPACE; }
    if (!row_ptr) { set_error("%s: NULL row_ptr", fn); return VB_ERR_ARG; }
    if (ne > 0 && !elems) { set_error("%s: NULL elems", fn); return VB_ERR_ARG; }
    if (elem_ld < ne) { set_error("%s: elem_ld < ne", fn); return VB_ERR_ARG; }
    if ((node_elem_ptr != nullptr) != (node_elem != nullptr) || (node_elem_slot && !node_elem)) {
        set_error("%s: node_elem_ptr, node_elem (and node_elem_slot) must be given together", fn);
        return VB_ERR_ARG;
    }
    w = carve(work, nn, ne, nv);
    cudaStream_t s = cs(stream);
    const Stamp mine{STAMP_MAGIC, nn, ne, nv, elem_ld, elems, {0, 0}};
    vb_status st = VB_OK;
    if (validate && ne > 0) {   // before any kernel indexes by vertex id (one read-back)
        long long* first = reinterpret_cast<long long*>(w.total) + 1;
        init_first_k<<<1, 1, 0, s>>>(first);
        validate_k<<<grid_for(ne, 256, 8), 256, 0, s>>>(ne, nv, nn, elems, elem_ld, first);
        if ((st = launch_check(fn)) != VB_OK) return st;
        long long bad = 0;
        if ((st = read_small(s, first, sizeof(bad), &bad, fn)) != VB_OK) return st;
        if (bad != 0x7fffffffffffffffll) {
            int32_t v = 0;
            const int64_t e = bad / nv, a = bad % nv;
            if ((st = read_small(s, elems + a * elem_ld + e, 4, &v, fn)) != VB_OK) return st;
            set_error("%s: vertex %lld of element %lld is %d, outside [0, nn=%lld)", fn, (long long)a, (long long)e, v,
                      (long long)nn);
            return VB_ERR_ARG;
        }
    }
#ifndef VB_PATTERN_BPS
#define VB_PATTERN_BPS 6   // resident row-kernel blocks per SM (32 KB of lists each: 6 fit); configs[4] pattern-only 2.11 (4) / 2.03 (5) / 1.98 (6) / 2.45 ms (7: a second wave)
#endif
    unsigned gr = grid_for(nn, BLOCK, VB_PATTERN_BPS);

    // 1. node -> element incidences (into work; the fill phase reuses them)
    auto incidences = [&]() -> vb_status {
        cudaMemsetAsync(w.cursor, 0, 4 * (nn + 1), s);
        unsigned ge = grid_for(ne, 256, 8);
        if (ne > 0) degree_k<<<ge, 256, 0, s>>>(ne, nv, elems, elem_ld, w.cursor);
        vb_status r = exclusive_scan_i32(w.cursor, w.nptr, nn, w.scan_tmp, s, nullptr);
        if (r != VB_OK) return r;
        cudaMemcpyAsync(w.cursor, w.nptr, 4 * (nn + 1), cudaMemcpyDeviceToDevice, s);
        if (ne > 0) bucket_fill_k<SH><<<ge, 256, 0, s>>>(ne, nv, elems, elem_ld, w.cursor, w.node_elem);
        if (nn > 0) sort_incidences_k<<<grid_for(nn, SORT_BLOCK, 8), SORT_BLOCK, 0, s>>>(nn, w.nptr, w.node_elem);
        return launch_check(fn);
    };

    if (!col_idx) {
        // count phase: incidences, row lists (kept for the fill phase), row_ptr, nnz
        cudaMemsetAsync(w.flags, 0, 64, s);
        Stamp none{};
        write_stamp_k<<<1, 1, 0, s>>>(w.stamp, none);
        if ((st = incidences()) != VB_OK) return st;
        if (nn > 0) row_count_k<SH, CAP, BLOCK><<<gr, BLOCK, 0, s>>>(nn, nv, elems, elem_ld, w.nptr, w.node_elem, w.row_len, w.ovf, w.rowlist, w.flags);
        row_count_big_k<SH><<<64, 32, 0, s>>>(nv, elems, elem_ld, w.nptr, w.node_elem, w.row_len, w.ovf, w.flags);
        if ((st = exclusive_scan_i32(w.row_len, row_ptr, nn, w.scan_tmp, s, w.total)) != VB_OK) return st;
        write_stamp_k<<<1, 1, 0, s>>>(w.stamp, mine);
        if ((st = launch_check(fn)) != VB_OK) return st;
        int64_t host[2] = {0, 0};
        int hflags[4] = {0, 0, 0, 0};
        if ((st = read_small(s, w.total, sizeof(int64_t), host, fn)) != VB_OK) return st;
        if ((st = read_small(s, w.flags, sizeof(hflags), hflags, fn)) != VB_OK) return st;
        if (hflags[FLAG_TOO_LONG]) { set_error("%s: a row has more than %d distinct columns", fn, ROW_CAP_BIG); return VB_ERR_UNSUPPORTED; }
        if (host[0] >= (1ll << 31)) { set_error("%s: nnz=%lld does not fit int32", fn, (long long)host[0]); return VB_ERR_OVERFLOW; }
        if (nnz_out) *nnz_out = host[0];
        return VB_OK;
    }
    // fill phase (row_ptr from the count phase); check the capacity before writing.
    // With the count phase's work buffer (stamp matches) its incidence lists and
    // row lists are reused; otherwise they are rebuilt here.
    int32_t nnz32 = 0;
    Stamp seen{};
    if ((st = read_small(s, row_ptr + nn, 4, &nnz32, fn)) != VB_OK) return st;
    if ((st = read_small(s, w.stamp, sizeof(Stamp), &seen, fn)) != VB_OK) return st;
    if (nnz32 < 0 || nnz32 > col_cap) { set_error("%s: col_cap=%lld < nnz=%d", fn, (long long)col_cap, nnz32); return VB_ERR_ARG; }
    const bool reuse = seen.magic == mine.magic && seen.nn == nn && seen.ne == ne && seen.nv == nv &&
                       seen.elem_ld == elem_ld && seen.elems == elems;
    cudaMemsetAsync(w.flags, 0, 64, s);
    if (!reuse && (st = incidences()) != VB_OK) return st;
    if (node_elem_ptr) {
        cudaMemcpyAsync(node_elem_ptr, w.nptr, 4 * (nn + 1), cudaMemcpyDeviceToDevice, s);
        if (ne > 0) cudaMemcpyAsync(node_elem, w.node_elem, 4 * (size_t)nv * ne, cudaMemcpyDeviceToDevice, s);
    }
    if (nn > 0) {
        // rows longer than CAP are collected by row_fill_k and filled by the fallback
        row_fill_k<SH, CAP, BLOCK><<<gr, BLOCK, 0, s>>>(nn, ne, nv, elems, elem_ld, w.nptr, w.node_elem, row_ptr, col_idx,
                                                        elem2nnz, node_elem_slot, reuse ? w.rowlist : nullptr,
                                                        w.ovf, w.flags);
        row_fill_big_k<SH><<<64, 32, 0, s>>>(ne, nv, elems, elem_ld, w.nptr, w.node_elem, row_ptr, col_idx, elem2nnz,
                                              node_elem_slot, w.ovf, w.flags);
    }
    if ((st = launch_check(fn)) != VB_OK) return st;
    int hflags[4] = {0, 0, 0, 0};
    if ((st = read_small(s, w.flags, sizeof(hflags), hflags, fn)) != VB_OK) return st;
    if (hflags[FLAG_TOO_LONG]) { set_error("%s: a row has more than %d distinct columns", fn, ROW_CAP_BIG); return VB_ERR_UNSUPPORTED; }
    if (hflags[FLAG_SLOT_RANGE]) { set_error("%s: a row has more than 255 entries; gather plan unsupported, use elem2nnz", fn); return VB_ERR_UNSUPPORTED; }
    if (nnz_out) *nnz_out = nnz32;
    return VB_OK;
}

}  // namespace
}  // namespace vb

using namespace vb;

extern "C" vb_status fem_p1_pattern(int dim, int64_t nn, int64_t ne, const int32_t* elems, int64_t elem_ld, void* work,
                                    size_t* work_bytes, int32_t* row_ptr, int32_t* col_idx, int64_t col_cap,
                                    int32_t* elem2nnz, int32_t* node_elem_ptr, int32_t* node_elem,
                                    uint32_t* node_elem_slot, int64_t* nnz_out, vb_stream_t stream) {
    clear_error();
    const bool validate = (dim & VB_PATTERN_VALIDATE) != 0;
    dim &= ~VB_PATTERN_VALIDATE;
    if (dim != 2 && dim != 3) { set_error("fem_p1_pattern: dim=%d, need 2 or 3", dim); return VB_ERR_UNSUPPORTED; }
    return pattern_impl<2, 64, 128>("fem_p1_pattern", dim + 1, nn, ne, elems, elem_ld, work, work_bytes, row_ptr,
                                    col_idx, col_cap, elem2nnz, node_elem_ptr, node_elem, node_elem_slot, nnz_out,
                                    stream, validate);
}

extern "C" vb_status fem_pattern(int nv, int64_t nn, int64_t ne, const int32_t* elems, int64_t elem_ld, void* work,
                                 size_t* work_bytes, int32_t* row_ptr, int32_t* col_idx, int64_t col_cap,
                                 int32_t* elem2nnz, int32_t* node_elem_ptr, int32_t* node_elem,
                                 uint32_t* node_elem_slot, int64_t* nnz_out, vb_stream_t stream) {
    clear_error();
    const bool validate = (nv & VB_PATTERN_VALIDATE) != 0;
    nv &= ~VB_PATTERN_VALIDATE;
    if (nv < 2 || nv > 16) { set_error("fem_pattern: nv=%d, need 2..16 nodes per element", nv); return VB_ERR_UNSUPPORTED; }
    return pattern_impl<4, 128, 64>("fem_pattern", nv, nn, ne, elems, elem_ld, work, work_bytes, row_ptr, col_idx,
                                    col_cap, elem2nnz, node_elem_ptr, node_elem, node_elem_slot, nnz_out, stream,
                                    validate);
}

// ------------------------------------------------------------------ plan statistics
namespace vb {
namespace {
// maxima over 32-row blocks: [0] row length, [1] CSR entries of a block, [2] incidences of a block
__global__ void plan_stats_k(int64_t nn, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ nptr,
                             int* __restrict__ out) {
    int m0 = 0, m1 = 0, m2 = 0;
    const int64_t nb = (nn + 31) / 32;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r0 = b * 32, r1 = r0 + 32 < nn ? r0 + 32 : nn;
        for (int64_t r = r0; r < r1; r++) m0 = max(m0, row_ptr[r + 1] - row_ptr[r]);
        m1 = max(m1, row_ptr[r1] - row_ptr[r0]);
        if (nptr) m2 = max(m2, nptr[r1] - nptr[r0]);
    }
    atomicMax(out, m0);
    atomicMax(out + 1, m1);
    atomicMax(out + 2, m2);
}
}  // namespace
}  // namespace vb

extern "C" vb_status fem_plan_stats(int64_t nn, const int32_t* row_ptr, const int32_t* node_elem_ptr, void* work,
                                    int64_t* stats_out, vb_stream_t stream) {
    clear_error();
    const char* fn = "fem_plan_stats";
    if (nn < 0) { set_error("%s: negative nn", fn); return VB_ERR_ARG; }
    if (!row_ptr || !work || !stats_out) { set_error("%s: NULL row_ptr, work or stats_out", fn); return VB_ERR_ARG; }
    cudaStream_t s = cs(stream);
    int* d = reinterpret_cast<int*>(work);
    cudaMemsetAsync(d, 0, 3 * sizeof(int), s);
    if (nn > 0) plan_stats_k<<<grid_for((nn + 31) / 32, 256, 4), 256, 0, s>>>(nn, row_ptr, node_elem_ptr, d);
    vb_status st = launch_check(fn);
    if (st != VB_OK) return st;
    int h[3] = {0, 0, 0};
    if ((st = read_small(s, d, sizeof(h), h, fn)) != VB_OK) return st;
    for (int i = 0; i < 3; i++) stats_out[i] = h[i];
    return VB_OK;
}

// ------------------------------------------------------------------ packed plan words
namespace vb {
namespace {
__global__ void pack_slots_k(int dim, int64_t n, const uint32_t* __restrict__ in, uint16_t* __restrict__ out,
                             int* __restrict__ bad) {
    int b = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t w = in[i];
        const uint32_t s1 = (w >> 8) & 0xff, s2 = (w >> 16) & 0xff, s3 = dim == 3 ? w >> 24 : 0;
        b |= (s1 | s2 | s3) >= 16;
        out[i] = (uint16_t)(s1 | (s2 << 4) | (s3 << 8));
    }
    if (b) atomicOr(bad, 1);
}
}  // namespace
}  // namespace vb

extern "C" vb_status fem_plan_pack_slots(int dim, int64_t n_inc, const uint32_t* node_elem_slot, uint16_t* packed,
                                         void* work, vb_stream_t stream) {
    clear_error();
    const char* fn = "fem_plan_pack_slots";
    if (dim != 2 && dim != 3) { set_error("%s: dim=%d, need 2 or 3", fn, dim); return VB_ERR_UNSUPPORTED; }
    if (n_inc < 0) { set_error("%s: negative n_inc", fn); return VB_ERR_ARG; }
    if (n_inc > 0 && (!node_elem_slot || !packed || !work)) { set_error("%s: NULL argument", fn); return VB_ERR_ARG; }
    if (n_inc == 0) return VB_OK;
    cudaStream_t s = cs(stream);
    int* d = reinterpret_cast<int*>(work);
    cudaMemsetAsync(d, 0, sizeof(int), s);
    pack_slots_k<<<grid_for(n_inc, 256, 8), 256, 0, s>>>(dim, n_inc, node_elem_slot, packed, d);
    vb_status st = launch_check(fn);
    if (st != VB_OK) return st;
    int bad = 0;
    if ((st = read_small(s, d, sizeof(int), &bad, fn)) != VB_OK) return st;
    if (bad) { set_error("%s: a row has more than 16 entries; the packed form needs offsets < 16", fn); return VB_ERR_UNSUPPORTED; }
    return VB_OK;
}
