// Row classes of the P1 gather plan (fem_plan_classes): rows whose assembly runs
// the identical sequence of operations, so that a warp can assemble 32 of them
// with a warp-uniform incidence loop and the row's K/M accumulators in registers
// (assemble_class_k, assemble.cu).
//
// The row of node v (the nnz of row v of sparse(X3D(:),Y3D(:),..))
// is assembled from its incidences (e, a), ascending e, each one contributing
// K_e[a][b] and M_e[a][b] to the row's in-row slots of the element's other
// vertices (the plan word of the incidence, fem_p1_pattern).  The signature of
// a row is (row length L, incidence count n, the n plan words in order): two
// rows with equal signatures differ only in their column ids and coordinates.
// On meshes built by uniform refinement (the paper's unit square / cube /
// sphere tables) almost every row falls into a handful of classes.
//
// Build (all on the GPU, deterministic): 63-bit hash of each signature -> radix
// sort of (hash, row) -> run-length encoding -> runs with fewer than MIN_CLASS
// rows, rows longer than the register budget and hash collisions (every row is
// compared word by word with its class's first row) are moved into one "mixed"
// class -> re-sort -> groups of up to 32 consecutive rows of one class.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>

#include "vb_internal.cuh"

namespace vb {
namespace {

constexpr uint64_t MIXED = ~0ull;   // key of rows outside every class (top bit set; class keys have it clear)
constexpr int MIN_CLASS = 8;        // smaller classes go to the mixed rows

__device__ __forceinline__ uint64_t fmix64(uint64_t h) {
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ull;
    h ^= h >> 33;
    return h;
}

__global__ void cls_hash_k(int64_t nn, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ nptr,
                           const uint32_t* __restrict__ nslot, int maxl, int maxn, uint64_t* __restrict__ keys,
                           int32_t* __restrict__ rows) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nn) return;
    const int L = row_ptr[v + 1] - row_ptr[v];
    const int i0 = nptr[v], n = nptr[v + 1] - i0;
    uint64_t key = MIXED;
    if (L >= 2 && L <= maxl && n > 0 && n <= maxn) {
        uint64_t h = fmix64(((uint64_t)L << 32) | (uint32_t)n);
        for (int i = 0; i < n; i++) h = (h ^ __ldg(nslot + i0 + i)) * 0x100000001b3ull + 0x9e3779b97f4a7c15ull;
        key = fmix64(h) >> 1;
    }
    keys[v] = key;
    rows[v] = (int32_t)v;
}

// run id of sorted position i: the last run whose offset is <= i (offsets ascending)
__device__ __forceinline__ int run_of(int64_t i, const int32_t* __restrict__ roff, int nruns) {
    int lo = 0, hi = nruns - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (roff[mid] <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ bool same_signature(int32_t a, int32_t b, const int32_t* __restrict__ row_ptr,
                                               const int32_t* __restrict__ nptr, const uint32_t* __restrict__ nslot) {
    if (row_ptr[a + 1] - row_ptr[a] != row_ptr[b + 1] - row_ptr[b]) return false;
    const int ia = nptr[a], ib = nptr[b], n = nptr[a + 1] - ia;
    if (nptr[b + 1] - ib != n) return false;
    for (int i = 0; i < n; i++)
        if (__ldg(nslot + ia + i) != __ldg(nslot + ib + i)) return false;
    return true;
}

// pass 1: rows of small runs and rows whose signature differs from their run's
// first row (hash collision) get the mixed key
__global__ void cls_demote_k(int64_t nn, const uint64_t* __restrict__ skeys, const int32_t* __restrict__ srows,
                             const int32_t* __restrict__ rcnt, const int* __restrict__ nruns_p,
                             const int32_t* __restrict__ roff, const int32_t* __restrict__ row_ptr,
                             const int32_t* __restrict__ nptr, const uint32_t* __restrict__ nslot,
                             uint64_t* __restrict__ keys2, int32_t* __restrict__ rows2) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn) return;
    uint64_t k = skeys[i];
    const int32_t v = srows[i];
    if (k != MIXED) {
        const int r = run_of(i, roff, *nruns_p);
        if (rcnt[r] < MIN_CLASS || !same_signature(v, srows[roff[r]], row_ptr, nptr, nslot)) k = MIXED;
    }
    keys2[i] = k;
    rows2[i] = v;
}

// groups per run: ceil(count / 32)
__global__ void cls_ngroups_k(const int* __restrict__ nruns_p, const int32_t* __restrict__ rcnt,
                              int32_t* __restrict__ ng, int64_t cap) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= cap) return;
    ng[r] = r < *nruns_p ? (rcnt[r] + 31) / 32 : 0;
}

// one thread per sorted position that starts a group
__global__ void cls_groups_k(int64_t nn, const uint64_t* __restrict__ skeys, const int32_t* __restrict__ srows,
                             const int* __restrict__ nruns_p, const int32_t* __restrict__ roff,
                             const int32_t* __restrict__ rcnt, const int32_t* __restrict__ gofs,
                             int4* __restrict__ groups, int64_t gcap) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn) return;
    const int r = run_of(i, roff, *nruns_p);
    const int64_t j = i - roff[r];
    if (j % 32) return;
    const int64_t g = gofs[r] + j / 32;
    if (g >= gcap) return;
    const int cnt = rcnt[r] - j < 32 ? (int)(rcnt[r] - j) : 32;
    groups[g] = make_int4((int)i, cnt, skeys[i] == MIXED ? -1 : srows[roff[r]], 0);
}

// stats: [0] groups, [1] classes (runs with a class key), [2] rows in classes,
// [3] longest row in a class
__global__ void cls_stats_k(const int* __restrict__ nruns_p, const uint64_t* __restrict__ ukeys,
                            const int32_t* __restrict__ rcnt, const int32_t* __restrict__ gofs,
                            const int32_t* __restrict__ roff, const int32_t* __restrict__ srows,
                            const int32_t* __restrict__ row_ptr, int64_t* __restrict__ out) {
    const int nr = *nruns_p;
    if (threadIdx.x == 0) {
        out[0] = gofs[nr];
        const bool mixed_last = nr > 0 && ukeys[nr - 1] == MIXED;
        out[1] = nr - (mixed_last ? 1 : 0);
        int64_t rows = 0, lmax = 0;
        for (int r = 0; r < nr - (mixed_last ? 1 : 0); r++) {
            rows += rcnt[r];
            const int32_t v = srows[roff[r]];
            const int64_t L = row_ptr[v + 1] - row_ptr[v];
            lmax = L > lmax ? L : lmax;
        }
        out[2] = rows;
        out[3] = lmax;
    }
}

struct ClsWork {
    uint64_t *k1, *k2, *uk;
    int32_t *r1, *r2, *cnt, *roff, *ng, *gofs;
    int* nruns;
    int64_t* stats;
    void* cub;
    size_t cub_bytes;
    void* scan;
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t cls_layout(int64_t nn, char* base, ClsWork* w) {
    size_t cub_sort = 0, cub_rle = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, cub_sort, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, (int)nn);
    cub::DeviceRunLengthEncode::Encode(nullptr, cub_rle, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                       (int32_t*)nullptr, (int*)nullptr, (int)nn);
    const size_t cubb = cub_sort > cub_rle ? cub_sort : cub_rle;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* p = base ? base + off : nullptr;
        off += align256(bytes);
        return p;
    };
    ClsWork W{};
    W.k1 = (uint64_t*)take(8 * nn);
    W.k2 = (uint64_t*)take(8 * nn);
    W.uk = (uint64_t*)take(8 * nn);
    W.r1 = (int32_t*)take(4 * nn);
    W.r2 = (int32_t*)take(4 * nn);
    W.cnt = (int32_t*)take(4 * nn);
    W.roff = (int32_t*)take(4 * (nn + 1));
    W.ng = (int32_t*)take(4 * nn);
    W.gofs = (int32_t*)take(4 * (nn + 1));
    W.nruns = (int*)take(8);
    W.stats = (int64_t*)take(8 * 4);
    W.cub = take(cubb);
    W.cub_bytes = cubb;
    W.scan = take(scan_tmp_bytes(nn));
    if (w) *w = W;
    return off;
}

// sort (keys, rows) and run-length encode the sorted keys: runs -> uk, cnt, roff
vb_status sort_rle(const ClsWork& W, int64_t nn, const uint64_t* kin, const int32_t* rin, uint64_t* kout,
                   int32_t* rout, cudaStream_t s, const char* fn) {
    size_t b = W.cub_bytes;
    if (cub::DeviceRadixSort::SortPairs(W.cub, b, kin, kout, rin, rout, (int)nn, 0, 64, s) != cudaSuccess) {
        set_error("%s: radix sort failed", fn);
        return VB_ERR_CUDA;
    }
    b = W.cub_bytes;
    if (cub::DeviceRunLengthEncode::Encode(W.cub, b, kout, W.uk, W.cnt, W.nruns, (int)nn, s) != cudaSuccess) {
        set_error("%s: run-length encode failed", fn);
        return VB_ERR_CUDA;
    }
    cls_ngroups_k<<<grid_for(nn, 256, 8, 64), 256, 0, s>>>(W.nruns, W.cnt, W.ng, nn);   // reused below for offsets
    return launch_check(fn);
}

}  // namespace
}  // namespace vb

using namespace vb;

extern "C" vb_status fem_plan_classes(int dim, int64_t nn, const int32_t* row_ptr, const int32_t* node_elem_ptr,
                                      const uint32_t* node_elem_slot, void* work, size_t* work_bytes,
                                      int32_t* class_rows, int32_t* groups, int64_t groups_cap,
                                      int64_t* stats_out, vb_stream_t stream) {
    const char* fn = "fem_plan_classes";
    clear_error();
    if (dim != 2 && dim != 3) { set_error("%s: dim=%d, need 2 or 3", fn, dim); return VB_ERR_UNSUPPORTED; }
    if (nn < 0 || !work_bytes) { set_error("%s: bad size or NULL work_bytes", fn); return VB_ERR_ARG; }
    if (nn >= (int64_t)1 << 30) { set_error("%s: nn=%lld too large", fn, (long long)nn); return VB_ERR_OVERFLOW; }
    const int64_t n1 = nn > 0 ? nn : 1;
    const size_t need = cls_layout(n1, nullptr, nullptr);
    if (!work) { *work_bytes = need; return VB_OK; }
    if (*work_bytes < need) { set_error("%s: work %zu < %zu bytes", fn, *work_bytes, need); return VB_ERR_WORKSPACE; }
    if (!row_ptr || !node_elem_ptr || !node_elem_slot || !class_rows || !groups || !stats_out) {
        set_error("%s: NULL argument", fn);
        return VB_ERR_ARG;
    }
    if (nn == 0) {
        stats_out[0] = stats_out[1] = stats_out[2] = stats_out[3] = 0;
        return VB_OK;
    }
    cudaStream_t s = cs(stream);
    ClsWork W;
    cls_layout(n1, static_cast<char*>(work), &W);
    const int maxl = dim == 3 ? 15 : 12;  // widest edge-vector buffer of assemble_class_k (columns per row)
    const int maxn = dim == 3 ? 32 : 16;  // its decoded plan-word table (incidences per row)
    const unsigned g = (unsigned)((nn + 255) / 256);
    vb_status st;
    cls_hash_k<<<g, 256, 0, s>>>(nn, row_ptr, node_elem_ptr, node_elem_slot, maxl, maxn, W.k1, W.r1);
    if ((st = launch_check(fn)) != VB_OK) return st;
    if ((st = sort_rle(W, nn, W.k1, W.r1, W.k2, W.r2, s, fn)) != VB_OK) return st;
    if ((st = exclusive_scan_i32(W.cnt, W.roff, nn, W.scan, s, nullptr)) != VB_OK) return st;
    cls_demote_k<<<g, 256, 0, s>>>(nn, W.k2, W.r2, W.cnt, W.nruns, W.roff, row_ptr, node_elem_ptr, node_elem_slot,
                                   W.k1, W.r1);
    if ((st = launch_check(fn)) != VB_OK) return st;
    // second pass: the mixed rows (largest key) end up last, in ascending row order
    if ((st = sort_rle(W, nn, W.k1, W.r1, W.k2, class_rows, s, fn)) != VB_OK) return st;
    if ((st = exclusive_scan_i32(W.cnt, W.roff, nn, W.scan, s, nullptr)) != VB_OK) return st;
    if ((st = exclusive_scan_i32(W.ng, W.gofs, nn, W.scan, s, nullptr)) != VB_OK) return st;
    cls_groups_k<<<g, 256, 0, s>>>(nn, W.k2, class_rows, W.nruns, W.roff, W.cnt, W.gofs,
                                   reinterpret_cast<int4*>(groups), groups_cap);
    if ((st = launch_check(fn)) != VB_OK) return st;
    cls_stats_k<<<1, 32, 0, s>>>(W.nruns, W.uk, W.cnt, W.gofs, W.roff, class_rows, row_ptr, W.stats);
    if ((st = launch_check(fn)) != VB_OK) return st;
    if ((st = read_small(s, W.stats, 4 * sizeof(int64_t), stats_out, fn)) != VB_OK) return st;
    if (stats_out[0] > groups_cap) {
        set_error("%s: %lld groups, groups_cap %lld", fn, (long long)stats_out[0], (long long)groups_cap);
        return VB_ERR_WORKSPACE;
    }
    return VB_OK;
}
