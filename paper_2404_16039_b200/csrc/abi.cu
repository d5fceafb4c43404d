// ABI glue: error reporting, device queries and the device-wide scan used by
// the pattern build ("built once on the GPU by sort/unique/scan").
#include <atomic>
#include <cstdarg>
#include <cstring>

#include "vb_internal.cuh"

namespace vb {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
void clear_error() { g_err[0] = 0; }

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cached[dev] = n;
    }
    return cached[dev];
}

// ------------------------------------------------------------------ small read-backs
namespace {
__global__ void read_small_k(const unsigned char* __restrict__ src, unsigned char* dst, int bytes) {
    for (int i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}
// One 4 KB pinned, mapped host buffer per device (64 slots of 64 bytes, taken and returned
// with an atomic bitmap), allocated on first use and freed at process exit: the only
// allocation of the library, bounded (not per host thread).  With all 64 slots busy a
// read-back falls back to a plain copy.
constexpr int RS_SLOTS = 64;
struct MappedPool {
    unsigned char* h = nullptr;
    unsigned char* d = nullptr;
    std::atomic<unsigned long long> busy{0};
    std::atomic<int> state{0};   // 0 none, 1 initialising, 2 ready, 3 unavailable
    ~MappedPool() {
        if (h) cudaFreeHost(h);   // best effort at exit (the context may already be gone)
    }
};
MappedPool g_pool[16];

int take_slot(MappedPool& P) {
    unsigned long long b = P.busy.load();
    while (~b) {
        const int i = __builtin_ctzll(~b);
        if (P.busy.compare_exchange_weak(b, b | (1ull << i))) return i;
    }
    return -1;
}
}  // namespace

vb_status read_small(cudaStream_t s, const void* src, size_t bytes, void* dst, const char* fn) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (bytes > 64) { set_error("%s: read_small of %zu bytes", fn, bytes); return VB_ERR_ARG; }
    MappedPool* P = (dev >= 0 && dev < 16) ? &g_pool[dev] : nullptr;
    if (P) {
        int st = P->state.load();
        if (st == 0 && P->state.compare_exchange_strong(st, 1)) {
            if (cudaHostAlloc((void**)&P->h, 64 * RS_SLOTS, cudaHostAllocMapped) != cudaSuccess ||
                cudaHostGetDevicePointer((void**)&P->d, P->h, 0) != cudaSuccess) {
                cudaGetLastError();
                if (P->h) cudaFreeHost(P->h);
                P->h = P->d = nullptr;
                P->state.store(3);
            } else {
                P->state.store(2);
            }
        }
        while (P->state.load() == 1) {
        }
    }
    const int slot = (P && P->state.load() == 2) ? take_slot(*P) : -1;
    cudaError_t e;
    if (slot >= 0) {
        read_small_k<<<1, 32, 0, s>>>(static_cast<const unsigned char*>(src), P->d + 64 * slot, (int)bytes);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e == cudaSuccess) memcpy(dst, (const void*)(P->h + 64 * slot), bytes);
        P->busy.fetch_and(~(1ull << slot));
    } else {   // no mapped memory (or all slots busy): plain copy
        e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    }
    if (e != cudaSuccess) { set_error("%s: %s", fn, cudaGetErrorString(e)); return VB_ERR_CUDA; }
    return VB_OK;
}

// ------------------------------------------------------------------ scan
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ long long block_sum_ll(long long v, long long* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    long long t = 0;
    if (threadIdx.x < 32) {
        t = (l < (int)(blockDim.x >> 5)) ? sh[l] : 0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    __syncthreads();
    return t;  // valid in thread 0
}

// exclusive scan of v across the block; returns the block total in *tot
__device__ __forceinline__ long long block_exscan_ll(long long v, long long* sh, long long* tot) {
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (l >= o) x += y;
    }
    if (l == 31) sh[w] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
        int nw = blockDim.x >> 5;
        long long s = (l < nw) ? sh[l] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(0xffffffffu, s, o);
            if (l >= o) s += y;
        }
        sh[32 + l] = s;  // inclusive scan of warp sums
    }
    __syncthreads();
    long long warp_off = (w > 0) ? sh[32 + w - 1] : 0;
    *tot = sh[32 + (blockDim.x >> 5) - 1];
    __syncthreads();
    return warp_off + x - v;
}

__global__ void scan_reduce_k(const int32_t* __restrict__ in, int64_t n, long long* __restrict__ part) {
    __shared__ long long sh[64];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    long long s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
        int64_t idx = base + (int64_t)i * SCAN_THREADS + threadIdx.x;
        if (idx < n) s += in[idx];
    }
    long long t = block_sum_ll(s, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void scan_partials_k(long long* __restrict__ part, int64_t nb, int64_t* __restrict__ total) {
    __shared__ long long sh[64];
    long long carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += blockDim.x) {
        int64_t i = b0 + threadIdx.x;
        long long v = (i < nb) ? part[i] : 0;
        long long tot;
        long long ex = block_exscan_ll(v, sh, &tot);
        if (i < nb) part[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void scan_down_k(const int32_t* __restrict__ in, int32_t* __restrict__ out, int64_t n,
                            const long long* __restrict__ part) {
    __shared__ long long sh[64];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int32_t v[SCAN_ITEMS];
    long long s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
        int64_t idx = base + i;
        v[i] = (idx < n) ? in[idx] : 0;
        s += v[i];
    }
    long long tot;
    long long off = part[blockIdx.x] + block_exscan_ll(s, sh, &tot);
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
        int64_t idx = base + i;
        if (idx < n) out[idx] = (int32_t)off;
        off += v[i];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = (int32_t)(part[blockIdx.x] + tot);
}

size_t scan_tmp_bytes(int64_t n) {
    int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (nb < 1) nb = 1;
    return (size_t)(nb * sizeof(long long) + 256) & ~(size_t)255;
}

vb_status exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, void* tmp, cudaStream_t s,
                             int64_t* total_dev) {
    int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (nb < 1) nb = 1;
    long long* part = reinterpret_cast<long long*>(tmp);
    scan_reduce_k<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, n, part);
    scan_partials_k<<<1, 1024, 0, s>>>(part, nb, total_dev);
    scan_down_k<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, out, n, part);
    return launch_check("exclusive_scan");
}

}  // namespace vb

extern "C" const char* vb_last_error(void) { return vb::g_err; }
extern "C" int vb_abi_version(void) { return 2; }
