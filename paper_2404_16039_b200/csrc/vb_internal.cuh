// Internal helpers shared by the libvb.so translation units (never by oracle/).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../../include/vb.h"

namespace vb {

// thread-local last-error message (vb_last_error)
void set_error(const char* fmt, ...);
void clear_error();

inline cudaStream_t cs(vb_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// SM count of the current device (cached per process; B200: 148).
int sm_count();

// Check the launch that was just enqueued.
inline vb_status launch_check(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: CUDA launch failed: %s", what, cudaGetErrorString(e));
        return VB_ERR_CUDA;
    }
    return VB_OK;
}

// Read `bytes` (<= 64) of device memory into host memory: enqueued on `s`, then
// synchronises `s`.  Goes through a small mapped pinned buffer written by a
// one-thread kernel, so the read-back never waits in a copy-engine queue behind
// large async copies that other streams have in flight (a pageable
// cudaMemcpyAsync would).  Returns VB_ERR_CUDA (message set) on failure.
vb_status read_small(cudaStream_t s, const void* src, size_t bytes, void* dst, const char* fn);

// Grid for a grid-stride kernel over `units` work items of `block` threads:
// never more than `waves` full waves of resident blocks.
inline unsigned grid_for(int64_t units, int block, int blocks_per_sm, int waves = 1) {
    int64_t need = (units + block - 1) / block;
    int64_t cap = (int64_t)sm_count() * blocks_per_sm * waves;
    if (need < 1) need = 1;
    return (unsigned)(need < cap ? need : cap);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Device-side bounds checks, compiled in only for the debug variant
// (tools/build_variant.py debug -DVB_DEBUG_BOUNDS): a failed check traps.
#ifdef VB_DEBUG_BOUNDS
#define VB_CHECK(cond)      \
    do {                    \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define VB_CHECK(cond) \
    do {               \
    } while (0)
#endif

// streaming (evict-first) loads/stores for data touched once
__device__ __forceinline__ double ldcs(const double* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ldcs2(const double* p) { return __ldcs(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ void stcs(double* p, double v) { __stcs(p, v); }
__device__ __forceinline__ void stcs2(double* p, double2 v) { __stcs(reinterpret_cast<double2*>(p), v); }

// device-wide exclusive scan of int32 counts (n values) into out (n+1 values:
// out[n] = total).  Uses `tmp` of scan_tmp_bytes(n).  Deterministic.
size_t scan_tmp_bytes(int64_t n);
vb_status exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, void* tmp, cudaStream_t s,
                             int64_t* total_dev /* optional: int64 total (overflow-safe) */);

}  // namespace vb
