// a6: fused surface geometry over a triangulated closed surface (config 3):
// gather the three vertices of each face, n = (b-a) x (c-a), |n|, nhat, area,
// and the divergence-theorem volume sum (1/6) sum a.n reduced with
// a fixed-shape tree (block partials in a fixed grid, then one block) so the
// volume is bitwise reproducible.
#include "vb_internal.cuh"

namespace vb {
namespace {

constexpr int SURF_BLOCK = 256;
constexpr int SURF_BLOCKS_PER_SM = 8;

__global__ void __launch_bounds__(SURF_BLOCK) tri_surface_k(int64_t nf, const int32_t* __restrict__ tri, int64_t tld,
                                                            const double* __restrict__ xyz, int64_t ns, int64_t cst,
                                                            double* __restrict__ n_out, double* __restrict__ nh_out,
                                                            double* __restrict__ area, double* __restrict__ part) {
    double vol = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += stride) {
        int64_t ia = __ldcs(tri + f), ib = __ldcs(tri + tld + f), ic = __ldcs(tri + 2 * tld + f);
        double a[3], u[3], w[3];
#pragma unroll
        for (int d = 0; d < 3; d++) {
            a[d] = __ldg(xyz + d * cst + ia * ns);
            u[d] = __ldg(xyz + d * cst + ib * ns) - a[d];
            w[d] = __ldg(xyz + d * cst + ic * ns) - a[d];
        }
        double n0 = fma(u[1], w[2], -u[2] * w[1]);
        double n1 = fma(u[2], w[0], -u[0] * w[2]);
        double n2 = fma(u[0], w[1], -u[1] * w[0]);
        double len = sqrt(fma(n0, n0, fma(n1, n1, n2 * n2)));
        if (n_out) {
            stcs(n_out + f, n0);
            stcs(n_out + nf + f, n1);
            stcs(n_out + 2 * nf + f, n2);
        }
        if (nh_out) {
            double r = 1.0 / len;
            stcs(nh_out + f, n0 * r);
            stcs(nh_out + nf + f, n1 * r);
            stcs(nh_out + 2 * nf + f, n2 * r);
        }
        if (area) stcs(area + f, 0.5 * len);
        vol += fma(a[0], n0, fma(a[1], n1, a[2] * n2));
    }
    if (part) {
        __shared__ double sh[SURF_BLOCK / 32];
        for (int o = 16; o > 0; o >>= 1) vol += __shfl_xor_sync(0xffffffffu, vol, o);
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = vol;
        __syncthreads();
        if (threadIdx.x < 32) {
            double t = (threadIdx.x < SURF_BLOCK / 32) ? sh[threadIdx.x] : 0.0;
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (threadIdx.x == 0) part[blockIdx.x] = t;
        }
    }
}

// the same, two consecutive faces per thread: index pairs loaded as int2, every output plane written with
// 128-bit stores, both faces' 18 gathers in flight together (nf even, planes 16-byte aligned)
#ifndef VB_SURF_MINB
#define VB_SURF_MINB 4   // 64 registers (12 bytes of spills): 32 warps per SM; 3: 0.345 ms, 4: 0.323 ms, 5: 0.384 ms on configs[2]
#endif
__global__ void __launch_bounds__(SURF_BLOCK, VB_SURF_MINB) tri_surface2_k(int64_t nf, const int32_t* __restrict__ tri, int64_t tld,
                                                             const double* __restrict__ xyz, int64_t ns, int64_t cst,
                                                             double* __restrict__ n_out, double* __restrict__ nh_out,
                                                             double* __restrict__ area, double* __restrict__ part) {
    double vol = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t npair = nf / 2;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < npair; t += stride) {
        const int64_t f = 2 * t;
        const int2 ia = __ldcs(reinterpret_cast<const int2*>(tri + f));
        const int2 ib = __ldcs(reinterpret_cast<const int2*>(tri + tld + f));
        const int2 ic = __ldcs(reinterpret_cast<const int2*>(tri + 2 * tld + f));
        const int64_t va[2] = {ia.x, ia.y}, vb_[2] = {ib.x, ib.y}, vc[2] = {ic.x, ic.y};
        double a[2][3], u[2][3], w[2][3];
#pragma unroll
        for (int k = 0; k < 2; k++)
#pragma unroll
            for (int d = 0; d < 3; d++) {
                a[k][d] = __ldg(xyz + d * cst + va[k] * ns);
                u[k][d] = __ldg(xyz + d * cst + vb_[k] * ns);
                w[k][d] = __ldg(xyz + d * cst + vc[k] * ns);
            }
        double nn[2][3], len[2];
#pragma unroll
        for (int k = 0; k < 2; k++) {
#pragma unroll
            for (int d = 0; d < 3; d++) {
                u[k][d] -= a[k][d];
                w[k][d] -= a[k][d];
            }
            nn[k][0] = fma(u[k][1], w[k][2], -u[k][2] * w[k][1]);
            nn[k][1] = fma(u[k][2], w[k][0], -u[k][0] * w[k][2]);
            nn[k][2] = fma(u[k][0], w[k][1], -u[k][1] * w[k][0]);
            len[k] = sqrt(fma(nn[k][0], nn[k][0], fma(nn[k][1], nn[k][1], nn[k][2] * nn[k][2])));
            vol += fma(a[k][0], nn[k][0], fma(a[k][1], nn[k][1], a[k][2] * nn[k][2]));
        }
        if (n_out) {
#pragma unroll
            for (int d = 0; d < 3; d++) stcs2(n_out + d * nf + f, make_double2(nn[0][d], nn[1][d]));
        }
        if (nh_out) {
            const double r0 = 1.0 / len[0], r1 = 1.0 / len[1];
#pragma unroll
            for (int d = 0; d < 3; d++) stcs2(nh_out + d * nf + f, make_double2(nn[0][d] * r0, nn[1][d] * r1));
        }
        if (area) stcs2(area + f, make_double2(0.5 * len[0], 0.5 * len[1]));
    }
    if (part) {
        __shared__ double sh[SURF_BLOCK / 32];
        for (int o = 16; o > 0; o >>= 1) vol += __shfl_xor_sync(0xffffffffu, vol, o);
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = vol;
        __syncthreads();
        if (threadIdx.x < 32) {
            double t = (threadIdx.x < SURF_BLOCK / 32) ? sh[threadIdx.x] : 0.0;
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (threadIdx.x == 0) part[blockIdx.x] = t;
        }
    }
}

__global__ void __launch_bounds__(1024) sum_parts_k(const double* __restrict__ part, int n, double* __restrict__ out) {
    __shared__ double sh[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = sh[threadIdx.x];
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) *out = t / 6.0;
    }
}

// NEXT-4: Code GI: value = sum_e sizes_e g_e with g_e = sum_c
// f_e(c) normals_e(c) (or f_e(0)) and f_e(c) = sum_q w_q fip(c, q, e) (amsv).
// One thread per page (grid-stride, streaming loads), the same fixed-shape
// reduction as the surface volume (bitwise reproducible).
constexpr int GI_MAXQ = 16;
struct GIW {
    double w[GI_MAXQ];
};

// D, Q > 0: compile-time shape (every load of a page issued before the arithmetic);
// 0: runtime d / nip
template <int D, int Q>
__global__ void __launch_bounds__(SURF_BLOCK) gi_k(int64_t ne, int d, int nip, const double* __restrict__ fip,
                                                   int64_t ld, GIW w, const double* __restrict__ sizes,
                                                   const double* __restrict__ normals, int64_t nld,
                                                   double* __restrict__ part) {
    double acc = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if constexpr (D > 0 && Q > 0) {
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += stride) {
            double v[D][Q], nv[D];
#pragma unroll
            for (int c = 0; c < D; c++)
#pragma unroll
                for (int q = 0; q < Q; q++) v[c][q] = __ldcs(fip + (int64_t)(c + q * D) * ld + e);
            if (normals)
#pragma unroll
                for (int c = 0; c < D; c++) nv[c] = __ldcs(normals + c * nld + e);
            const double sz = __ldcs(sizes + e);
            double g = 0.0;
#pragma unroll
            for (int c = 0; c < D; c++) {
                double f = 0.0;
#pragma unroll
                for (int q = 0; q < Q; q++) f = fma(v[c][q], w.w[q], f);
                g = normals ? fma(f, nv[c], g) : f;
            }
            acc = fma(sz, g, acc);
        }
    } else {
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += stride) {
            double g = 0.0;
            for (int c = 0; c < d; c++) {
                double f = 0.0;
                for (int q = 0; q < nip; q++) f = fma(__ldcs(fip + (int64_t)(c + q * d) * ld + e), w.w[q], f);
                g = normals ? fma(f, __ldcs(normals + c * nld + e), g) : f;
            }
            acc = fma(__ldcs(sizes + e), g, acc);
        }
    }
    __shared__ double sh[SURF_BLOCK / 32];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = (threadIdx.x < SURF_BLOCK / 32) ? sh[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) part[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) gi_sum_k(const double* __restrict__ part, int n, double* __restrict__ out) {
    __shared__ double sh[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = sh[threadIdx.x];
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) *out = t;
    }
}

}  // namespace
}  // namespace vb

using namespace vb;

extern "C" vb_status vb_gi(int64_t npages, int d, int nip, const double* fip, int64_t ldf, const double* w,
                           const double* sizes, const double* normals, int64_t ldn, double* value, void* work,
                           size_t* work_bytes, vb_stream_t stream) {
    const char* fn = "vb_gi";
    clear_error();
    if (npages < 0) { set_error("%s: negative npages", fn); return VB_ERR_ARG; }
    if (d < 1 || d > 4) { set_error("%s: d=%d, need 1..4", fn, d); return VB_ERR_UNSUPPORTED; }
    if (nip < 1 || nip > GI_MAXQ) { set_error("%s: nip=%d, need 1..%d", fn, nip, GI_MAXQ); return VB_ERR_UNSUPPORTED; }
    const unsigned g = grid_for(npages, SURF_BLOCK, SURF_BLOCKS_PER_SM);
    const size_t need = ((size_t)g * sizeof(double) + 255) & ~(size_t)255;
    if (!work) {   // size query: needs only npages
        if (!work_bytes) { set_error("%s: work and work_bytes both NULL", fn); return VB_ERR_ARG; }
        *work_bytes = need;
        return VB_OK;
    }
    if (!normals && d != 1) { set_error("%s: d=%d needs normals (a vector field is integrated against them)", fn, d); return VB_ERR_DIM; }
    if (work_bytes && *work_bytes < need) { set_error("%s: work buffer too small (%zu < %zu)", fn, *work_bytes, need); return VB_ERR_WORKSPACE; }
    if (!value || !w) { set_error("%s: NULL value or w", fn); return VB_ERR_ARG; }
    if (npages > 0 && (!fip || !sizes)) { set_error("%s: NULL fip or sizes", fn); return VB_ERR_ARG; }
    if (ldf < npages || (normals && ldn < npages)) { set_error("%s: leading dimension < npages", fn); return VB_ERR_ARG; }
    auto s = cs(stream);
    if (npages == 0) {
        cudaMemsetAsync(value, 0, sizeof(double), s);
        return launch_check(fn);
    }
    GIW ww{};
    for (int q = 0; q < nip; q++) ww.w[q] = w[q];
    double* part = reinterpret_cast<double*>(work);
    auto k = gi_k<0, 0>;   // the shapes of the paper's integrals: scalar densities at 1 / 3 / 4 points, fields at 1
    if (d == 1 && nip == 1) k = gi_k<1, 1>;
    else if (d == 1 && nip == 3) k = gi_k<1, 3>;
    else if (d == 1 && nip == 4) k = gi_k<1, 4>;
    else if (d == 3 && nip == 1) k = gi_k<3, 1>;
    else if (d == 2 && nip == 1) k = gi_k<2, 1>;
    k<<<g, SURF_BLOCK, 0, s>>>(npages, d, nip, fip, ldf, ww, sizes, normals, ldn, part);
    gi_sum_k<<<1, 1024, 0, s>>>(part, (int)g, value);
    return launch_check(fn);
}

extern "C" vb_status vb_tri_surface(int64_t nf, const int32_t* tri, int64_t tri_ld, int64_t nverts, const double* xyz,
                                    int64_t node_stride, int64_t comp_stride, double* n, double* nhat, double* area,
                                    double* volume, void* work, size_t* work_bytes, vb_stream_t stream) {
    clear_error();
    if (nf < 0 || nverts < 0) { set_error("vb_tri_surface: negative size"); return VB_ERR_ARG; }
    unsigned g = grid_for(nf, SURF_BLOCK, SURF_BLOCKS_PER_SM);
    size_t need = volume ? ((size_t)g * sizeof(double) + 255) & ~(size_t)255 : 0;
    if (!work) {
        if (!work_bytes) { set_error("vb_tri_surface: work and work_bytes both NULL"); return VB_ERR_ARG; }
        *work_bytes = need;
        return VB_OK;
    }
    if (work_bytes && *work_bytes < need) { set_error("vb_tri_surface: work buffer too small (%zu < %zu)", *work_bytes, need); return VB_ERR_WORKSPACE; }
    if (nf > 0 && (!tri || !xyz)) { set_error("vb_tri_surface: NULL %s", !tri ? "tri" : "xyz"); return VB_ERR_ARG; }
    if (tri_ld < nf) { set_error("vb_tri_surface: tri_ld < nf"); return VB_ERR_ARG; }
    auto s = cs(stream);
    double* part = volume ? reinterpret_cast<double*>(work) : nullptr;
    // pairs of faces with 128-bit accesses when every plane allows it (same values; the volume's partial
    // sums group differently, each path bitwise reproducible)
#ifndef VB_SURF_SCALAR
#define VB_SURF_SCALAR 0   // 1: always the one-face-per-thread kernel (A/B timing)
#endif
    const bool vec = !VB_SURF_SCALAR && (nf & 1) == 0 && (tri_ld & 1) == 0 && (reinterpret_cast<uintptr_t>(tri) & 7u) == 0 &&
                     (!n || aligned16(n)) && (!nhat || aligned16(nhat)) && (!area || aligned16(area));
    if (nf > 0 && vec) tri_surface2_k<<<g, SURF_BLOCK, 0, s>>>(nf, tri, tri_ld, xyz, node_stride, comp_stride, n, nhat, area, part);
    else if (nf > 0) tri_surface_k<<<g, SURF_BLOCK, 0, s>>>(nf, tri, tri_ld, xyz, node_stride, comp_stride, n, nhat, area, part);
    if (volume) {
        if (nf == 0) { cudaMemsetAsync(volume, 0, sizeof(double), s); return launch_check("vb_tri_surface"); }
        sum_parts_k<<<1, 1024, 0, s>>>(part, (int)g, volume);
    }
    return launch_check("vb_tri_surface");
}
