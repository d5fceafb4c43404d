// NEXT-2: P1 load vector (Code rhs_vectorP1) and the page-wise
// bilinear form avtamav (eq:layeredBilin P:292-301) used for the
// element energies J_{i,k}.
#include "vb_internal.cuh"

namespace vb {
namespace {

// intquad(gqo, dim) in barycentric form: gqo = 1 centroid, gqo = 2 the
// symmetric degree-2 rules (point q = ALPHA at vertex q, BETA elsewhere)
// (reading: DESIGN.md §4).
struct Rule {
    int nip;
    double lam[4][4];
    double w[4];
};

bool make_rule(int dim, int gqo, Rule& R) {
    const int nv = dim + 1;
    const double dfact = dim == 2 ? 2.0 : (dim == 3 ? 6.0 : 1.0);
    if (gqo == 1) {
        R.nip = 1;
        for (int a = 0; a < nv; a++) R.lam[0][a] = 1.0 / nv;
        R.w[0] = 1.0 / dfact;
        return true;
    }
    if (gqo == 2 && (dim == 2 || dim == 3)) {
        const double al = dim == 2 ? 2.0 / 3.0 : 0.58541019662496845446;
        const double be = dim == 2 ? 1.0 / 6.0 : 0.13819660112501051518;
        R.nip = nv;
        for (int q = 0; q < nv; q++) {
            for (int a = 0; a < nv; a++) R.lam[q][a] = a == q ? al : be;
            R.w[q] = 1.0 / (dfact * nv);
        }
        return true;
    }
    return false;
}

template <int DIM>
__device__ __forceinline__ void rhs_elem(int64_t e, int64_t ne, const double* __restrict__ coords, int64_t ns,
                                         int64_t cst, const int32_t* __restrict__ elems, int64_t eld,
                                         const double* __restrict__ fq, const Rule& R, double* __restrict__ b2D,
                                         double* __restrict__ b) {
    constexpr int NV = DIM + 1;
    {
        // the streamed f values first: in flight while the vertex gather (elems -> coords) runs
        double fv[NV];
#pragma unroll
        for (int i = 0; i < NV; i++) fv[i] = i < R.nip ? __ldcs(fq + (int64_t)i * ne + e) : 0.0;
        int32_t vid[NV];
        double x[NV][DIM];
#pragma unroll
        for (int a = 0; a < NV; a++) {
            vid[a] = __ldg(elems + a * eld + e);
#pragma unroll
            for (int c = 0; c < DIM; c++) x[a][c] = __ldg(coords + c * cst + (int64_t)vid[a] * ns);
        }
        double det;
        if constexpr (DIM == 2) {
            det = fma(x[1][0] - x[0][0], x[2][1] - x[0][1], -(x[1][1] - x[0][1]) * (x[2][0] - x[0][0]));
        } else {
            double J[3][3];
#pragma unroll
            for (int r = 0; r < 3; r++)
#pragma unroll
                for (int c = 0; c < 3; c++) J[r][c] = x[r + 1][c] - x[0][c];
            det = J[0][0] * fma(J[1][1], J[2][2], -J[1][2] * J[2][1]) +
                  J[0][1] * fma(J[1][2], J[2][0], -J[1][0] * J[2][2]) +
                  J[0][2] * fma(J[1][0], J[2][1], -J[1][1] * J[2][0]);
        }
        const double ad = fabs(det);
        double loc[NV];
#pragma unroll
        for (int a = 0; a < NV; a++) loc[a] = 0.0;
#pragma unroll
        for (int i = 0; i < NV; i++) {
            if (i >= R.nip) break;
            const double fw = R.w[i] * ad * fv[i];
#pragma unroll
            for (int a = 0; a < NV; a++) loc[a] = fma(fw, R.lam[i][a], loc[a]);
        }
#pragma unroll
        for (int a = 0; a < NV; a++) {
            if (b2D) stcs(b2D + (int64_t)a * ne + e, loc[a]);
            if (b) atomicAdd(b + vid[a], loc[a]);
        }
    }
}

// two elements per thread and step: both elements' loads in flight together
template <int DIM>
__global__ void __launch_bounds__(256) rhs_elem_k(int64_t ne, const double* __restrict__ coords, int64_t ns, int64_t cst,
                                                  const int32_t* __restrict__ elems, int64_t eld,
                                                  const double* __restrict__ fq, const Rule R, double* __restrict__ b2D,
                                                  double* __restrict__ b) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += 2 * stride) {
        rhs_elem<DIM>(e, ne, coords, ns, cst, elems, eld, fq, R, b2D, b);
        if (e + stride < ne) rhs_elem<DIM>(e + stride, ne, coords, ns, cst, elems, eld, fq, R, b2D, b);
    }
}

// The same for two ADJACENT elements per thread (ne even, planes 16-byte aligned): index pairs as int2, f and
// b2D planes with 128-bit accesses, both elements' gathers in flight together.
#ifndef VB_RHS_MINB
#define VB_RHS_MINB 3   // config-5 rhs: 2 blocks 0.339 ms, 3: 0.319, 4 (64 registers, spills): 0.321; scalar kernel 0.371
#endif
template <int DIM>
__global__ void __launch_bounds__(256, VB_RHS_MINB) rhs_elem2_k(int64_t ne, const double* __restrict__ coords, int64_t ns,
                                                      int64_t cst, const int32_t* __restrict__ elems, int64_t eld,
                                                      const double* __restrict__ fq, const Rule R,
                                                      double* __restrict__ b2D, double* __restrict__ b) {
    constexpr int NV = DIM + 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t npair = ne / 2;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < npair; t += stride) {
        const int64_t e = 2 * t;
        double fv[2][NV];
#pragma unroll
        for (int i = 0; i < NV; i++) {
            const double2 f2 = i < R.nip ? ldcs2(fq + (int64_t)i * ne + e) : make_double2(0.0, 0.0);
            fv[0][i] = f2.x;
            fv[1][i] = f2.y;
        }
        int32_t vid[2][NV];
#pragma unroll
        for (int a = 0; a < NV; a++) {
            const int2 p = __ldg(reinterpret_cast<const int2*>(elems + a * eld + e));
            vid[0][a] = p.x;
            vid[1][a] = p.y;
        }
        double x[2][NV][DIM];
#pragma unroll
        for (int k = 0; k < 2; k++)
#pragma unroll
            for (int a = 0; a < NV; a++)
#pragma unroll
                for (int c = 0; c < DIM; c++) x[k][a][c] = __ldg(coords + c * cst + (int64_t)vid[k][a] * ns);
        double loc[2][NV];
#pragma unroll
        for (int k = 0; k < 2; k++) {
            double det;
            if constexpr (DIM == 2) {
                det = fma(x[k][1][0] - x[k][0][0], x[k][2][1] - x[k][0][1],
                          -(x[k][1][1] - x[k][0][1]) * (x[k][2][0] - x[k][0][0]));
            } else {
                double J[3][3];
#pragma unroll
                for (int r = 0; r < 3; r++)
#pragma unroll
                    for (int c = 0; c < 3; c++) J[r][c] = x[k][r + 1][c] - x[k][0][c];
                det = J[0][0] * fma(J[1][1], J[2][2], -J[1][2] * J[2][1]) +
                      J[0][1] * fma(J[1][2], J[2][0], -J[1][0] * J[2][2]) +
                      J[0][2] * fma(J[1][0], J[2][1], -J[1][1] * J[2][0]);
            }
            const double ad = fabs(det);
#pragma unroll
            for (int a = 0; a < NV; a++) loc[k][a] = 0.0;
#pragma unroll
            for (int i = 0; i < NV; i++) {
                if (i >= R.nip) break;
                const double fw = R.w[i] * ad * fv[k][i];
#pragma unroll
                for (int a = 0; a < NV; a++) loc[k][a] = fma(fw, R.lam[i][a], loc[k][a]);
            }
        }
#pragma unroll
        for (int a = 0; a < NV; a++) {
            if (b2D) stcs2(b2D + (int64_t)a * ne + e, make_double2(loc[0][a], loc[1][a]));
            if (b) {
                atomicAdd(b + vid[0][a], loc[0][a]);
                atomicAdd(b + vid[1][a], loc[1][a]);
            }
        }
    }
}

// accumarray, deterministic: b_v = sum over v's incidences (ascending e) of b2D(a, e)
__global__ void __launch_bounds__(256) rhs_gather_k(int64_t nn, int64_t ne, const int32_t* __restrict__ nptr,
                                                    const int32_t* __restrict__ nelem, const double* __restrict__ b2D,
                                                    double* __restrict__ b) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nn; v += stride) {
        // 8 incidences at a time: their ids, then their values, are loaded before the (ordered) additions
        double s = 0.0;
        for (int i = __ldg(nptr + v), i1 = __ldg(nptr + v + 1); i < i1; i += 8) {
            int32_t ea[8];
            double val[8];
#pragma unroll
            for (int k = 0; k < 8; k++) ea[k] = i + k < i1 ? __ldg(nelem + i + k) : -1;
#pragma unroll
            for (int k = 0; k < 8; k++) val[k] = ea[k] >= 0 ? __ldg(b2D + (int64_t)(ea[k] & 3) * ne + (ea[k] >> 2)) : 0.0;
#pragma unroll
            for (int k = 0; k < 8; k++)
                if (ea[k] >= 0) s += val[k];
        }
        b[v] = s;
    }
}

__global__ void zero_k(double* __restrict__ a, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = 0.0;
}


}  // namespace
}  // namespace vb

using namespace vb;

extern "C" int vb_quad_rule(int dim, int gqo, double* lam, double* w) {
    clear_error();
    Rule R;
    if (!make_rule(dim, gqo, R)) {
        set_error("vb_quad_rule: no rule for dim=%d gqo=%d", dim, gqo);
        return VB_ERR_UNSUPPORTED;
    }
    for (int q = 0; q < R.nip; q++) {
        for (int a = 0; a <= dim; a++)
            if (lam) lam[q * (dim + 1) + a] = R.lam[q][a];
        if (w) w[q] = R.w[q];
    }
    return R.nip;
}

extern "C" vb_status fem_p1_rhs(int dim, int64_t nn, int64_t ne, const double* coords, int64_t node_stride,
                                int64_t comp_stride, const int32_t* elems, int64_t elem_ld, int gqo, const double* fq,
                                double* b2D, double* b, const int32_t* node_elem_ptr, const int32_t* node_elem,
                                int mode, vb_stream_t stream) {
    clear_error();
    if (dim != 2 && dim != 3) { set_error("fem_p1_rhs: dim=%d, need 2 or 3", dim); return VB_ERR_UNSUPPORTED; }
    if (nn < 0 || ne < 0) { set_error("fem_p1_rhs: negative size"); return VB_ERR_ARG; }
    Rule R;
    if (!make_rule(dim, gqo, R)) { set_error("fem_p1_rhs: gqo=%d unsupported", gqo); return VB_ERR_UNSUPPORTED; }
    if (mode != VB_ASSEMBLE_ATOMIC && mode != VB_ASSEMBLE_GATHER) { set_error("fem_p1_rhs: unknown mode %d", mode); return VB_ERR_ARG; }
    if (ne > 0 && (!coords || !elems || !fq)) { set_error("fem_p1_rhs: NULL coords, elems or fq"); return VB_ERR_ARG; }
    if (elem_ld < ne) { set_error("fem_p1_rhs: elem_ld < ne"); return VB_ERR_ARG; }
    if (mode == VB_ASSEMBLE_GATHER && b && (!b2D || !node_elem_ptr || !node_elem)) {
        set_error("fem_p1_rhs: gather mode needs b2D, node_elem_ptr and node_elem");
        return VB_ERR_ARG;
    }
    cudaStream_t s = cs(stream);
    const bool atomic = mode == VB_ASSEMBLE_ATOMIC;
    if (b && atomic && nn > 0) zero_k<<<grid_for(nn, 256, 8), 256, 0, s>>>(b, nn);
    if (ne > 0 && (b2D || (b && atomic))) {
        unsigned g = grid_for(ne, 256, 8);
        double* bb = atomic ? b : nullptr;
#ifndef VB_RHS_SCALAR
#define VB_RHS_SCALAR 0   // 1: always the scalar element kernel (A/B timing)
#endif
        const bool vec = !VB_RHS_SCALAR && (ne & 1) == 0 && (elem_ld & 1) == 0 && (reinterpret_cast<uintptr_t>(elems) & 7u) == 0 &&
                         aligned16(fq) && (!b2D || aligned16(b2D));
        if (vec) {
            g = grid_for(ne / 2, 256, VB_RHS_MINB);
            if (dim == 2) rhs_elem2_k<2><<<g, 256, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, fq, R, b2D, bb);
            else rhs_elem2_k<3><<<g, 256, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, fq, R, b2D, bb);
        } else if (dim == 2) rhs_elem_k<2><<<g, 256, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, fq, R, b2D, bb);
        else rhs_elem_k<3><<<g, 256, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, fq, R, b2D, bb);
    }
    if (b && !atomic && nn > 0)
        rhs_gather_k<<<grid_for(nn, 256, 8), 256, 0, s>>>(nn, ne, node_elem_ptr, node_elem, b2D, b);
    return launch_check("fem_p1_rhs");
}

