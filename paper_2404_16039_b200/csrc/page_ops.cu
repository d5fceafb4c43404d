// Page-wise fp64 kernels: products with
// transposes, transpose, determinant, adjugate inverse, cross product and the
// coords3D gather.  HBM-bound streaming kernels: struct-of-arrays planes, one
// thread per PAIR of pages (128-bit ld/st of two neighbouring pages of a
// plane), pages held in registers, grid-stride over the batch.
#include "vb_internal.cuh"

namespace vb {
namespace {

constexpr int PAGE_BLOCK = 256;
constexpr int PAGE_BLOCKS_PER_SM = 8;  // 2048 threads / SM

// load entry `plane` of pages (p, p+1) into v[0], v[1]
__device__ __forceinline__ void ld_pair(const double* __restrict__ base, int64_t ld, int plane,
                                        int64_t p, int64_t np, bool vec, double& v0, double& v1) {
    if (ld == 0) {  // eq:copy broadcast: one contiguous object
        v0 = v1 = __ldg(base + plane);
        return;
    }
    const double* q = base + (int64_t)plane * ld + p;
    if (vec && p + 1 < np) {
        double2 t = ldcs2(q);
        v0 = t.x;
        v1 = t.y;
    } else {
        v0 = ldcs(q);
        v1 = (p + 1 < np) ? ldcs(q + 1) : 0.0;
    }
}

__device__ __forceinline__ void st_pair(double* __restrict__ base, int64_t ld, int plane, int64_t p,
                                        int64_t np, bool vec, double v0, double v1) {
    double* q = base + (int64_t)plane * ld + p;
    if (vec && p + 1 < np) {
        stcs2(q, make_double2(v0, v1));
    } else {
        stcs(q, v0);
        if (p + 1 < np) stcs(q + 1, v1);
    }
}

// ------------------------------------------------------------ a1 mtimes
// Z_k (M x N) = op(X_k) (M x KK) * op(Y_k) (KK x N); l ascending, fused multiply-add.
template <int M, int KK, int N>
__global__ void __launch_bounds__(PAGE_BLOCK) mtimes_k(int64_t np, const double* __restrict__ X, int64_t ldx, int tX,
                                                       const double* __restrict__ Y, int64_t ldy, int tY,
                                                       double* __restrict__ Z, int64_t ldz, bool vec) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
    for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; p < np; p += stride) {
        double x[M][KK][2], y[KK][N][2];
#pragma unroll
        for (int i = 0; i < M; i++)
#pragma unroll
            for (int l = 0; l < KK; l++) {
                int plane = tX ? (l + i * KK) : (i + l * M);   // stored X is KK x M when transposed
                ld_pair(X, ldx, plane, p, np, vec, x[i][l][0], x[i][l][1]);
            }
#pragma unroll
        for (int l = 0; l < KK; l++)
#pragma unroll
            for (int j = 0; j < N; j++) {
                int plane = tY ? (j + l * N) : (l + j * KK);   // stored Y is N x KK when transposed
                ld_pair(Y, ldy, plane, p, np, vec, y[l][j][0], y[l][j][1]);
            }
#pragma unroll
        for (int j = 0; j < N; j++)
#pragma unroll
            for (int i = 0; i < M; i++) {
                double s0 = x[i][0][0] * y[0][j][0], s1 = x[i][0][1] * y[0][j][1];
#pragma unroll
                for (int l = 1; l < KK; l++) {
                    s0 = fma(x[i][l][0], y[l][j][0], s0);
                    s1 = fma(x[i][l][1], y[l][j][1], s1);
                }
                st_pair(Z, ldz, i + j * M, p, np, vec, s0, s1);
            }
    }
}

typedef void (*mtimes_fn)(int64_t, const double*, int64_t, int, const double*, int64_t, int, double*, int64_t, bool);

template <int M, int KK>
mtimes_fn pick_n(int n) {
    switch (n) {
        case 1: return mtimes_k<M, KK, 1>;
        case 2: return mtimes_k<M, KK, 2>;
        case 3: return mtimes_k<M, KK, 3>;
        default: return mtimes_k<M, KK, 4>;
    }
}
template <int M>
mtimes_fn pick_k(int k, int n) {
    switch (k) {
        case 1: return pick_n<M, 1>(n);
        case 2: return pick_n<M, 2>(n);
        case 3: return pick_n<M, 3>(n);
        default: return pick_n<M, 4>(n);
    }
}
mtimes_fn pick_mtimes(int m, int k, int n) {
    switch (m) {
        case 1: return pick_k<1>(k, n);
        case 2: return pick_k<2>(k, n);
        case 3: return pick_k<3>(k, n);
        default: return pick_k<4>(k, n);
    }
}

// ------------------------------------------------------------ a2 transpose
// A page transpose in SoA layout is a permutation of planes: Z plane (j + i*cols)
// = X plane (i + j*rows).  blockIdx.y picks the plane, threads stream pairs of
// pages of it (128-bit loads and stores), so every access is coalesced and there
// is no per-page register array.
__global__ void __launch_bounds__(PAGE_BLOCK) transpose_k(int64_t np, const double* __restrict__ X, int rows, int cols,
                                                          int64_t ldx, double* __restrict__ Z, int64_t ldz, bool vec) {
    const int q = blockIdx.y;
    const int i = q % rows, j = q / rows;   // X(i, j) -> Z(j, i), Z is cols x rows
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
    for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; p < np; p += stride) {
        double v0, v1;
        ld_pair(X, ldx, q, p, np, vec, v0, v1);
        st_pair(Z, ldz, j + i * cols, p, np, vec, v0, v1);
    }
}

// ------------------------------------------------------------ avtamav (NEXT-2)
// s_k = a_k^T M_k b_k = sum_i a_i (sum_j M_ij b_j) (eq:layeredBilin
// P:292-301): every plane of a pair of pages loaded first (128-bit), then the
// arithmetic.  a is n x 1, M is n x m, b is m x 1; ld 0 broadcasts.
template <int N, int M>
__global__ void __launch_bounds__(PAGE_BLOCK) bilinear_k(int64_t np, const double* __restrict__ A, int64_t lda,
                                                         const double* __restrict__ Mx, int64_t ldm,
                                                         const double* __restrict__ B, int64_t ldb,
                                                         double* __restrict__ s, bool vec) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
    for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; p < np; p += stride) {
        double a[N][2], b[M][2], m[N][M][2];
#pragma unroll
        for (int i = 0; i < N; i++) ld_pair(A, lda, i, p, np, vec, a[i][0], a[i][1]);
#pragma unroll
        for (int j = 0; j < M; j++) ld_pair(B, ldb, j, p, np, vec, b[j][0], b[j][1]);
#pragma unroll
        for (int j = 0; j < M; j++)
#pragma unroll
            for (int i = 0; i < N; i++) ld_pair(Mx, ldm, i + j * N, p, np, vec, m[i][j][0], m[i][j][1]);
        double acc[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            double r = 0.0;
#pragma unroll
            for (int i = 0; i < N; i++) {
                double t = 0.0;
#pragma unroll
                for (int j = 0; j < M; j++) t = fma(m[i][j][h], b[j][h], t);
                r = fma(a[i][h], t, r);
            }
            acc[h] = r;
        }
        st_pair(s, np, 0, p, np, vec, acc[0], acc[1]);
    }
}

typedef void (*bil_fn)(int64_t, const double*, int64_t, const double*, int64_t, const double*, int64_t, double*, bool);
template <int N>
bil_fn pick_bil_m(int m) {
    switch (m) {
        case 1: return bilinear_k<N, 1>;
        case 2: return bilinear_k<N, 2>;
        case 3: return bilinear_k<N, 3>;
        default: return bilinear_k<N, 4>;
    }
}
bil_fn pick_bilinear(int n, int m) {
    switch (n) {
        case 1: return pick_bil_m<1>(m);
        case 2: return pick_bil_m<2>(m);
        case 3: return pick_bil_m<3>(m);
        default: return pick_bil_m<4>(m);
    }
}

// ------------------------------------------------------------ closed forms
template <int n>
struct Page {
    double a[n][n];
};

template <int n>
__device__ __forceinline__ void load_page2(const double* __restrict__ X, int64_t ldx, int64_t p, int64_t np,
                                           bool vec, Page<n>& A0, Page<n>& A1) {
#pragma unroll
    for (int j = 0; j < n; j++)
#pragma unroll
        for (int i = 0; i < n; i++) ld_pair(X, ldx, i + j * n, p, np, vec, A0.a[i][j], A1.a[i][j]);
}

// determinant and adjugate (adj = det * inverse); b may be nullptr-like (not computed) via template
template <int n, bool ADJ>
__device__ __forceinline__ double det_adj(const Page<n>& A, Page<n>& B) {
    const auto& a = A.a;
    if constexpr (n == 1) {
        if (ADJ) B.a[0][0] = 1.0;
        return a[0][0];
    } else if constexpr (n == 2) {
        if (ADJ) {
            B.a[0][0] = a[1][1];
            B.a[0][1] = -a[0][1];
            B.a[1][0] = -a[1][0];
            B.a[1][1] = a[0][0];
        }
        return fma(a[0][0], a[1][1], -a[0][1] * a[1][0]);
    } else if constexpr (n == 3) {
        // cofactors C_ij; adj(i,j) = C_ji
        double c00 = fma(a[1][1], a[2][2], -a[1][2] * a[2][1]);
        double c01 = fma(a[1][2], a[2][0], -a[1][0] * a[2][2]);
        double c02 = fma(a[1][0], a[2][1], -a[1][1] * a[2][0]);
        double d = fma(a[0][0], c00, fma(a[0][1], c01, a[0][2] * c02));
        if (ADJ) {
            B.a[0][0] = c00;
            B.a[1][0] = c01;
            B.a[2][0] = c02;
            B.a[0][1] = fma(a[0][2], a[2][1], -a[0][1] * a[2][2]);
            B.a[1][1] = fma(a[0][0], a[2][2], -a[0][2] * a[2][0]);
            B.a[2][1] = fma(a[0][1], a[2][0], -a[0][0] * a[2][1]);
            B.a[0][2] = fma(a[0][1], a[1][2], -a[0][2] * a[1][1]);
            B.a[1][2] = fma(a[0][2], a[1][0], -a[0][0] * a[1][2]);
            B.a[2][2] = fma(a[0][0], a[1][1], -a[0][1] * a[1][0]);
        }
        return d;
    } else {
        // Laplace expansion by the 2x2 minors of rows (0,1) and rows (2,3)
        double s0 = fma(a[0][0], a[1][1], -a[1][0] * a[0][1]);
        double s1 = fma(a[0][0], a[1][2], -a[1][0] * a[0][2]);
        double s2 = fma(a[0][0], a[1][3], -a[1][0] * a[0][3]);
        double s3 = fma(a[0][1], a[1][2], -a[1][1] * a[0][2]);
        double s4 = fma(a[0][1], a[1][3], -a[1][1] * a[0][3]);
        double s5 = fma(a[0][2], a[1][3], -a[1][2] * a[0][3]);
        double c5 = fma(a[2][2], a[3][3], -a[3][2] * a[2][3]);
        double c4 = fma(a[2][1], a[3][3], -a[3][1] * a[2][3]);
        double c3 = fma(a[2][1], a[3][2], -a[3][1] * a[2][2]);
        double c2 = fma(a[2][0], a[3][3], -a[3][0] * a[2][3]);
        double c1 = fma(a[2][0], a[3][2], -a[3][0] * a[2][2]);
        double c0 = fma(a[2][0], a[3][1], -a[3][0] * a[2][1]);
        double d = s0 * c5 - s1 * c4 + s2 * c3 + s3 * c2 - s4 * c1 + s5 * c0;
        if (ADJ) {
            B.a[0][0] = a[1][1] * c5 - a[1][2] * c4 + a[1][3] * c3;
            B.a[0][1] = -a[0][1] * c5 + a[0][2] * c4 - a[0][3] * c3;
            B.a[0][2] = a[3][1] * s5 - a[3][2] * s4 + a[3][3] * s3;
            B.a[0][3] = -a[2][1] * s5 + a[2][2] * s4 - a[2][3] * s3;
            B.a[1][0] = -a[1][0] * c5 + a[1][2] * c2 - a[1][3] * c1;
            B.a[1][1] = a[0][0] * c5 - a[0][2] * c2 + a[0][3] * c1;
            B.a[1][2] = -a[3][0] * s5 + a[3][2] * s2 - a[3][3] * s1;
            B.a[1][3] = a[2][0] * s5 - a[2][2] * s2 + a[2][3] * s1;
            B.a[2][0] = a[1][0] * c4 - a[1][1] * c2 + a[1][3] * c0;
            B.a[2][1] = -a[0][0] * c4 + a[0][1] * c2 - a[0][3] * c0;
            B.a[2][2] = a[3][0] * s4 - a[3][1] * s2 + a[3][3] * s0;
            B.a[2][3] = -a[2][0] * s4 + a[2][1] * s2 - a[2][3] * s0;
            B.a[3][0] = -a[1][0] * c3 + a[1][1] * c1 - a[1][2] * c0;
            B.a[3][1] = a[0][0] * c3 - a[0][1] * c1 + a[0][2] * c0;
            B.a[3][2] = -a[3][0] * s3 + a[3][1] * s1 - a[3][2] * s0;
            B.a[3][3] = a[2][0] * s3 - a[2][1] * s1 + a[2][2] * s0;
        }
        return d;
    }
}

// ------------------------------------------------------------ a3 det
template <int n>
__global__ void __launch_bounds__(PAGE_BLOCK) det_k(int64_t np, const double* __restrict__ X, int64_t ldx,
                                                    double* __restrict__ det, bool vec) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
    for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; p < np; p += stride) {
        Page<n> A0, A1, dummy;
        load_page2<n>(X, ldx, p, np, vec, A0, A1);
        double d0 = det_adj<n, false>(A0, dummy);
        double d1 = det_adj<n, false>(A1, dummy);
        st_pair(det, 0, 0, p, np, vec, d0, d1);
    }
}

// ------------------------------------------------------------ a4 inverse
template <int n>
__device__ __forceinline__ double norm_inf(const Page<n>& A) {
    double m = 0.0;
#pragma unroll
    for (int i = 0; i < n; i++) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < n; j++) s += fabs(A.a[i][j]);
        m = fmax(m, s);
    }
    return m;
}

template <int n>
__device__ __forceinline__ bool singular_nrm(double d, double nrm, double tol) {
    double pw = 1.0;
#pragma unroll
    for (int k = 0; k < n; k++) pw *= nrm;
    return !(fabs(d) > tol * pw);  // also flags nan
}

template <int n>
__global__ void __launch_bounds__(PAGE_BLOCK) inv_k(int64_t np, const double* __restrict__ X, int64_t ldx,
                                                    double* __restrict__ Xi, int64_t ldi, double* __restrict__ det,
                                                    unsigned long long* __restrict__ first_sing, double tol, bool vec) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
    for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; p < np; p += stride) {
        Page<n> A0, A1, B0, B1;
        load_page2<n>(X, ldx, p, np, vec, A0, A1);
        // the singularity test needs only ||A||_inf: take it now so the pages die early
        // (4x4: 244 -> fewer registers, more resident warps)
        const double nrm0 = first_sing ? norm_inf<n>(A0) : 0.0, nrm1 = first_sing ? norm_inf<n>(A1) : 0.0;
        double d0 = det_adj<n, true>(A0, B0);
        double d1 = det_adj<n, true>(A1, B1);
        double r0 = 1.0 / d0, r1 = 1.0 / d1;
#pragma unroll
        for (int j = 0; j < n; j++)
#pragma unroll
            for (int i = 0; i < n; i++) st_pair(Xi, ldi, i + j * n, p, np, vec, B0.a[i][j] * r0, B1.a[i][j] * r1);
        if (det) st_pair(det, 0, 0, p, np, vec, d0, d1);
        if (first_sing) {
            if (singular_nrm<n>(d0, nrm0, tol)) atomicMin(first_sing, (unsigned long long)p);
            else if (p + 1 < np && singular_nrm<n>(d1, nrm1, tol)) atomicMin(first_sing, (unsigned long long)(p + 1));
        }
    }
}

__global__ void set_i64_k(int64_t* p, int64_t v) { *p = v; }

// ------------------------------------------------------------ a5 cross
__global__ void __launch_bounds__(PAGE_BLOCK) cross_k(int64_t np, const double* __restrict__ A, int64_t lda,
                                                      const double* __restrict__ B, int64_t ldb,
                                                      double* __restrict__ Cc, int64_t ldc, bool vec) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
    for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; p < np; p += stride) {
        double a[3][2], b[3][2];
#pragma unroll
        for (int i = 0; i < 3; i++) {
            ld_pair(A, lda, i, p, np, vec, a[i][0], a[i][1]);
            ld_pair(B, ldb, i, p, np, vec, b[i][0], b[i][1]);
        }
        double c[3][2];
#pragma unroll
        for (int q = 0; q < 2; q++) {
            c[0][q] = fma(a[1][q], b[2][q], -a[2][q] * b[1][q]);
            c[1][q] = fma(a[2][q], b[0][q], -a[0][q] * b[2][q]);
            c[2][q] = fma(a[0][q], b[1][q], -a[1][q] * b[0][q]);
        }
#pragma unroll
        for (int i = 0; i < 3; i++) st_pair(Cc, ldc, i, p, np, vec, c[i][0], c[i][1]);
    }
}

// ------------------------------------------------------------ a7 gather
template <int DIM, int NV>
__global__ void __launch_bounds__(PAGE_BLOCK) gather_k(int64_t ne, const double* __restrict__ coords, int64_t ns,
                                                       int64_t cs_, const int32_t* __restrict__ elems, int64_t eld,
                                                       double* __restrict__ c3, double* __restrict__ v3) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += stride) {
        double x[NV][DIM];
#pragma unroll
        for (int a = 0; a < NV; a++) {
            int64_t v = __ldcs(elems + a * eld + e);
#pragma unroll
            for (int c = 0; c < DIM; c++) x[a][c] = __ldg(coords + c * cs_ + v * ns);
        }
        if (c3) {
#pragma unroll
            for (int a = 0; a < NV; a++)
#pragma unroll
                for (int c = 0; c < DIM; c++) stcs(c3 + (int64_t)(c + a * DIM) * ne + e, x[a][c]);
        }
        if (v3) {
#pragma unroll
            for (int a = 0; a < NV - 1; a++)
#pragma unroll
                for (int c = 0; c < DIM; c++) stcs(v3 + (int64_t)(c + a * DIM) * ne + e, x[a][c] - x[NV - 1][c]);
        }
    }
}

// the same for two adjacent elements per thread: index pairs as int2, every plane written with 128-bit stores
// (ne even, planes 16-byte aligned)
#ifndef VB_GATHER_MINB
#define VB_GATHER_MINB 3
#endif
template <int DIM, int NV>
__global__ void __launch_bounds__(PAGE_BLOCK, VB_GATHER_MINB) gather2_k(int64_t ne, const double* __restrict__ coords, int64_t ns,
                                                           int64_t cs_, const int32_t* __restrict__ elems, int64_t eld,
                                                           double* __restrict__ c3, double* __restrict__ v3) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t npair = ne / 2;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < npair; t += stride) {
        const int64_t e = 2 * t;
        int64_t v[2][NV];
#pragma unroll
        for (int a = 0; a < NV; a++) {
            const int2 p = __ldcs(reinterpret_cast<const int2*>(elems + a * eld + e));
            v[0][a] = p.x;
            v[1][a] = p.y;
        }
        double x[2][NV][DIM];
#pragma unroll
        for (int k = 0; k < 2; k++)
#pragma unroll
            for (int a = 0; a < NV; a++)
#pragma unroll
                for (int c = 0; c < DIM; c++) x[k][a][c] = __ldg(coords + c * cs_ + v[k][a] * ns);
        if (c3) {
#pragma unroll
            for (int a = 0; a < NV; a++)
#pragma unroll
                for (int c = 0; c < DIM; c++)
                    stcs2(c3 + (int64_t)(c + a * DIM) * ne + e, make_double2(x[0][a][c], x[1][a][c]));
        }
        if (v3) {
#pragma unroll
            for (int a = 0; a < NV - 1; a++)
#pragma unroll
                for (int c = 0; c < DIM; c++)
                    stcs2(v3 + (int64_t)(c + a * DIM) * ne + e,
                          make_double2(x[0][a][c] - x[0][NV - 1][c], x[1][a][c] - x[1][NV - 1][c]));
        }
    }
}

bool ld_ok(int64_t ld, int64_t np, bool input) { return ld >= np || (input && ld == 0); }

bool vec_ok(std::initializer_list<std::pair<const void*, int64_t>> ops) {
    for (auto& o : ops) {
        if (o.second == 0) continue;  // broadcast operands are loaded scalar
        if (!aligned16(o.first) || (o.second & 1)) return false;
    }
    return true;
}

}  // namespace
}  // namespace vb

using namespace vb;

extern "C" vb_status vb_page_mtimes(int64_t npages, const double* X, int xrows, int xcols, int64_t ldx, int transX,
                                    const double* Y, int yrows, int ycols, int64_t ldy, int transY, double* Z,
                                    int64_t ldz, vb_stream_t stream) {
    clear_error();
    if (npages < 0) { set_error("vb_page_mtimes: npages < 0"); return VB_ERR_ARG; }
    int m = transX ? xcols : xrows, kx = transX ? xrows : xcols;
    int ky = transY ? ycols : yrows, n = transY ? yrows : ycols;
    for (int d : {xrows, xcols, yrows, ycols})
        if (d < 1 || d > 4) { set_error("vb_page_mtimes: page dimensions must be 1..4 (got X %dx%d, Y %dx%d)", xrows, xcols, yrows, ycols); return VB_ERR_UNSUPPORTED; }
    if (kx != ky) {
        set_error("vb_page_mtimes: inner dimension mismatch: op(X) has %d columns, op(Y) has %d rows", kx, ky);
        return VB_ERR_DIM;
    }
    if (npages == 0) return VB_OK;
    if (!X || !Y || !Z) { set_error("vb_page_mtimes: NULL %s", !X ? "X" : !Y ? "Y" : "Z"); return VB_ERR_ARG; }
    if (!ld_ok(ldx, npages, true) || !ld_ok(ldy, npages, true) || !ld_ok(ldz, npages, false)) {
        set_error("vb_page_mtimes: leading dimension smaller than npages (ldx=%lld ldy=%lld ldz=%lld npages=%lld)",
                  (long long)ldx, (long long)ldy, (long long)ldz, (long long)npages);
        return VB_ERR_ARG;
    }
    bool vec = vec_ok({{X, ldx}, {Y, ldy}, {Z, ldz}});
    unsigned g = grid_for((npages + 1) / 2, PAGE_BLOCK, PAGE_BLOCKS_PER_SM);
    pick_mtimes(m, kx, n)<<<g, PAGE_BLOCK, 0, cs(stream)>>>(npages, X, ldx, transX ? 1 : 0, Y, ldy, transY ? 1 : 0,
                                                            Z, ldz, vec);
    return launch_check("vb_page_mtimes");
}

extern "C" vb_status vb_page_transpose(int64_t npages, const double* X, int rows, int cols, int64_t ldx, double* Z,
                                       int64_t ldz, vb_stream_t stream) {
    clear_error();
    if (npages < 0) { set_error("vb_page_transpose: npages < 0"); return VB_ERR_ARG; }
    if (rows < 1 || rows > 4 || cols < 1 || cols > 4) { set_error("vb_page_transpose: rows/cols must be 1..4"); return VB_ERR_UNSUPPORTED; }
    if (npages == 0) return VB_OK;
    if (!X || !Z) { set_error("vb_page_transpose: NULL %s", !X ? "X" : "Z"); return VB_ERR_ARG; }
    if (!ld_ok(ldx, npages, true) || !ld_ok(ldz, npages, false)) { set_error("vb_page_transpose: ld < npages"); return VB_ERR_ARG; }
    bool vec = vec_ok({{X, ldx}, {Z, ldz}});
    // rows*cols planes side by side in grid.y; about PAGE_BLOCKS_PER_SM resident CTAs per SM in all
    const int nplanes = rows * cols;
    const int bps = PAGE_BLOCKS_PER_SM / nplanes > 0 ? PAGE_BLOCKS_PER_SM / nplanes : 1;
    const dim3 g(grid_for((npages + 1) / 2, PAGE_BLOCK, bps, nplanes < PAGE_BLOCKS_PER_SM ? 1 : 2), nplanes);
    transpose_k<<<g, PAGE_BLOCK, 0, cs(stream)>>>(npages, X, rows, cols, ldx, Z, ldz, vec);
    return launch_check("vb_page_transpose");
}

extern "C" vb_status vb_page_det(int64_t npages, int n, const double* X, int64_t ldx, double* det, vb_stream_t stream) {
    clear_error();
    if (npages < 0) { set_error("vb_page_det: npages < 0"); return VB_ERR_ARG; }
    if (n < 1 || n > 4) { set_error("vb_page_det: page size n=%d outside 1..4", n); return VB_ERR_UNSUPPORTED; }
    if (npages == 0) return VB_OK;
    if (!X || !det) { set_error("vb_page_det: NULL %s", !X ? "X" : "det"); return VB_ERR_ARG; }
    if (!ld_ok(ldx, npages, true)) { set_error("vb_page_det: ldx < npages"); return VB_ERR_ARG; }
    bool vec = vec_ok({{X, ldx}, {det, 2}});
    unsigned g = grid_for((npages + 1) / 2, PAGE_BLOCK, PAGE_BLOCKS_PER_SM);
    auto s = cs(stream);
    switch (n) {
        case 1: det_k<1><<<g, PAGE_BLOCK, 0, s>>>(npages, X, ldx, det, vec); break;
        case 2: det_k<2><<<g, PAGE_BLOCK, 0, s>>>(npages, X, ldx, det, vec); break;
        case 3: det_k<3><<<g, PAGE_BLOCK, 0, s>>>(npages, X, ldx, det, vec); break;
        default: det_k<4><<<g, PAGE_BLOCK, 0, s>>>(npages, X, ldx, det, vec); break;
    }
    return launch_check("vb_page_det");
}

extern "C" vb_status vb_page_inv(int64_t npages, int n, const double* X, int64_t ldx, double* Xinv, int64_t ldinv,
                                 double* det, int64_t* first_singular, double sing_tol, vb_stream_t stream) {
    clear_error();
    if (npages < 0) { set_error("vb_page_inv: npages < 0"); return VB_ERR_ARG; }
    if (n < 1 || n > 4) { set_error("vb_page_inv: page size n=%d outside 1..4", n); return VB_ERR_UNSUPPORTED; }
    auto s = cs(stream);
    if (first_singular) {
        set_i64_k<<<1, 1, 0, s>>>(first_singular, npages);
        if (launch_check("vb_page_inv") != VB_OK) return VB_ERR_CUDA;
    }
    if (npages == 0) return VB_OK;
    if (!X || !Xinv) { set_error("vb_page_inv: NULL %s", !X ? "X" : "Xinv"); return VB_ERR_ARG; }
    if (!ld_ok(ldx, npages, true) || !ld_ok(ldinv, npages, false)) { set_error("vb_page_inv: ld < npages"); return VB_ERR_ARG; }
    bool vec = vec_ok({{X, ldx}, {Xinv, ldinv}}) && (!det || aligned16(det));
    unsigned g = grid_for((npages + 1) / 2, PAGE_BLOCK, PAGE_BLOCKS_PER_SM);
    auto fs = reinterpret_cast<unsigned long long*>(first_singular);
    switch (n) {
        case 1: inv_k<1><<<g, PAGE_BLOCK, 0, s>>>(npages, X, ldx, Xinv, ldinv, det, fs, sing_tol, vec); break;
        case 2: inv_k<2><<<g, PAGE_BLOCK, 0, s>>>(npages, X, ldx, Xinv, ldinv, det, fs, sing_tol, vec); break;
        case 3: inv_k<3><<<g, PAGE_BLOCK, 0, s>>>(npages, X, ldx, Xinv, ldinv, det, fs, sing_tol, vec); break;
        default: inv_k<4><<<g, PAGE_BLOCK, 0, s>>>(npages, X, ldx, Xinv, ldinv, det, fs, sing_tol, vec); break;
    }
    return launch_check("vb_page_inv");
}

extern "C" vb_status vb_page_cross(int64_t npages, const double* A, int64_t lda, const double* B, int64_t ldb,
                                   double* C, int64_t ldc, vb_stream_t stream) {
    clear_error();
    if (npages < 0) { set_error("vb_page_cross: npages < 0"); return VB_ERR_ARG; }
    if (npages == 0) return VB_OK;
    if (!A || !B || !C) { set_error("vb_page_cross: NULL %s", !A ? "A" : !B ? "B" : "C"); return VB_ERR_ARG; }
    if (!ld_ok(lda, npages, true) || !ld_ok(ldb, npages, true) || !ld_ok(ldc, npages, false)) { set_error("vb_page_cross: ld < npages"); return VB_ERR_ARG; }
    bool vec = vec_ok({{A, lda}, {B, ldb}, {C, ldc}});
    unsigned g = grid_for((npages + 1) / 2, PAGE_BLOCK, PAGE_BLOCKS_PER_SM);
    cross_k<<<g, PAGE_BLOCK, 0, cs(stream)>>>(npages, A, lda, B, ldb, C, ldc, vec);
    return launch_check("vb_page_cross");
}

extern "C" vb_status vb_create_coords3D(int dim, int nv, int64_t ne, const double* coords, int64_t node_stride,
                                        int64_t comp_stride, const int32_t* elems, int64_t elem_ld, double* coords3D,
                                        double* vectors3D, vb_stream_t stream) {
    clear_error();
    if (ne < 0) { set_error("vb_create_coords3D: ne < 0"); return VB_ERR_ARG; }
    if (dim < 1 || dim > 3 || nv < 2 || nv > 4) { set_error("vb_create_coords3D: need dim in 1..3, nv in 2..4"); return VB_ERR_UNSUPPORTED; }
    if (ne == 0) return VB_OK;
    if (!coords || !elems || (!coords3D && !vectors3D)) { set_error("vb_create_coords3D: NULL argument"); return VB_ERR_ARG; }
    if (elem_ld < ne) { set_error("vb_create_coords3D: elem_ld < ne"); return VB_ERR_ARG; }
    unsigned g = grid_for(ne, PAGE_BLOCK, PAGE_BLOCKS_PER_SM);
    auto s = cs(stream);
    bool vec = (ne & 1) == 0 && (elem_ld & 1) == 0 && (reinterpret_cast<uintptr_t>(elems) & 7u) == 0 &&
               (!coords3D || aligned16(coords3D)) && (!vectors3D || aligned16(vectors3D));
    #ifndef VB_GATHER_SCALAR
#define VB_GATHER_SCALAR 0
#endif
    // measured on the configs[4] mesh (tools/time_gather.py): one output 0.236 (scalar) -> 0.201 ms (paired, 3 blocks
    // per SM); both outputs 0.452 (scalar) vs 0.465 (paired): the paired kernel takes the one-output calls only
    if (VB_GATHER_SCALAR || (coords3D && vectors3D)) vec = false;
    if (vec) g = grid_for(ne / 2, PAGE_BLOCK, VB_GATHER_MINB);
#define VB_GATHER(D, V)                                                                                                     \
    do {                                                                                                                    \
        if (vec) gather2_k<D, V><<<g, PAGE_BLOCK, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, coords3D, vectors3D); \
        else gather_k<D, V><<<g, PAGE_BLOCK, 0, s>>>(ne, coords, node_stride, comp_stride, elems, elem_ld, coords3D, vectors3D);      \
    } while (0)
    if (dim == 1) {
        if (nv == 2) VB_GATHER(1, 2); else if (nv == 3) VB_GATHER(1, 3); else VB_GATHER(1, 4);
    } else if (dim == 2) {
        if (nv == 2) VB_GATHER(2, 2); else if (nv == 3) VB_GATHER(2, 3); else VB_GATHER(2, 4);
    } else {
        if (nv == 2) VB_GATHER(3, 2); else if (nv == 3) VB_GATHER(3, 3); else VB_GATHER(3, 4);
    }
#undef VB_GATHER
    return launch_check("vb_create_coords3D");
}

extern "C" vb_status vb_page_bilinear(int64_t npages, int n, int m, const double* A, int64_t lda, const double* Mx,
                                      int64_t ldm, const double* B, int64_t ldb, double* s, vb_stream_t stream) {
    clear_error();
    if (npages < 0) { set_error("vb_page_bilinear: npages < 0"); return VB_ERR_ARG; }
    if (n < 1 || n > 4 || m < 1 || m > 4) { set_error("vb_page_bilinear: n, m must be 1..4"); return VB_ERR_UNSUPPORTED; }
    if (npages == 0) return VB_OK;
    if (!A || !Mx || !B || !s) { set_error("vb_page_bilinear: NULL argument"); return VB_ERR_ARG; }
    if (!ld_ok(lda, npages, true) || !ld_ok(ldm, npages, true) || !ld_ok(ldb, npages, true)) {
        set_error("vb_page_bilinear: leading dimension < npages");
        return VB_ERR_ARG;
    }
    const bool vec = vec_ok({{A, lda}, {Mx, ldm}, {B, ldb}, {s, npages}});
    const unsigned g = grid_for((npages + 1) / 2, PAGE_BLOCK, PAGE_BLOCKS_PER_SM);
    pick_bilinear(n, m)<<<g, PAGE_BLOCK, 0, cs(stream)>>>(npages, A, lda, Mx, ldm, B, ldb, s, vec);
    return launch_check("vb_page_bilinear");
}
