/*
 * ORACLE -- plain, slow, single-threaded CPU reference for the hot path of
 * arXiv 2404.16039 ("vectorized" page-wise linear algebra + P1 FEM assembly).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product (paper_2404_16039_b200/, include/vb.h, libvb.so) never links,
 * includes or calls anything here, and nothing here includes product code.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (oracle/build.py).
 * fp64 throughout (the paper's MATLAB default, P:461 / BASELINE.md).
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * O1..O12 = SURVEY.md §8(c) oracle algorithm rows.
 *
 * Page layout (O1): entry (i,j) of page k of a
 * rows x cols page array lives at p[(i + j*rows)*ld + k]; ld == 0 means the
 * single object is broadcast to every page (eq:copy).
 *
 * Every function below writes the plain definition out; there is no blocking,
 * fusion or reordering.  Parity pins live in tests/test_oracle_*.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_DIM (-2)
#define ORC_ERR_ARG (-1)

/* O1: page accessor (P:248-266 with W as the page index).  ld == 0 is the
 * copy map eq:copy: ONE rows x cols object, stored column-major
 * and contiguous, is used as every page. */
static double at(const double* p, int64_t ld, int rows, int i, int j, int64_t k) {
    if (ld == 0) return p[i + j * rows];
    return p[(int64_t)(i + j * rows) * ld + k];
}

/* O2: page-wise matrix multiplication Z_k = op(X_k) op(Y_k)
 * (eq:pagewisemultGeneral / layeredMultiplication; pagemtimes
 * semantics P:391).  op = transpose when tX/tY != 0.  Sum over l ascending,
 * plain multiply-then-add (no FMA: -ffp-contract=off). */
int orc_page_mtimes(int64_t np, const double* X, int xr, int xc, int64_t ldx, int tX,
                    const double* Y, int yr, int yc, int64_t ldy, int tY,
                    double* Z, int64_t ldz) {
    int m = tX ? xc : xr, kx = tX ? xr : xc;
    int ky = tY ? yc : yr, n = tY ? yr : yc;
    if (kx != ky) return ORC_ERR_DIM;
    for (int64_t k = 0; k < np; k++)
        for (int i = 0; i < m; i++)
            for (int j = 0; j < n; j++) {
                double s = 0.0;
                for (int l = 0; l < kx; l++) {
                    double a = tX ? at(X, ldx, xr, l, i, k) : at(X, ldx, xr, i, l, k);
                    double b = tY ? at(Y, ldy, yr, j, l, k) : at(Y, ldy, yr, l, j, k);
                    s = s + a * b;
                }
                Z[(int64_t)(i + j * m) * ldz + k] = s;
            }
    return ORC_OK;
}

/* O3: page-wise transpose (layeredTransposeHom/Ten). */
int orc_page_transpose(int64_t np, const double* X, int rows, int cols, int64_t ldx,
                       double* Z, int64_t ldz) {
    for (int64_t k = 0; k < np; k++)
        for (int i = 0; i < rows; i++)
            for (int j = 0; j < cols; j++)
                Z[(int64_t)(j + i * cols) * ldz + k] = at(X, ldx, rows, i, j, k);
    return ORC_OK;
}

/* O4: determinant by Laplace (cofactor) expansion along row 0 with recursive
 * minors -- the textbook definition (layeredDeterminant). a is an
 * n x n matrix stored a[i*4 + j] (row-major scratch, n <= 4). */
static double det_laplace(const double* a, int n) {
    if (n == 1) return a[0];
    if (n == 2) return a[0 * 4 + 0] * a[1 * 4 + 1] - a[0 * 4 + 1] * a[1 * 4 + 0];
    double s = 0.0;
    for (int c = 0; c < n; c++) {
        double sub[16];
        for (int i = 1; i < n; i++) {
            int jj = 0;
            for (int j = 0; j < n; j++) {
                if (j == c) continue;
                sub[(i - 1) * 4 + jj] = a[i * 4 + j];
                jj++;
            }
        }
        double cof = det_laplace(sub, n - 1);
        double term = a[0 * 4 + c] * cof;
        s = (c % 2 == 0) ? s + term : s - term;
    }
    return s;
}

/* minor(r, c): determinant of a with row r and column c removed. */
static double minor_rc(const double* a, int n, int r, int c) {
    double sub[16];
    int ii = 0;
    for (int i = 0; i < n; i++) {
        if (i == r) continue;
        int jj = 0;
        for (int j = 0; j < n; j++) {
            if (j == c) continue;
            sub[ii * 4 + jj] = a[i * 4 + j];
            jj++;
        }
        ii++;
    }
    return det_laplace(sub, n - 1);
}

static void load_page(const double* X, int64_t ldx, int n, int64_t k, double* a) {
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) a[i * 4 + j] = at(X, ldx, n, i, j, k);
}

int orc_page_det(int64_t np, int n, const double* X, int64_t ldx, double* det) {
    if (n < 1 || n > 4) return ORC_ERR_DIM;
    double a[16];
    for (int64_t k = 0; k < np; k++) {
        load_page(X, ldx, n, k, a);
        det[k] = det_laplace(a, n);
    }
    return ORC_OK;
}

/* O5: inverse by the adjugate, inv(i,j) = (-1)^(i+j) minor(j,i) / det
 * (layeredInverse; aminv returns the determinant too).
 * Singular pages follow IEEE (division by zero), SURVEY B3. */
int orc_page_inv(int64_t np, int n, const double* X, int64_t ldx,
                 double* Xinv, int64_t ldinv, double* det) {
    if (n < 1 || n > 4) return ORC_ERR_DIM;
    double a[16];
    for (int64_t k = 0; k < np; k++) {
        load_page(X, ldx, n, k, a);
        double d = det_laplace(a, n);
        for (int i = 0; i < n; i++)
            for (int j = 0; j < n; j++) {
                double cof = (n == 1) ? 1.0 : minor_rc(a, n, j, i);
                if ((i + j) % 2) cof = -cof;
                Xinv[(int64_t)(i + j * n) * ldinv + k] = cof / d;
            }
        if (det) det[k] = d;
    }
    return ORC_OK;
}

/* O6: cross product c = a x b of 3-vector pages (BASELINE.json north_star;
 * the columns of cof(A) are cross products of A's columns). */
int orc_page_cross(int64_t np, const double* A, int64_t lda, const double* B, int64_t ldb,
                   double* C, int64_t ldc) {
    for (int64_t k = 0; k < np; k++) {
        double a1 = at(A, lda, 3, 0, 0, k), a2 = at(A, lda, 3, 1, 0, k), a3 = at(A, lda, 3, 2, 0, k);
        double b1 = at(B, ldb, 3, 0, 0, k), b2 = at(B, ldb, 3, 1, 0, k), b3 = at(B, ldb, 3, 2, 0, k);
        C[0 * ldc + k] = a2 * b3 - a3 * b2;
        C[1 * ldc + k] = a3 * b1 - a1 * b3;
        C[2 * ldc + k] = a1 * b2 - a2 * b1;
    }
    return ORC_OK;
}

/* O8: gather, create_coords3D (Code coords3D): coords3D(:,a,e) =
 * coords(elems(e,a),:) and vectors3D(:,a,e) = coords3D(:,a,e) - coords3D(:,end,e).
 * Outputs are page arrays (dim x nv and dim x (nv-1) pages, ld = ne). */
int orc_create_coords3D(int dim, int nv, int64_t ne, const double* coords, int64_t node_stride,
                        int64_t comp_stride, const int32_t* elems, int64_t elem_ld,
                        double* coords3D, double* vectors3D) {
    for (int64_t e = 0; e < ne; e++)
        for (int a = 0; a < nv; a++) {
            int64_t v = elems[a * elem_ld + e];
            for (int c = 0; c < dim; c++) {
                double x = coords[c * comp_stride + v * node_stride];
                if (coords3D) coords3D[(int64_t)(c + a * dim) * ne + e] = x;
            }
        }
    if (vectors3D)
        for (int64_t e = 0; e < ne; e++) {
            int64_t vl = elems[(nv - 1) * elem_ld + e];
            for (int a = 0; a < nv - 1; a++) {
                int64_t v = elems[a * elem_ld + e];
                for (int c = 0; c < dim; c++)
                    vectors3D[(int64_t)(c + a * dim) * ne + e] =
                        coords[c * comp_stride + v * node_stride] - coords[c * comp_stride + vl * node_stride];
            }
        }
    return ORC_OK;
}

/* O7: surface geometry of a triangulated closed surface (config 3):
 * n = (b-a) x (c-a); |n| = sqrt(n.n); nhat = n/|n|; area = |n|/2;
 * volume = sum_f (1/6) a.n, the divergence theorem with F = x/3
 * (surf_int), summed in face order with Neumaier compensation. */
int orc_tri_surface(int64_t nf, const int32_t* tri, int64_t tri_ld, const double* xyz,
                    int64_t node_stride, int64_t comp_stride, double* n_out, double* nhat_out,
                    double* area_out, double* volume_out) {
    double s = 0.0, comp = 0.0;
    for (int64_t f = 0; f < nf; f++) {
        int64_t va = tri[0 * tri_ld + f], vb = tri[1 * tri_ld + f], vc = tri[2 * tri_ld + f];
        double a[3], b[3], c[3], u[3], w[3], n[3];
        for (int d = 0; d < 3; d++) {
            a[d] = xyz[d * comp_stride + va * node_stride];
            b[d] = xyz[d * comp_stride + vb * node_stride];
            c[d] = xyz[d * comp_stride + vc * node_stride];
            u[d] = b[d] - a[d];
            w[d] = c[d] - a[d];
        }
        n[0] = u[1] * w[2] - u[2] * w[1];
        n[1] = u[2] * w[0] - u[0] * w[2];
        n[2] = u[0] * w[1] - u[1] * w[0];
        double len = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
        for (int d = 0; d < 3; d++) {
            if (n_out) n_out[d * nf + f] = n[d];
            if (nhat_out) nhat_out[d * nf + f] = n[d] / len;
        }
        if (area_out) area_out[f] = len / 2.0;
        double x = (a[0] * n[0] + a[1] * n[1] + a[2] * n[2]) / 6.0;
        double t = s + x;  /* Neumaier */
        if (fabs(s) >= fabs(x)) comp += (s - t) + x;
        else comp += (x - t) + s;
        s = t;
    }
    if (volume_out) *volume_out = s + comp;
    return ORC_OK;
}

/* ---------------------------------------------------------------- FEM P1 */

static int64_t factorial(int d) { int64_t f = 1; for (int i = 2; i <= d; i++) f *= i; return f; }

/* O9: P1 element matrices with c_K = c_M = 1 (eq:K_M P:967-975 with the
 * RV2013 case c = 1; Code phider P:929-947; Code stiff_scalar_P1 P:978-1004):
 *   tjac = D * X^T, i.e. J[r][c] = x_{r+1}[c] - x_0[c]     (smamt)
 *   detJ (O4), |T| = |detJ| / d!
 *   Jinv = adjugate / detJ (O5)                             (aminv)
 *   G = Jinv * D, D = [-1 | I]                              (amsm)
 *   K_e[a][b] = |T| * sum_r G[r][a] G[r][b]  (r ascending)   (amtam)
 *   M_e[a][b] = |T| / ((d+1)(d+2)) * (1 + delta_ab)          (BASELINE north_star)
 * X is the element's vertex coordinates, X[c*nv + a] = coordinate c of vertex a.
 * Ke, Me are nv x nv, stored Ke[a*nv + b]. */
void orc_p1_local(int dim, const double* X, double* Ke, double* Me) {
    int nv = dim + 1;
    double J[16], Jinv[16], G[4 * 4];
    for (int r = 0; r < dim; r++)
        for (int c = 0; c < dim; c++) J[r * 4 + c] = X[c * nv + (r + 1)] - X[c * nv + 0];
    double detJ = det_laplace(J, dim);
    double T = fabs(detJ) / (double)factorial(dim);
    for (int i = 0; i < dim; i++)
        for (int j = 0; j < dim; j++) {
            double cof = (dim == 1) ? 1.0 : minor_rc(J, dim, j, i);
            if ((i + j) % 2) cof = -cof;
            Jinv[i * 4 + j] = cof / detJ;
        }
    /* G = Jinv * D with D[r][0] = -1, D[r][a] = delta_{r, a-1} */
    for (int r = 0; r < dim; r++)
        for (int a = 0; a < nv; a++) {
            double s = 0.0;
            for (int l = 0; l < dim; l++) {
                double dla = (a == 0) ? -1.0 : (l == a - 1 ? 1.0 : 0.0);
                s = s + Jinv[r * 4 + l] * dla;
            }
            G[r * 4 + a] = s;
        }
    double mscale = T / (double)((dim + 1) * (dim + 2));
    for (int a = 0; a < nv; a++)
        for (int b = 0; b < nv; b++) {
            double s = 0.0;
            for (int r = 0; r < dim; r++) s = s + G[r * 4 + a] * G[r * 4 + b];
            Ke[a * nv + b] = T * s;
            Me[a * nv + b] = mscale * (a == b ? 2.0 : 1.0);
        }
}

/* Local matrices of all elements as page arrays K3D/M3D (nv x nv pages,
 * ld = ne), the second output of stiffness_matrixP1. */
int orc_p1_local_all(int dim, int64_t ne, const double* coords, int64_t node_stride,
                     int64_t comp_stride, const int32_t* elems, int64_t elem_ld,
                     double* K3D, double* M3D) {
    int nv = dim + 1;
    for (int64_t e = 0; e < ne; e++) {
        double X[16], Ke[16], Me[16];
        for (int a = 0; a < nv; a++) {
            int64_t v = elems[a * elem_ld + e];
            for (int c = 0; c < dim; c++) X[c * nv + a] = coords[c * comp_stride + v * node_stride];
        }
        orc_p1_local(dim, X, Ke, Me);
        for (int a = 0; a < nv; a++)
            for (int b = 0; b < nv; b++) {
                if (K3D) K3D[(int64_t)(a + b * nv) * ne + e] = Ke[a * nv + b];
                if (M3D) M3D[(int64_t)(a + b * nv) * ne + e] = Me[a * nv + b];
            }
    }
    return ORC_OK;
}

static int cmp_i32(const void* x, const void* y) {
    int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
    return (a > b) - (a < b);
}

/* O10: topological CSR pattern of sparse(X3D(:),Y3D(:),...):
 * for e, a, b: push elems[e][b] into rows[elems[e][a]]; per row sort + unique
 * (explicit zeros kept); row_ptr = exclusive scan of row sizes.
 * Returns nnz.  With col_idx == NULL only row_ptr is written.  orc_pattern
 * takes the number of nodes per element (P2: 6 or 10). */
int64_t orc_pattern(int nv, int64_t nn, int64_t ne, const int32_t* elems, int64_t elem_ld,
                    int32_t* row_ptr, int32_t* col_idx);
int64_t orc_p1_pattern(int dim, int64_t nn, int64_t ne, const int32_t* elems, int64_t elem_ld,
                       int32_t* row_ptr, int32_t* col_idx) {
    return orc_pattern(dim + 1, nn, ne, elems, elem_ld, row_ptr, col_idx);
}
int64_t orc_pattern(int nv, int64_t nn, int64_t ne, const int32_t* elems, int64_t elem_ld,
                    int32_t* row_ptr, int32_t* col_idx) {
    int64_t* cnt = calloc((size_t)nn + 1, sizeof(int64_t));
    if (!cnt) return -1;
    for (int64_t e = 0; e < ne; e++)
        for (int a = 0; a < nv; a++) cnt[elems[a * elem_ld + e] + 1] += nv;
    for (int64_t v = 0; v < nn; v++) cnt[v + 1] += cnt[v];
    int32_t* push = malloc((size_t)(cnt[nn] ? cnt[nn] : 1) * sizeof(int32_t));
    int64_t* fill = malloc((size_t)(nn ? nn : 1) * sizeof(int64_t));
    if (!push || !fill) { free(cnt); free(push); free(fill); return -1; }
    for (int64_t v = 0; v < nn; v++) fill[v] = cnt[v];
    for (int64_t e = 0; e < ne; e++)
        for (int a = 0; a < nv; a++) {
            int64_t r = elems[a * elem_ld + e];
            for (int b = 0; b < nv; b++) push[fill[r]++] = elems[b * elem_ld + e];
        }
    int64_t nnz = 0;
    for (int64_t v = 0; v < nn; v++) {
        int32_t* seg = push + cnt[v];
        int64_t len = cnt[v + 1] - cnt[v];
        qsort(seg, (size_t)len, sizeof(int32_t), cmp_i32);
        int64_t u = 0;
        for (int64_t i = 0; i < len; i++)
            if (i == 0 || seg[i] != seg[i - 1]) seg[u++] = seg[i];
        row_ptr[v] = (int32_t)nnz;
        if (col_idx) memcpy(col_idx + nnz, seg, (size_t)u * sizeof(int32_t));
        nnz += u;
    }
    row_ptr[nn] = (int32_t)nnz;
    free(cnt); free(push); free(fill);
    return nnz;
}

static int64_t find_col(const int32_t* row_ptr, const int32_t* col_idx, int64_t r, int32_t c) {
    int64_t lo = row_ptr[r], hi = row_ptr[r + 1];
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (col_idx[mid] < c) lo = mid + 1; else hi = mid;
    }
    return (lo < row_ptr[r + 1] && col_idx[lo] == c) ? lo : -1;
}

/* O11: assembly = MATLAB sparse() with duplicates summed:
 * zero K, M; for e ascending, a ascending, b ascending:
 *   p = position of col elems[e][b] in row elems[e][a] (binary search);
 *   K[p] += K_e[a][b]; M[p] += M_e[a][b].
 * If row_mask != NULL only rows with row_mask[r] != 0 are accumulated (the
 * same sums, restricted; used for sampled parity at full size) and only
 * elements touching such a row are evaluated.  K or M may be NULL.
 * Returns 0, or -3 if a (row, col) pair is missing from the pattern. */
int orc_p1_assemble(int dim, int64_t nn, int64_t ne, const double* coords, int64_t node_stride,
                    int64_t comp_stride, const int32_t* elems, int64_t elem_ld,
                    const int32_t* row_ptr, const int32_t* col_idx,
                    double* K, double* M, const uint8_t* row_mask) {
    int nv = dim + 1;
    int64_t nnz = row_ptr[nn];
    if (K) for (int64_t p = 0; p < nnz; p++) K[p] = 0.0;
    if (M) for (int64_t p = 0; p < nnz; p++) M[p] = 0.0;
    for (int64_t e = 0; e < ne; e++) {
        int32_t vid[4];
        int touch = 0;
        for (int a = 0; a < nv; a++) {
            vid[a] = elems[a * elem_ld + e];
            if (!row_mask || row_mask[vid[a]]) touch = 1;
        }
        if (!touch) continue;
        double X[16], Ke[16], Me[16];
        for (int a = 0; a < nv; a++)
            for (int c = 0; c < dim; c++) X[c * nv + a] = coords[c * comp_stride + (int64_t)vid[a] * node_stride];
        orc_p1_local(dim, X, Ke, Me);
        for (int a = 0; a < nv; a++) {
            if (row_mask && !row_mask[vid[a]]) continue;
            for (int b = 0; b < nv; b++) {
                int64_t p = find_col(row_ptr, col_idx, vid[a], vid[b]);
                if (p < 0) return -3;
                if (K) K[p] += Ke[a * nv + b];
                if (M) M[p] += Me[a * nv + b];
            }
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------- NEXT-1: coefficients */

/* intquad(gqo, dim): quadrature on the reference simplex as
 * barycentric points lam[q*(dim+1) + a] and weights w[q] summing to |T_ref| =
 * 1/d!.  The paper's own point sets are not printed; reading:
 * gqo = 1: the centroid; gqo = 2: the symmetric degree-2 rules -- 2D: the three
 * points (2/3, 1/6, 1/6) and permutations, w = 1/6; 3D: the four points
 * (a, b, b, b) and permutations, a = (5 + 3 sqrt5)/20, b = (5 - sqrt5)/20,
 * w = 1/24.  Returns nip, or -1 if (dim, gqo) is not supported. */
int orc_quad_rule(int dim, int gqo, double* lam, double* w) {
    int nv = dim + 1;
    if (gqo == 1) {
        for (int a = 0; a < nv; a++) lam[a] = 1.0 / (double)nv;
        w[0] = 1.0 / (double)factorial(dim);
        return 1;
    }
    if (gqo == 2 && dim == 2) {
        for (int q = 0; q < 3; q++) {
            for (int a = 0; a < 3; a++) lam[q * 3 + a] = (a == q) ? 2.0 / 3.0 : 1.0 / 6.0;
            w[q] = 1.0 / 6.0;
        }
        return 3;
    }
    if (gqo == 2 && dim == 3) {
        double pa = (5.0 + 3.0 * sqrt(5.0)) / 20.0, pb = (5.0 - sqrt(5.0)) / 20.0;
        for (int q = 0; q < 4; q++) {
            for (int a = 0; a < 4; a++) lam[q * 4 + a] = (a == q) ? pa : pb;
            w[q] = 1.0 / 24.0;
        }
        return 4;
    }
    /* gqo = 4 (P2): degree-4 rules -- 2D: Dunavant's 6 points,
     * (1-2a, a, a) and permutations for (a, w) = (0.44594849091596488632,
     * 0.22338158967801146570/2), (0.09157621350977074346, 0.10995174365532186764/2);
     * 3D: Keast's 11 points -- centroid with w = -74/5625, (11/14, 1/14, 1/14, 1/14)
     * and permutations with w = 343/45000, (a, a, b, b) and permutations with
     * a = (1 + sqrt(5/14))/4, b = (1 - sqrt(5/14))/4, w = 56/2250. */
    if (gqo == 4 && dim == 2) {
        const double as[2] = {0.44594849091596488632, 0.09157621350977074346};
        const double ws[2] = {0.22338158967801146570, 0.10995174365532186764};
        int q = 0;
        for (int k = 0; k < 2; k++)
            for (int p = 0; p < 3; p++) {
                for (int a = 0; a < 3; a++) lam[q * 3 + a] = (a == p) ? 1.0 - 2.0 * as[k] : as[k];
                w[q] = ws[k] / 2.0;
                q++;
            }
        return 6;
    }
    if (gqo == 4 && dim == 3) {
        int q = 0;
        for (int a = 0; a < 4; a++) lam[a] = 0.25;
        w[q++] = -74.0 / 5625.0;
        for (int p = 0; p < 4; p++) {
            for (int a = 0; a < 4; a++) lam[q * 4 + a] = (a == p) ? 11.0 / 14.0 : 1.0 / 14.0;
            w[q++] = 343.0 / 45000.0;
        }
        const double pa = (1.0 + sqrt(5.0 / 14.0)) / 4.0, pb = (1.0 - sqrt(5.0 / 14.0)) / 4.0;
        for (int i = 0; i < 4; i++)
            for (int j = i + 1; j < 4; j++) {
                for (int a = 0; a < 4; a++) lam[q * 4 + a] = (a == i || a == j) ? pa : pb;
                w[q++] = 56.0 / 2250.0;
            }
        return 11;
    }
    return -1;
}

/* c(x) = ca * exp(cb . x): the coefficient functions of eq:K_M;
 * c = 1 is ca = 1, cb = 0; the paper's benchmarks use ca = 1, cb = (1,..,1)
 * (c = e^{x1+x2(+x3)}).  coeffs_in_ip evaluates it at
 * the quadrature points x_q = sum_a lam_qa x_a. */
static double coef_eval(int dim, double ca, const double* cb, const double* x) {
    double s = 0.0;
    for (int c = 0; c < dim; c++) s = s + cb[c] * x[c];
    return ca * exp(s);
}

/* Element matrices with coefficients, step by step as Code stiff_scalar_P1
 * and the mass analogue of Code mass_scalar_P2:
 *   for each quadrature point q:  K_e += w_q * (|det| * (c_K(x_q) * G^T G))
 *                                  M_e += w_q * (|det| * (c_M(x_q) * phi_q phi_q^T))
 * with G = tjac^{-1} D from phider, phi_q = lam_q for P1. */
int orc_p1_local_coef(int dim, const double* X, int gqo, double cKa, const double* cKb, double cMa,
                      const double* cMb, double* Ke, double* Me) {
    int nv = dim + 1;
    double lam[64], w[16];
    int nip = orc_quad_rule(dim, gqo, lam, w);
    if (nip < 0) return ORC_ERR_ARG;
    double J[16], Jinv[16], G[16];
    for (int r = 0; r < dim; r++)
        for (int c = 0; c < dim; c++) J[r * 4 + c] = X[c * nv + (r + 1)] - X[c * nv + 0];
    double detJ = det_laplace(J, dim);
    double adet = fabs(detJ);
    for (int i = 0; i < dim; i++)
        for (int j = 0; j < dim; j++) {
            double cof = minor_rc(J, dim, j, i);
            if ((i + j) % 2) cof = -cof;
            Jinv[i * 4 + j] = cof / detJ;
        }
    for (int r = 0; r < dim; r++)
        for (int a = 0; a < nv; a++) {
            double s = 0.0;
            for (int l = 0; l < dim; l++) {
                double dla = (a == 0) ? -1.0 : (l == a - 1 ? 1.0 : 0.0);
                s = s + Jinv[r * 4 + l] * dla;
            }
            G[r * 4 + a] = s;
        }
    for (int p = 0; p < nv * nv; p++) {
        Ke[p] = 0.0;
        Me[p] = 0.0;
    }
    for (int q = 0; q < nip; q++) {
        double xq[3];
        for (int c = 0; c < dim; c++) {
            double s = 0.0;
            for (int a = 0; a < nv; a++) s = s + lam[q * nv + a] * X[c * nv + a];
            xq[c] = s;
        }
        double cK = coef_eval(dim, cKa, cKb, xq), cM = coef_eval(dim, cMa, cMb, xq);
        for (int a = 0; a < nv; a++)
            for (int b = 0; b < nv; b++) {
                double gtg = 0.0;
                for (int r = 0; r < dim; r++) gtg = gtg + G[r * 4 + a] * G[r * 4 + b];
                Ke[a * nv + b] = Ke[a * nv + b] + w[q] * (adet * (cK * gtg));
                Me[a * nv + b] = Me[a * nv + b] + w[q] * (adet * (cM * (lam[q * nv + a] * lam[q * nv + b])));
            }
    }
    return ORC_OK;
}

/* Assembly with coefficients: O11 with orc_p1_local_coef in place of O9. */
int orc_p1_assemble_coef(int dim, int64_t nn, int64_t ne, const double* coords, int64_t node_stride,
                         int64_t comp_stride, const int32_t* elems, int64_t elem_ld,
                         const int32_t* row_ptr, const int32_t* col_idx, int gqo, double cKa,
                         const double* cKb, double cMa, const double* cMb, double* K, double* M) {
    int nv = dim + 1;
    int64_t nnz = row_ptr[nn];
    for (int64_t p = 0; p < nnz; p++) {
        K[p] = 0.0;
        M[p] = 0.0;
    }
    for (int64_t e = 0; e < ne; e++) {
        int32_t vid[4];
        double X[16], Ke[16], Me[16];
        for (int a = 0; a < nv; a++) vid[a] = elems[a * elem_ld + e];
        for (int a = 0; a < nv; a++)
            for (int c = 0; c < dim; c++) X[c * nv + a] = coords[c * comp_stride + (int64_t)vid[a] * node_stride];
        int rc = orc_p1_local_coef(dim, X, gqo, cKa, cKb, cMa, cMb, Ke, Me);
        if (rc) return rc;
        for (int a = 0; a < nv; a++)
            for (int b = 0; b < nv; b++) {
                int64_t p = find_col(row_ptr, col_idx, vid[a], vid[b]);
                if (p < 0) return -3;
                K[p] += Ke[a * nv + b];
                M[p] += Me[a * nv + b];
            }
    }
    return ORC_OK;
}

/* ------------------------------------------------------- NEXT-2: rhs, energies */

/* avtamav (eq:layeredBilin P:292-301): s_k = a_k^T M_k b_k for
 * pages a (n x 1), M (n x m), b (m x 1); computed as sum_i a_i (sum_j M_ij b_j),
 * j and i ascending. */
int orc_page_bilinear(int64_t np, int n, int m, const double* A, int64_t lda, const double* Mx, int64_t ldm,
                      const double* B, int64_t ldb, double* s) {
    for (int64_t k = 0; k < np; k++) {
        double acc = 0.0;
        for (int i = 0; i < n; i++) {
            double t = 0.0;
            for (int j = 0; j < m; j++) t = t + at(Mx, ldm, n, i, j, k) * at(B, ldb, m, j, 0, k);
            acc = acc + at(A, lda, n, i, 0, k) * t;
        }
        s[k] = acc;
    }
    return ORC_OK;
}

/* Code rhs_vectorP1: b2D(j, e) = sum_i w_i |det_e| f(x_ie) phi_j(ip_i)
 * (loop over integration points as written: b2D = b2D + w(i)*detj_abs'.*integrand_i,
 * detj_abs = sizes*factorial(dim)), then b = accumarray(elems(:), b2D(:)) (e
 * ascending, local vertex ascending).  fq holds f at the integration points,
 * plane i (ld = ne), in the point order of orc_quad_rule.  b2D (nv planes of
 * ne) and b (nn) are nullable. */
int orc_p1_rhs(int dim, int64_t nn, int64_t ne, const double* coords, int64_t node_stride, int64_t comp_stride,
               const int32_t* elems, int64_t elem_ld, int gqo, const double* fq, double* b2D, double* b) {
    int nv = dim + 1;
    double lam[64], w[16];
    int nip = orc_quad_rule(dim, gqo, lam, w);
    if (nip < 0) return ORC_ERR_ARG;
    if (b)
        for (int64_t v = 0; v < nn; v++) b[v] = 0.0;
    for (int64_t e = 0; e < ne; e++) {
        double X[16], J[16];
        for (int a = 0; a < nv; a++) {
            int64_t v = elems[a * elem_ld + e];
            for (int c = 0; c < dim; c++) X[c * nv + a] = coords[c * comp_stride + v * node_stride];
        }
        for (int r = 0; r < dim; r++)
            for (int c = 0; c < dim; c++) J[r * 4 + c] = X[c * nv + (r + 1)] - X[c * nv + 0];
        double detj_abs = fabs(det_laplace(J, dim));
        double loc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int i = 0; i < nip; i++)
            for (int a = 0; a < nv; a++) {
                double integrand = fq[(int64_t)i * ne + e] * lam[i * nv + a];
                loc[a] = loc[a] + w[i] * (detj_abs * integrand);
            }
        for (int a = 0; a < nv; a++) {
            if (b2D) b2D[(int64_t)a * ne + e] = loc[a];
            if (b) b[elems[a * elem_ld + e]] += loc[a];
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------- NEXT-3: P2 elements */

static const int P2_EDGE_2D[3][2] = {{0, 1}, {1, 2}, {0, 2}};
static const int P2_EDGE_3D[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

/* shapefun / shapeder for P2: vertex a: lam_a (2 lam_a - 1); edge
 * (i, j): 4 lam_i lam_j (node order: vertices, then edges in the canonical
 * order of SPEC S:304).  Reference coordinates xi_r = lam_{r+1}, lam_0 = 1 - sum xi;
 * dshape[r][k] = d phi_k / d xi_r. */
static void p2_shape(int dim, const double* lam, double* phi, double* dshape /* dim x nlb, [r*10 + k] */) {
    int nv = dim + 1, ne = dim == 2 ? 3 : 6;
    const int(*E)[2] = dim == 2 ? P2_EDGE_2D : P2_EDGE_3D;
    double dl[10][4];  /* d phi_k / d lam_b */
    for (int k = 0; k < 10; k++)
        for (int b = 0; b < 4; b++) dl[k][b] = 0.0;
    for (int a = 0; a < nv; a++) {
        phi[a] = lam[a] * (2.0 * lam[a] - 1.0);
        dl[a][a] = 4.0 * lam[a] - 1.0;
    }
    for (int k = 0; k < ne; k++) {
        int i = E[k][0], j = E[k][1];
        phi[nv + k] = 4.0 * lam[i] * lam[j];
        dl[nv + k][i] = 4.0 * lam[j];
        dl[nv + k][j] = 4.0 * lam[i];
    }
    for (int r = 0; r < dim; r++)
        for (int k = 0; k < nv + ne; k++) dshape[r * 10 + k] = dl[k][r + 1] - dl[k][0];
}

/* Element matrices of stiffness_matrixP2 / mass_matrixP2, point by
 * point as Code phider and Code mass_scalar_P2:
 *   tjac = dshape * X^T over all nlb nodes (the iso-parametric map), jacinv, detj,
 *   dphi = jacinv * dshape;  K_e += w_q (|det| (c_K(x_q) dphi^T dphi));
 *   M_e += w_q (|det| (c_M(x_q) phi phi^T)),  x_q = sum_k phi_k(q) x_k.
 * X[c*nlb + k]: coordinate c of node k.  Ke, Me: nlb x nlb row-major. */
int orc_p2_local_coef(int dim, const double* X, int gqo, double cKa, const double* cKb, double cMa,
                      const double* cMb, double* Ke, double* Me) {
    int nv = dim + 1, nlb = dim == 2 ? 6 : 10;
    double lam[64], w[16];
    int nip = orc_quad_rule(dim, gqo, lam, w);
    if (nip < 0) return ORC_ERR_ARG;
    for (int p = 0; p < nlb * nlb; p++) {
        Ke[p] = 0.0;
        Me[p] = 0.0;
    }
    for (int q = 0; q < nip; q++) {
        double phi[10], ds[30], J[16], Jinv[16], dphi[30];
        p2_shape(dim, lam + q * nv, phi, ds);
        for (int r = 0; r < dim; r++)
            for (int c = 0; c < dim; c++) {
                double s = 0.0;
                for (int k = 0; k < nlb; k++) s = s + ds[r * 10 + k] * X[c * nlb + k];
                J[r * 4 + c] = s;
            }
        double detJ = det_laplace(J, dim);
        for (int i = 0; i < dim; i++)
            for (int j = 0; j < dim; j++) {
                double cof = minor_rc(J, dim, j, i);
                if ((i + j) % 2) cof = -cof;
                Jinv[i * 4 + j] = cof / detJ;
            }
        for (int r = 0; r < dim; r++)
            for (int k = 0; k < nlb; k++) {
                double s = 0.0;
                for (int l = 0; l < dim; l++) s = s + Jinv[r * 4 + l] * ds[l * 10 + k];
                dphi[r * 10 + k] = s;
            }
        double xq[3];
        for (int c = 0; c < dim; c++) {
            double s = 0.0;
            for (int k = 0; k < nlb; k++) s = s + phi[k] * X[c * nlb + k];
            xq[c] = s;
        }
        double cK = coef_eval(dim, cKa, cKb, xq), cM = coef_eval(dim, cMa, cMb, xq);
        double adet = fabs(detJ);
        for (int a = 0; a < nlb; a++)
            for (int b = 0; b < nlb; b++) {
                double gtg = 0.0;
                for (int r = 0; r < dim; r++) gtg = gtg + dphi[r * 10 + a] * dphi[r * 10 + b];
                Ke[a * nlb + b] = Ke[a * nlb + b] + w[q] * (adet * (cK * gtg));
                Me[a * nlb + b] = Me[a * nlb + b] + w[q] * (adet * (cM * (phi[a] * phi[b])));
            }
    }
    return ORC_OK;
}

/* P2 assembly: sparse() of the nlb x nlb element matrices, O11 order. */
int orc_p2_assemble_coef(int dim, int64_t nn, int64_t ne, const double* coords, int64_t node_stride,
                         int64_t comp_stride, const int32_t* elems, int64_t elem_ld,
                         const int32_t* row_ptr, const int32_t* col_idx, int gqo, double cKa,
                         const double* cKb, double cMa, const double* cMb, double* K, double* M) {
    int nlb = dim == 2 ? 6 : 10;
    int64_t nnz = row_ptr[nn];
    for (int64_t p = 0; p < nnz; p++) {
        K[p] = 0.0;
        M[p] = 0.0;
    }
    for (int64_t e = 0; e < ne; e++) {
        int32_t vid[10];
        double X[30], Ke[100], Me[100];
        for (int a = 0; a < nlb; a++) vid[a] = elems[a * elem_ld + e];
        for (int a = 0; a < nlb; a++)
            for (int c = 0; c < dim; c++) X[c * nlb + a] = coords[c * comp_stride + (int64_t)vid[a] * node_stride];
        int rc = orc_p2_local_coef(dim, X, gqo, cKa, cKb, cMa, cMb, Ke, Me);
        if (rc) return rc;
        for (int a = 0; a < nlb; a++)
            for (int b = 0; b < nlb; b++) {
                int64_t p = find_col(row_ptr, col_idx, vid[a], vid[b]);
                if (p < 0) return -3;
                K[p] += Ke[a * nlb + b];
                M[p] += Me[a * nlb + b];
            }
    }
    return ORC_OK;
}

/* ------------------------------------------------- NEXT-4: GI */

/* Code GI as written:
 *   f_elems(e, c) = sum_q fip(c, q, e) w(q)             (amsv(fip, w), q ascending)
 *   with normals:  g_e = sum_c f_elems(e, c) normals(e, c)   (c ascending)
 *   without:       g_e = f_elems(e, 0)                  (d must be 1)
 *   value = sum_e sizes(e) g_e                          (sum over e ascending, Neumaier-compensated)
 * fip: d x nip pages, entry (c, q) of page e at fip[(c + q*d)*ld + e]; normals:
 * d planes of ne (plane stride nld), NULL for a scalar integrand.
 * Returns 0, or -1 for d != 1 without normals. */
int orc_gi(int64_t ne, int d, int nip, const double* fip, int64_t ld, const double* w, const double* sizes,
           const double* normals, int64_t nld, double* value) {
    if (!normals && d != 1) return -1;
    double s = 0.0, comp = 0.0;
    for (int64_t e = 0; e < ne; e++) {
        double g = 0.0;
        for (int c = 0; c < d; c++) {
            double f = 0.0;
            for (int q = 0; q < nip; q++) f = f + at(fip, ld, d, c, q, e) * w[q];
            g = normals ? g + f * normals[c * nld + e] : f;
        }
        double x = sizes[e] * g;
        double t = s + x;
        if (fabs(s) >= fabs(x)) comp += (s - t) + x;
        else comp += (x - t) + s;
        s = t;
    }
    *value = s + comp;
    return ORC_OK;
}
