// Element-once 3D P1 K+M assembly on Kuhn lattices (the headline path of
// SURVEY §8(a) a7-a17 for BASELINE configs[4]).
//
// What is computed is exactly fem_p1_assemble's K and M with c = 1 (eq:K_M
// P:967-975, Code stiff_scalar_P1 P:978-1004, mass P:1007, accumulated as
// sparse(X3D(:), Y3D(:), K3D(:)) P:1001-1003): per element tjac = D X^T
// (P:941), |T| = |det|/6, G = tjac^{-1} D, K_e = |T| G^T G
// (P:996), M_e = |T|/20 (1 + delta_ab); here K_e[a][b] = (h_a . h_b) / (6 |det|)
// with h_r the adjugate columns (h_1 = f_2 x f_3, h_2 = f_3 x f_1,
// h_3 = f_1 x f_2, h_0 = -(h_1 + h_2 + h_3); f_r = x_r - x_0), the same
// quantity as |T| grad(phi_a) . grad(phi_b) (Remark rem:phider P:955-965: the
// whole chain is page-wise per element).
//
// The mesh is a Kuhn lattice: nodes (i, j, k), 0 <= i <= nx, ..., numbered
// id = i + (nx+1)(j + (ny+1) k); each cell split into the 6 tetrahedra of the
// monotone paths of one cell diagonal (SURVEY §8(d) config 5 recipe; any of
// the four diagonals, any element order, any vertex order inside an element).
// fem_plan_lattice verifies that once per mesh (every element is one Kuhn
// tetrahedron, no two are the same; the CSR pattern is the lattice stencil),
// so the numeric phase reads no connectivity: the element list is implicit.
// Working in canonical lattice coordinates (axes mirrored so that the split
// diagonal runs from (0,0,0) to (1,1,1)), node p owns its 7 "up" edges
// +x, +y, +z, +xy, +xz, +yz, +xyz (every mesh edge exactly once).  Cell c
// (corner 000 at node c) contributes to 19 of them: the 7 of its own corner
// 000 and 3 / 3 / 3 / 1 / 1 / 1 of corners 100 / 010 / 001 / 110 / 101 / 011.
//
// Kernel (assemble_lattice_k): a CTA holds a tile of 32 lanes (x) x LR warp
// rows (y) of lattice columns and marches along z, one node layer per step,
// evaluating every cell (6 tets) ONCE.  Contributions move to the owning node
// by warp shuffle (x), shared memory (y) and registers (z).  The first lane of
// every x segment and row 0 of every band after the first are halos (their
// cells are recomputed by the neighbouring tile); a halo lane left of x = 0 is
// a virtual node whose (absent) cells contribute exact zeros, so no received
// value needs masking.  Rows of CSR are assembled in registers (14 edges;
// diagonals by the partition of unity, K_pp = -sum_q K_pq, M_pp = (2/3)
// sum_q M_pq, as the gather variants), staged in shared memory and leave as
// TMA bulk copies (cp.async.bulk; K and M of a segment in one statement issued by
// one elected lane, committed a step later).  The CTAs' ranges of the tile-layer
// sequence are cost-balanced once per mesh and kept in the plan (lat_ranges).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "vb_internal.cuh"

namespace vb {
namespace {

#ifndef VB_LAT_R
#define VB_LAT_R 12
#endif
#ifndef VB_LAT_MINB
#define VB_LAT_MINB 1
#endif
#ifndef VB_LAT_KO
#define VB_LAT_KO 0   // timing knock-outs (wrong results; tools/ab_time.sh): 1 no bulk stores, 2 no cell arithmetic, 3 both
#endif
constexpr int LR = VB_LAT_R;      // warp rows per tile (row 0 may be a halo line)
constexpr int LCOLS = 40;         // coordinate columns per row (lanes + one gap per segment)
#ifndef VB_LAT_NBUF
#define VB_LAT_NBUF 5
#endif
constexpr int LNBUF = VB_LAT_NBUF;   // coordinate layer buffers: layer Lz + LNBUF - 1 is fetched at the start of step Lz
constexpr int LDIST = LNBUF - 1;     // (configs[4]: 3 buffers 0.1725 ms, 4 buffers 0.1622, 5 buffers 0.1601; issuing the
                                     // fetch behind the bulk wait, which shares its scoreboard, changed nothing)
constexpr int LSTG = 31 * 15 + 3;    // staging doubles per matrix and warp row: 31 rows + the parity offset, 16-byte multiple
constexpr int LTHREADS = 32 * LR;
constexpr int LMAXCTA = 1024;     // CTA ranges kept in the plan
constexpr uint32_t LAT_MAGIC = 0x4c415431u;   // "LAT1"

// stencil directions: 0 self, 1..7 = +x +y +z +xy +xz +yz +xyz, 8..14 the negatives
__host__ __device__ constexpr int dir_dx(int d) { return d == 0 ? 0 : (d <= 7 ? 1 : -1) * ((d - 1) % 7 == 0 || (d - 1) % 7 == 3 || (d - 1) % 7 == 4 || (d - 1) % 7 == 6); }
__host__ __device__ constexpr int dir_dy(int d) { return d == 0 ? 0 : (d <= 7 ? 1 : -1) * ((d - 1) % 7 == 1 || (d - 1) % 7 == 3 || (d - 1) % 7 == 5 || (d - 1) % 7 == 6); }
__host__ __device__ constexpr int dir_dz(int d) { return d == 0 ? 0 : (d <= 7 ? 1 : -1) * ((d - 1) % 7 == 2 || (d - 1) % 7 == 4 || (d - 1) % 7 == 5 || (d - 1) % 7 == 6); }

// CSR column order of the stencil for orientation (FY, FZ) (canonical x never mirrored): column ids
// id0 + I + sy (nx+1) J + sz (nx+1)(ny+1) K sort lexicographically by (sz dz, sy dy, dx) when nx, ny >= 2;
// fem_plan_lattice refuses lattices where the real order differs.  LOW[d] = directions before d.
__host__ __device__ constexpr long long lex_off(int d, int FY, int FZ) {
    return dir_dx(d) + (FY ? -4 : 4) * dir_dy(d) + (FZ ? -16 : 16) * dir_dz(d);
}
template <int FY, int FZ>
struct Order {
    uint32_t low[15];
    int slot[15];   // position in an interior row (all 15 present)
    __host__ __device__ constexpr Order() : low(), slot() {
        for (int d = 0; d < 15; d++) {
            uint32_t m = 0;
            int c = 0;
            for (int e = 0; e < 15; e++)
                if (lex_off(e, FY, FZ) < lex_off(d, FY, FZ)) { m |= 1u << e; c++; }
            low[d] = m;
            slot[d] = c;
        }
    }
};

struct LatParams {
    int nx, ny, nz, T;            // cells per axis, tiles
    int64_t L;                    // T * (nz + 1) tile-layers
    int id0, dJ, dK;              // node id of canonical (I, J, K) = id0 + I + dJ J + dK K
    const double* X;
    int64_t ns, cs;               // coordinate addressing X[c*cs + v*ns]
    const int32_t* row_ptr;
    double* Kv;
    double* Mv;
    const int4* lanes;            // T x 32 lane descriptors
    const uint32_t* token;        // plan token (LAT_MAGIC ^ hash) written by fem_plan_lattice
    uint32_t want;
    int bulk;                     // K, M 16-byte aligned: rows leave as bulk copies
    const int32_t* range;         // plan: CTA c owns tile-layers [range[c], range[c+1]) (cost-balanced)
};

// lane descriptor (int4): x = I (canonical x of the lane's node, -1 for the virtual halo left of x = 0,
// -2: idle lane), y = J0 (canonical y of row 0), z = flags | col << 8 | first owned lane << 16 |
// last lane << 24, w = staging base of the segment
enum : int { LF_OWNX = 1, LF_XPLUS = 4, LF_ROW0 = 8, LF_HEAD = 16, LF_BULK = 32 };

struct LatSmem {
    double X[LNBUF][3][LR + 1][LCOLS];   // node coordinates of a layer, [comp][row][column]
    double P[LR][10][32];                // cell -> next row: c010 (+x,+z,+xz), c110 (+z), c011 (+x); K then M
    double Ein[LR][4][32];               // finished in-plane edges for the next row: +y, +xy (K, M)
    double Ez[2][LR][4][32];             // finished z-edges for the next row, by layer parity: +yz, +xyz
    double S[LR][2][LSTG];               // CSR staging (K, M) of a warp row
};

__device__ __forceinline__ uint32_t smem_u32l(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cpa8(double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32l(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// K and M rows of one segment as two bulk copies in ONE statement: every operand is in its (uniform) register
// before the first copy issues; two statements made the second one's operand setup wait for the first copy to
// release the registers it shares
__device__ __forceinline__ void bulk_st2(double* dk, const double* sk, double* dm, const double* sm, int bytes) {
    asm volatile(
        "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %4;\n"
        "cp.async.bulk.global.shared::cta.bulk_group [%2], [%3], %4;" ::"l"(dk),
        "r"(smem_u32l(sk)), "l"(dm), "r"(smem_u32l(sm)), "r"(bytes)
        : "memory");
}
__device__ __forceinline__ void bulk_st(double* dst, const double* src, int bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32l(src)),
                 "r"(bytes)
                 : "memory");
}

// 1/x: hardware seed and two Newton steps (as the gather kernels)
__device__ __forceinline__ double rcp2(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(y, fma(-x, y, 1.0), y);
    y = fma(y, fma(-x, y, 1.0), y);
    return y;
}
__device__ __forceinline__ void crs(const double (&a)[3], const double (&b)[3], double (&c)[3]) {
    c[0] = fma(a[1], b[2], -a[2] * b[1]);
    c[1] = fma(a[2], b[0], -a[0] * b[2]);
    c[2] = fma(a[0], b[1], -a[1] * b[0]);
}
__device__ __forceinline__ double dot3(const double (&a)[3], const double (&b)[3]) {
    return fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
}

struct Tet {
    double k01, k02, k03, k12, k13, k23, m;
};
// One tetrahedron v0, v1 = v0 + f1, v2 = v0 + f2, v3 = v0 + f3 (tjac rows f_r) with
// h1 = f2 x f3 and h2 = f3 x f1 given (shared between the cell's tets): K_e off-diagonals and
// the mass off-diagonal |T|/20 = |det|/120.  CHK: live = false (no such cell) gives exact zeros
// (the coordinates are finite, s = 0).
template <bool CHK>
__device__ __forceinline__ Tet tet(const double (&f1)[3], const double (&f2)[3], const double (&h1)[3],
                                   const double (&h2)[3], bool live) {
    double h3[3];
    crs(f1, f2, h3);
    const double det = dot3(f1, h1);
    const double ad = CHK ? (live ? fabs(det) : 0.0) : fabs(det);
    const double r = rcp2(6.0 * ad);
    const double s = CHK ? (live ? r : 0.0) : r;
    double h0[3];
#pragma unroll
    for (int c = 0; c < 3; c++) h0[c] = -(h1[c] + h2[c] + h3[c]);
    Tet t;
    t.k01 = s * dot3(h0, h1);
    t.k02 = s * dot3(h0, h2);
    t.k03 = s * dot3(h0, h3);
    t.k12 = s * dot3(h1, h2);
    t.k13 = s * dot3(h1, h3);
    t.k23 = s * dot3(h2, h3);
    t.m = ad * (1.0 / 120.0);
    return t;
}

// The 6 Kuhn tetrahedra of one cell (corner 000 at x0[0], layer buffers x0 / x1 of the cell's bottom /
// top nodes, columns +1 = +x, +LCOLS = +y), each evaluated once, routed to the 19 up edges the cell
// touches (corner 000: e, corners 100: c100, 010 / 110 / 011: o, 101: c101, 001: c001).  Paths in
// lexicographic order: (x,y,z) (x,z,y) (y,x,z) (y,z,x) (z,x,y) (z,y,x); t.m = |det|/120 of each.
struct Cell {
    double e[7];      // +x +y +z +xy +xz +yz +xyz
    double c100[3];   // +y +z +yz
    double o[5];      // c010: +x +z +xz, c110: +z, c011: +x
    double c101;      // +y
    double c001[3];   // +x +y +xy
};
template <bool CHK>
__device__ __forceinline__ void cell(const double* x0, const double* x1, bool live, Cell& K, Cell& M) {
    double x000[3], ux[3], uy[3], uz[3], wxy[3], wxz[3], wyz[3], bd[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
        x000[c] = x0[c * ((LR + 1) * LCOLS)];
        ux[c] = x0[c * ((LR + 1) * LCOLS) + 1] - x000[c];
        uy[c] = x0[c * ((LR + 1) * LCOLS) + LCOLS] - x000[c];
        wxy[c] = x0[c * ((LR + 1) * LCOLS) + LCOLS + 1] - x000[c];
        uz[c] = x1[c * ((LR + 1) * LCOLS)] - x000[c];
        wxz[c] = x1[c * ((LR + 1) * LCOLS) + 1] - x000[c];
        wyz[c] = x1[c * ((LR + 1) * LCOLS) + LCOLS] - x000[c];
        bd[c] = x1[c * ((LR + 1) * LCOLS) + LCOLS + 1] - x000[c];
    }
    double hxy[3], hxz[3], hyz[3];
    crs(wxy, bd, hxy);
    crs(wxz, bd, hxz);
    crs(wyz, bd, hyz);
    double mxyz, mxzy, myxz, myzx, mzxy, mzyx;
    {   // paths starting along x
        double h2[3];
        crs(bd, ux, h2);
        const Tet a = tet<CHK>(ux, wxy, hxy, h2, live);
        const Tet b = tet<CHK>(ux, wxz, hxz, h2, live);
        K.e[0] = a.k01 + b.k01;
        K.e[3] = a.k02;
        K.e[4] = b.k02;
        K.e[6] = a.k03 + b.k03;
        K.c100[0] = a.k12;
        K.c100[1] = b.k12;
        K.c100[2] = a.k13 + b.k13;
        K.o[3] = a.k23;
        K.c101 = b.k23;
        mxyz = a.m;
        mxzy = b.m;
    }
    {   // (y,x,z), (y,z,x)
        double h2[3];
        crs(bd, uy, h2);
        const Tet a = tet<CHK>(uy, wxy, hxy, h2, live);
        const Tet b = tet<CHK>(uy, wyz, hyz, h2, live);
        K.e[1] = a.k01 + b.k01;
        K.e[3] += a.k02;
        K.e[5] = b.k02;
        K.e[6] += a.k03 + b.k03;
        K.o[0] = a.k12;
        K.o[1] = b.k12;
        K.o[2] = a.k13 + b.k13;
        K.o[3] += a.k23;
        K.o[4] = b.k23;
        myxz = a.m;
        myzx = b.m;
    }
    {   // (z,x,y), (z,y,x)
        double h2[3];
        crs(bd, uz, h2);
        const Tet a = tet<CHK>(uz, wxz, hxz, h2, live);
        const Tet b = tet<CHK>(uz, wyz, hyz, h2, live);
        K.e[2] = a.k01 + b.k01;
        K.e[4] += a.k02;
        K.e[5] += b.k02;
        K.e[6] += a.k03 + b.k03;
        K.c001[0] = a.k12;
        K.c001[1] = b.k12;
        K.c001[2] = a.k13 + b.k13;
        K.c101 += a.k23;
        K.o[4] += b.k23;
        mzxy = a.m;
        mzyx = b.m;
    }
    // every edge of a tetrahedron carries its |det|/120: the same routing with six values
    const double px = mxyz + mxzy, py = myxz + myzx, pz = mzxy + mzyx;
    const double qxy = mxyz + myxz, qxz = mxzy + mzxy, qyz = myzx + mzyx;
    M.e[0] = px; M.e[1] = py; M.e[2] = pz; M.e[3] = qxy; M.e[4] = qxz; M.e[5] = qyz; M.e[6] = (px + py) + pz;
    M.c100[0] = mxyz; M.c100[1] = mxzy; M.c100[2] = px;
    M.o[0] = myxz; M.o[1] = myzx; M.o[2] = py; M.o[3] = qxy; M.o[4] = qyz;
    M.c101 = qxz;
    M.c001[0] = mzxy; M.c001[1] = mzyx; M.c001[2] = pz;
}

// edge slots of the owned-edge arrays: +x +y +z +xy +xz +yz +xyz
enum { EX = 0, EY, EZ, EXY, EXZ, EYZ, EXYZ };

__device__ __forceinline__ double shup(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }

constexpr int XB = 3 * (LR + 1) * LCOLS;   // doubles per coordinate layer buffer
constexpr int XC = (LR + 1) * LCOLS;       // doubles per component plane

// 12 warps: 3 per SM sub-partition, whose 16 K registers allow 168 per thread; a 13th warp (4 on one
// sub-partition) would cap the kernel at 128 registers (ptxas then spills) and 16 rows do not fit 227 KB.
template <int FY, int FZ>
__global__ void __launch_bounds__(LTHREADS, VB_LAT_MINB) assemble_lattice_k(const LatParams p) {
    constexpr Order<FY, FZ> ORD{};
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LatSmem& S = *reinterpret_cast<LatSmem*>(smem_raw);
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    if (*p.token != p.want) return;   // plan of another mesh / not verified: write nothing
    // coordinates of nodes never loaded must be finite: zero the layer buffers once
    for (int i = threadIdx.x; i < LNBUF * XB; i += LTHREADS) (&S.X[0][0][0][0])[i] = 0.0;
#ifdef VB_LAT_PROF
    long long t_start = clock64();
#endif

    const int64_t g0 = __ldg(p.range + blockIdx.x), g1 = __ldg(p.range + blockIdx.x + 1);
    VB_CHECK(g0 >= 0 && g0 <= g1 && g1 <= p.L);
    const int NK = p.nz + 1;
    const int64_t plane = p.dK;   // node id step per layer
    double* const SK = S.S[w][0];
    double* const SM = S.S[w][1];
    int64_t g = g0;
    while (g < g1) {
        const int tau = (int)(g / NK);
        const int ka = (int)(g % NK);
        const int64_t gend = (int64_t)(tau + 1) * NK < g1 ? (int64_t)(tau + 1) * NK : g1;
        const int kb = (int)(gend - (int64_t)tau * NK);   // node layers [ka, kb)
        g = gend;

        const int4 ds = p.lanes[tau * 32 + lane];
        const int I = ds.x;
        const int J = ds.y + w;
        const int fl = ds.z & 0xff;
        const int col = (ds.z >> 8) & 0xff;
        const int lfirst = (ds.z >> 16) & 0xff;
        const int llast = (ds.z >> 24) & 0xff;
        const bool node = I >= 0 && J <= p.ny;                      // a real lattice node
        const bool owned = node && (fl & LF_OWNX) && (w > 0 || (fl & LF_ROW0));
        const bool cellxy = node && I < p.nx && J < p.ny;           // cell (I, J, .) exists
        const bool xplus = node && (fl & LF_XPLUS) && I < p.nx;
        const int idIJ = p.id0 + I + p.dJ * J;                      // valid where node
        const double* xg = p.X + (int64_t)idIJ * p.ns;              // own node, layer 0
        double* const xs = &S.X[0][0][w][col];

        // coordinate prefetch of node layer Lz into buffer Lz % LNBUF: own node, the +x node of a
        // segment's last lane, and row LR (J + 1) for the last warp row
        auto fetch = [&](int Lz) {
            if (Lz > p.nz) return;
            double* d = xs + (Lz % LNBUF) * XB;
            const double* sg = xg + (int64_t)Lz * plane * p.ns;
            if (node) {
#pragma unroll
                for (int c = 0; c < 3; c++) cpa8(d + c * XC, sg + c * p.cs);
                if (xplus)
#pragma unroll
                    for (int c = 0; c < 3; c++) cpa8(d + c * XC + 1, sg + c * p.cs + p.ns);
            }
            if (w == LR - 1 && I >= 0 && J + 1 <= p.ny) {
                const double* s2 = sg + (int64_t)p.dJ * p.ns;
#pragma unroll
                for (int c = 0; c < 3; c++) cpa8(d + c * XC + LCOLS, s2 + c * p.cs);
                if (xplus)
#pragma unroll
                    for (int c = 0; c < 3; c++) cpa8(d + c * XC + LCOLS + 1, s2 + c * p.cs + p.ns);
            }
        };

        const int Ls = ka > 0 ? ka - 1 : ka;   // one halo layer when the range starts inside the tile
        __syncthreads();                       // previous range's readers of every buffer are done
        static_assert(LDIST >= 2 && LDIST <= 4, "prefetch distance");
        fetch(Ls);
        fetch(Ls + 1);
        cpa_commit();
#pragma unroll
        for (int l = 2; l < LDIST; l++) {   // LDIST - 1 groups in flight
            fetch(Ls + l);
            cpa_commit();
        }
        cpa_wait<LDIST - 2>();
        __syncthreads();

        // carries along z: zc = in-plane up edges (+x, +y, +xy) of this node at the next layer from the
        // cells below it; ez / exz = this node's +z / +xz edge of the previous layer
        double zcK0 = 0, zcK1 = 0, zcK2 = 0, zcM0 = 0, zcM1 = 0, zcM2 = 0;
        double ezK = 0, ezM = 0, exzK = 0, exzM = 0;
        const int32_t* rpp = p.row_ptr + idIJ;
        int rp_next = (Ls >= ka && owned) ? __ldg(rpp + (int64_t)Ls * plane) : 0;   // row_ptr, one step ahead

        for (int Lz = Ls; Lz < kb; Lz++) {
            fetch(Lz + LDIST);
            cpa_commit();
            const bool out = Lz >= ka;
            const int rp = rp_next;
            if (Lz + 1 < kb && owned) rp_next = __ldg(rpp + (int64_t)(Lz + 1) * plane);

            // ---- phase A: the cell (I, J, Lz) -> owned edges eK/eM (+ carries) and outgoing parts
            Cell CK, CM;
            {
                const double* x0 = xs + (Lz % LNBUF) * XB;
                const double* x1 = xs + ((Lz + 1) % LNBUF) * XB;
                const bool live = cellxy && Lz < p.nz;   // the top layer has no cells (coordinates still finite)
#if VB_LAT_KO >= 2
                {
                    const double v = x0[0] + x1[XC + 1 + LCOLS];
                    for (int i = 0; i < 7; i++) CK.e[i] = CM.e[i] = v;
                    for (int i = 0; i < 3; i++) CK.c100[i] = CM.c100[i] = CK.c001[i] = CM.c001[i] = v;
                    for (int i = 0; i < 5; i++) CK.o[i] = CM.o[i] = v;
                    CK.c101 = CM.c101 = v;
                }
#else
                if (__all_sync(0xffffffffu, live)) cell<false>(x0, x1, true, CK, CM);
                else cell<true>(x0, x1, live, CK, CM);
#endif
            }
            double eK[7], eM[7];
            eK[EX] = zcK0 + CK.e[0]; eK[EY] = zcK1 + CK.e[1]; eK[EXY] = zcK2 + CK.e[3];
            eM[EX] = zcM0 + CM.e[0]; eM[EY] = zcM1 + CM.e[1]; eM[EXY] = zcM2 + CM.e[3];
            eK[EZ] = CK.e[2]; eK[EXZ] = CK.e[4]; eK[EYZ] = CK.e[5]; eK[EXYZ] = CK.e[6];
            eM[EZ] = CM.e[2]; eM[EXZ] = CM.e[4]; eM[EYZ] = CM.e[5]; eM[EXYZ] = CM.e[6];
            // ---- phase B: x neighbours by shuffle, the next row through shared memory
            eK[EY] += shup(CK.c100[0]);  eM[EY] += shup(CM.c100[0]);
            eK[EZ] += shup(CK.c100[1]);  eM[EZ] += shup(CM.c100[1]);
            eK[EYZ] += shup(CK.c100[2]); eM[EYZ] += shup(CM.c100[2]);
            zcK0 = CK.c001[0]; zcK1 = CK.c001[1] + shup(CK.c101); zcK2 = CK.c001[2];
            zcM0 = CM.c001[0]; zcM1 = CM.c001[1] + shup(CM.c101); zcM2 = CM.c001[2];
#pragma unroll
            for (int e = 0; e < 5; e++) {
                S.P[w][e][lane] = CK.o[e];
                S.P[w][5 + e][lane] = CM.o[e];
            }
            __syncthreads();

            // ---- phase C: contributions of the row below; publish the finished edges
            if (w > 0) {
                const double* Pb = &S.P[w - 1][0][0];
                eK[EX] += Pb[0 * 32 + lane];  eM[EX] += Pb[5 * 32 + lane];
                eK[EZ] += Pb[1 * 32 + lane] + Pb[3 * 32 + lane - 1];
                eM[EZ] += Pb[6 * 32 + lane] + Pb[8 * 32 + lane - 1];
                eK[EXZ] += Pb[2 * 32 + lane]; eM[EXZ] += Pb[7 * 32 + lane];
                zcK0 += Pb[4 * 32 + lane];    zcM0 += Pb[9 * 32 + lane];
            }
            S.Ein[w][0][lane] = eK[EY];
            S.Ein[w][1][lane] = eM[EY];
            S.Ein[w][2][lane] = eK[EXY];
            S.Ein[w][3][lane] = eM[EXY];
            S.Ez[Lz & 1][w][0][lane] = eK[EYZ];
            S.Ez[Lz & 1][w][1][lane] = eM[EYZ];
            S.Ez[Lz & 1][w][2][lane] = eK[EXYZ];
            S.Ez[Lz & 1][w][3][lane] = eM[EXYZ];
            cpa_wait<LDIST - 2>();   // layer Lz + 2 has landed
            __syncthreads();

            // ---- phase D: the CSR rows of this layer's owned nodes
            // incoming edges (the up edges of the lower neighbours): -x, -y, -z, -xy, -xz, -yz, -xyz
            double iK[7], iM[7];
            iK[0] = shup(eK[EX]);  iM[0] = shup(eM[EX]);
            iK[4] = shup(exzK);    iM[4] = shup(exzM);
            iK[2] = ezK;           iM[2] = ezM;
            if (w > 0) {
                iK[1] = S.Ein[w - 1][0][lane];
                iM[1] = S.Ein[w - 1][1][lane];
                iK[3] = (&S.Ein[w - 1][2][0])[lane - 1];
                iM[3] = (&S.Ein[w - 1][3][0])[lane - 1];
                if (Lz > 0) {
                    const int q = (Lz - 1) & 1;
                    iK[5] = S.Ez[q][w - 1][0][lane];
                    iM[5] = S.Ez[q][w - 1][1][lane];
                    iK[6] = (&S.Ez[q][w - 1][2][0])[lane - 1];
                    iM[6] = (&S.Ez[q][w - 1][3][0])[lane - 1];
                } else {
                    iK[5] = iK[6] = iM[5] = iM[6] = 0.0;
                }
            } else {
                iK[1] = iK[3] = iK[5] = iK[6] = iM[1] = iM[3] = iM[5] = iM[6] = 0.0;
            }
            ezK = eK[EZ]; ezM = eM[EZ]; exzK = eK[EXZ]; exzM = eM[EXZ];

            if (out) {
                // segment of this lane: CSR base = row_ptr of its first owned lane; the staging offset keeps
                // the parity of the CSR position (16-byte aligned bodies for the bulk copies)
                const int a_seg = __shfl_sync(0xffffffffu, rp, lfirst);
                const int soff = ds.w + ((fl & LF_BULK) ? (a_seg & 1) : 0);
                const bool px = I < p.nx, mx = I > 0, py = J < p.ny, my = J > 0, pz = Lz < p.nz, mz = Lz > 0;
                int rlen = 0;
                // the last step's copies are committed here, a step after their issue (a commit right behind them
                // waited for the TMA unit to take them: 0.1642 -> 0.1622 ms with bulk_st2); then: staging read
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
                if (owned) {
                    double sK = 0.0, sM = 0.0;
#pragma unroll
                    for (int e = 0; e < 7; e++) { sK += eK[e] + iK[e]; sM += eM[e] + iM[e]; }
                    double* rk = SK + soff + (rp - a_seg);
                    double* rm = SM + soff + (rp - a_seg);
                    VB_CHECK(rp >= a_seg && soff + (rp - a_seg) + 15 <= LSTG);   // the row lies in the staging strip
                    if (px && mx && py && my && pz && mz) {   // interior row: all 15 columns
                        rlen = 15;
                        rk[ORD.slot[0]] = -sK;
                        rm[ORD.slot[0]] = sM * (2.0 / 3.0);
#pragma unroll
                        for (int e = 0; e < 7; e++) {
                            rk[ORD.slot[1 + e]] = eK[e];
                            rm[ORD.slot[1 + e]] = eM[e];
                            rk[ORD.slot[8 + e]] = iK[e];
                            rm[ORD.slot[8 + e]] = iM[e];
                        }
                    } else if (px && !mx && py && my && pz && mz) {
                        // a row of the face x = 0 (no -x, -xy, -xz, -xyz columns), one lane of every tile that
                        // starts a line: compile-time slots as well (the general path below, run by the whole
                        // warp for that one lane, made these tiles 13 % slower)
                        constexpr uint32_t PX0 = 0x7fffu & ~(1u << 8 | 1u << 11 | 1u << 12 | 1u << 14);
                        rlen = 11;
                        rk[__popc(PX0 & ORD.low[0])] = -sK;
                        rm[__popc(PX0 & ORD.low[0])] = sM * (2.0 / 3.0);
#pragma unroll
                        for (int e = 0; e < 7; e++) {
                            rk[__popc(PX0 & ORD.low[1 + e])] = eK[e];
                            rm[__popc(PX0 & ORD.low[1 + e])] = eM[e];
                            if (PX0 >> (8 + e) & 1) {
                                rk[__popc(PX0 & ORD.low[8 + e])] = iK[e];
                                rm[__popc(PX0 & ORD.low[8 + e])] = iM[e];
                            }
                        }
                    } else {   // boundary row: the present columns, same order
                        uint32_t pres = 1u;
                        pres |= (uint32_t)px << 1 | (uint32_t)py << 2 | (uint32_t)pz << 3 |
                                (uint32_t)(px && py) << 4 | (uint32_t)(px && pz) << 5 | (uint32_t)(py && pz) << 6 |
                                (uint32_t)(px && py && pz) << 7;
                        pres |= (uint32_t)mx << 8 | (uint32_t)my << 9 | (uint32_t)mz << 10 |
                                (uint32_t)(mx && my) << 11 | (uint32_t)(mx && mz) << 12 |
                                (uint32_t)(my && mz) << 13 | (uint32_t)(mx && my && mz) << 14;
                        rlen = __popc(pres);
                        rk[__popc(pres & ORD.low[0])] = -sK;
                        rm[__popc(pres & ORD.low[0])] = sM * (2.0 / 3.0);
#pragma unroll
                        for (int e = 0; e < 7; e++) {
                            if (pres >> (1 + e) & 1) {
                                const int s = __popc(pres & ORD.low[1 + e]);
                                rk[s] = eK[e];
                                rm[s] = eM[e];
                            }
                            if (pres >> (8 + e) & 1) {
                                const int s = __popc(pres & ORD.low[8 + e]);
                                rk[s] = iK[e];
                                rm[s] = iM[e];
                            }
                        }
                    }
                }
                // segment range [a_seg, end of its last owned lane's row)
                const int segend = __shfl_sync(0xffffffffu, rp + rlen, llast);
                const bool tma = p.bulk && (fl & LF_BULK);   // full segment (the whole warp): rows leave through TMA
                if (tma && owned) {
                    // the 16-byte aligned body [a_seg + (a_seg & 1), segend - (segend & 1)) leaves as bulk copies; an
                    // odd first / last entry is stored by the lane that staged it (its own staging row: no fence
                    // needed), ahead of the fence so that its latency overlaps the bulk issue
                    const double* rk = SK + soff + (rp - a_seg);
                    const double* rm = SM + soff + (rp - a_seg);
                    if (lane == lfirst && (rp & 1) && rlen > 0) {
                        if (p.Kv) __stcs(p.Kv + rp, rk[0]);
                        if (p.Mv) __stcs(p.Mv + rp, rm[0]);
                    }
                    if (lane == llast && (segend & 1) && segend - 1 > a_seg) {
                        if (p.Kv) __stcs(p.Kv + segend - 1, rk[rlen - 1]);
                        if (p.Mv) __stcs(p.Mv + segend - 1, rm[rlen - 1]);
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (tma) {
                    const int a = a_seg + (a_seg & 1), e = segend - (segend & 1);
                    // one elected lane issues both copies (elect.sync: the compiler keeps the operands in uniform
                    // registers; a lane == 0 test made it loop over the "active lanes": 0.1662 -> 0.1642 ms)
                    uint32_t el = 0;
                    asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(el));
                    if (el && e > a) {
#if VB_LAT_KO != 1 && VB_LAT_KO != 3
                        if (p.Kv && p.Mv)
                            bulk_st2(p.Kv + a, SK + soff + (a - a_seg), p.Mv + a, SM + soff + (a - a_seg), (e - a) * 8);
                        else if (p.Kv) bulk_st(p.Kv + a, SK + soff + (a - a_seg), (e - a) * 8);
                        else if (p.Mv) bulk_st(p.Mv + a, SM + soff + (a - a_seg), (e - a) * 8);
#endif
                    }
                } else {
                    // packed tiles (several short segments per warp) and unaligned K / M: one segment at a time
                    // (warp-uniform), plain coalesced stores
                    uint32_t heads = __ballot_sync(0xffffffffu, owned && (fl & LF_HEAD));
                    while (heads) {
                        const int hd = __ffs(heads) - 1;
                        heads &= heads - 1;
                        const int a0 = __shfl_sync(0xffffffffu, a_seg, hd);
                        const int e0 = __shfl_sync(0xffffffffu, segend, hd);
                        const int s0 = __shfl_sync(0xffffffffu, soff, hd);
                        for (int q = a0 + lane; q < e0; q += 32) {
                            if (p.Kv) p.Kv[q] = SK[s0 + (q - a0)];
                            if (p.Mv) p.Mv[q] = SM[s0 + (q - a0)];
                        }
                    }
                }
            }
        }
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#ifdef VB_LAT_PROF
    if (threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        printf("LATPROF cta %d sm %u cycles %lld ns 0 g0 %lld g1 %lld\n", blockIdx.x, smid, clock64() - t_start,
               (long long)g0, (long long)g1);
    }
#endif
}

// Degenerate tetrahedra of the lattice (fem_p1_assemble_lattice's optional counter; a pass of its own so that the
// assembly kernel carries none of it): the determinant exactly as the kernel evaluates it (f1 . (f2 x f3) with
// the fused cross and dot products above) is 0, or two vertices of the tet have identical coordinates (a
// determinant that is 0 in exact arithmetic may be evaluated as a rounding residual).  One thread per cell.
__global__ void lattice_degenerate_k(int nx, int ny, int nz, int id0, int dJ, int dK, const double* __restrict__ X,
                                     int64_t ns, int64_t cs_, unsigned long long* __restrict__ out) {
    const int64_t ncell = (int64_t)nx * ny * nz;
    int mine = 0;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell; c += (int64_t)gridDim.x * blockDim.x) {
        const int I = (int)(c % nx), J = (int)((c / nx) % ny), K = (int)(c / ((int64_t)nx * ny));
        double cx[8][3];   // corners by bits x = 1, y = 2, z = 4
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int64_t v = id0 + (I + (q & 1)) + (int64_t)dJ * (J + ((q >> 1) & 1)) + (int64_t)dK * (K + (q >> 2));
#pragma unroll
            for (int d = 0; d < 3; d++) cx[q][d] = X[d * cs_ + v * ns];
        }
        double f[8][3];
#pragma unroll
        for (int q = 1; q < 8; q++)
#pragma unroll
            for (int d = 0; d < 3; d++) f[q][d] = cx[q][d] - cx[0][d];
        auto same = [&](int a, int b) { return cx[a][0] == cx[b][0] && cx[a][1] == cx[b][1] && cx[a][2] == cx[b][2]; };
        constexpr int mid[6][2] = {{1, 3}, {1, 5}, {2, 3}, {2, 6}, {4, 5}, {4, 6}};   // paths xyz xzy yxz yzx zxy zyx
#pragma unroll
        for (int t = 0; t < 6; t++) {
            const int a = mid[t][0], b = mid[t][1];
            double h1[3];
            crs(f[b], f[7], h1);   // the kernel's h1 = f2 x f3 (f3 = the cell diagonal), det = f1 . h1
            const double det = dot3(f[a], h1);
            mine += det == 0.0 || same(0, a) || same(0, b) || same(0, 7) || same(a, b) || same(a, 7) || same(b, 7);
        }
    }
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(out, (unsigned long long)mine);
}

// ------------------------------------------------------------------ plan: verification kernels
struct LatOrder {
    int dir[15];   // stencil directions in ascending column order
};
struct LatGeom {
    int nx, ny, nz;
    int fx, fy, fz;
    int64_t NX1, NY1;
};
__device__ __forceinline__ void canon(const LatGeom& g, int64_t id, int& I, int& J, int& K) {
    // node ids are below 2^31 (checked by the callers): 32-bit divisions (the 64-bit ones were most of the
    // element check's time)
#ifndef VB_LAT_FDIV
#define VB_LAT_FDIV 1   // quotients through an fp64 reciprocal with one correction (0: 32-bit integer divisions)
#endif
    const uint32_t u = (uint32_t)id, nx1 = (uint32_t)g.NX1, ny1 = (uint32_t)g.NY1;
#if VB_LAT_FDIV
    // u < 2^31 is exact in fp64 and u * (1/d) is within 2^-52 relative of u/d: the floor is the quotient or,
    // when u/d is an integer, one below it -- one comparison puts it right
    const double ix = 1.0 / (double)nx1, iy = 1.0 / (double)ny1;   // loop-invariant (kernel parameters)
    uint32_t q = __double2uint_rd((double)u * ix);
    uint32_t i = u - q * nx1;
    if (i >= nx1) { q++; i -= nx1; }
    uint32_t k = __double2uint_rd((double)q * iy);
    uint32_t j = q - k * ny1;
    if (j >= ny1) { k++; j -= ny1; }
#else
    const uint32_t q = u / nx1;
    const uint32_t i = u - q * nx1, k = q / ny1, j = q - k * ny1;
#endif
    I = (int)(g.fx ? g.nx - i : i);
    J = (int)(g.fy ? g.ny - j : j);
    K = (int)(g.fz ? g.nz - k : k);
}

// (cell, path) code of one element, or -1 if it is not a Kuhn tetrahedron of the canonical lattice
__device__ __forceinline__ int64_t lattice_elem_code(const LatGeom& g, int64_t nn, const int32_t (&vid)[4]) {
    int I[4], J[4], K[4];
    bool bad = false;
#pragma unroll
    for (int a = 0; a < 4; a++) {
        const int32_t v = vid[a];
        if (v < 0 || v >= nn) { bad = true; I[a] = J[a] = K[a] = 0; continue; }
        canon(g, v, I[a], J[a], K[a]);
    }
    int I0 = min(min(I[0], I[1]), min(I[2], I[3])), J0 = min(min(J[0], J[1]), min(J[2], J[3]));
    int K0 = min(min(K[0], K[1]), min(K[2], K[3]));
    // order the vertices by level (offset sum 0..3), each level exactly once (selects, no indexed array:
    // an array indexed by the level went to local memory)
    int at0 = -1, at1 = -1, at2 = -1, at3 = -1;
#pragma unroll
    for (int a = 0; a < 4; a++) {
        const int ox = I[a] - I0, oy = J[a] - J0, oz = K[a] - K0;
        if (ox < 0 || ox > 1 || oy < 0 || oy > 1 || oz < 0 || oz > 1) { bad = true; continue; }
        const int lev = ox + oy + oz, cd = ox | oy << 1 | oz << 2;
        const int prev = lev == 0 ? at0 : (lev == 1 ? at1 : (lev == 2 ? at2 : at3));
        if (prev >= 0) bad = true;
        at0 = lev == 0 ? cd : at0;
        at1 = lev == 1 ? cd : at1;
        at2 = lev == 2 ? cd : at2;
        at3 = lev == 3 ? cd : at3;
    }
    if (!bad && (at0 != 0 || at3 != 7)) bad = true;
    if (I0 >= g.nx || J0 >= g.ny || K0 >= g.nz) bad = true;
    if (bad) return -1;
    const int s0 = at1, s1 = at2 & ~at1;   // first and second unit steps
    if (__popc(s0) != 1 || __popc(at2) != 2 || (at2 & s0) != s0) return -1;
    const int p0 = __ffs(s0) - 1, p1 = __ffs(s1) - 1;
    const int path = p0 * 2 + ((p1 == (p0 + 1) % 3) ? 0 : 1);   // 6 paths
    return (((int64_t)K0 * g.ny + J0) * g.nx + I0) * 6 + path;
}

// every element is one Kuhn tetrahedron of the canonical lattice; its (cell, path) code is marked in a
// bitset, a code seen twice or a non-Kuhn element sets flags[0]
constexpr int LCHK_U = 4;   // groups of 32 elements per warp and step: their loads, then their atomics, in flight together
__global__ void lattice_check_elems_k(int64_t ne, int64_t nn, const int32_t* __restrict__ elems, int64_t eld,
                                      LatGeom g, uint32_t* __restrict__ bits, int* __restrict__ flags) {
    const int lane = threadIdx.x & 31;
    // whole warps run the loop: the bitset update is aggregated per word (elements in cell order put a warp's
    // 32 codes into one or two words: 2 atomics instead of 32; 0.39 -> 0.23 ms on configs[4]); a step was one
    // dependent chain load -> code -> atomic (old word back) per warp, so LCHK_U groups run side by side
    for (int64_t eb = (blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) * LCHK_U; eb < ne;
         eb += (int64_t)gridDim.x * blockDim.x * LCHK_U) {
        int32_t vid[LCHK_U][4];
        bool valid[LCHK_U];
#pragma unroll
        for (int u = 0; u < LCHK_U; u++) {
            valid[u] = eb + u * 32 + lane < ne;
            const int64_t e = valid[u] ? eb + u * 32 + lane : ne - 1;
#pragma unroll
            for (int a = 0; a < 4; a++) vid[u][a] = elems[a * eld + e];
        }
        int64_t code[LCHK_U];
        uint32_t old[LCHK_U], bit[LCHK_U];
        unsigned peers[LCHK_U];
#pragma unroll
        for (int u = 0; u < LCHK_U; u++) {
            code[u] = lattice_elem_code(g, nn, vid[u]);
            const bool mark = valid[u] && code[u] >= 0;
            // lanes of one word: OR their bits, one atomic by the lowest lane, the old word back to all of them;
            // a code twice inside the warp shows as two lanes with the same bit
            const long long key = mark ? (long long)(code[u] >> 5) : -1 - lane;
            peers[u] = __match_any_sync(0xffffffffu, key);
            bit[u] = mark ? 1u << (code[u] & 31) : 0u;
            const uint32_t all = __reduce_or_sync(peers[u], bit[u]);
            old[u] = 0;
            if (mark && lane == __ffs(peers[u]) - 1) old[u] = atomicOr(bits + (code[u] >> 5), all);
        }
        bool bad = false;
#pragma unroll
        for (int u = 0; u < LCHK_U; u++) {
            const bool mark = valid[u] && code[u] >= 0;
            const uint32_t o = __shfl_sync(peers[u], old[u], __ffs(peers[u]) - 1);
            if (mark) {
                const unsigned same = __match_any_sync(peers[u], bit[u]);
                if ((o & bit[u]) || __popc(same) > 1) bad = true;
            }
            if (valid[u] && code[u] < 0) bad = true;
        }
        if (bad) atomicExch(flags, 1);
    }
}

// the CSR pattern is the lattice stencil: row lengths and sorted column ids
__global__ void lattice_check_csr_k(int64_t nn, int64_t nnz, const int32_t* __restrict__ row_ptr,
                                    const int32_t* __restrict__ col_idx, LatGeom g, int64_t id0, int64_t dI,
                                    int64_t dJ, int64_t dK, LatOrder ord, int* __restrict__ flags) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
        int I, J, K;
        canon(g, v, I, J, K);
        const int64_t b = row_ptr[v], e = row_ptr[v + 1];
        bool bad = (v == 0 && b != 0) || (v == nn - 1 && e != nnz) || e < b;
        int64_t q = b;
        for (int r = 0; r < 15 && !bad; r++) {
            const int d = ord.dir[r];
            const int x = I + dir_dx(d), y = J + dir_dy(d), z = K + dir_dz(d);
            if (x < 0 || x > g.nx || y < 0 || y > g.ny || z < 0 || z > g.nz) continue;
            const int64_t want = id0 + dI * x + dJ * y + dK * z;
            if (q >= e || col_idx[q] != want) bad = true;
            q++;
        }
        if (!bad && q != e) bad = true;
        if (bad) atomicExch(flags + 1, 1);
    }
}


// the lattice stencil written out as a CSR pattern (fem_lattice_pattern): row lengths, then the columns of
// every row in ascending order (ord: stencil directions by ascending column id)
__global__ void lattice_rowlen_k(int64_t nn, LatGeom g, int32_t* __restrict__ row_len) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
        int I, J, K;
        canon(g, v, I, J, K);
        int n = 0;
#pragma unroll
        for (int d = 0; d < 15; d++) {
            const int x = I + dir_dx(d), y = J + dir_dy(d), z = K + dir_dz(d);
            n += x >= 0 && x <= g.nx && y >= 0 && y <= g.ny && z >= 0 && z <= g.nz;
        }
        row_len[v] = n;
    }
}
// 256 consecutive rows per block: every thread puts its row's columns into shared memory at the row's offset
// in the block's contiguous piece of col_idx, then the block writes the piece coalesced (one thread writing its
// own 15 ints, 60 bytes apart from its neighbour's: 0.169 ms on configs[4])
constexpr int LCOLS_BLOCK = 256;
__global__ void __launch_bounds__(LCOLS_BLOCK) lattice_cols_k(int64_t nn, LatGeom g, int64_t id0, int64_t dI, int64_t dJ,
                                                              int64_t dK, LatOrder ord,
                                                              const int32_t* __restrict__ row_ptr,
                                                              int32_t* __restrict__ col_idx) {
    __shared__ int32_t buf[LCOLS_BLOCK * 15];
    for (int64_t vb = blockIdx.x * (int64_t)LCOLS_BLOCK; vb < nn; vb += (int64_t)gridDim.x * LCOLS_BLOCK) {
        const int64_t v = vb + threadIdx.x;
        const int64_t vend = vb + LCOLS_BLOCK < nn ? vb + LCOLS_BLOCK : nn;
        const int64_t base = row_ptr[vb];
        const int len = (int)(row_ptr[vend] - base);
        if (v < nn) {
            int I, J, K;
            canon(g, v, I, J, K);
            int q = (int)(row_ptr[v] - base);
#pragma unroll
            for (int r = 0; r < 15; r++) {
                const int d = ord.dir[r];
                const int x = I + dir_dx(d), y = J + dir_dy(d), z = K + dir_dz(d);
                if (x < 0 || x > g.nx || y < 0 || y > g.ny || z < 0 || z > g.nz) continue;
                buf[q++] = (int32_t)(id0 + dI * x + dJ * y + dK * z);
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < len; i += LCOLS_BLOCK) col_idx[base + i] = buf[i];
        __syncthreads();
    }
}

__global__ void lattice_elem0_k(const int32_t* __restrict__ elems, int64_t eld, int32_t* __restrict__ out) {
    out[threadIdx.x] = elems[threadIdx.x * eld];
}

__global__ void lattice_token_k(const int* __restrict__ flags, uint32_t* __restrict__ token, uint32_t want) {
    *token = (flags[0] == 0 && flags[1] == 0) ? want : 0u;
}

// ------------------------------------------------------------------ host: geometry, tiling, token
struct LatHost {
    int nx, ny, nz, fx, fy, fz;
    int64_t id0, dI, dJ, dK;
    uint16_t lower[16];
    LatOrder ord;
};

bool lat_host(int nx, int ny, int nz, const int* flip, LatHost& h) {
    h.nx = nx; h.ny = ny; h.nz = nz;
    h.fx = flip[0] ? 1 : 0; h.fy = flip[1] ? 1 : 0; h.fz = flip[2] ? 1 : 0;
    if (h.fx) {   // mirroring all three axes maps a Kuhn lattice onto itself: keep x unmirrored
        h.fx = 0; h.fy ^= 1; h.fz ^= 1;
    }
    const int64_t NX1 = nx + 1, NY1 = ny + 1;
    if (NX1 * NY1 * (nz + 1) >= ((int64_t)1 << 31)) return false;
    h.id0 = NX1 * ((h.fy ? ny : 0) + NY1 * (int64_t)(h.fz ? nz : 0));
    h.dI = 1;
    h.dJ = (h.fy ? -1 : 1) * NX1;
    h.dK = (h.fz ? -1 : 1) * NX1 * NY1;
    int64_t off[15];
    for (int d = 0; d < 15; d++) off[d] = h.dI * dir_dx(d) + h.dJ * dir_dy(d) + h.dK * dir_dz(d);
    for (int d = 0; d < 16; d++) h.lower[d] = 0;
    for (int d = 0; d < 15; d++)
        for (int e = 0; e < 15; e++) {
            if (e != d && off[e] == off[d]) return false;   // two stencil columns with one id
            if (off[e] < off[d]) h.lower[d] |= (uint16_t)(1u << e);
        }
    // the kernel's compile-time column order must be the real one (it is for nx, ny >= 2)
    const Order<0, 0> o00{};
    const Order<0, 1> o01{};
    const Order<1, 0> o10{};
    const Order<1, 1> o11{};
    const uint32_t* low = h.fy ? (h.fz ? o11.low : o10.low) : (h.fz ? o01.low : o00.low);
    for (int d = 0; d < 15; d++)
        if (low[d] != h.lower[d]) return false;
    int idx[15];
    for (int d = 0; d < 15; d++) idx[d] = d;
    std::sort(idx, idx + 15, [&](int x, int y) { return off[x] < off[y]; });
    for (int r = 0; r < 15; r++) h.ord.dir[r] = idx[r];
    return true;
}

uint32_t lat_want(const LatHost& h, int64_t nn, int64_t nnz, int G) {
    uint64_t z = 0x9E3779B97F4A7C15ull;
    auto mix = [&](uint64_t v) {
        z ^= v + 0x9E3779B97F4A7C15ull + (z << 6) + (z >> 2);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
    };
    mix(h.nx); mix(h.ny); mix(h.nz); mix(h.fx | h.fy << 1 | h.fz << 2); mix(nn); mix(nnz); mix(G);
    const uint32_t t = LAT_MAGIC ^ (uint32_t)z ^ (uint32_t)(z >> 32);
    return t ? t : 1u;
}

// Cost of one tile-layer in SM cycles (measured on B200 with the per-CTA clock64 of the VB_LAT_PROF build,
// tools/latprof_run.py + latprof_sum.py, configs[4], refitted after every kernel change): a fixed part
// (barriers and the latency chains of a step) and a part per warp row holding nodes: 12 rows 6230, 7 rows
// 5160; a band without a halo row owns all its rows (the boundary row J = 0: +255).  A tile whose segment
// holds x = 0 or x = nx runs the masked cell path (absent cells) and a boundary-row path in every warp:
// x 1.11.  Packed tiles (always holding x = nx; plain stores, one pass per segment): x 1.0 with 2
// segments, x 1.7 with 5.
int lat_cost(int rows, int row0_owned, int xbnd = 0, int nseg = 0) {   // nseg > 0: a packed tile
    const int c = 3662 + 214 * rows + (row0_owned ? 255 : 0);
    const int packed = 765 + 235 * (nseg - 1);   // per mille
    return (int)((int64_t)c * (xbnd ? 111 : 100) / 100 * (nseg > 0 ? packed : 1000) / 1000);
}

// short segments (W lanes: a halo and W - 1 owned nodes) packed into one tile: as many as the lanes and the
// staging area (15 (W - 1) + 1 doubles and up to 15 of padding each) hold, at most 7 (coordinate columns)
int lat_per(int W) {
    int per = std::min(7, 32 / W);
    while (per > 1 && per * (15 * (W - 1) + 16) > LSTG) per--;
    return per;
}

// Tiles of 32 lanes.  x segments: a halo lane and 31 owned nodes (segment 0's halo is the virtual
// node x = -1); y bands of LR rows (the first owns LR lines, the next a halo line + LR - 1).  The
// short last segment of every band is packed with those of other bands.  work[t] = warp rows of
// tile t that hold a node (the cost weight of its layers).
void lat_tiles(int nx, int ny, std::vector<int4>& lanes, std::vector<int>& work, int& T) {
    struct Seg { int I0, nown; };
    std::vector<Seg> full, shortv;
    for (int x0 = 0; x0 <= nx; x0 += 31) {
        const int n = std::min(31, nx + 1 - x0);
        (n == 31 ? full : shortv).push_back({x0 - 1, n});
    }
    std::vector<std::pair<int, int>> bands;   // (J0, row 0 owned)
    bands.push_back({0, 1});
    for (int covered = LR - 1; covered < ny; covered += LR - 1) bands.push_back({covered, 0});
    auto rows_of = [&](int J0) { return std::min(LR, ny - J0 + 1); };
    lanes.clear();
    work.clear();
    auto lane_of = [](const Seg& sg, int J0, int row0, int lo, int k, int base, int l) {
        const int W = sg.nown + 1;
        int fl = W == 32 ? LF_BULK : 0;   // full segments leave through TMA bulk copies
        if (l > lo) fl |= LF_OWNX;
        if (l == lo + W - 1) fl |= LF_XPLUS;
        if (row0) fl |= LF_ROW0;
        if (l == lo + 1) fl |= LF_HEAD;
        const int col = l + k, first = lo + 1, last = lo + W - 1;
        return make_int4(sg.I0 + (l - lo), J0, fl | col << 8 | first << 16 | last << 24, base);
    };
    const int4 idle = make_int4(-2, 0, 0, 0);
    for (auto& b : bands)
        for (auto& sg : full) {
            for (int l = 0; l < 32; l++) lanes.push_back(lane_of(sg, b.first, b.second, 0, 0, 0, l));
            work.push_back(lat_cost(rows_of(b.first), b.second, sg.I0 < 0 || sg.I0 + sg.nown >= nx));
        }
    if (!shortv.empty()) {
        // at most one short segment per band (the last one), all of the same width
        const int W = shortv[0].nown + 1;
        const int per = lat_per(W);
        for (size_t b0 = 0; b0 < bands.size(); b0 += per) {
            int4 t[32];
            for (int l = 0; l < 32; l++) t[l] = idle;
            int end = 0, rows = 0;
            for (int k = 0; k < per && b0 + k < bands.size(); k++) {
                const int lo = k * W;
                // staging base = -lo - 1 (mod 16), so that the rows of the lanes of a half warp (15 doubles
                // apart) start in distinct bank pairs (packed tiles store with plain coalesced stores)
                const int base = end + ((16 - ((end + lo + 1) & 15)) & 15);
                for (int l = lo; l < lo + W; l++)
                    t[l] = lane_of(shortv[0], bands[b0 + k].first, bands[b0 + k].second, lo, k, base, l);
                end = base + 15 * shortv[0].nown + 1;
                rows = std::max(rows, rows_of(bands[b0 + k].first));
            }
            for (int l = 0; l < 32; l++) lanes.push_back(t[l]);
            const int nseg = (int)std::min<size_t>(per, bands.size() - b0);
            work.push_back(lat_cost(rows, b0 == 0, 1, nseg));
        }
    }
    T = (int)(lanes.size() / 32);
}

// the number of tiles lat_tiles makes (the assembly call needs only the count)
int lat_tile_count(int nx, int ny) {
    int nfull = 0, nshort = 0;
    for (int x0 = 0; x0 <= nx; x0 += 31) {
        const int n = std::min(31, nx + 1 - x0);
        if (n == 31) nfull++;
        else nshort = n;
    }
    int bands = 1;
    for (int covered = LR - 1; covered < ny; covered += LR - 1) bands++;
    int T = bands * nfull;
    if (nshort) {
        const int per = lat_per(nshort + 1);
        T += (bands + per - 1) / per;
    }
    return T;
}

// CTA ranges over the tile-layer sequence (tile-major): contiguous, with the smallest possible maximum
// cost per CTA.  A CTA pays work[t] per layer, LAT_START per tile it enters (prologue: barriers and the
// latency of the first coordinate layers) and one more layer when its range starts inside a tile (the
// halo layer below it).  Smallest feasible budget by bisection, each trial a greedy fill.
constexpr int LAT_START = 4000;
void lat_ranges(const std::vector<int>& work, int nz, int G, int* range) {
    const int NK = nz + 1;
    const int64_t L = (int64_t)work.size() * NK;
    auto fill = [&](int64_t budget, int* out) {   // true if G CTAs cover everything within the budget
        int64_t pos = 0;
        for (int c = 0; c < G; c++) {
            if (out) out[c] = (int)pos;
            int64_t cost = 0;
            while (pos < L) {
                const int t = (int)(pos / NK), k = (int)(pos % NK);
                int64_t add = work[t];
                if (cost == 0) add += LAT_START + (k > 0 ? work[t] : 0);
                else if (k == 0) add += LAT_START;
                if (cost > 0 && cost + add > budget) break;   // a CTA takes at least one layer
                cost += add;
                pos++;
            }
        }
        if (out) out[G] = (int)L;
        return pos >= L;
    };
    int64_t lo = 0, hi = 0;
    for (int w : work) hi += (int64_t)(w + 1) * NK + LAT_START;
    hi += LAT_START;
    while (lo + 1 < hi) {   // fill(hi) holds, fill(lo) fails
        const int64_t mid = (lo + hi) / 2;
        if (fill(mid, nullptr)) hi = mid;
        else lo = mid;
    }
    fill(hi, range);
    range[G] = (int)L;
}

constexpr int LAT_HDR = 16;   // plan header ints (token, dims, flips, tiles, CTAs), then the lane descriptors (T x 32
                              // int4) and the CTA ranges (LMAXCTA + 1 ints)
// one CTA per SM of the current device (the plan's ranges are for this grid: the token covers it)
int lat_grid(int T, int nz) {
    int64_t L = (int64_t)T * (nz + 1);
    int g = std::min(sm_count() * VB_LAT_MINB, LMAXCTA);
    return (int)std::min<int64_t>(g, L);
}

}  // namespace

// ------------------------------------------------------------------ exports
extern "C" VB_API vb_status fem_plan_lattice(int64_t nn, int64_t ne, const int32_t* elems, int64_t elem_ld,
                                             const int32_t* row_ptr, const int32_t* col_idx, int64_t nnz, int nx,
                                             int ny, int nz, void* work, size_t* work_bytes, int32_t* plan,
                                             int64_t* plan_ints, int64_t* stats_out, vb_stream_t stream) {
    const char* fn = "fem_plan_lattice";
    clear_error();
    if (nx < 1 || ny < 1 || nz < 1 || !work_bytes || !plan_ints) {
        set_error("%s: nx, ny, nz must be >= 1 and work_bytes, plan_ints non-NULL", fn);
        return VB_ERR_ARG;
    }
    const int64_t nn_want = (int64_t)(nx + 1) * (ny + 1) * (nz + 1), ne_want = (int64_t)6 * nx * ny * nz;
    std::vector<int4> lanes;
    std::vector<int> twork;
    int T = 0;
    lat_tiles(nx, ny, lanes, twork, T);
    if (T != lat_tile_count(nx, ny)) { set_error("%s: internal tile count mismatch", fn); return VB_ERR_UNSUPPORTED; }
    const int64_t need_ints = LAT_HDR + (int64_t)T * 32 * 4 + LMAXCTA + 1;
    const size_t wb = 256 + (size_t)((ne_want + 31) / 32) * 4;
    if (!work) {
        *work_bytes = wb;
        *plan_ints = need_ints;
        return VB_OK;
    }
    if (*work_bytes < wb) { set_error("%s: work_bytes %zu < %zu", fn, *work_bytes, wb); return VB_ERR_WORKSPACE; }
    if (!plan || *plan_ints < need_ints) {
        set_error("%s: plan needs %lld ints", fn, (long long)need_ints);
        return VB_ERR_WORKSPACE;
    }
    if (!stats_out || !elems || (row_ptr == nullptr) != (col_idx == nullptr) || elem_ld < ne) {
        set_error("%s: NULL argument, only one of row_ptr / col_idx, or elem_ld < ne", fn);
        return VB_ERR_ARG;
    }
    if (!aligned16(plan)) { set_error("%s: plan must be 16-byte aligned", fn); return VB_ERR_ARG; }
    stats_out[0] = 0;
    stats_out[1] = T;
    stats_out[2] = 0;
    if (nn != nn_want || ne != ne_want) {
        stats_out[2] = 1;   // counts are not those of an nx x ny x nz Kuhn lattice
        return VB_OK;
    }
    cudaStream_t s = cs(stream);
    // orientation from element 0: the vertex pair at lattice distance 3 is the split diagonal
    int32_t v0[4];
    {   // the four vertex ids of element 0 in one read-back
        lattice_elem0_k<<<1, 4, 0, s>>>(elems, elem_ld, reinterpret_cast<int32_t*>(work));
        vb_status st = launch_check(fn);
        if (st == VB_OK) st = read_small(s, work, sizeof(v0), v0, fn);
        if (st != VB_OK) return st;
    }
    int flip[3] = {0, 0, 0};
    {
        const int64_t NX1 = nx + 1, NY1 = ny + 1;
        int best = -1, bi = 0, bj = 0;
        for (int a = 0; a < 4; a++)
            for (int b = 0; b < 4; b++) {
                if (v0[a] < 0 || v0[a] >= nn || v0[b] < 0 || v0[b] >= nn) { stats_out[2] = 2; return VB_OK; }
                const int64_t dx = v0[b] % NX1 - v0[a] % NX1, dy = (v0[b] / NX1) % NY1 - (v0[a] / NX1) % NY1,
                              dz = v0[b] / (NX1 * NY1) - v0[a] / (NX1 * NY1);
                const int dist = (int)(std::llabs(dx) + std::llabs(dy) + std::llabs(dz));
                if (dist > best && dx > 0) { best = dist; bi = a; bj = b; }
            }
        if (best != 3) { stats_out[2] = 2; return VB_OK; }
        const int64_t dy = (v0[bj] / NX1) % NY1 - (v0[bi] / NX1) % NY1, dz = v0[bj] / (NX1 * NY1) - v0[bi] / (NX1 * NY1);
        flip[1] = dy < 0;
        flip[2] = dz < 0;
    }
    if (nx < 2 || ny < 2) { stats_out[2] = 3; return VB_OK; }   // the kernel's column order needs nx, ny >= 2
    LatHost h;
    if (!lat_host(nx, ny, nz, flip, h)) { stats_out[2] = 3; return VB_OK; }
    LatGeom g{nx, ny, nz, h.fx, h.fy, h.fz, (int64_t)nx + 1, (int64_t)ny + 1};
    int* flags = reinterpret_cast<int*>(work);
    uint32_t* bits = reinterpret_cast<uint32_t*>(static_cast<char*>(work) + 256);
    cudaError_t e = cudaMemsetAsync(work, 0, wb, s);
    if (e != cudaSuccess) { set_error("%s: %s", fn, cudaGetErrorString(e)); return VB_ERR_CUDA; }
    lattice_check_elems_k<<<grid_for(ne, 256, 8), 256, 0, s>>>(ne, nn, elems, elem_ld, g, bits, flags);
    vb_status st = launch_check(fn);
    if (st != VB_OK) return st;
    if (row_ptr) {   // NULL, NULL: the pattern comes from fem_lattice_pattern (the stencil by construction)
        lattice_check_csr_k<<<grid_for(nn, 256, 8), 256, 0, s>>>(nn, nnz, row_ptr, col_idx, g, h.id0, h.dI, h.dJ, h.dK,
                                                                 h.ord, flags);
        if ((st = launch_check(fn)) != VB_OK) return st;
    }
    // header + lanes
    int32_t hdr[LAT_HDR] = {0};
    hdr[1] = nx; hdr[2] = ny; hdr[3] = nz;
    hdr[4] = h.fx; hdr[5] = h.fy; hdr[6] = h.fz; hdr[7] = T;
    const int G = lat_grid(T, nz);
    hdr[8] = G;
    std::vector<int> range(LMAXCTA + 1, (int)((int64_t)T * (nz + 1)));
    lat_ranges(twork, nz, G, range.data());
    e = cudaMemcpyAsync(plan, hdr, sizeof(hdr), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(plan + LAT_HDR, lanes.data(), lanes.size() * sizeof(int4), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(plan + LAT_HDR + (int64_t)T * 128, range.data(), range.size() * sizeof(int),
                            cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) { set_error("%s: %s", fn, cudaGetErrorString(e)); return VB_ERR_CUDA; }
    lattice_token_k<<<1, 1, 0, s>>>(flags, reinterpret_cast<uint32_t*>(plan), lat_want(h, nn, nnz, G));
    if ((st = launch_check(fn)) != VB_OK) return st;
    int fl2[2];
    if ((st = read_small(s, flags, 8, fl2, fn)) != VB_OK) return st;   // synchronises: host arrays outlive
    if (fl2[0]) stats_out[2] = 4;       // an element is not a Kuhn tetrahedron of this lattice (or twice)
    else if (fl2[1]) stats_out[2] = 5;  // the CSR pattern is not the lattice stencil
    else stats_out[0] = 1;
    stats_out[3] = h.fx | h.fy << 1 | h.fz << 2 | (int64_t)G << 8;   // orientation, and the grid the ranges are for
    return VB_OK;
}

// nnz of the lattice stencil: direction d is present at (nx+1-|dx|)(ny+1-|dy|)(nz+1-|dz|) nodes
static int64_t lat_nnz(int nx, int ny, int nz) {
    int64_t n = 0;
    for (int d = 0; d < 15; d++)
        n += (int64_t)(nx + 1 - std::abs(dir_dx(d))) * (ny + 1 - std::abs(dir_dy(d))) * (nz + 1 - std::abs(dir_dz(d)));
    return n;
}

extern "C" VB_API vb_status fem_lattice_pattern(int64_t nn, int nx, int ny, int nz, int flips, void* work,
                                                size_t* work_bytes, int32_t* row_ptr, int32_t* col_idx,
                                                int64_t col_cap, int64_t* nnz_out, vb_stream_t stream) {
    const char* fn = "fem_lattice_pattern";
    clear_error();
    if (nx < 1 || ny < 1 || nz < 1 || (int64_t)(nx + 1) * (ny + 1) * (nz + 1) != nn || !work_bytes) {
        set_error("%s: nx, ny, nz >= 1, nn = (nx+1)(ny+1)(nz+1) and work_bytes non-NULL are required", fn);
        return VB_ERR_ARG;
    }
    const int64_t nnz = lat_nnz(nx, ny, nz);
    if (nnz >= ((int64_t)1 << 31)) { set_error("%s: nnz=%lld does not fit int32", fn, (long long)nnz); return VB_ERR_OVERFLOW; }
    if (nnz_out) *nnz_out = nnz;
    const size_t len_bytes = ((size_t)(nn + 1) * 4 + 255) & ~(size_t)255;
    const size_t wb = len_bytes + scan_tmp_bytes(nn);
    if (!work) {
        *work_bytes = wb;
        return VB_OK;
    }
    if (*work_bytes < wb) { set_error("%s: work_bytes %zu < %zu", fn, *work_bytes, wb); return VB_ERR_WORKSPACE; }
    if (!row_ptr || !col_idx || col_cap < nnz) { set_error("%s: NULL row_ptr / col_idx or col_cap < nnz=%lld", fn, (long long)nnz); return VB_ERR_ARG; }
    const int fl[3] = {flips & 1, (flips >> 1) & 1, (flips >> 2) & 1};
    LatHost h;
    if (nx < 2 || ny < 2 || !lat_host(nx, ny, nz, fl, h)) {
        set_error("%s: lattice outside the kernel's limits (nx, ny >= 2)", fn);
        return VB_ERR_UNSUPPORTED;
    }
    LatGeom g{nx, ny, nz, h.fx, h.fy, h.fz, (int64_t)nx + 1, (int64_t)ny + 1};
    cudaStream_t s = cs(stream);
    int32_t* row_len = reinterpret_cast<int32_t*>(work);
    void* scan_tmp = static_cast<char*>(work) + len_bytes;
    lattice_rowlen_k<<<grid_for(nn, 256, 8), 256, 0, s>>>(nn, g, row_len);
    vb_status st = launch_check(fn);
    if (st != VB_OK) return st;
    if ((st = exclusive_scan_i32(row_len, row_ptr, nn, scan_tmp, s, nullptr)) != VB_OK) return st;
    lattice_cols_k<<<grid_for(nn, LCOLS_BLOCK, 8), LCOLS_BLOCK, 0, s>>>(nn, g, h.id0, h.dI, h.dJ, h.dK, h.ord, row_ptr, col_idx);
    return launch_check(fn);
}

extern "C" VB_API vb_status fem_p1_assemble_lattice(int64_t nn, const double* coords, int64_t node_stride,
                                                    int64_t comp_stride, const int32_t* row_ptr, int64_t nnz,
                                                    const int32_t* plan, int nx, int ny, int nz, int flips,
                                                    double* K_vals, double* M_vals, int64_t* degenerate,
                                                    vb_stream_t stream) {
    const char* fn = "fem_p1_assemble_lattice";
    clear_error();
    if (nx < 1 || ny < 1 || nz < 1 || (int64_t)(nx + 1) * (ny + 1) * (nz + 1) != nn) {
        set_error("%s: nn != (nx+1)(ny+1)(nz+1)", fn);
        return VB_ERR_ARG;
    }
    if (!coords || !row_ptr || !plan || nnz < 0 || nnz >= ((int64_t)1 << 31)) {
        set_error("%s: NULL coords/row_ptr/plan or bad nnz", fn);
        return VB_ERR_ARG;
    }
    if (!aligned16(plan)) { set_error("%s: plan must be 16-byte aligned", fn); return VB_ERR_ARG; }
    if (!K_vals && !M_vals && !degenerate) return VB_OK;
    const int g_plan = flips >> 8;   // 0: not given (orientation only)
    const int fl[3] = {flips & 1, (flips >> 1) & 1, (flips >> 2) & 1};
    LatHost h;
    if (nx < 2 || ny < 2 || !lat_host(nx, ny, nz, fl, h)) {
        set_error("%s: lattice outside the kernel's limits (nx, ny >= 2)", fn);
        return VB_ERR_ARG;
    }
    const int T = lat_tile_count(nx, ny);
    LatParams p;
    p.nx = nx; p.ny = ny; p.nz = nz; p.T = T;
    p.L = (int64_t)T * (nz + 1);
    p.id0 = (int)h.id0; p.dJ = (int)h.dJ; p.dK = (int)h.dK;
    p.X = coords; p.ns = node_stride; p.cs = comp_stride;
    p.row_ptr = row_ptr;
    p.Kv = K_vals; p.Mv = M_vals;
    p.lanes = reinterpret_cast<const int4*>(plan + LAT_HDR);
    p.token = reinterpret_cast<const uint32_t*>(plan);
    const int grid = lat_grid(T, nz);
    if (g_plan && g_plan != grid) {
        set_error("%s: the plan was built for a device with another SM count (%d CTAs, this device: %d)", fn, g_plan,
                  grid);
        return VB_ERR_ARG;
    }
    p.range = plan + LAT_HDR + (int64_t)T * 128;
    p.want = lat_want(h, nn, nnz, grid);
    p.bulk = (!K_vals || aligned16(K_vals)) && (!M_vals || aligned16(M_vals));
    if (degenerate) {   // a pass of its own over the cells, with the kernel's determinant expressions
        cudaError_t e = cudaMemsetAsync(degenerate, 0, sizeof(int64_t), cs(stream));
        if (e != cudaSuccess) { set_error("%s: %s", fn, cudaGetErrorString(e)); return VB_ERR_CUDA; }
        const int64_t ncell = (int64_t)nx * ny * nz;
        lattice_degenerate_k<<<grid_for(ncell, 256, 8), 256, 0, cs(stream)>>>(
            nx, ny, nz, (int)h.id0, (int)h.dJ, (int)h.dK, coords, node_stride, comp_stride,
            reinterpret_cast<unsigned long long*>(degenerate));
        vb_status st = launch_check(fn);
        if (st != VB_OK) return st;
    }
    if (!K_vals && !M_vals) return VB_OK;
    const size_t smem = sizeof(LatSmem);
    static bool smem_set[64] = {};   // the attribute is per device (idempotent: a race only repeats the calls)
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !smem_set[dev]) {
        cudaFuncSetAttribute(assemble_lattice_k<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(assemble_lattice_k<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(assemble_lattice_k<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(assemble_lattice_k<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (dev >= 0 && dev < 64) smem_set[dev] = true;
    }
    auto launch = [&](void (*kern)(LatParams)) { kern<<<grid, LTHREADS, smem, cs(stream)>>>(p); };
    switch (h.fy | h.fz << 1) {
        case 0: launch(assemble_lattice_k<0, 0>); break;
        case 1: launch(assemble_lattice_k<1, 0>); break;
        case 2: launch(assemble_lattice_k<0, 1>); break;
        default: launch(assemble_lattice_k<1, 1>); break;
    }
    return launch_check(fn);
}

}  // namespace vb
