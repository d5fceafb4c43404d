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
// Kernel (assemble_lattice_k): a CTA holds a tile of 32 lanes (x) x R warp
// rows (y) of lattice columns and marches along z, one node layer per step,
// evaluating every cell (6 tets) ONCE.  Contributions move to the owning node
// by warp shuffle (x), shared memory (y) and registers (z).  Row 0 of a tile
// and the first lane of an x segment are halos (their cells are recomputed by
// the neighbouring tile, ~15% of the cells); everything else is owned.  Rows of
// CSR are assembled in registers (14 edges; diagonals by the partition of unity,
// K_pp = -sum_q K_pq, M_pp = (2/3) sum_q M_pq, as the gather variants) and leave
// through a shared-memory staging buffer with coalesced stores.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "vb_internal.cuh"

namespace vb {
namespace {

constexpr int LR = 12;            // warp rows per tile (row 0 may be a halo line)
constexpr int LCOLS = 40;         // coordinate columns per row (lanes + one gap per segment)
constexpr int LNBUF = 3;          // coordinate layer buffers (prefetch distance 2)
constexpr int LSTG = 32 * 15 + 16;   // staging doubles per matrix and warp row
constexpr int LTHREADS = 32 * LR;
constexpr uint32_t LAT_MAGIC = 0x4c415431u;   // "LAT1"

// stencil directions: 0 self, 1..7 = +x +y +z +xy +xz +yz +xyz, 8..14 the negatives
__host__ __device__ constexpr int dir_dx(int d) { return d == 0 ? 0 : (d <= 7 ? 1 : -1) * ((d - 1) % 7 == 0 || (d - 1) % 7 == 3 || (d - 1) % 7 == 4 || (d - 1) % 7 == 6); }
__host__ __device__ constexpr int dir_dy(int d) { return d == 0 ? 0 : (d <= 7 ? 1 : -1) * ((d - 1) % 7 == 1 || (d - 1) % 7 == 3 || (d - 1) % 7 == 5 || (d - 1) % 7 == 6); }
__host__ __device__ constexpr int dir_dz(int d) { return d == 0 ? 0 : (d <= 7 ? 1 : -1) * ((d - 1) % 7 == 2 || (d - 1) % 7 == 4 || (d - 1) % 7 == 5 || (d - 1) % 7 == 6); }

struct LatParams {
    int nx, ny, nz, T;            // cells per axis, tiles
    int64_t L;                    // T * (nz + 1) tile-layers
    int64_t id0, dI, dJ, dK;      // node id of canonical (I, J, K) = id0 + dI I + dJ J + dK K
    const double* X;
    int64_t ns, cs;               // coordinate addressing X[c*cs + v*ns]
    const int32_t* row_ptr;
    double* Kv;
    double* Mv;
    const int4* lanes;            // T x 32 lane descriptors
    const uint32_t* token;        // plan token (LAT_MAGIC ^ hash) written by fem_plan_lattice
    uint32_t want;
    uint16_t lower[16];           // lower[d]: directions whose id offset is below d's (CSR slot order)
};

// lane descriptor (int4): x = I (canonical x of the lane's node; -1: idle lane), y = J0 (canonical y of
// row 0), z = flags | col << 8 | first owned lane << 16 | last lane << 24, w = staging base of the segment
enum : int { LF_OWNX = 1, LF_LEFT = 2, LF_XPLUS = 4, LF_ROW0 = 8, LF_HEAD = 16 };

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
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

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
// the mass off-diagonal |T|/20 = |det|/120.
__device__ __forceinline__ Tet tet(const double (&f1)[3], const double (&f2)[3], const double (&h1)[3],
                                   const double (&h2)[3]) {
    double h3[3];
    crs(f1, f2, h3);
    const double det = dot3(f1, h1);
    const double ad = fabs(det);
    const double s = rcp2(6.0 * ad);
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

// edge slots of the owned-edge arrays: +x +y +z +xy +xz +yz +xyz
enum { EX = 0, EY, EZ, EXY, EXZ, EYZ, EXYZ };

__device__ __forceinline__ double shup(double v, bool ok) {   // value of lane - 1 (0 if not the -x neighbour)
    const double r = __shfl_up_sync(0xffffffffu, v, 1);
    return ok ? r : 0.0;
}

__global__ void __launch_bounds__(LTHREADS, 1) assemble_lattice_k(const LatParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LatSmem& S = *reinterpret_cast<LatSmem*>(smem_raw);
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    if (*p.token != p.want) return;   // plan of another mesh / not verified: write nothing

    const int64_t g0 = p.L * blockIdx.x / gridDim.x, g1 = p.L * (blockIdx.x + 1) / gridDim.x;
    const int NK = p.nz + 1;
    int64_t g = g0;
    while (g < g1) {
        const int tau = (int)(g / NK);
        const int ka = (int)(g % NK);
        const int64_t gend = (int64_t)(tau + 1) * NK < g1 ? (int64_t)(tau + 1) * NK : g1;
        const int kb = (int)(gend - (int64_t)tau * NK);   // node layers [ka, kb)
        g += kb - ka;

        const int4 ds = p.lanes[tau * 32 + lane];
        const int I = ds.x;
        const int J = ds.y + w;
        const int fl = ds.z & 0xff;
        const int col = (ds.z >> 8) & 0xff;
        const int lfirst = (ds.z >> 16) & 0xff;
        const int llast = (ds.z >> 24) & 0xff;
        const bool valid = I >= 0 && J <= p.ny;
        const bool left = (fl & LF_LEFT) != 0;
        const bool owned = valid && (fl & LF_OWNX) && (w > 0 || (fl & LF_ROW0));
        const bool cellxy = valid && I < p.nx && J < p.ny;
        const bool xplus = valid && (fl & LF_XPLUS) && I < p.nx;
        const int64_t idIJ = p.id0 + p.dI * I + p.dJ * J;

        // coordinate prefetch of node layer Lz into buffer Lz % 3: own node, the +x node of a segment's
        // last lane, and row LR (J + 1) for the last warp row
        auto fetch = [&](int Lz) {
            if (Lz > p.nz) return;
            const int b = Lz % LNBUF;
            const int64_t v = idIJ + p.dK * Lz;
            if (valid) {
#pragma unroll
                for (int c = 0; c < 3; c++) cpa8(&S.X[b][c][w][col], p.X + c * p.cs + v * p.ns);
                if (xplus)
#pragma unroll
                    for (int c = 0; c < 3; c++) cpa8(&S.X[b][c][w][col + 1], p.X + c * p.cs + (v + p.dI) * p.ns);
            }
            if (w == LR - 1 && I >= 0 && J + 1 <= p.ny) {
                const int64_t v2 = v + p.dJ;
#pragma unroll
                for (int c = 0; c < 3; c++) cpa8(&S.X[b][c][LR][col], p.X + c * p.cs + v2 * p.ns);
                if (xplus)
#pragma unroll
                    for (int c = 0; c < 3; c++)
                        cpa8(&S.X[b][c][LR][col + 1], p.X + c * p.cs + (v2 + p.dI) * p.ns);
            }
        };

        const int Ls = ka > 0 ? ka - 1 : ka;   // one halo layer when the range starts inside the tile
        __syncthreads();                       // previous range's readers of every buffer are done
        fetch(Ls);
        fetch(Ls + 1);
        cpa_commit();
        cpa_wait_all();
        __syncthreads();

        // carries along z: zc = in-plane up edges (+x, +y, +xy) of this node at the next layer from the
        // cells below it; ez / exz = this node's +z / +xz edge of the previous layer
        double zcK[3] = {0, 0, 0}, zcM[3] = {0, 0, 0};
        double ezK = 0, ezM = 0, exzK = 0, exzM = 0;

        for (int Lz = Ls; Lz < kb; Lz++) {
            fetch(Lz + 2);
            cpa_commit();
            const bool out = Lz >= ka;
            int rp = 0;
            if (out && owned) rp = __ldg(p.row_ptr + idIJ + p.dK * Lz);

            // ---- phase A: the cell (I, J, Lz) -> owned edges eK/eM (+ carries) and outgoing parts
            double eK[7], eM[7];
#pragma unroll
            for (int e = 0; e < 7; e++) eK[e] = eM[e] = 0.0;
            eK[EX] = zcK[0]; eK[EY] = zcK[1]; eK[EXY] = zcK[2];
            eM[EX] = zcM[0]; eM[EY] = zcM[1]; eM[EXY] = zcM[2];
            double oK[10], oM[10];   // to the next row: c010 (x, z, xz), c110 (z), c011 (x) -- slots 0..4
            double c101K = 0, c101M = 0;
            double c100K[3] = {0, 0, 0}, c100M[3] = {0, 0, 0};
#pragma unroll
            for (int e = 0; e < 5; e++) oK[e] = oM[e] = 0.0;
            double c001K[3] = {0, 0, 0}, c001M[3] = {0, 0, 0};
            if (cellxy && Lz < p.nz) {
                const int b0 = Lz % LNBUF, b1 = (Lz + 1) % LNBUF;
                double x000[3], ux[3], uy[3], uz[3], wxy[3], wxz[3], wyz[3], bd[3];
#pragma unroll
                for (int c = 0; c < 3; c++) {
                    x000[c] = S.X[b0][c][w][col];
                    ux[c] = S.X[b0][c][w][col + 1] - x000[c];
                    uy[c] = S.X[b0][c][w + 1][col] - x000[c];
                    wxy[c] = S.X[b0][c][w + 1][col + 1] - x000[c];
                    uz[c] = S.X[b1][c][w][col] - x000[c];
                    wxz[c] = S.X[b1][c][w][col + 1] - x000[c];
                    wyz[c] = S.X[b1][c][w + 1][col] - x000[c];
                    bd[c] = S.X[b1][c][w + 1][col + 1] - x000[c];
                }
                double hxy[3], hxz[3], hyz[3];
                crs(wxy, bd, hxy);
                crs(wxz, bd, hxz);
                crs(wyz, bd, hyz);
                {   // paths starting along x: (x,y,z), (x,z,y)
                    double h2[3];
                    crs(bd, ux, h2);
                    const Tet a = tet(ux, wxy, hxy, h2);
                    const Tet b = tet(ux, wxz, hxz, h2);
                    eK[EX] += a.k01 + b.k01;   eM[EX] += a.m + b.m;
                    eK[EXY] += a.k02;          eM[EXY] += a.m;
                    eK[EXZ] += b.k02;          eM[EXZ] += b.m;
                    eK[EXYZ] += a.k03 + b.k03; eM[EXYZ] += a.m + b.m;
                    c100K[0] = a.k12;          c100M[0] = a.m;          // corner 100: +y
                    c100K[1] = b.k12;          c100M[1] = b.m;          //             +z
                    c100K[2] = a.k13 + b.k13;  c100M[2] = a.m + b.m;    //             +yz
                    oK[3] = a.k23;             oM[3] = a.m;             // corner 110: +z
                    c101K = b.k23;             c101M = b.m;             // corner 101: +y
                }
                {   // (y,x,z), (y,z,x)
                    double h2[3];
                    crs(bd, uy, h2);
                    const Tet a = tet(uy, wxy, hxy, h2);
                    const Tet b = tet(uy, wyz, hyz, h2);
                    eK[EY] += a.k01 + b.k01;   eM[EY] += a.m + b.m;
                    eK[EXY] += a.k02;          eM[EXY] += a.m;
                    eK[EYZ] += b.k02;          eM[EYZ] += b.m;
                    eK[EXYZ] += a.k03 + b.k03; eM[EXYZ] += a.m + b.m;
                    oK[0] = a.k12;             oM[0] = a.m;             // corner 010: +x
                    oK[1] = b.k12;             oM[1] = b.m;             //             +z
                    oK[2] = a.k13 + b.k13;     oM[2] = a.m + b.m;       //             +xz
                    oK[3] += a.k23;            oM[3] += a.m;            // corner 110: +z
                    oK[4] = b.k23;             oM[4] = b.m;             // corner 011: +x
                }
                {   // (z,x,y), (z,y,x)
                    double h2[3];
                    crs(bd, uz, h2);
                    const Tet a = tet(uz, wxz, hxz, h2);
                    const Tet b = tet(uz, wyz, hyz, h2);
                    eK[EZ] += a.k01 + b.k01;   eM[EZ] += a.m + b.m;
                    eK[EXZ] += a.k02;          eM[EXZ] += a.m;
                    eK[EYZ] += b.k02;          eM[EYZ] += b.m;
                    eK[EXYZ] += a.k03 + b.k03; eM[EXYZ] += a.m + b.m;
                    c001K[0] = a.k12;          c001M[0] = a.m;          // corner 001: +x
                    c001K[1] = b.k12;          c001M[1] = b.m;          //             +y
                    c001K[2] = a.k13 + b.k13;  c001M[2] = a.m + b.m;    //             +xy
                    c101K += a.k23;            c101M += a.m;            // corner 101: +y
                    oK[4] += b.k23;            oM[4] += b.m;            // corner 011: +x
                }
            }
            // ---- phase B: x neighbours by shuffle, the next row through shared memory
            eK[EY] += shup(c100K[0], left);  eM[EY] += shup(c100M[0], left);
            eK[EZ] += shup(c100K[1], left);  eM[EZ] += shup(c100M[1], left);
            eK[EYZ] += shup(c100K[2], left); eM[EYZ] += shup(c100M[2], left);
            zcK[0] = c001K[0]; zcK[1] = c001K[1] + shup(c101K, left); zcK[2] = c001K[2];
            zcM[0] = c001M[0]; zcM[1] = c001M[1] + shup(c101M, left); zcM[2] = c001M[2];
#pragma unroll
            for (int e = 0; e < 5; e++) {
                S.P[w][e][lane] = oK[e];
                S.P[w][5 + e][lane] = oM[e];
            }
            __syncthreads();

            // ---- phase C: contributions of the row below; publish the finished edges
            if (w > 0) {
                const double* Pb = &S.P[w - 1][0][0];
                eK[EX] += Pb[0 * 32 + lane];  eM[EX] += Pb[5 * 32 + lane];
                eK[EZ] += Pb[1 * 32 + lane];  eM[EZ] += Pb[6 * 32 + lane];
                eK[EXZ] += Pb[2 * 32 + lane]; eM[EXZ] += Pb[7 * 32 + lane];
                if (left) { eK[EZ] += Pb[3 * 32 + lane - 1]; eM[EZ] += Pb[8 * 32 + lane - 1]; }
                zcK[0] += Pb[4 * 32 + lane];  zcM[0] += Pb[9 * 32 + lane];
            }
            S.Ein[w][0][lane] = eK[EY];
            S.Ein[w][1][lane] = eM[EY];
            S.Ein[w][2][lane] = eK[EXY];
            S.Ein[w][3][lane] = eM[EXY];
            S.Ez[Lz & 1][w][0][lane] = eK[EYZ];
            S.Ez[Lz & 1][w][1][lane] = eM[EYZ];
            S.Ez[Lz & 1][w][2][lane] = eK[EXYZ];
            S.Ez[Lz & 1][w][3][lane] = eM[EXYZ];
            cpa_wait_all();
            __syncthreads();

            // ---- phase D: the CSR rows of this layer's owned nodes
            // incoming edges (the up edges of the lower neighbours): -x, -y, -z, -xy, -xz, -yz, -xyz
            double iK[7], iM[7];
            iK[0] = shup(eK[EX], left);  iM[0] = shup(eM[EX], left);
            iK[4] = shup(exzK, left);    iM[4] = shup(exzM, left);
            iK[2] = ezK;                 iM[2] = ezM;
            iK[1] = iK[3] = iK[5] = iK[6] = 0.0;
            iM[1] = iM[3] = iM[5] = iM[6] = 0.0;
            if (w > 0) {
                iK[1] = S.Ein[w - 1][0][lane];
                iM[1] = S.Ein[w - 1][1][lane];
                if (left) { iK[3] = S.Ein[w - 1][2][lane - 1]; iM[3] = S.Ein[w - 1][3][lane - 1]; }
                if (Lz > 0) {
                    const int q = (Lz - 1) & 1;
                    iK[5] = S.Ez[q][w - 1][0][lane];
                    iM[5] = S.Ez[q][w - 1][1][lane];
                    if (left) { iK[6] = S.Ez[q][w - 1][2][lane - 1]; iM[6] = S.Ez[q][w - 1][3][lane - 1]; }
                }
            }
            ezK = eK[EZ]; ezM = eM[EZ]; exzK = eK[EXZ]; exzM = eM[EXZ];

            if (out) {
                double* SK = S.S[w][0];
                double* SM = S.S[w][1];
                // segment of this lane: CSR base = row_ptr of its first owned lane; the staging offset keeps
                // the parity of the CSR position (16-byte alignment for bulk copies)
                const int a_seg = __shfl_sync(0xffffffffu, rp, lfirst);
                const int soff = ds.w + (a_seg & 1);
                int rlen = 0;
                if (owned) {
                    // stencil presence (canonical bounds) and slots in ascending column order
                    const bool px = I < p.nx, mx = I > 0, py = J < p.ny, my = J > 0, pz = Lz < p.nz, mz = Lz > 0;
                    uint32_t pres = 1u;
                    pres |= (uint32_t)px << 1 | (uint32_t)py << 2 | (uint32_t)pz << 3 | (uint32_t)(px && py) << 4 |
                            (uint32_t)(px && pz) << 5 | (uint32_t)(py && pz) << 6 | (uint32_t)(px && py && pz) << 7;
                    pres |= (uint32_t)mx << 8 | (uint32_t)my << 9 | (uint32_t)mz << 10 | (uint32_t)(mx && my) << 11 |
                            (uint32_t)(mx && mz) << 12 | (uint32_t)(my && mz) << 13 | (uint32_t)(mx && my && mz) << 14;
                    rlen = __popc(pres);
                    double sK = 0.0, sM = 0.0;
#pragma unroll
                    for (int e = 0; e < 7; e++) { sK += eK[e] + iK[e]; sM += eM[e] + iM[e]; }
                    const int base = soff + (rp - a_seg);
                    SK[base + __popc(pres & p.lower[0])] = -sK;
                    SM[base + __popc(pres & p.lower[0])] = sM * (2.0 / 3.0);
#pragma unroll
                    for (int e = 0; e < 7; e++) {
                        if (pres >> (1 + e) & 1) {
                            const int s = base + __popc(pres & p.lower[1 + e]);
                            SK[s] = eK[e];
                            SM[s] = eM[e];
                        }
                        if (pres >> (8 + e) & 1) {
                            const int s = base + __popc(pres & p.lower[8 + e]);
                            SK[s] = iK[e];
                            SM[s] = iM[e];
                        }
                    }
                }
                __syncwarp();
                // coalesced write-out, one segment at a time (the owned lanes of a segment are contiguous)
                uint32_t heads = __ballot_sync(0xffffffffu, owned && (fl & LF_HEAD));
                const int rend = rp + rlen;
                while (heads) {
                    const int h = __ffs(heads) - 1;
                    heads &= heads - 1;
                    const int a = __shfl_sync(0xffffffffu, rp, h);
                    const int hl = __shfl_sync(0xffffffffu, llast, h);
                    const int so = __shfl_sync(0xffffffffu, soff, h);
                    const int n = __shfl_sync(0xffffffffu, rend, hl) - a;
                    if (p.Kv)
                        for (int q = lane; q < n; q += 32) __stcs(p.Kv + a + q, SK[so + q]);
                    if (p.Mv)
                        for (int q = lane; q < n; q += 32) __stcs(p.Mv + a + q, SM[so + q]);
                }
            }
        }
    }
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
    const int64_t i = id % g.NX1, j = (id / g.NX1) % g.NY1, k = id / (g.NX1 * g.NY1);
    I = (int)(g.fx ? g.nx - i : i);
    J = (int)(g.fy ? g.ny - j : j);
    K = (int)(g.fz ? g.nz - k : k);
}

// every element is one Kuhn tetrahedron of the canonical lattice; its (cell, path) code is marked in a
// bitset, a code seen twice or a non-Kuhn element sets flags[0]
__global__ void lattice_check_elems_k(int64_t ne, int64_t nn, const int32_t* __restrict__ elems, int64_t eld,
                                      LatGeom g, uint32_t* __restrict__ bits, int* __restrict__ flags) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
        int I[4], J[4], K[4];
        bool bad = false;
#pragma unroll
        for (int a = 0; a < 4; a++) {
            const int32_t v = elems[a * eld + e];
            if (v < 0 || v >= nn) { bad = true; I[a] = J[a] = K[a] = 0; continue; }
            canon(g, v, I[a], J[a], K[a]);
        }
        int I0 = min(min(I[0], I[1]), min(I[2], I[3])), J0 = min(min(J[0], J[1]), min(J[2], J[3]));
        int K0 = min(min(K[0], K[1]), min(K[2], K[3]));
        // order the vertices by level (offset sum 0..3), each level exactly once
        int at[4] = {-1, -1, -1, -1};
#pragma unroll
        for (int a = 0; a < 4; a++) {
            const int ox = I[a] - I0, oy = J[a] - J0, oz = K[a] - K0;
            if (ox < 0 || ox > 1 || oy < 0 || oy > 1 || oz < 0 || oz > 1) { bad = true; continue; }
            const int lev = ox + oy + oz;
            if (at[lev] >= 0) bad = true;
            at[lev] = ox | oy << 1 | oz << 2;
        }
        if (!bad && (at[0] != 0 || at[3] != 7)) bad = true;
        if (I0 >= g.nx || J0 >= g.ny || K0 >= g.nz) bad = true;
        if (!bad) {
            const int s0 = at[1], s1 = at[2] & ~at[1];   // first and second unit steps
            if (__popc(s0) != 1 || __popc(at[2]) != 2 || (at[2] & s0) != s0) bad = true;
            else {
                const int p0 = __ffs(s0) - 1, p1 = __ffs(s1) - 1;
                const int path = p0 * 2 + ((p1 == (p0 + 1) % 3) ? 0 : 1);   // 6 paths
                const int64_t code = (((int64_t)K0 * g.ny + J0) * g.nx + I0) * 6 + path;
                const uint32_t bit = 1u << (code & 31);
                const uint32_t old = atomicOr(bits + (code >> 5), bit);
                if (old & bit) bad = true;
            }
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
    const int64_t NX1 = nx + 1, NY1 = ny + 1;
    h.id0 = (h.fx ? nx : 0) + NX1 * ((h.fy ? ny : 0) + NY1 * (int64_t)(h.fz ? nz : 0));
    h.dI = h.fx ? -1 : 1;
    h.dJ = (h.fy ? -1 : 1) * NX1;
    h.dK = (h.fz ? -1 : 1) * NX1 * NY1;
    int64_t off[15];
    for (int d = 0; d < 15; d++) off[d] = h.dI * dir_dx(d) + h.dJ * dir_dy(d) + h.dK * dir_dz(d);
    for (int d = 0; d < 16; d++) h.lower[d] = 0;
    for (int d = 0; d < 15; d++)
        for (int e = 0; e < 15; e++) {
            if (e != d && off[e] == off[d]) return false;   // two stencil columns with one id
            if (off[e] < off[d]) h.lower[d] |= (uint16_t)(1u << (e == 0 ? 0 : e));
        }
    // pres bit of direction d is bit d (self = bit 0); lower uses the same bits
    int idx[15];
    for (int d = 0; d < 15; d++) idx[d] = d;
    std::sort(idx, idx + 15, [&](int a, int b) { return off[a] < off[b]; });
    for (int r = 0; r < 15; r++) h.ord.dir[r] = idx[r];
    return true;
}

uint32_t lat_want(const LatHost& h, int64_t nn, int64_t nnz) {
    uint64_t z = 0x9E3779B97F4A7C15ull;
    auto mix = [&](uint64_t v) {
        z ^= v + 0x9E3779B97F4A7C15ull + (z << 6) + (z >> 2);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
    };
    mix(h.nx); mix(h.ny); mix(h.nz); mix(h.fx | h.fy << 1 | h.fz << 2); mix(nn); mix(nnz);
    const uint32_t t = LAT_MAGIC ^ (uint32_t)z ^ (uint32_t)(z >> 32);
    return t ? t : 1u;
}

// tiles of 32 lanes: x segments (the first owns 32 nodes, the next a halo lane + 31), y bands of LR rows
// (the first owns LR lines, the next a halo line + LR - 1); short segments of all bands packed together
void lat_tiles(int nx, int ny, std::vector<int4>& lanes, int& T) {
    struct Seg { int I0, halo, nown; };
    std::vector<Seg> full, shortv;
    {
        int nown = std::min(32, nx + 1);
        (nown == 32 ? full : shortv).push_back({0, 0, nown});
        int covered = nown - 1;
        while (covered < nx) {
            const int n = std::min(31, nx - covered);
            (n == 31 ? full : shortv).push_back({covered, 1, n});
            covered += n;
        }
    }
    std::vector<std::pair<int, int>> bands;   // (J0, row 0 owned)
    bands.push_back({0, 1});
    for (int covered = LR - 1; covered < ny; covered += LR - 1) bands.push_back({covered, 0});
    lanes.clear();
    auto lane_of = [](const Seg& sg, int J0, int row0, int lo, int k, int base, int l) {
        const int W = sg.nown + sg.halo;
        int fl = 0;
        if (!(sg.halo && l == lo)) fl |= LF_OWNX;
        if (l > lo) fl |= LF_LEFT;
        if (l == lo + W - 1) fl |= LF_XPLUS;
        if (row0) fl |= LF_ROW0;
        if (l == lo + sg.halo) fl |= LF_HEAD;
        const int col = l + k, first = lo + sg.halo, last = lo + W - 1;
        return make_int4(sg.I0 + (l - lo), J0, fl | col << 8 | first << 16 | last << 24, base);
    };
    const int4 idle = make_int4(-1, 0, (LCOLS - 1) << 8, 0);
    for (auto& b : bands)
        for (auto& sg : full)
            for (int l = 0; l < 32; l++) lanes.push_back(lane_of(sg, b.first, b.second, 0, 0, 0, l));
    if (!shortv.empty()) {
        // at most one short segment per band (the last one); all of the same width
        const int W = shortv[0].nown + shortv[0].halo;
        const int per = std::min(8, 32 / W);
        for (size_t b0 = 0; b0 < bands.size(); b0 += per) {
            int4 t[32];
            for (int l = 0; l < 32; l++) t[l] = idle;
            int base = 0;
            for (int k = 0; k < per && b0 + k < bands.size(); k++) {
                const int lo = k * W;
                for (int l = lo; l < lo + W; l++)
                    t[l] = lane_of(shortv[0], bands[b0 + k].first, bands[b0 + k].second, lo, k, base, l);
                base += 15 * shortv[0].nown + 2;
            }
            for (int l = 0; l < 32; l++) lanes.push_back(t[l]);
        }
    }
    T = (int)(lanes.size() / 32);
}

constexpr int LAT_HDR = 16;   // plan header ints (token, dims, flips, tiles), then the lane descriptors

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
    int T = 0;
    lat_tiles(nx, ny, lanes, T);
    const int64_t need_ints = LAT_HDR + (int64_t)T * 32 * 4;
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
    if (!stats_out || !elems || !row_ptr || !col_idx || elem_ld < ne) {
        set_error("%s: NULL argument or elem_ld < ne", fn);
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
    for (int a = 0; a < 4; a++) {
        vb_status st = read_small(s, elems + a * elem_ld, 4, &v0[a], fn);
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
    lattice_check_csr_k<<<grid_for(nn, 256, 8), 256, 0, s>>>(nn, nnz, row_ptr, col_idx, g, h.id0, h.dI, h.dJ, h.dK,
                                                             h.ord, flags);
    if ((st = launch_check(fn)) != VB_OK) return st;
    // header + lanes
    int32_t hdr[LAT_HDR] = {0};
    hdr[1] = nx; hdr[2] = ny; hdr[3] = nz;
    hdr[4] = h.fx; hdr[5] = h.fy; hdr[6] = h.fz; hdr[7] = T;
    e = cudaMemcpyAsync(plan, hdr, sizeof(hdr), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(plan + LAT_HDR, lanes.data(), lanes.size() * sizeof(int4), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) { set_error("%s: %s", fn, cudaGetErrorString(e)); return VB_ERR_CUDA; }
    lattice_token_k<<<1, 1, 0, s>>>(flags, reinterpret_cast<uint32_t*>(plan), lat_want(h, nn, nnz));
    if ((st = launch_check(fn)) != VB_OK) return st;
    int fl2[2];
    if ((st = read_small(s, flags, 8, fl2, fn)) != VB_OK) return st;   // synchronises: host arrays outlive
    if (fl2[0]) stats_out[2] = 4;       // an element is not a Kuhn tetrahedron of this lattice (or twice)
    else if (fl2[1]) stats_out[2] = 5;  // the CSR pattern is not the lattice stencil
    else stats_out[0] = 1;
    stats_out[3] = h.fx | h.fy << 1 | h.fz << 2;
    return VB_OK;
}

extern "C" VB_API vb_status fem_p1_assemble_lattice(int64_t nn, const double* coords, int64_t node_stride,
                                                    int64_t comp_stride, const int32_t* row_ptr, int64_t nnz,
                                                    const int32_t* plan, int nx, int ny, int nz, int flips,
                                                    double* K_vals, double* M_vals, vb_stream_t stream) {
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
    if (!K_vals && !M_vals) return VB_OK;
    const int fl[3] = {flips & 1, (flips >> 1) & 1, (flips >> 2) & 1};
    LatHost h;
    if (!lat_host(nx, ny, nz, fl, h)) { set_error("%s: degenerate lattice", fn); return VB_ERR_ARG; }
    std::vector<int4> lanes;
    int T = 0;
    lat_tiles(nx, ny, lanes, T);
    LatParams p;
    p.nx = nx; p.ny = ny; p.nz = nz; p.T = T;
    p.L = (int64_t)T * (nz + 1);
    p.id0 = h.id0; p.dI = h.dI; p.dJ = h.dJ; p.dK = h.dK;
    p.X = coords; p.ns = node_stride; p.cs = comp_stride;
    p.row_ptr = row_ptr;
    p.Kv = K_vals; p.Mv = M_vals;
    p.lanes = reinterpret_cast<const int4*>(plan + LAT_HDR);
    p.token = reinterpret_cast<const uint32_t*>(plan);
    p.want = lat_want(h, nn, nnz);
    for (int d = 0; d < 16; d++) p.lower[d] = h.lower[d];
    static int smem_set = 0;
    const size_t smem = sizeof(LatSmem);
    if (!smem_set) {
        cudaFuncSetAttribute(assemble_lattice_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        smem_set = 1;
    }
    int grid = sm_count();
    if (grid > p.L) grid = (int)p.L;
    assemble_lattice_k<<<grid, LTHREADS, smem, cs(stream)>>>(p);
    return launch_check(fn);
}

}  // namespace vb
