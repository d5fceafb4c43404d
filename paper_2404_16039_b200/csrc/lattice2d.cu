// Element-once 2D P1 K+M assembly on triangulated rectangular lattices (SURVEY §8(a) a7-a17 for BASELINE
// configs[0] and configs[3]; the 2D counterpart of lattice.cu).
//
// What is computed is exactly fem_p1_assemble's K and M with c = 1 in 2D (eq:K_M P:967-975, Code
// stiff_scalar_P1 P:978-1004, mass P:1007, sparse(X3D(:), Y3D(:), K3D(:)) P:1001-1003): per triangle
// tjac = D X^T, |T| = |det|/2, G = tjac^{-1} D, K_e = |T| G^T G, M_e = |T|/12 (1 + delta_ab); here
// K_e[a][b] = (h_a . h_b) / (2 |det|) with the adjugate columns h_1 = (f_2y, -f_2x), h_2 = (-f_1y, f_1x),
// h_0 = -(h_1 + h_2), f_r = x_r - x_0.
//
// The mesh: nodes (i, j), 0 <= i <= nx, 0 <= j <= ny, id = i + (nx+1) j; every cell split into two
// triangles by the same diagonal (either one; element order and vertex order free).  fem_plan_lattice2d
// verifies that once per mesh (every element is one of the two triangles of its cell, none twice; the CSR
// pattern is the 7-point stencil), so the numeric phase reads no connectivity.  In canonical coordinates
// (y mirrored so that the diagonal runs from (0,0) to (1,1)) node p owns its up edges +x, +y, +xy; the cell
// at p has the triangles A = (p, p+x, p+xy) and B = (p, p+y, p+xy): A gives +x and +xy of p and +y of p+x,
// B gives +y and +xy of p and +x of p+y.
//
// Kernel: a WARP holds one x segment (lane 0 a halo, 30 owned nodes, lane 31 their right neighbour, whose
// coordinates are all it contributes) and marches along y, one node row per
// step: both triangles of its cell once, the +y part of p+x by shuffle, the +x part of p+y and the finished
// +y, +xy edges carried in registers to the next row.  No shared-memory exchange and no barrier: warps are
// independent.  Rows (7 columns; diagonals by the partition of unity K_pp = -sum_q K_pq, M_pp = sum_q M_pq)
// are staged in CSR order and leave as TMA bulk copies.  Warps take contiguous ranges of the (segment, row)
// sequence (warps that run together cover whole x lines); a range that starts inside a segment recomputes one
// halo row.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "vb_internal.cuh"

namespace vb {
namespace {

constexpr int L2_WARPS = 4;                  // warps per CTA (27 KB of static staging)
constexpr int L2_THREADS = 32 * L2_WARPS;
constexpr int L2_OWN = 30;                   // owned nodes per segment (lanes 1..30)
constexpr int L2_STG = L2_OWN * 7 + 2;       // staging doubles per matrix, warp and buffer (parity offset, 16-byte multiple)
constexpr int L2_PF = 4;                     // coordinate rows in flight (registers)
constexpr int L2_MAXW = 1 << 15;             // most warp ranges a plan holds
constexpr uint32_t LAT2_MAGIC = 0x4c415432u;   // "LAT2"
constexpr int LAT2_HDR = 16;

// stencil directions: 0 self, 1 +x, 2 +y, 3 +xy, 4 -x, 5 -y, 6 -xy
__host__ __device__ constexpr int d2x(int d) { return d == 0 ? 0 : (d <= 3 ? 1 : -1) * ((d - 1) % 3 != 1); }
__host__ __device__ constexpr int d2y(int d) { return d == 0 ? 0 : (d <= 3 ? 1 : -1) * ((d - 1) % 3 != 0); }

// column order for orientation FY (canonical y mirrored or not): ids id0 + I + sy (nx+1) J sort by (sy dy, dx)
template <int FY>
struct Order2 {
    uint32_t low[7];
    int slot[7];
    __host__ __device__ constexpr Order2() : low(), slot() {
        for (int d = 0; d < 7; d++) {
            uint32_t m = 0;
            int c = 0;
            for (int e = 0; e < 7; e++) {
                const int od = d2x(d) + (FY ? -4 : 4) * d2y(d), oe = d2x(e) + (FY ? -4 : 4) * d2y(e);
                if (oe < od) { m |= 1u << e; c++; }
            }
            low[d] = m;
            slot[d] = c;
        }
    }
};

struct Lat2Params {
    int nx, ny, S;                // cells per axis, x segments
    int id0, dJ;                  // node id of canonical (I, J) = id0 + I + dJ J
    const double* X;
    int64_t ns, cs;
    const int32_t* row_ptr;
    double* Kv;
    double* Mv;
    const uint32_t* token;
    uint32_t want;
    int bulk;
    const int32_t* range;         // plan: warp w owns items [range[2w], range[2w+1]) of the (segment, row) sequence
    int nwarps;
};

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double rcp2d(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(y, fma(-x, y, 1.0), y);
    y = fma(y, fma(-x, y, 1.0), y);
    return y;
}
__device__ __forceinline__ double shu(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double shd(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }

struct Tri {
    double k01, k02, k12, m;
};
// triangle x0, x0 + f1, x0 + f2: off-diagonal K_e entries and |T|/12 = |det|/24; live = false gives zeros
__device__ __forceinline__ Tri tri(double f1x, double f1y, double f2x, double f2y, bool live) {
    const double det = fma(f1x, f2y, -f1y * f2x);
    const double ad = live ? fabs(det) : 0.0;
    const double s = live ? rcp2d(2.0 * ad) : 0.0;
    const double h1x = f2y, h1y = -f2x, h2x = -f1y, h2y = f1x;
    const double h0x = -(h1x + h2x), h0y = -(h1y + h2y);
    Tri t;
    t.k01 = s * fma(h0y, h1y, h0x * h1x);
    t.k02 = s * fma(h0y, h2y, h0x * h2x);
    t.k12 = s * fma(h1y, h2y, h1x * h2x);
    t.m = ad * (1.0 / 24.0);
    return t;
}

template <int FY>
__global__ void __launch_bounds__(L2_THREADS) assemble_lattice2d_k(const Lat2Params p) {
    constexpr Order2<FY> ORD{};
    __shared__ __align__(16) double stage[L2_WARPS][2][2][L2_STG];   // [warp][step parity][K, M]
    const int lane = threadIdx.x & 31;
    const int wl = threadIdx.x >> 5;
    const int gw = blockIdx.x * L2_WARPS + wl;
    if (*p.token != p.want || gw >= p.nwarps) return;   // plan of another mesh / not verified: write nothing
    int nst = 0;   // output steps of this warp: staging buffer = parity
    const int NJ = p.ny + 1;
    int64_t g = __ldg(p.range + 2 * gw);
    const int64_t g1 = __ldg(p.range + 2 * gw + 1);
    VB_CHECK(g >= 0 && g <= g1 && g1 <= (int64_t)p.S * NJ);
    while (g < g1) {
        const int sgm = (int)(g / NJ);
        const int ja = (int)(g % NJ);
        const int64_t gend = (int64_t)(sgm + 1) * NJ < g1 ? (int64_t)(sgm + 1) * NJ : g1;
        const int jb = (int)(gend - (int64_t)sgm * NJ);   // node rows [ja, jb)
        g = gend;
        const int nown = min(L2_OWN, p.nx + 1 - L2_OWN * sgm);
        const int I = L2_OWN * sgm - 1 + lane;             // lane 0: the halo node (virtual left of x = 0)
        const bool node = I >= 0 && I <= p.nx && lane <= nown + 1;
        const bool owned = lane >= 1 && lane <= nown;
        const bool cellx = node && I < p.nx && lane <= nown;
        const double* xg = p.X + (int64_t)(p.id0 + I) * p.ns;
        const int32_t* rpp = p.row_ptr + p.id0 + I;
        // predicated loads pinned where they are written (volatile): issued when the ring slot's old value is
        // dead, so that the load lands in the slot's register (no move of an in-flight register)
        auto ldrow = [&](int J, double& x, double& y) {
            const double* q = xg + (int64_t)J * p.dJ * p.ns;
            const int ok = J <= p.ny && node;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\nmov.f64 %0, 0d0000000000000000;\nmov.f64 %1, 0d0000000000000000;\n"
                "@p ld.global.nc.f64 %0, [%2];\n@p ld.global.nc.f64 %1, [%3];\n}\n"
                : "+d"(x), "+d"(y)   // in place: the slot keeps its register
                : "l"(q), "l"(q + p.cs), "r"(ok));
        };
        const int Ls = ja > 0 ? ja - 1 : ja;   // one halo row when the range starts inside the segment
        // A ring of L2_PF rows (coordinates and row_ptr) in registers: row J + L2_PF is requested in step J and
        // first used in step J + L2_PF - 1.  The loop is unrolled over the ring so that no in-flight register is
        // ever moved (a rotating array made every step wait for the youngest load: half of all stall samples).
        double xr[L2_PF], yr[L2_PF];
        int rpr[L2_PF];
        auto ldrp = [&](int J, int& r) {
            const int ok = J >= ja && J < jb && owned;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %2, 0;\nmov.b32 %0, 0;\n@p ld.global.nc.b32 %0, [%1];\n}\n"
                         : "+r"(r)
                         : "l"(rpp + (int64_t)J * p.dJ), "r"(ok));
        };
#pragma unroll
        for (int k = 0; k < L2_PF; k++) {
            xr[k] = yr[k] = 0.0;
            rpr[k] = 0;
            ldrow(Ls + k, xr[k], yr[k]);
            ldrp(Ls + k, rpr[k]);
        }
        double cxK = 0, cxM = 0, pyK = 0, pyM = 0, pxyK = 0, pxyM = 0;   // carries from the row below
        for (int Jb = Ls; Jb < jb; Jb += L2_PF) {
#pragma unroll
          for (int u = 0; u < L2_PF; u++) {
            const int J = Jb + u;
            if (J >= jb) break;
            const double x0 = xr[u], y0 = yr[u], x1 = xr[(u + 1) % L2_PF], y1 = yr[(u + 1) % L2_PF];
            const int rp = rpr[u];
            const bool out = J >= ja;
            // the cell at p: corners p (x0,y0), p+x, p+y (x1,y1), p+xy
            const double ax = shd(x0), ay = shd(y0), bx = shd(x1), by = shd(y1);
            const bool live = cellx && J < p.ny;
            const double ux = ax - x0, uy = ay - y0, vx = x1 - x0, vy = y1 - y0, wx = bx - x0, wy = by - y0;
            const int a_seg_ = __shfl_sync(0xffffffffu, rp, 1);   // the slot's old values are dead from here on
            ldrow(J + L2_PF, xr[u], yr[u]);
            ldrp(J + L2_PF, rpr[u]);
            const Tri A = tri(ux, uy, wx, wy, live);   // (p, p+x, p+xy)
            const Tri B = tri(vx, vy, wx, wy, live);   // (p, p+y, p+xy)
            // this node's up edges
            const double eXK = cxK + A.k01, eXM = cxM + A.m;
            const double eYK = B.k01 + shu(A.k12), eYM = B.m + shu(A.m);
            const double eXYK = A.k02 + B.k02, eXYM = A.m + B.m;
            // incoming edges: the up edges of the lower neighbours
            const double iXK = shu(eXK), iXM = shu(eXM);
            const double iYK = pyK, iYM = pyM;
            const double iXYK = shu(pxyK), iXYM = shu(pxyM);
            cxK = B.k12; cxM = B.m;
            pyK = eYK; pyM = eYM; pxyK = eXYK; pxyM = eXYM;
            if (out) {
                double* const SK = stage[wl][nst & 1][0];
                double* const SM = stage[wl][nst & 1][1];
                nst++;
                const int lfirst = 1, llast = nown;
                const int a_seg = a_seg_;
                const int soff = a_seg & 1;   // staging keeps the parity of the CSR position
                const bool px = I < p.nx, mx = I > 0, py = J < p.ny, my = J > 0;
                int rlen = 0;
                // the last step's copies are committed here; this buffer was read by the copies of two steps ago
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp();
                if (owned) {
                    const double sK = ((eXK + iXK) + (eYK + iYK)) + (eXYK + iXYK);
                    const double sM = ((eXM + iXM) + (eYM + iYM)) + (eXYM + iXYM);
                    double* rk = SK + soff + (rp - a_seg);
                    double* rm = SM + soff + (rp - a_seg);
                    VB_CHECK(rp >= a_seg && soff + (rp - a_seg) + 7 <= L2_STG);   // the row lies in the staging strip
                    if (px && mx && py && my) {   // interior row: all 7 columns
                        rlen = 7;
                        rk[ORD.slot[0]] = -sK;   rm[ORD.slot[0]] = sM;
                        rk[ORD.slot[1]] = eXK;   rm[ORD.slot[1]] = eXM;
                        rk[ORD.slot[2]] = eYK;   rm[ORD.slot[2]] = eYM;
                        rk[ORD.slot[3]] = eXYK;  rm[ORD.slot[3]] = eXYM;
                        rk[ORD.slot[4]] = iXK;   rm[ORD.slot[4]] = iXM;
                        rk[ORD.slot[5]] = iYK;   rm[ORD.slot[5]] = iYM;
                        rk[ORD.slot[6]] = iXYK;  rm[ORD.slot[6]] = iXYM;
                    } else {   // boundary row: the present columns, same order
                        const uint32_t pres = 1u | (uint32_t)px << 1 | (uint32_t)py << 2 | (uint32_t)(px && py) << 3 |
                                              (uint32_t)mx << 4 | (uint32_t)my << 5 | (uint32_t)(mx && my) << 6;
                        rlen = __popc(pres);
                        const double vk[7] = {-sK, eXK, eYK, eXYK, iXK, iYK, iXYK};
                        const double vm[7] = {sM, eXM, eYM, eXYM, iXM, iYM, iXYM};
#pragma unroll
                        for (int d = 0; d < 7; d++)
                            if (pres >> d & 1) {
                                const int s = __popc(pres & ORD.low[d]);
                                rk[s] = vk[d];
                                rm[s] = vm[d];
                            }
                    }
                }
                const int segend = __shfl_sync(0xffffffffu, rp + rlen, llast);
                if (p.bulk == 1) {
                    if (owned) {   // odd first / last entries: plain stores by the lanes that staged them
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
                    const int a = a_seg + (a_seg & 1), e = segend - (segend & 1);   // 16-byte aligned body
                    uint32_t el = 0;
                    asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(el));
                    if (el && e > a) {
                        const int bytes = (e - a) * 8;
                        if (p.Kv && p.Mv)
                            asm volatile(
                                "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %4;\n"
                                "cp.async.bulk.global.shared::cta.bulk_group [%2], [%3], %4;" ::"l"(p.Kv + a),
                                "r"(s32(SK + soff + (a - a_seg))), "l"(p.Mv + a), "r"(s32(SM + soff + (a - a_seg))),
                                "r"(bytes)
                                : "memory");
                        else if (p.Kv)
                            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p.Kv + a),
                                         "r"(s32(SK + soff + (a - a_seg))), "r"(bytes)
                                         : "memory");
                        else if (p.Mv)
                            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p.Mv + a),
                                         "r"(s32(SM + soff + (a - a_seg))), "r"(bytes)
                                         : "memory");
                    }
                } else if (p.bulk == 2) {   // aligned K, M: 128-bit plain stores of the body, odd ends by two lanes
                    __syncwarp();
                    const int a = a_seg + (a_seg & 1), e = segend - (segend & 1);
                    for (int q = a + 2 * lane; q < e; q += 64) {
                        if (p.Kv) __stcs(reinterpret_cast<double2*>(p.Kv + q), *reinterpret_cast<const double2*>(SK + soff + (q - a_seg)));
                        if (p.Mv) __stcs(reinterpret_cast<double2*>(p.Mv + q), *reinterpret_cast<const double2*>(SM + soff + (q - a_seg)));
                    }
                    if (lane == 0 && (a_seg & 1) && a_seg < segend) {
                        if (p.Kv) __stcs(p.Kv + a_seg, SK[soff]);
                        if (p.Mv) __stcs(p.Mv + a_seg, SM[soff]);
                    }
                    if (lane == 1 && (segend & 1) && segend - 1 > a_seg) {
                        if (p.Kv) __stcs(p.Kv + segend - 1, SK[soff + (segend - 1 - a_seg)]);
                        if (p.Mv) __stcs(p.Mv + segend - 1, SM[soff + (segend - 1 - a_seg)]);
                    }
                    __syncwarp();
                } else {
                    __syncwarp();
                    for (int q = a_seg + lane; q < segend; q += 32) {
                        if (p.Kv) p.Kv[q] = SK[soff + (q - a_seg)];
                        if (p.Mv) p.Mv[q] = SM[soff + (q - a_seg)];
                    }
                    __syncwarp();
                }
            }
          }
        }
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Degenerate triangles of the lattice (the optional counter; a pass of its own): the determinant exactly as the
// kernel evaluates it is 0, or two vertices of the triangle have identical coordinates.  One thread per cell.
__global__ void lattice2d_degenerate_k(int nx, int ny, int id0, int dJ, const double* __restrict__ X, int64_t ns,
                                       int64_t cs_, unsigned long long* __restrict__ out) {
    const int64_t ncell = (int64_t)nx * ny;
    int mine = 0;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell; c += (int64_t)gridDim.x * blockDim.x) {
        const int I = (int)(c % nx), J = (int)(c / nx);
        double x[4], y[4];   // corners p, p+x, p+y, p+xy
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int64_t v = id0 + (I + (q & 1)) + (int64_t)dJ * (J + (q >> 1));
            x[q] = X[v * ns];
            y[q] = X[cs_ + v * ns];
        }
        auto same = [&](int a, int b) { return x[a] == x[b] && y[a] == y[b]; };
        const double wx = x[3] - x[0], wy = y[3] - y[0];
#pragma unroll
        for (int t = 0; t < 2; t++) {   // A = (p, p+x, p+xy), B = (p, p+y, p+xy): det = f1x f2y - f1y f2x as in tri()
            const int a = t + 1;
            const double f1x = x[a] - x[0], f1y = y[a] - y[0];
            const double det = fma(f1x, wy, -f1y * wx);
            mine += det == 0.0 || same(0, a) || same(0, 3) || same(a, 3);
        }
    }
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(out, (unsigned long long)mine);
}

// ------------------------------------------------------------------ plan: verification kernels
struct Lat2Geom {
    int nx, ny, fy;
    int64_t NX1;
};
__device__ __forceinline__ void canon2(const Lat2Geom& g, int64_t id, int& I, int& J) {
    const int64_t i = id % g.NX1, j = id / g.NX1;
    I = (int)i;
    J = (int)(g.fy ? g.ny - j : j);
}
struct Lat2Order {
    int dir[7];
};

__global__ void lattice2d_check_elems_k(int64_t ne, int64_t nn, const int32_t* __restrict__ elems, int64_t eld,
                                        Lat2Geom g, uint32_t* __restrict__ bits, int* __restrict__ flags) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
        int I[3], J[3];
        bool bad = false;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            const int32_t v = elems[a * eld + e];
            if (v < 0 || v >= nn) { bad = true; I[a] = J[a] = 0; continue; }
            canon2(g, v, I[a], J[a]);
        }
        const int I0 = min(I[0], min(I[1], I[2])), J0 = min(J[0], min(J[1], J[2]));
        int have = 0;   // bit of offset code ox | oy << 1
#pragma unroll
        for (int a = 0; a < 3; a++) {
            const int ox = I[a] - I0, oy = J[a] - J0;
            if (ox < 0 || ox > 1 || oy < 0 || oy > 1) { bad = true; continue; }
            const int bit = 1 << (ox | oy << 1);
            if (have & bit) bad = true;
            have |= bit;
        }
        // corners 00 and 11 and one of 10 (triangle A) / 01 (triangle B)
        if (!bad && have != (1 | 8 | 2) && have != (1 | 8 | 4)) bad = true;
        if (I0 >= g.nx || J0 >= g.ny) bad = true;
        if (!bad) {
            const int64_t code = ((int64_t)J0 * g.nx + I0) * 2 + (have == (1 | 8 | 4));
            const uint32_t bit = 1u << (code & 31);
            if (atomicOr(bits + (code >> 5), bit) & bit) bad = true;
        }
        if (bad) atomicExch(flags, 1);
    }
}

__global__ void lattice2d_check_csr_k(int64_t nn, int64_t nnz, const int32_t* __restrict__ row_ptr,
                                      const int32_t* __restrict__ col_idx, Lat2Geom g, int64_t id0, int64_t dJ,
                                      Lat2Order ord, int* __restrict__ flags) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
        int I, J;
        canon2(g, v, I, J);
        const int64_t b = row_ptr[v], e = row_ptr[v + 1];
        bool bad = (v == 0 && b != 0) || (v == nn - 1 && e != nnz) || e < b;
        int64_t q = b;
        for (int r = 0; r < 7 && !bad; r++) {
            const int d = ord.dir[r];
            const int x = I + d2x(d), y = J + d2y(d);
            if (x < 0 || x > g.nx || y < 0 || y > g.ny) continue;
            if (q >= e || col_idx[q] != id0 + x + dJ * y) bad = true;
            q++;
        }
        if (!bad && q != e) bad = true;
        if (bad) atomicExch(flags + 1, 1);
    }
}

// the 7-point stencil written out as a CSR pattern (fem_lattice2d_pattern)
__global__ void lattice2d_rowlen_k(int64_t nn, Lat2Geom g, int32_t* __restrict__ row_len) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
        int I, J;
        canon2(g, v, I, J);
        int n = 0;
#pragma unroll
        for (int d = 0; d < 7; d++) {
            const int x = I + d2x(d), y = J + d2y(d);
            n += x >= 0 && x <= g.nx && y >= 0 && y <= g.ny;
        }
        row_len[v] = n;
    }
}
__global__ void lattice2d_cols_k(int64_t nn, Lat2Geom g, int64_t id0, int64_t dJ, Lat2Order ord,
                                 const int32_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
        int I, J;
        canon2(g, v, I, J);
        int64_t q = row_ptr[v];
#pragma unroll
        for (int r = 0; r < 7; r++) {
            const int d = ord.dir[r];
            const int x = I + d2x(d), y = J + d2y(d);
            if (x < 0 || x > g.nx || y < 0 || y > g.ny) continue;
            col_idx[q++] = (int32_t)(id0 + x + dJ * y);
        }
    }
}

__global__ void lattice2d_elem0_k(const int32_t* __restrict__ elems, int64_t eld, int32_t* __restrict__ out) {
    out[threadIdx.x] = elems[threadIdx.x * eld];
}
__global__ void lattice2d_token_k(const int* __restrict__ flags, uint32_t* __restrict__ token, uint32_t want) {
    *token = (flags[0] == 0 && flags[1] == 0) ? want : 0u;
}

// ------------------------------------------------------------------ host
struct Lat2Host {
    int nx, ny, fy;
    int64_t id0, dJ;
    Lat2Order ord;
};
bool lat2_host(int nx, int ny, int fy, Lat2Host& h) {
    h.nx = nx; h.ny = ny; h.fy = fy ? 1 : 0;
    const int64_t NX1 = nx + 1;
    if (NX1 * (ny + 1) >= ((int64_t)1 << 31) || nx < 2 || ny < 1) return false;
    h.id0 = h.fy ? NX1 * ny : 0;
    h.dJ = h.fy ? -NX1 : NX1;
    int64_t off[7];
    for (int d = 0; d < 7; d++) off[d] = d2x(d) + h.dJ * d2y(d);
    const Order2<0> o0{};
    const Order2<1> o1{};
    const uint32_t* low = h.fy ? o1.low : o0.low;
    for (int d = 0; d < 7; d++) {
        uint32_t m = 0;
        for (int e = 0; e < 7; e++) {
            if (e != d && off[e] == off[d]) return false;
            if (off[e] < off[d]) m |= 1u << e;
        }
        if (m != low[d]) return false;   // the kernel's compile-time column order must be the real one
    }
    int idx[7];
    for (int d = 0; d < 7; d++) idx[d] = d;
    std::sort(idx, idx + 7, [&](int a, int b) { return off[a] < off[b]; });
    for (int r = 0; r < 7; r++) h.ord.dir[r] = idx[r];
    return true;
}
uint32_t lat2_want(const Lat2Host& h, int64_t nn, int64_t nnz, int nwarps) {
    uint64_t z = 0x9E3779B97F4A7C15ull;
    auto mix = [&](uint64_t v) {
        z ^= v + 0x9E3779B97F4A7C15ull + (z << 6) + (z >> 2);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
    };
    mix(h.nx); mix(h.ny); mix(h.fy); mix(nn); mix(nnz); mix(nwarps);
    const uint32_t t = LAT2_MAGIC ^ (uint32_t)z ^ (uint32_t)(z >> 32);
    return t ? t : 1u;
}
int lat2_segments(int nx) { return (nx + 1 + L2_OWN - 1) / L2_OWN; }

// resident warps of the current device (the plan's ranges are for this many: the token covers it)
int lat2_warps(int nx, int ny) {
    static int occ_dev[64] = {};   // per device (idempotent)
    int dev = 0;
    cudaGetDevice(&dev);
    int occ = (dev >= 0 && dev < 64) ? occ_dev[dev] : 0;
    if (!occ) {
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, assemble_lattice2d_k<0>, L2_THREADS, 0) != cudaSuccess || o < 1)
            o = 1;
        occ = o;
        if (dev >= 0 && dev < 64) occ_dev[dev] = o;
    }
    const int64_t items = (int64_t)lat2_segments(nx) * (ny + 1);
    int64_t w = (int64_t)sm_count() * occ * L2_WARPS;
    w = std::min<int64_t>(w, L2_MAXW);
    // at least ~8 rows per warp (a range start costs a halo row)
    w = std::min<int64_t>(w, std::max<int64_t>(1, items / 8));
    return (int)w;
}

// Warp w = (row chunk c, segment s), s fastest: [start, end) in the (segment, row) item sequence.  Warps that
// run together then write the same node rows: whole x lines of K and M (DRAM pages written in full) instead of
// one 1.7 KB piece of thousands of different lines.  Meshes with fewer rows than warps per segment fall back to
// splitting the sequence evenly.
void lat2_ranges(int S, int NJ, int W, int* range) {
    const int chunks = W / S;
    for (int w = 0; w < W; w++) range[2 * w] = range[2 * w + 1] = 0;
    if (chunks >= 1) {
        const int R = (NJ + chunks - 1) / chunks;
        for (int c = 0; c < chunks; c++)
            for (int sg = 0; sg < S; sg++) {
                const int w = c * S + sg;
                const int j0 = std::min(NJ, c * R), j1 = std::min(NJ, (c + 1) * R);
                range[2 * w] = sg * NJ + j0;
                range[2 * w + 1] = sg * NJ + j1;
            }
        return;
    }
    const int64_t L = (int64_t)S * NJ;   // more segments than warps: contiguous pieces of the sequence
    for (int w = 0; w < W; w++) {
        range[2 * w] = (int)(L * w / W);
        range[2 * w + 1] = (int)(L * (w + 1) / W);
    }
}

}  // namespace

// ------------------------------------------------------------------ exports
extern "C" VB_API vb_status fem_plan_lattice2d(int64_t nn, int64_t ne, const int32_t* elems, int64_t elem_ld,
                                               const int32_t* row_ptr, const int32_t* col_idx, int64_t nnz, int nx,
                                               int ny, void* work, size_t* work_bytes, int32_t* plan,
                                               int64_t* plan_ints, int64_t* stats_out, vb_stream_t stream) {
    const char* fn = "fem_plan_lattice2d";
    clear_error();
    if (nx < 1 || ny < 1 || !work_bytes || !plan_ints) {
        set_error("%s: nx, ny must be >= 1 and work_bytes, plan_ints non-NULL", fn);
        return VB_ERR_ARG;
    }
    const int64_t nn_want = (int64_t)(nx + 1) * (ny + 1), ne_want = (int64_t)2 * nx * ny;
    const int64_t need_ints = LAT2_HDR + 2 * L2_MAXW;
    const size_t wb = 256 + (size_t)((ne_want + 31) / 32) * 4;
    if (!work) {
        *work_bytes = wb;
        *plan_ints = need_ints;
        return VB_OK;
    }
    if (*work_bytes < wb) { set_error("%s: work_bytes %zu < %zu", fn, *work_bytes, wb); return VB_ERR_WORKSPACE; }
    if (!plan || *plan_ints < need_ints) { set_error("%s: plan needs %lld ints", fn, (long long)need_ints); return VB_ERR_WORKSPACE; }
    if (!stats_out || !elems || (row_ptr == nullptr) != (col_idx == nullptr) || elem_ld < ne) {
        set_error("%s: NULL argument, only one of row_ptr / col_idx, or elem_ld < ne", fn);
        return VB_ERR_ARG;
    }
    stats_out[0] = stats_out[1] = stats_out[2] = stats_out[3] = 0;
    if (nn != nn_want || ne != ne_want) { stats_out[2] = 1; return VB_OK; }
    cudaStream_t s = cs(stream);
    int32_t v0[3];
    {
        lattice2d_elem0_k<<<1, 3, 0, s>>>(elems, elem_ld, reinterpret_cast<int32_t*>(work));
        vb_status st = launch_check(fn);
        if (st == VB_OK) st = read_small(s, work, sizeof(v0), v0, fn);
        if (st != VB_OK) return st;
    }
    // orientation from element 0: its longest edge is the cell diagonal, (1, 1) or (1, -1)
    int fy = -1;
    {
        const int64_t NX1 = nx + 1;
        for (int a = 0; a < 3 && fy < 0; a++)
            for (int b = 0; b < 3; b++) {
                if (v0[a] < 0 || v0[a] >= nn || v0[b] < 0 || v0[b] >= nn) { stats_out[2] = 2; return VB_OK; }
                const int64_t dx = v0[b] % NX1 - v0[a] % NX1, dy = v0[b] / NX1 - v0[a] / NX1;
                if (dx == 1 && (dy == 1 || dy == -1)) { fy = dy < 0; break; }
            }
        if (fy < 0) { stats_out[2] = 2; return VB_OK; }
    }
    Lat2Host h;
    if (!lat2_host(nx, ny, fy, h)) { stats_out[2] = 3; return VB_OK; }   // nx < 2 or ids that do not order as the kernel assumes
    Lat2Geom g{nx, ny, h.fy, (int64_t)nx + 1};
    int* flags = reinterpret_cast<int*>(work);
    uint32_t* bits = reinterpret_cast<uint32_t*>(static_cast<char*>(work) + 256);
    cudaError_t e = cudaMemsetAsync(work, 0, wb, s);
    if (e != cudaSuccess) { set_error("%s: %s", fn, cudaGetErrorString(e)); return VB_ERR_CUDA; }
    lattice2d_check_elems_k<<<grid_for(ne, 256, 8), 256, 0, s>>>(ne, nn, elems, elem_ld, g, bits, flags);
    vb_status st = launch_check(fn);
    if (st != VB_OK) return st;
    if (row_ptr) {   // NULL, NULL: the pattern comes from fem_lattice2d_pattern (the stencil by construction)
        lattice2d_check_csr_k<<<grid_for(nn, 256, 8), 256, 0, s>>>(nn, nnz, row_ptr, col_idx, g, h.id0, h.dJ, h.ord,
                                                                   flags);
        if ((st = launch_check(fn)) != VB_OK) return st;
    }
    const int S = lat2_segments(nx), W = lat2_warps(nx, ny);
    int32_t hdr[LAT2_HDR] = {0};
    hdr[1] = nx; hdr[2] = ny; hdr[3] = h.fy; hdr[4] = S; hdr[5] = W;
    std::vector<int> range(2 * L2_MAXW, 0);
    lat2_ranges(S, ny + 1, W, range.data());
    e = cudaMemcpyAsync(plan, hdr, sizeof(hdr), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(plan + LAT2_HDR, range.data(), range.size() * sizeof(int), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) { set_error("%s: %s", fn, cudaGetErrorString(e)); return VB_ERR_CUDA; }
    lattice2d_token_k<<<1, 1, 0, s>>>(flags, reinterpret_cast<uint32_t*>(plan), lat2_want(h, nn, nnz, W));
    if ((st = launch_check(fn)) != VB_OK) return st;
    int fl2[2];
    if ((st = read_small(s, flags, 8, fl2, fn)) != VB_OK) return st;   // synchronises: host arrays outlive
    if (fl2[0]) stats_out[2] = 4;
    else if (fl2[1]) stats_out[2] = 5;
    else stats_out[0] = 1;
    stats_out[1] = S;
    stats_out[3] = h.fy | (int64_t)W << 8;
    return VB_OK;
}

extern "C" VB_API vb_status fem_lattice2d_pattern(int64_t nn, int nx, int ny, int flips, void* work, size_t* work_bytes,
                                                  int32_t* row_ptr, int32_t* col_idx, int64_t col_cap,
                                                  int64_t* nnz_out, vb_stream_t stream) {
    const char* fn = "fem_lattice2d_pattern";
    clear_error();
    if (nx < 1 || ny < 1 || (int64_t)(nx + 1) * (ny + 1) != nn || !work_bytes) {
        set_error("%s: nx, ny >= 1, nn = (nx+1)(ny+1) and work_bytes non-NULL are required", fn);
        return VB_ERR_ARG;
    }
    int64_t nnz = 0;   // direction d is present at (nx+1-|dx|)(ny+1-|dy|) nodes
    for (int d = 0; d < 7; d++) nnz += (int64_t)(nx + 1 - std::abs(d2x(d))) * (ny + 1 - std::abs(d2y(d)));
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
    Lat2Host h;
    if (!lat2_host(nx, ny, flips & 1, h)) { set_error("%s: lattice outside the kernel's limits (nx >= 2)", fn); return VB_ERR_UNSUPPORTED; }
    Lat2Geom g{nx, ny, h.fy, (int64_t)nx + 1};
    cudaStream_t s = cs(stream);
    int32_t* row_len = reinterpret_cast<int32_t*>(work);
    lattice2d_rowlen_k<<<grid_for(nn, 256, 8), 256, 0, s>>>(nn, g, row_len);
    vb_status st = launch_check(fn);
    if (st != VB_OK) return st;
    if ((st = exclusive_scan_i32(row_len, row_ptr, nn, static_cast<char*>(work) + len_bytes, s, nullptr)) != VB_OK) return st;
    lattice2d_cols_k<<<grid_for(nn, 256, 8), 256, 0, s>>>(nn, g, h.id0, h.dJ, h.ord, row_ptr, col_idx);
    return launch_check(fn);
}

extern "C" VB_API vb_status fem_p1_assemble_lattice2d(int64_t nn, const double* coords, int64_t node_stride,
                                                      int64_t comp_stride, const int32_t* row_ptr, int64_t nnz,
                                                      const int32_t* plan, int nx, int ny, int flips, double* K_vals,
                                                      double* M_vals, int64_t* degenerate, vb_stream_t stream) {
    const char* fn = "fem_p1_assemble_lattice2d";
    clear_error();
    if (nx < 1 || ny < 1 || (int64_t)(nx + 1) * (ny + 1) != nn) { set_error("%s: nn != (nx+1)(ny+1)", fn); return VB_ERR_ARG; }
    if (!coords || !row_ptr || !plan || nnz < 0 || nnz >= ((int64_t)1 << 31)) {
        set_error("%s: NULL coords/row_ptr/plan or bad nnz", fn);
        return VB_ERR_ARG;
    }
    if (!K_vals && !M_vals && !degenerate) return VB_OK;
    Lat2Host h;
    if (!lat2_host(nx, ny, flips & 1, h)) { set_error("%s: lattice outside the kernel's limits (nx >= 2)", fn); return VB_ERR_ARG; }
    const int W = lat2_warps(nx, ny), w_plan = flips >> 8;
    if (w_plan && w_plan != W) {
        set_error("%s: the plan was built for another device (%d warps, this device: %d)", fn, w_plan, W);
        return VB_ERR_ARG;
    }
    Lat2Params p;
    p.nx = nx; p.ny = ny; p.S = lat2_segments(nx);
    p.id0 = (int)h.id0; p.dJ = (int)h.dJ;
    p.X = coords; p.ns = node_stride; p.cs = comp_stride;
    p.row_ptr = row_ptr;
    p.Kv = K_vals; p.Mv = M_vals;
    p.token = reinterpret_cast<const uint32_t*>(plan);
    p.want = lat2_want(h, nn, nnz, W);
    p.bulk = (!K_vals || aligned16(K_vals)) && (!M_vals || aligned16(M_vals));
#ifdef VB_LAT2_PLAIN
    if (p.bulk) p.bulk = 2;
#endif
    p.range = plan + LAT2_HDR;
    p.nwarps = W;
    if (degenerate) {   // a pass of its own over the cells, with the kernel's determinant expression
        cudaError_t e = cudaMemsetAsync(degenerate, 0, sizeof(int64_t), cs(stream));
        if (e != cudaSuccess) { set_error("%s: %s", fn, cudaGetErrorString(e)); return VB_ERR_CUDA; }
        lattice2d_degenerate_k<<<grid_for((int64_t)nx * ny, 256, 8), 256, 0, cs(stream)>>>(
            nx, ny, (int)h.id0, (int)h.dJ, coords, node_stride, comp_stride,
            reinterpret_cast<unsigned long long*>(degenerate));
        vb_status st = launch_check(fn);
        if (st != VB_OK) return st;
    }
    if (!K_vals && !M_vals) return VB_OK;
    const int grid = (W + L2_WARPS - 1) / L2_WARPS;
    if (h.fy) assemble_lattice2d_k<1><<<grid, L2_THREADS, 0, cs(stream)>>>(p);
    else assemble_lattice2d_k<0><<<grid, L2_THREADS, 0, cs(stream)>>>(p);
    return launch_check(fn);
}

}  // namespace vb
