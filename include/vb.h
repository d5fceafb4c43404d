/*
 * vb.h -- C ABI of the B200-native page-wise fp64 linear algebra and P1 FEM
 * assembly library (libvb.so), the hot path of arXiv 2404.16039.
 *
 * Citation keys: P:n = PAPER.md line n (arXiv 2404.16039 LaTeX source);
 * S:n = SPEC.md line n; SURVEY.md §8 rows a1..a17.
 *
 * ------------------------------------------------------------------ conventions
 * Memory.  Every array argument is a DEVICE pointer owned by the caller.  The
 *   library never allocates device memory, never frees, and keeps no pointer
 *   after a call returns.  Scratch space is passed as (work, work_bytes): call
 *   once with work == NULL to query *work_bytes, then again with a buffer of at
 *   least that size (16-byte aligned).
 * Streams.  All work is enqueued on `stream` (a cudaStream_t; NULL = legacy
 *   default stream).  Calls return after enqueueing, except where a host
 *   synchronisation is documented (fem_p1_pattern's count phase reads nnz).
 *   Calls on different streams with disjoint buffers are thread-safe.
 * Devices.  Calls act on the current CUDA device of the calling thread; the
 *   intended use is one process per GPU (the library caches launch attributes
 *   of its larger kernels per process; the lattice entry points per device).
 * Page layout (SURVEY B2, P:248-266 with the index space W as the page index,
 *   S:32): a batch of N pages of r x c matrices is stored struct-of-arrays:
 *   entry (i, j) of page k is at  p[(i + j*r) * ld + k]  (column-major entry
 *   order as in MATLAB, one contiguous plane of N values per entry), ld >= N.
 *   ld == 0 is the copy map eq:copy: ONE r x c object stored
 *   column-major and contiguous (p[i + j*r]) is used for every page -- this is
 *   how amsm/amsv/smamt/svamt broadcast single objects.
 *   A contiguous torch tensor of shape (c, r, N) is a valid operand, ld = N.
 *   Fast paths need 16-byte aligned planes and even ld; other inputs take a
 *   scalar path of the same kernels (no other backend exists).
 * Outputs are overwritten, never accumulated, and must not alias any input.
 * Indices are 0-based int32 (MATLAB is 1-based).  Vertex indices
 *   out of [0, nn) are a precondition violation and are not checked on the
 *   hot path.
 * Errors.  Argument/shape errors return a negative vb_status synchronously
 *   and set a thread-local message (vb_last_error) naming the offending
 *   argument.  Numerical singularity is NOT an error (inverse_W is only
 *   defined where det != 0): results follow IEEE arithmetic and
 *   are flagged where documented.  VB_ERR_CUDA reports a launch failure.
 */
#ifndef VB_H_
#define VB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define VB_API __attribute__((visibility("default")))
#else
#define VB_API
#endif

typedef struct CUstream_st* vb_stream_t; /* == cudaStream_t */

typedef enum {
    VB_OK = 0,
    VB_ERR_ARG = -1,         /* NULL pointer, negative size, bad flag, bad ld   */
    VB_ERR_DIM = -2,         /* inner dimensions disagree / page not square     */
    VB_ERR_UNSUPPORTED = -3, /* page size outside 1..4, dim outside {2,3}, ...  */
    VB_ERR_OVERFLOW = -4,    /* a count does not fit int32 (nnz, ne*nv*nv, ...) */
    VB_ERR_WORKSPACE = -5,   /* work buffer missing or smaller than queried     */
    VB_ERR_CUDA = -6         /* a CUDA launch or copy failed                    */
} vb_status;

/* Message of the last failing call on this host thread ("" if none). */
VB_API const char* vb_last_error(void);
/* ABI version, currently 2 (work / degenerate arguments of the assembly calls). */
VB_API int vb_abi_version(void);

/* ---------------------------------------------------------- a1 page product
 * Z_k = op(X_k) * op(Y_k) for k = 0..npages-1, op(A) = A or A^T by the flag.
 * Page-wise matrix multiplication eq:pagewisemultGeneral / layeredMultiplication
 * = MATLAB pagemtimes(X, tX, Y, tY).  Every library
 * product of P:380-411 is one call: amtam = (tX=1, tY=0) (reading B1),
 * avtam/avtav = X of r x 1 pages with tX=1, astam = X of 1 x 1 pages,
 * amsm/amsv = ldy 0, smamt = ldx 0 with tY=1, svamt = ldx 0, tX=1, tY=1.
 * xrows/xcols, yrows/ycols describe the STORED X, Y (each 1..4).
 * Z is (rows of op(X)) x (cols of op(Y)), ldz >= npages.
 * Errors: VB_ERR_DIM if the inner dimensions of op(X), op(Y) differ;
 * VB_ERR_UNSUPPORTED if any dimension is outside 1..4; VB_ERR_ARG for ld < npages
 * (other than 0 on an input) or NULL pointers with npages > 0. npages == 0 is a no-op. */
VB_API vb_status vb_page_mtimes(int64_t npages,
                         const double* X, int xrows, int xcols, int64_t ldx, int transX,
                         const double* Y, int yrows, int ycols, int64_t ldy, int transY,
                         double* Z, int64_t ldz, vb_stream_t stream);

/* ---------------------------------------------------------- a2 page transpose
 * Z_k = X_k^T (layeredTransposeHom/Ten P:268-279; amt = pagetranspose P:415).
 * X is rows x cols (1..4 each), Z is cols x rows.  Exact (a permutation of
 * planes).  ldx may be 0 (broadcast). */
VB_API vb_status vb_page_transpose(int64_t npages, const double* X, int rows, int cols, int64_t ldx,
                            double* Z, int64_t ldz, vb_stream_t stream);

/* ---------------------------------------------------------- a3 page determinant
 * det[k] = det X_k for n x n pages, n in 1..4 (layeredDeterminant P:331-336;
 * amdet P:418-420).  Closed forms: n<=3 cofactor expansion, n=4 Laplace
 * expansion by the 2x2 minors of rows (0,1) and (2,3).  det is one plane of
 * npages values. */
VB_API vb_status vb_page_det(int64_t npages, int n, const double* X, int64_t ldx,
                      double* det, vb_stream_t stream);

/* ---------------------------------------------------------- a4 page inverse
 * Xinv_k = adj(X_k) / det X_k (layeredInverse P:338-352; aminv P:414, which
 * also returns the determinant), n in 1..4, one reciprocal per page.
 * det (nullable) receives the signed determinants (reading B6).
 * first_singular (nullable, DEVICE int64 scalar): set in-stream to the
 * smallest page index k with |det X_k| <= sing_tol * ||X_k||_inf^n, or to
 * npages if there is none (SPEC S:141 uses sing_tol = 1e-14).  Singular pages
 * still produce IEEE results (inf/nan). */
VB_API vb_status vb_page_inv(int64_t npages, int n, const double* X, int64_t ldx,
                      double* Xinv, int64_t ldinv, double* det,
                      int64_t* first_singular, double sing_tol, vb_stream_t stream);

/* ---------------------------------------------------------- a5 page cross product
 * C_k = A_k x B_k for 3-vector pages (3 x 1; BASELINE.json north_star; the
 * cofactor columns of eq:transformNormal P:354-374 are such products). */
VB_API vb_status vb_page_cross(int64_t npages, const double* A, int64_t lda, const double* B, int64_t ldb,
                        double* C, int64_t ldc, vb_stream_t stream);

/* ---------------------------------------------------------- a7 gather (coords3D)
 * create_coords3D (Code coords3D): coords3D is a dim x nv page
 * array (ld = ne) with column a of page e = coordinates of vertex elems[a][e];
 * vectors3D (nullable) is dim x (nv-1) with column a = x_a - x_{nv-1}
 * (vectors from the LAST local node).  coords are addressed
 * coords[c*comp_stride + v*node_stride] (SoA: node_stride 1, comp_stride nn;
 * AoS/padded AoS: node_stride dim or 4, comp_stride 1).  elems[a*elem_ld + e].
 * dim in {2,3}, nv in 2..4. */
VB_API vb_status vb_create_coords3D(int dim, int nv, int64_t ne,
                             const double* coords, int64_t node_stride, int64_t comp_stride,
                             const int32_t* elems, int64_t elem_ld,
                             double* coords3D, double* vectors3D, vb_stream_t stream);

/* NEXT-4, fused: signed sizes and (not normalised) outer normals of every simplex
 * in one pass over coords and elems, the paper's two scripts
 *   [~, vectors3D] = create_coords3D(coords, elems);
 *   meass = amdet(vectors3D) / factorial(dim);
 *   normals3D = amsm(amt(aminv(vectors3D)), normalsRef);
 * without the intermediate page arrays (the chain of page calls above gives the
 * same values and remains available).  dim in {2, 3}; elems: dim+1 vertex
 * planes (elems[a*elem_ld + e]); coords strided as in vb_create_coords3D.
 * meass (DEVICE, ne; nullable): det[v_0 .. v_{d-1}] / d!, v_a = x_a - x_d (vectors
 * from the LAST local node); its sign is the orientation, meas =
 * norm(meass, 1).  normals3D (DEVICE, nullable): dim x (dim+1) pages,
 * entry (c, j) of page e at normals3D[(c + j*dim)*ldn + e], ldn >= ne; column
 * j is the outer normal of the face opposite local node j, of length (face
 * size) / (d |T|) (normalsRef = [-I | 1]; in 2D the same
 * construction).  At least one output is required.  Planes that are 16-byte
 * aligned with even ldn / elem_ld take the 128-bit path; any other layout is
 * handled with scalar accesses (same values).  A degenerate element (det = 0)
 * gives meass = 0 and non-finite normals, as aminv does; no
 * validation of vertex ids.  Asynchronous on `stream`; errors as above. */
VB_API vb_status vb_simplex_geometry(int dim, int64_t ne,
                              const double* coords, int64_t node_stride, int64_t comp_stride,
                              const int32_t* elems, int64_t elem_ld,
                              double* meass, double* normals3D, int64_t ldn, vb_stream_t stream);

/* ---------------------------------------------------------- a6 surface geometry
 * For each triangle f = (a, b, c) (tri[v*tri_ld + f], v = 0..2) of a closed
 * surface with vertex coordinates xyz (strided as above):
 *   n_f = (b-a) x (c-a)        (3 planes, ld = nf; nullable)
 *   nhat_f = n_f / |n_f|       (3 planes, ld = nf; nullable)
 *   area_f = |n_f| / 2         (1 plane; nullable)
 *   *volume = sum_f (1/6) a . n_f   (DEVICE scalar, nullable): the divergence
 *   theorem with F = x/3 (surf_int).  The sum uses a fixed-shape
 *   tree (per-block then one block), so it is bitwise reproducible run to run.
 * Requires work (query with work == NULL) when volume != NULL. */
VB_API vb_status vb_tri_surface(int64_t nf, const int32_t* tri, int64_t tri_ld, int64_t nverts,
                         const double* xyz, int64_t node_stride, int64_t comp_stride,
                         double* n, double* nhat, double* area, double* volume,
                         void* work, size_t* work_bytes, vb_stream_t stream);

/* ---------------------------------------------------------- a14/a15 pattern + plans
 * Topological CSR pattern of K = sparse(X3D(:), Y3D(:), K3D(:), nn, nn)
 * (reading B12: every pair (i, j) of vertices sharing an element,
 * diagonal included, kept even where the value cancels), columns ascending.
 * dim in {2,3} (nv = dim+1 vertices per element), elems[a*elem_ld + e].
 *
 * Count phase (col_idx == NULL): writes row_ptr[0..nn], then SYNCHRONISES the
 *   stream and stores nnz in *nnz_out (host int64).
 * Fill phase (col_idx != NULL, col_cap >= nnz, row_ptr from the count phase;
 *   also synchronises the stream, to check col_cap and the row-length flags).
 *   Given the count phase's work buffer (same elems pointer, sizes and elem_ld,
 *   recorded there by the count phase), it reuses the node->element incidence
 *   lists and the row lists the count phase left in work; with any other work
 *   buffer it rebuilds them (same results, slower).  elems must therefore not
 *   change between a count and a fill call that share a work buffer.  Writes:
 *   writes col_idx[0..nnz) and the optional scatter plans:
 *   elem2nnz (nullable): int32, nv*nv planes of ne: plane (a*nv + b) entry e is
 *     the position in col_idx of column elems[b][e] in row elems[a][e]
 *     (the scatter map of VB_ASSEMBLE_ATOMIC);
 *   node_elem_ptr (nullable, nn+1 int32) / node_elem (nv*ne int32) /
 *     node_elem_slot (nv*ne uint32): the gather plan of VB_ASSEMBLE_GATHER:
 *     for row v, entries node_elem_ptr[v]..node_elem_ptr[v+1]-1 list the
 *     incidences (e, a) with elems[a][e] == v, packed e*4 + a, ascending e;
 *     node_elem_slot packs in-row offsets (positions within row v's columns):
 *     byte 0 = offset of v itself (the diagonal), bytes 1..nv-1 = offsets of
 *     the element's other vertices elems[b][e], b != a, in ascending b (so
 *     rows must have <= 255 entries; VB_ERR_UNSUPPORTED otherwise).
 * Validation mode: dim | VB_PATTERN_VALIDATE checks every vertex id against
 *   [0, nn) before anything else (one more read-back) and returns VB_ERR_ARG
 *   naming the first offending element and vertex (without it, out-of-range
 *   ids are a precondition violation, not checked).
 * Errors: VB_ERR_OVERFLOW if nnz >= 2^31 or ne*nv*nv >= 2^31 or ne >= 2^29;
 *   VB_ERR_UNSUPPORTED if a row has more than 4096 distinct columns;
 *   VB_ERR_ARG if col_cap < nnz.  Deterministic: identical outputs every run. */
#define VB_PATTERN_VALIDATE 0x100
VB_API vb_status fem_p1_pattern(int dim, int64_t nn, int64_t ne,
                         const int32_t* elems, int64_t elem_ld,
                         void* work, size_t* work_bytes,
                         int32_t* row_ptr, int32_t* col_idx, int64_t col_cap,
                         int32_t* elem2nnz,
                         int32_t* node_elem_ptr, int32_t* node_elem, uint32_t* node_elem_slot,
                         int64_t* nnz_out, vb_stream_t stream);

/* Plan statistics for choosing the gather kernel's shared-memory budget
 * (VB_GATHER_HINT_COMPACT): stats_out (HOST, 3 values) = maximum row length,
 * maximum CSR entries of a 32-row block, maximum incidences of a 32-row block
 * (node_elem_ptr nullable: then 0).  work: DEVICE scratch of >= 16 bytes.
 * Synchronises the stream. */
VB_API vb_status fem_plan_stats(int64_t nn, const int32_t* row_ptr, const int32_t* node_elem_ptr, void* work,
                                int64_t* stats_out, vb_stream_t stream);

/* Packed 16-bit form of the P1 gather plan words, required with
 * VB_GATHER_HINT_COMPACT: packed[i] = o1 | o2 << 4 | o3 << 8 (2D: o1 | o2 << 4)
 * with o_j the in-row offsets of the incidence's other vertices (bytes 1..nv-1
 * of node_elem_slot[i]).  packed (n_inc uint16, DEVICE) must be readable up to
 * the next multiple of 8 entries.  work: DEVICE scratch of >= 16 bytes.
 * VB_ERR_UNSUPPORTED if an offset is >= 16 (a row with more than 16 entries).
 * Synchronises the stream. */
VB_API vb_status fem_plan_pack_slots(int dim, int64_t n_inc, const uint32_t* node_elem_slot, uint16_t* packed,
                                     void* work, vb_stream_t stream);

/* Row classes of the P1 gather plan (the plan of the class variant,
 * fem_p1_assemble_classes).  The row of node v is assembled from its
 * incidences (plan words node_elem_slot[node_elem_ptr[v] ..], ascending
 * element); its signature is (row length, incidence count, plan
 * words).  Rows with equal signatures run the same operations on different
 * coordinates, so a warp assembles up to 32 of them with one uniform loop.
 * Outputs (DEVICE, caller-owned):
 *   class_rows (nn int32): all rows, grouped by class (ascending row id within
 *     a class); rows in classes of fewer than 8 rows, rows with more than 15
 *     (3D) / 12 (2D) entries or more than 32 (3D) / 16 (2D) incidences and rows
 *     without incidences form the last,
 *     "mixed" class;
 *   groups (groups_cap x 4 int32): group g = (first position in class_rows,
 *     row count <= 32, first row of its class or -1 for the mixed class, 0).
 * stats_out (HOST, 4 int64): number of groups, number of classes (mixed
 * excluded), rows in classes, longest row in a class (the c = 1 kernel takes
 * 2D classes of up to 8 entries and assembles longer ones like mixed rows).  work: DEVICE scratch; work == NULL queries its
 * size into *work_bytes.  VB_ERR_WORKSPACE if the groups do not fit groups_cap
 * (stats_out[0] then holds the count needed).  Deterministic; synchronises the
 * stream (one small read-back). */
VB_API vb_status fem_plan_classes(int dim, int64_t nn, const int32_t* row_ptr, const int32_t* node_elem_ptr,
                                  const uint32_t* node_elem_slot, void* work, size_t* work_bytes,
                                  int32_t* class_rows, int32_t* groups, int64_t groups_cap,
                                  int64_t* stats_out, vb_stream_t stream);

/* ---------------------------------------------------------- a7..a17 assembly
 * Global P1 stiffness and mass matrices with c_K = c_M = 1 (eq:K_M P:967-975,
 * stiffness_matrixP1 P:978-1004, mass_matrixP1 P:1007), written
 * as CSR values on the pattern of fem_p1_pattern.  Per element:
 *   tjac = D X^T  (J[r][c] = x_{r+1}[c] - x_0[c]),  |T| = |det tjac| / d!,
 *   G = tjac^{-1} D (D = [-1 | I]),  K_e = |T| G^T G,
 *   M_e = |T| / ((d+1)(d+2)) (1 + delta_ab).
 * mode VB_ASSEMBLE_ATOMIC: one thread per element, K_e/M_e added into
 *   K_vals/M_vals through elem2nnz with fp64 atomics (targets are zero-filled
 *   by the call); summation order unspecified (reading B13).
 * mode VB_ASSEMBLE_GATHER: deterministic segmented reduction: one thread per
 *   row v sums the contributions of its incidences in ascending element order
 *   (the oracle's order) in on-chip memory and writes each CSR entry once; no
 *   atomics, no zero-fill.  Needs col_idx, node_elem_ptr and node_elem_slot
 *   (node_elem is not read).  col_idx and node_elem_slot are streamed with
 *   16-byte TMA bulk copies: both must be 16-byte aligned (VB_ERR_ARG
 *   otherwise) and readable up to the next multiple of 4 entries (torch
 *   allocations satisfy this).
 *   Diagonals follow from the partition of unity sum_b phi_b = 1
 *   (K_vv = -sum_{w!=v} K_vw, M_vv = (2/d) sum_{w!=v} M_vw).
 *   Bitwise reproducible.
 * K_vals / M_vals (nnz each) are nullable (skip that matrix).
 * K_local / M_local (nullable): K3D / M3D page arrays (nv x nv pages, ld = ne),
 *   the second outputs of stiffness_matrixP1 / mass_matrixP1.
 * coords strided as in vb_create_coords3D.
 * work (DEVICE, caller-owned, 16-byte aligned, >= *work_bytes = 16 bytes):
 *   holds this launch's block counter of the gather kernels' dynamic schedule
 *   (zeroed in-stream by the call), so concurrent calls on different streams
 *   are independent when each has its own work buffer.  work == NULL with
 *   work_bytes != NULL is a size query (nothing else happens); work == NULL
 *   with work_bytes == NULL runs the static block schedule (no counter).
 * degenerate (nullable DEVICE int64): receives the number of elements with
 *   det tjac = 0 (outside the domain of inverse_W; tjac rows
 *   x_{r+1} - x_0, det by cofactor expansion along row 0) as the kernel
 *   evaluates it, or with two vertices of identical coordinates (whose exact
 *   determinant 0 may be evaluated as a rounding residual); the same rule in
 *   every kernel that takes this argument -- an extra pass over the elements
 *   when requested.  Degenerate elements still propagate
 *   inf/nan into K/M (IEEE; not an error code). */
#define VB_ASSEMBLE_ATOMIC 0
#define VB_ASSEMBLE_GATHER 1
/* Hint OR'ed into a gather mode (3D; ignored otherwise): every 32-row block of
 * the plan has rows of <= 15 columns, <= 16*32 CSR entries and <= 25*32
 * incidences (fem_p1_pattern's stats_out tells; Kuhn cubes qualify).  The
 * kernel then runs with a smaller shared-memory budget (9 instead of 7 CTAs
 * per SM) and node_elem_slot must point to the packed 16-bit plan words of
 * fem_plan_pack_slots.  Blocks that do not fit the budget are still assembled
 * correctly (in place in HBM), only slower. */
#define VB_GATHER_HINT_COMPACT 0x100
VB_API vb_status fem_p1_assemble(int dim, int64_t nn, int64_t ne,
                          const double* coords, int64_t node_stride, int64_t comp_stride,
                          const int32_t* elems, int64_t elem_ld,
                          const int32_t* row_ptr, const int32_t* col_idx, int64_t nnz,
                          const int32_t* elem2nnz,
                          const int32_t* node_elem_ptr, const int32_t* node_elem,
                          const uint32_t* node_elem_slot,
                          double* K_vals, double* M_vals,
                          double* K_local, double* M_local,
                          int mode, void* work, size_t* work_bytes, int64_t* degenerate,
                          vb_stream_t stream);

/* The gather variant of fem_p1_assemble (c_K = c_M = 1; same arithmetic and
 * ownership, diagonal from the partition of unity) driven by the row classes of fem_plan_classes: a warp
 * takes one group (<= 32 rows of one class) and keeps each row's K and M sums
 * in registers.  Rows of the mixed class are assembled in place in HBM.
 * Arguments as fem_p1_assemble (node_elem_slot: the 32-bit plan words) plus
 * class_rows, groups, ngroups from fem_plan_classes on the same plan.
 * K_vals / M_vals (nnz, nullable) are overwritten.  work / work_bytes: the
 * launch's group counter, as fem_p1_assemble (16 bytes; NULL, NULL: static
 * group schedule).  Deterministic: the same bits as every run of this call
 * (per entry, the order is ascending pair order of build_pairs: the two
 * incidences of a pair are added together first, DESIGN.md §3.4 -- equal to
 * fem_p1_assemble's ascending element order within rounding, not bitwise). */
VB_API vb_status fem_p1_assemble_classes(int dim, int64_t nn, const double* coords, int64_t node_stride,
                                         int64_t comp_stride, const int32_t* row_ptr, const int32_t* col_idx,
                                         int64_t nnz, const int32_t* node_elem_ptr, const uint32_t* node_elem_slot,
                                         const int32_t* class_rows, const int32_t* groups, int64_t ngroups,
                                         double* K_vals, double* M_vals, void* work, size_t* work_bytes,
                                         vb_stream_t stream);

/* ---------------------------------------------------------- tile variant
 * Element-once deterministic assembly (same K, M as fem_p1_assemble, c = 1:
 * eq:K_M P:967-975, stiffness_matrixP1 P:978-1004, mass_matrixP1 P:1007,
 * accumulated as sparse(X3D(:),Y3D(:),..) P:1001-1003).  The rows are ordered
 * along a Morton curve of the node coordinates and cut into tiles of
 * VB_TILE_ROWS rows; every element is evaluated once per tile it has a vertex
 * in, and adds its off-diagonal K_e/M_e entries into the tile's rows in shared
 * memory, in the color order of the plan (elements of one color update
 * disjoint entries).  Diagonals from the partition of unity (K_vv = -sum_{w!=v}
 * K_vw, M_vv = (2/d) sum_{w!=v} M_vw).  Each CSR entry is written once, no
 * atomics; bitwise reproducible.
 *
 * fem_plan_tiles builds the plan from the CSR pattern of fem_p1_pattern
 * (row_ptr, col_idx) and the mesh; the coordinates only choose the tiles (any
 * coordinates give a correct plan; near ones give compact tiles).  Outputs
 * (DEVICE, caller-owned; ntiles = ceil(nn / VB_TILE_ROWS)):
 *   tile_meta   (ntiles x 4 int32): owned rows, local nodes, colors, first entry;
 *   tile_nodes  (ntiles x VB_TILE_NLOC int32): local node table (owned rows in
 *               tile order, then the halo in ascending node id);
 *   tile_rows   (ntiles x VB_TILE_ROWS x 2 int32): row_ptr[v], L | diag slot << 8;
 *   tile_colors (ntiles x (VB_TILE_MAXC + 1) int32): entry offsets per color;
 *   tile_elems  (elems_cap x 4 uint32): one entry per (tile, element): the
 *               local ids of the element's vertices and the in-row slots.
 * stats_out (HOST, 6 int64): entries, max elements per tile, max local nodes
 * (pass it as nloc_max), max colors, refusal reason (0 = none), ntiles.
 * VB_ERR_WORKSPACE when the entries do not fit elems_cap (stats_out[0] holds
 * the count; nv * ne always suffices); VB_ERR_UNSUPPORTED when a row has more
 * than 16 entries or a tile needs more than 3072 elements, VB_TILE_NLOC local
 * nodes or VB_TILE_MAXC colors (unstructured meshes with long rows: use the
 * other variants).  work: DEVICE scratch, work == NULL queries its size.
 * Synchronises the stream (two small read-backs). */
#define VB_TILE_ROWS 128
#define VB_TILE_NLOC 1024
#define VB_TILE_MAXC 32
VB_API vb_status fem_plan_tiles(int dim, int64_t nn, int64_t ne, const double* coords, int64_t node_stride,
                                int64_t comp_stride, const int32_t* elems, int64_t elem_ld,
                                const int32_t* row_ptr, const int32_t* col_idx, void* work, size_t* work_bytes,
                                int32_t* tile_meta, int32_t* tile_nodes, int32_t* tile_rows,
                                int32_t* tile_colors, uint32_t* tile_elems, int64_t elems_cap,
                                int64_t* stats_out, vb_stream_t stream);
/* K_vals / M_vals (nnz each, nullable) overwritten; coords strided as in
 * vb_create_coords3D; plan arrays, nloc_max (stats_out[2], <= VB_TILE_NLOC)
 * and elems_max (stats_out[1]: sizes the shared-memory staging of a tile's
 * entries) from fem_plan_tiles on the same mesh and pattern.  tile_elems must
 * be 16-byte aligned (bulk copies). */
VB_API vb_status fem_p1_assemble_tiles(int dim, int64_t nn, const double* coords, int64_t node_stride,
                                       int64_t comp_stride, int64_t nnz, const int32_t* tile_meta,
                                       const int32_t* tile_nodes, const int32_t* tile_rows,
                                       const int32_t* tile_colors, const uint32_t* tile_elems, int nloc_max,
                                       int elems_max, double* K_vals, double* M_vals, vb_stream_t stream);

/* ---------------------------------------------------------- Kuhn-lattice (element-once) variant
 * The same K, M (c = 1; eq:K_M P:967-975, stiffness_matrixP1 P:978-1004,
 * mass_matrixP1 P:1007, K_e = |T| G^T G with G = tjac^{-1} D from phider
 * P:929-947, accumulated as sparse(X3D(:),Y3D(:),..) P:1001-1003) for meshes
 * that are Kuhn lattices: nodes (i, j, k), 0 <= i <= nx, 0 <= j <= ny,
 * 0 <= k <= nz, numbered id = i + (nx+1)(j + (ny+1)k) (coordinates arbitrary,
 * e.g. jittered), every cell split into the 6 tetrahedra of the monotone paths
 * along one of its 4 diagonals (the same diagonal in every cell; element order
 * and vertex order inside an element are free) -- the paper's unit-cube meshes
 * and BASELINE configs[4].
 *
 * fem_plan_lattice verifies this ONCE per mesh on the GPU: every element is a
 * Kuhn tetrahedron of the nx x ny x nz lattice, no two elements are the same
 * tetrahedron (so the ne = 6 nx ny nz elements are exactly the lattice's), and
 * row_ptr/col_idx (from fem_p1_pattern) is the lattice stencil (15 columns in
 * the interior; row_ptr = col_idx = NULL skips this last check for a pattern
 * that fem_lattice_pattern writes).  It writes the plan (caller-owned DEVICE int32 array of
 * *plan_ints entries, 16-byte aligned: a token, the dims, the kernel's tile
 * descriptors and the cost-balanced range of tile layers of every CTA, one CTA
 * per SM of the current device -- the plan is for the device it was built on)
 * and reports in stats_out (HOST, 4 int64): [0] 1 if the mesh is
 * such a lattice (else 0 and nothing may be assembled with the plan), [1] the
 * number of tiles, [2] the refusal reason (1 counts, 2 element 0, 3 nx or
 * ny < 2 or degenerate ordering, 4 an element, 5 the pattern), [3] the
 * value to pass as `flips` to fem_p1_assemble_lattice (bits 0-2 the
 * orientation, bits 8.. the number of CTAs the plan's ranges are for).  work: DEVICE scratch
 * (ne/8 + 256 bytes); work == NULL queries *work_bytes and *plan_ints.
 * Synchronises the stream (small read-backs).  Refusal is not an error.
 *
 * fem_p1_assemble_lattice then reads no connectivity at all: one CTA per SM
 * marches along z through tiles of 32 x 12 lattice columns and evaluates every
 * tetrahedron ONCE (the row-owner variants evaluate it once per vertex);
 * contributions reach the owning rows by warp shuffles, shared memory and
 * registers; rows are assembled on chip (diagonals by the partition of unity,
 * K_pp = -sum_{q != p} K_pq, M_pp = (2/3) sum_{q != p} M_pq, reading "new" in
 * DESIGN.md §4) and written once (TMA bulk copies when K, M are 16-byte
 * aligned).  Deterministic: bitwise reproducible run to run.  Arguments: nx,
 * ny, nz and flips as planned (stats_out[3]), coords strided as in
 * vb_create_coords3D, row_ptr of the planned pattern, nnz, K_vals / M_vals
 * (nnz each, nullable; overwritten), degenerate (nullable DEVICE int64: the
 * number of tetrahedra with det = 0 as the kernel evaluates it or with two
 * vertices of identical coordinates, fem_p1_assemble's rule; a pass of its own
 * over the cells when requested).  VB_ERR_ARG for NULL coords / row_ptr /
 * plan, nn != (nx+1)(ny+1)(nz+1), nx or ny < 2, or a plan built for a device
 * with another SM count (flips bits 8..).  A plan of another mesh (token
 * mismatch, checked on the device) makes the kernel write nothing. */
VB_API vb_status fem_plan_lattice(int64_t nn, int64_t ne, const int32_t* elems, int64_t elem_ld,
                                  const int32_t* row_ptr, const int32_t* col_idx, int64_t nnz, int nx, int ny,
                                  int nz, void* work, size_t* work_bytes, int32_t* plan, int64_t* plan_ints,
                                  int64_t* stats_out, vb_stream_t stream);
/* The CSR pattern of such a lattice written directly (sparse(X3D(:),Y3D(:),..)'s
 * structure P:1001-1003 in closed form: the 15-point stencil, columns ascending,
 * explicit diagonal): bit-identical to what fem_p1_pattern builds from the
 * elements, in ~0.1 ms instead of ~2.3 ms on configs[4].  flips: the orientation
 * (bits 0-2 of fem_plan_lattice's stats_out[3]; higher bits ignored).  Query
 * with work == NULL: *work_bytes and *nnz_out (HOST; closed form).  Then
 * row_ptr (nn+1) and col_idx (col_cap >= nnz) DEVICE, caller-owned, are
 * overwritten; work: DEVICE scratch.  No read-back, no synchronisation.
 * Intended order: fem_plan_lattice with row_ptr = col_idx = NULL (verifies the
 * elements only, passing nnz from this query), then this call; a mesh that
 * fem_plan_lattice refuses takes fem_p1_pattern.  VB_ERR_ARG for inconsistent
 * sizes, VB_ERR_UNSUPPORTED for nx or ny < 2, VB_ERR_WORKSPACE. */
VB_API vb_status fem_lattice_pattern(int64_t nn, int nx, int ny, int nz, int flips, void* work, size_t* work_bytes,
                                     int32_t* row_ptr, int32_t* col_idx, int64_t col_cap, int64_t* nnz_out,
                                     vb_stream_t stream);
VB_API vb_status fem_p1_assemble_lattice(int64_t nn, const double* coords, int64_t node_stride,
                                         int64_t comp_stride, const int32_t* row_ptr, int64_t nnz,
                                         const int32_t* plan, int nx, int ny, int nz, int flips, double* K_vals,
                                         double* M_vals, int64_t* degenerate, vb_stream_t stream);

/* ---------------------------------------------------------- 2D lattice (element-once) variant
 * The 2D counterpart of the Kuhn-lattice variant, for BASELINE configs[0] and
 * configs[3]: the same K, M as fem_p1_assemble (dim = 2, c = 1; eq:K_M
 * P:967-975) for meshes whose nodes are (i, j), 0 <= i <= nx,
 * 0 <= j <= ny, id = i + (nx+1) j (coordinates arbitrary, e.g. jittered), every
 * cell split into two triangles by the same diagonal (either one; element
 * order and vertex order free).  fem_plan_lattice2d verifies that once per
 * mesh (elements and the 7-point CSR stencil) and writes the plan (token,
 * dims, the range of (x segment, node row) items of every resident warp of the
 * current device); arguments, work / plan query, stats_out ([0] accepted, [1]
 * x segments, [2] refusal reason 1 counts, 2 element 0, 3 nx < 2, 4 an
 * element, 5 the pattern, [3] the `flips` value for the assembly: bit 0 the
 * diagonal, bits 8.. the number of warps) and errors as fem_plan_lattice.
 * fem_p1_assemble_lattice2d: a warp marches along y over one x segment (31
 * nodes), both triangles of a cell evaluated once, contributions passed by
 * shuffle (x) and registers (y), no shared-memory exchange, no barrier; rows
 * (diagonals by the partition of unity, K_pp = -sum K_pq, M_pp = sum M_pq)
 * staged in CSR order and written once by TMA bulk copies (K, M 16-byte
 * aligned; plain stores otherwise).  Deterministic, bitwise reproducible.
 * degenerate: nullable DEVICE int64, the number of triangles with det = 0 as
 * evaluated or two identical vertices (fem_p1_assemble's rule; its own pass). */
VB_API vb_status fem_plan_lattice2d(int64_t nn, int64_t ne, const int32_t* elems, int64_t elem_ld,
                                    const int32_t* row_ptr, const int32_t* col_idx, int64_t nnz, int nx, int ny,
                                    void* work, size_t* work_bytes, int32_t* plan, int64_t* plan_ints,
                                    int64_t* stats_out, vb_stream_t stream);
/* The 7-point stencil pattern of such a lattice in closed form, bit-identical to
 * fem_p1_pattern's: arguments, query and errors as fem_lattice_pattern (flips:
 * bit 0 of fem_plan_lattice2d's stats_out[3]); fem_plan_lattice2d accepts
 * row_ptr = col_idx = NULL (elements only) for a pattern written by this call. */
VB_API vb_status fem_lattice2d_pattern(int64_t nn, int nx, int ny, int flips, void* work, size_t* work_bytes,
                                       int32_t* row_ptr, int32_t* col_idx, int64_t col_cap, int64_t* nnz_out,
                                       vb_stream_t stream);
VB_API vb_status fem_p1_assemble_lattice2d(int64_t nn, const double* coords, int64_t node_stride,
                                           int64_t comp_stride, const int32_t* row_ptr, int64_t nnz,
                                           const int32_t* plan, int nx, int ny, int flips, double* K_vals,
                                           double* M_vals, int64_t* degenerate, vb_stream_t stream);

/* ---------------------------------------------------------- exact-order check
 * The verification path of SURVEY §8(c) ("bitwise mode"): K and M (c = 1) with
 * every operation of the definition as an IEEE round-to-nearest fp64
 * operation (no FMA contraction) in the written order -- tjac = D X^T,
 * det by Laplace expansion along row 0, |T| = |det|/d!,
 * Jinv = adjugate/det, G = Jinv D, K_e = |T| sum_r G_ra G_rb
 * (P:996), M_e = |T|/((d+1)(d+2)) (1+delta_ab) -- and duplicates
 * summed per CSR entry from 0 in ascending element id.  Any
 * plain IEEE fp64 program doing the same gets the same bits.  One thread per
 * row over node_elem (fem_p1_pattern's gather plan, entries e*4 + a, ascending
 * e); slow by design, for checking the fast variants.  K_vals / M_vals (nnz,
 * nullable) overwritten; coords and elems strided as fem_p1_assemble. */
VB_API vb_status fem_p1_assemble_exact(int dim, int64_t nn, const double* coords, int64_t node_stride,
                                       int64_t comp_stride, const int32_t* elems, int64_t elem_ld,
                                       const int32_t* row_ptr, const int32_t* col_idx,
                                       const int32_t* node_elem_ptr, const int32_t* node_elem, double* K_vals,
                                       double* M_vals, vb_stream_t stream);

/* ---------------------------------------------------------- NEXT-4: GI
 * Code GI, the Gauss integration of the paper's volume and
 * surface integrals:
 *   f_e(c) = sum_q w_q fip(c, q, e)                      (amsv(fip, w))
 *   g_e = sum_c f_e(c) normals(c, e)  (normals given: a vector field against
 *         outer normals), else g_e = f_e(0)               (d must be 1)
 *   *value = sum_e sizes_e g_e
 * fip: npages d x nip pages (SoA, entry (c, q) of page e at fip[(c + q d) ldf
 * + e]); w: HOST array of nip weights (GI averages: they sum to 1 when sizes
 * are element measures; reading B20); sizes: npages values; normals: d planes
 * (plane stride ldn) or NULL; value: DEVICE scalar.  d in 1..4, nip in 1..16.
 * work: DEVICE scratch, work == NULL queries its size.  The reduction has a
 * fixed shape: bitwise reproducible.  VB_ERR_DIM for d != 1 without normals. */
VB_API vb_status vb_gi(int64_t npages, int d, int nip, const double* fip, int64_t ldf, const double* w,
                       const double* sizes, const double* normals, int64_t ldn, double* value, void* work,
                       size_t* work_bytes, vb_stream_t stream);

/* ---------------------------------------------------------- NEXT-1: coefficients
 * As fem_p1_assemble, with the coefficient functions of eq:K_M
 *   c_K(x) = cK_a * exp(cK_b . x),   c_M(x) = cM_a * exp(cM_b . x)
 * (cK_b, cM_b: HOST arrays of dim doubles, NULL = 0; c = 1 is a = 1, b = 0; the
 * paper's benchmarks use a = 1, b = (1, .., 1)) integrated with
 * intquad(gqo) as Code stiff_scalar_P1:
 *   K_e = sum_q w_q |det| c_K(x_q) G^T G,   M_e = sum_q w_q |det| c_M(x_q) phi_q phi_q^T,
 * gqo = 1 (centroid) or 2 (symmetric degree-2 rules: 3 points in 2D, 4 in 3D;
 * reading in DESIGN.md §4).  Both modes; in gather mode the diagonal of M is
 * the row sum of M_e (sum_b phi_b = 1) minus the off-diagonals.  work,
 * work_bytes, degenerate as fem_p1_assemble.
 * Errors as fem_p1_assemble, plus VB_ERR_UNSUPPORTED for other gqo. */
VB_API vb_status fem_p1_assemble_coef(int dim, int64_t nn, int64_t ne,
                          const double* coords, int64_t node_stride, int64_t comp_stride,
                          const int32_t* elems, int64_t elem_ld,
                          const int32_t* row_ptr, const int32_t* col_idx, int64_t nnz,
                          const int32_t* elem2nnz,
                          const int32_t* node_elem_ptr, const int32_t* node_elem,
                          const uint32_t* node_elem_slot,
                          int gqo, double cK_a, const double* cK_b, double cM_a, const double* cM_b,
                          double* K_vals, double* M_vals,
                          double* K_local, double* M_local,
                          int mode, void* work, size_t* work_bytes, int64_t* degenerate,
                          vb_stream_t stream);

/* NEXT-1 through the row classes: fem_p1_assemble_classes with c_K = c_M =
 * c_a exp(c_b . x) (c_b: HOST array of dim doubles, NULL = 0) and the gqo = 2
 * rule of fem_p1_assemble_coef (Code stiff_scalar_P1 P:978-1004, the paper's
 * benchmark case P:1149-1176; c_b: dim doubles).  The coefficient at a
 * quadrature point is formed from per-node factors P = exp(beta c_b.x), R = exp((alpha - beta) c_b.x)
 * computed into work (DEVICE, 2 nn + 2 doubles, caller-owned, 16-byte aligned;
 * the last 16 bytes hold the launch's group counter) at the start of the call.  gqo = 2 only (VB_ERR_UNSUPPORTED otherwise: use
 * fem_p1_assemble_coef).  Other arguments and guarantees as
 * fem_p1_assemble_classes. */
VB_API vb_status fem_p1_assemble_classes_coef(int dim, int64_t nn, const double* coords, int64_t node_stride,
                                              int64_t comp_stride, const int32_t* row_ptr, const int32_t* col_idx,
                                              int64_t nnz, const int32_t* node_elem_ptr,
                                              const uint32_t* node_elem_slot, const int32_t* class_rows,
                                              const int32_t* groups, int64_t ngroups, int gqo, double c_a,
                                              const double* c_b, double* work, double* K_vals, double* M_vals,
                                              vb_stream_t stream);

/* ---------------------------------------------------------- NEXT-2: rhs, energies
 * intquad(gqo, dim) as used by the kernels: writes the barycentric
 * points lam[q*(dim+1) + a] and weights w[q] (HOST arrays, nullable; at most 4
 * points) and returns nip, or a negative vb_status.  gqo 1: centroid; gqo 2:
 * symmetric degree-2 rules (reading).  Weights sum to 1/d!. */
VB_API int vb_quad_rule(int dim, int gqo, double* lam, double* w);

/* P1 load vector, Code rhs_vectorP1:
 *   b2D(a, e) = sum_q w_q |det_e| f(x_qe) phi_a(ip_q),   b = accumarray(elems, b2D)
 * fq: f at the integration points of intquad(gqo) (nip planes of ne values,
 * point order of vb_quad_rule; the caller evaluates f there, e.g. at
 * X_ip = amsm(coords3D, lam^T) via vb_create_coords3D + vb_page_mtimes, as the
 * paper's Code surface_integral does).  b2D (nv planes of ne) and
 * b (nn) are nullable outputs.  mode VB_ASSEMBLE_ATOMIC: fp64 atomics into b
 * (zero-filled by the call); VB_ASSEMBLE_GATHER: deterministic per-node sums
 * in ascending element order, needs b2D, node_elem_ptr and node_elem (the plan
 * of fem_p1_pattern). */
VB_API vb_status fem_p1_rhs(int dim, int64_t nn, int64_t ne,
                            const double* coords, int64_t node_stride, int64_t comp_stride,
                            const int32_t* elems, int64_t elem_ld, int gqo, const double* fq,
                            double* b2D, double* b,
                            const int32_t* node_elem_ptr, const int32_t* node_elem,
                            int mode, vb_stream_t stream);

/* avtamav (page-wise bilinear form eq:layeredBilin P:292-301):
 * s_k = a_k^T M_k b_k for pages a (n x 1), M (n x m), b (m x 1), n, m in 1..4;
 * ld = 0 broadcasts a single object.  With a = b = the element restriction of
 * a nodal vector (vb_create_coords3D with dim = 1) and M = K3D this gives the
 * element energies 2 J_{1,k} of eq:Jk_comps. */
VB_API vb_status vb_page_bilinear(int64_t npages, int n, int m, const double* A, int64_t lda,
                                  const double* Mx, int64_t ldm, const double* B, int64_t ldb,
                                  double* s, vb_stream_t stream);

/* ---------------------------------------------------------- NEXT-3: P2 elements
 * Topological CSR pattern (as fem_p1_pattern, same two phases, synchronisation,
 * work-buffer reuse and validation flag, OR'ed into nv) for elements with nv nodes, 2 <= nv <= 16 (P2: 6 in
 * 2D, 10 in 3D; sparse() of P:1033-1036).  Requires ne < 2^27.  Optional plans:
 *   elem2nnz (nullable): the nv^2-plane element-to-nnz map (atomic scatter);
 *   node_elem_ptr (nn+1) / node_elem (nv*ne, packed e*16 + a, ascending e per
 *     node) / node_elem_slot (nullable; W = ceil(nv/4) uint32 words per
 *     incidence, byte b of the W words = in-row offset of node b of the
 *     element, natural order; rows must have <= 255 entries): the gather plan
 *     of VB_ASSEMBLE_GATHER in fem_p2_assemble.  Given together or not at all
 *     (node_elem_slot may be NULL). */
VB_API vb_status fem_pattern(int nv, int64_t nn, int64_t ne,
                             const int32_t* elems, int64_t elem_ld,
                             void* work, size_t* work_bytes,
                             int32_t* row_ptr, int32_t* col_idx, int64_t col_cap,
                             int32_t* elem2nnz,
                             int32_t* node_elem_ptr, int32_t* node_elem, uint32_t* node_elem_slot,
                             int64_t* nnz_out, vb_stream_t stream);

/* P2 stiffness and mass matrices (stiffness_matrixP2 / mass_matrixP2,
 * P:1009-1049) with c_K = cK_a exp(cK_b . x), c_M = cM_a exp(cM_b . x) (host
 * arrays, NULL = 0) and intquad(gqo), gqo in {1, 2, 4} (4: Dunavant's 6-point
 * rule in 2D, Keast's 11-point rule in 3D; the paper uses 4; reading in
 * DESIGN.md §4).  elems: nlb = 6 (2D) / 10 (3D) node planes, vertices first,
 * then edge midpoints in the order (1,2),(2,3),(1,3) / (1,2),(1,3),(1,4),(2,3),
 * (2,4),(3,4); edges must be straight (midpoints exact).
 * mode VB_ASSEMBLE_ATOMIC: K_vals/M_vals (nnz, nullable) are zero-filled and
 *   accumulated with fp64 atomics through elem2nnz (fem_pattern); work unused.
 * mode VB_ASSEMBLE_GATHER: deterministic.  Call with work == NULL to query
 *   *work_bytes (2 nlb^2 ne doubles + 16; nothing else happens).  The element
 *   matrices are computed once into `work` (element-major), then every row
 *   sums its incidences' rows of them (a few rows per warp, nlb lanes each)
 *   in ascending element order (the oracle's order) and writes each CSR entry
 *   once.  Needs row_ptr, node_elem_ptr, node_elem and node_elem_slot of
 *   fem_pattern (elem2nnz unused).  Bitwise reproducible.
 * K_local/M_local (nullable): nlb x nlb page arrays (ld = ne). */
VB_API vb_status fem_p2_assemble(int dim, int64_t nn, int64_t ne,
                                 const double* coords, int64_t node_stride, int64_t comp_stride,
                                 const int32_t* elems, int64_t elem_ld,
                                 const int32_t* row_ptr, const int32_t* elem2nnz, int64_t nnz,
                                 const int32_t* node_elem_ptr, const int32_t* node_elem,
                                 const uint32_t* node_elem_slot,
                                 int gqo, double cK_a, const double* cK_b, double cM_a, const double* cM_b,
                                 double* K_vals, double* M_vals, double* K_local, double* M_local,
                                 int mode, void* work, size_t* work_bytes, vb_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* VB_H_ */
