/*
 * fo.h -- C ABI of the B200-native first-order (Blatter-Pattyn) Stokes
 * assembly library (libfo.so).
 *
 * What it computes.  PAPER.md = arXiv 2204.04321 (Watkins et al., MALI);
 * "P:n" = line n of /root/reference/PAPER.md.
 *   - the discrete residual F(U; phi, grad phi, H, beta, ...) of eq:residual
 *      for the first-order velocity equations eq:FOStokes
 *     with the strain rates of P:90-100, Glen's law eq:effvisc / eq:effeps
 *      regularised by eps_reg (reading L1), driving stress
 *     rho g grad s, basal linear sliding (Robin) BC and the
 *     stress-free upper surface, discretised with low-order 6-node
 *     prismatic (wedge) elements on the extrusion of a triangulated footprint
 *     (P:80);
 *   - the exact Newton Jacobian dF/dU of eq:linearsystem -- the
 *     quantity the paper obtains with Sacado forward AD --
 *     scattered into a fixed CSR graph;
 *   - the ghost-row sum of a footprint-partitioned assembly (the paper's
 *     Tpetra Export) and the ghost import of U.
 *
 * Numbering (fixed): footprint vertex c = extruded column;
 * node(c, k) = c*(L+1) + k for levels k = 0 (bed) .. L (surface); DOF
 * 2*node + a with a = 0 for u, 1 for v; wedge (t, k) = t*L + k.  CSR rows are
 * DOFs in ascending order; the columns of a row are ascending DOF ids; every
 * DOF pair that shares a wedge is structural.  row_ptr is int64, col_idx int32.
 *
 * Ownership.  Host arrays passed to *_create are copied; the caller may free
 * them on return.  Device pointers (d_*) are caller-owned fp64 device buffers
 * on the mesh's device (e.g. PyTorch tensors); the library never frees or
 * retains them.  `stream` is a cudaStream_t passed as void* (NULL = legacy
 * default stream).  Assembly calls enqueue work on `stream` and do not
 * synchronise the host.
 *
 * Errors.  Every call returns fo_status; 0 = FO_OK.  On error the outputs are
 * unspecified and fo_last_error() (thread-local) describes the failure.  The
 * library never aborts and never falls back to a CPU path.
 */
#ifndef FO_H
#define FO_H
#include <stdint.h>

#if defined(__GNUC__)
#define FO_API __attribute__((visibility("default")))
#else
#define FO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FO_OK = 0,
  FO_EINVAL = -1,   /* NULL argument, size mismatch, bad parameter */
  FO_EMESH = -2,    /* CW/degenerate triangle, isolated vertex, H < H_min,
                       sigma not strictly ascending from 0 to 1, index range */
  FO_ECUDA = -3,    /* CUDA runtime error (no device, launch failure, ...) */
  FO_ENCCL = -4,    /* NCCL error */
  FO_ENOMEM = -5,   /* device or host allocation failed */
  FO_ESTATE = -6    /* objects do not belong together (graph of another mesh) */
} fo_status;

typedef struct fo_mesh_s* fo_mesh;    /* owns device copies of geometry and fields */
typedef struct fo_graph_s* fo_graph;  /* owns the device CSR pattern               */
typedef struct fo_halo_s* fo_halo;    /* owns the NCCL communicator and halo maps  */

typedef struct {
  double rho;      /* ice density, kg m^-3 (910; reading L3)            */
  double g;        /* gravity, m s^-2 (9.81)                                      */
  double rho_w;    /* sea-water density, kg m^-3 (1028), floating mask only       */
  double glen_n;   /* Glen exponent n; 3 is the fast path, any n > 0 ok   */
  double eps_reg;  /* regularisation of eps_e^2, a^-2 (1e-10; reading L1)         */
  double A;        /* flow factor, Pa^-n a^-1 (1e-16), used when A_elem == NULL   */
  double H_min;    /* columns thinner than this are rejected (1 m; reading L17)   */
} fo_params;

/* Fills the defaults listed above. */
FO_API fo_status fo_params_default(fo_params* p);

/* Extruded mesh from a triangulated footprint.
 *   xy[n_vert][2] (m); tri[n_tri][3] 0-based CCW vertex ids (P1 footprint,
 *   reading L16: CW or degenerate -> FO_EMESH; a vertex in no triangle ->
 *   FO_EMESH); n_layers L >= 1; sigma[L+1] level fractions 0 = bed .. 1 =
 *   surface, strictly ascending (NULL = uniform); thickness H, surface s,
 *   beta (basal friction, Pa a m^-1) per vertex; bed b per vertex or NULL:
 *   when given, beta is zeroed where the column floats, rho H < -rho_w b
 *   (reading L9); A_elem[n_tri*L] per-wedge flow factor or NULL.
 *   Node heights z(c,k) = (s_c - H_c) + sigma_k H_c.
 *   n_vert = n_tri = 0 gives a valid empty mesh.  Synchronous. */
FO_API fo_status fo_mesh_create(const fo_params* p, int64_t n_vert, const double* xy,
                         int64_t n_tri, const int32_t* tri, int32_t n_layers,
                         const double* sigma, const double* thickness,
                         const double* surface, const double* bed,
                         const double* beta, const double* A_elem, int device,
                         fo_mesh* out);

/* Local mesh of part `my_part` of a footprint partition (part_of_tri[n_tri],
 * values in [0, n_parts)): local triangles are those of my_part; local columns
 * are numbered owned-first (class A: columns whose minimum incident part is
 * my_part, ascending global id), then ghost columns touched by local triangles
 * (class B, grouped by owner part ascending, global id inside a group), then
 * column-only couplings (class C).  Owned rows carry the full global row
 * pattern; DOFs [0, n_owned_dofs) are the owned prefix.
 * Same array arguments as fo_mesh_create (GLOBAL footprint).  Synchronous. */
FO_API fo_status fo_mesh_create_part(const fo_params* p, int64_t n_vert, const double* xy,
                              int64_t n_tri, const int32_t* tri, int32_t n_layers,
                              const double* sigma, const double* thickness,
                              const double* surface, const double* bed,
                              const double* beta, const double* A_elem,
                              const int32_t* part_of_tri, int32_t my_part,
                              int32_t n_parts, int device, fo_mesh* out);

/* NEXT-f3: temperature-dependent flow factor
 *   A = A0 exp(-Q / (R T*)),  R = 8.314462618 J mol^-1 K^-1,
 * per wedge, evaluated inside the assembly kernels (8 bytes of T* per wedge;
 * DESIGN.md reading L21).  T_star[n_tri*L] (K, pressure-corrected, wedge
 * t*L+k of the GLOBAL footprint for a part mesh) is copied to the device
 * (the caller may free it on return); A0 in Pa^-n a^-1, Q in J mol^-1.
 * Replaces p->A / A_elem for later assemblies; T_star == NULL reverts to them.
 * FO_EINVAL: mesh NULL, A0 <= 0 or some T* <= 0.  Synchronous. */
FO_API fo_status fo_mesh_set_temperature(fo_mesh m, const double* T_star, double A0, double Q);

/* NEXT-f4: hexahedral mesh from a QUADRILATERAL footprint:
 * quad[n_quad][4] 0-based CCW corners of convex quads (FO_EMESH otherwise),
 * every other argument as fo_mesh_create (A_elem[n_quad*L]).  Each layer
 * element is an 8-node trilinear hexahedron (reading L23: 2x2x2 Gauss,
 * isoparametric, exact Jacobian; basal term with 2x2 Gauss on the bilinear
 * bottom face).  Graph, SpMV, line preconditioner, A(T) apply unchanged.  The
 * default R + J scatter is the owner-computes quad-patch kernel (KH-patch:
 * Hilbert-ordered patches of <= 96 quads, boundary columns zero-filled
 * in-kernel and RED, multi columns by a fix-up; bitwise reproducible);
 * FO_SCATTER_ATOMIC selects the coloured read-modify-write ablation (quads
 * sharing a corner never run concurrently; a fixed launch order makes it
 * deterministic), which also computes the residual alone.  Single-domain;
 * no lateral term, no fo_set_element.  Synchronous. */
FO_API fo_status fo_mesh_create_quad(const fo_params* p, int64_t n_vert, const double* xy,
                                     int64_t n_quad, const int32_t* quad, int32_t n_layers,
                                     const double* sigma, const double* thickness,
                                     const double* surface, const double* bed, const double* beta,
                                     const double* A_elem, int device, fo_mesh* out);

/* Contiguous partition of the (Hilbert-ordered) triangle list:
 * part_of_tri[t] = floor(t * n_parts / n_tri).  Host only. */
FO_API fo_status fo_partition(int64_t n_tri, int32_t n_parts, int32_t* part_of_tri);

/* Sizes of a (local) mesh.  Any pointer may be NULL. */
FO_API fo_status fo_mesh_info(fo_mesh m, int64_t* n_nodes, int64_t* n_dofs, int64_t* n_elems,
                       int64_t* n_owned_dofs);

/* Local -> global column ids of a local mesh (identity for fo_mesh_create),
 * and the column class counts (A, B, C).  glob[n_local_columns]. */
FO_API fo_status fo_mesh_columns(fo_mesh m, int64_t* n_cols, int64_t* n_owned, int64_t* n_ghost,
                          int64_t* n_colonly, int64_t* glob);

/* Fixed CSR graph of the (local) mesh (FeCrs-style owned rows first).
 * Synchronous. */
FO_API fo_status fo_graph_build(fo_mesh m, fo_graph* out);
FO_API fo_status fo_graph_info(fo_graph g, int64_t* n_rows, int64_t* nnz);
/* device pointers owned by the graph (valid until fo_graph_destroy) */
FO_API fo_status fo_graph_arrays(fo_graph g, const int64_t** d_row_ptr, const int32_t** d_col_idx);
/* copies the pattern to host arrays row_ptr[n_rows+1], col_idx[nnz]. Synchronous. */
FO_API fo_status fo_graph_to_host(fo_graph g, int64_t* row_ptr, int32_t* col_idx);

/* Host-only graph construction with the library's algorithm (no device):
 * the same pattern fo_graph_build uploads.  Call with col_idx == NULL to get
 * nnz.  row_ptr[2*n_vert*(L+1)+1]. */
FO_API fo_status fo_graph_host(int64_t n_vert, int64_t n_tri, const int32_t* tri, int32_t n_layers,
                        int64_t* row_ptr, int32_t* col_idx, int64_t* nnz);

/* Host-only check of the owner-computes scatter plan (no device; tests):
 * builds the (part) mesh's patch plan as fo_mesh_create would and verifies
 * that every coupling-list slot and residual of a column with rows is written
 * by exactly one store (interior pair / multi-column fix-up) or by RED partial
 * sums onto a zero-filled column, and that every element entry is gathered
 * exactly once.  stats[8] = {patches, pairs, contributions, zero-filled
 * columns, multi columns, slot violations, element violations, largest plan
 * bytes}.  part_of_tri NULL: single domain.  Synchronous. */
FO_API fo_status fo_plan_check_host(int64_t n_vert, const double* xy, int64_t n_tri, const int32_t* tri,
                                    int32_t n_layers, const int32_t* part_of_tri, int32_t my_part,
                                    int32_t n_parts, int64_t* stats);

/* The same host-only check for the quadrilateral footprint of a hexahedral
 * mesh (fo_mesh_create_quad, NEXT-f4): the quad-patch plan of KH-patch, every
 * element entry (q, j, j2) of the 4 x 4 corner pairs gathered exactly once,
 * every slot / residual written once or RED onto a zero fill, the zero
 * fill's lead / wait lists consistent.  stats[8] as fo_plan_check_host
 * (contributions: 16 corner pairs per quad). */
FO_API fo_status fo_plan_check_quad_host(int64_t n_vert, const double* xy, int64_t n_quad, const int32_t* quad,
                                         int32_t n_layers, int64_t* stats);

/* R = F(U): overwrites d_R[n_dofs].  d_U[n_dofs] fp64. */
FO_API fo_status fo_assemble_residual(fo_mesh m, const double* d_U, double* d_R, void* stream);

/* vals = dF/dU in the CSR order of g (overwritten); d_R (nullable) = F(U)
 * overwritten in the same pass.  The kernel computes CSR
 * positions from the column structure; it does not read col_idx.
 * Assembly calls on ONE mesh must be ordered (one stream, or synchronised):
 * the mesh owns their scratch (multi-column partial sums, the in-kernel zero
 * fill's flags and patch ticket).  Different meshes may run concurrently. */
FO_API fo_status fo_assemble_jacobian(fo_mesh m, fo_graph g, const double* d_U, double* d_R,
                               double* d_vals, void* stream);

/* The same with HOST buffers: copies h_U in, assembles, copies R and vals out
 * on `stream` and synchronises it.  Host buffers should be pinned for full
 * copy bandwidth.  h_R may be NULL. */
FO_API fo_status fo_assemble_jacobian_host(fo_mesh m, fo_graph g, const double* h_U, double* h_R,
                                    double* h_vals, void* stream);

/* NEXT-f4: element of the prism layers.  FO_ELEM_WEDGE (default) is
 * the 6-node wedge (reading L5); FO_ELEM_TET3 splits every prism into three
 * P1 tetrahedra by GLOBAL vertex id (reading L22: with corners a < b < c,
 * {a,b,c,c'}, {a,b,b',c'}, {a,a',b',c'}), one quadrature point each, exact
 * Jacobian; it assembles into the same graph (3 of the 15 node pairs of a
 * prism become structural zeros) with the owner-computes scatter only.
 * FO_EINVAL for an unknown type, for TET3 with the lateral term enabled
 * (fo_set_lateral) or with FO_SCATTER_ATOMIC. */
typedef enum { FO_ELEM_WEDGE = 0, FO_ELEM_TET3 = 1 } fo_element;
FO_API fo_status fo_set_element(fo_mesh m, fo_element type);

/* ---- NEXT-f2: the Newton consumer of the assembled Jacobian ----
 * Single-domain meshes only (FO_ESTATE for a part mesh).  All buffers are
 * caller-owned contiguous fp64 device arrays of n_dofs entries unless stated;
 * work is enqueued on `stream`, no host synchronisation.
 *
 * y = J x, J the CSR values d_vals of fo_assemble_jacobian for graph g.  Every
 * value position comes from the column structure (row (c,k,a) couples slot s
 * of c's sorted neighbour list, levels k-1..k+1, comps 0..1), so col_idx is
 * never read.  One writer per y entry (deterministic). */
FO_API fo_status fo_spmv(fo_mesh m, fo_graph g, const double* d_vals, const double* d_x, double* d_y,
                         void* stream);
/* Vertical-line preconditioner: factor, for every column, the 2x2-block
 * tridiagonal block of J coupling the column's own 2(L+1) DOFs (block Thomas;
 * factors kept in the mesh; d_vals must stay valid until the next factor).
 * fo_line_solve: z = M^-1 r with M = those column blocks (block Jacobi over
 * vertical lines).  FO_ESTATE if fo_line_factor was not called. */
FO_API fo_status fo_line_factor(fo_mesh m, fo_graph g, const double* d_vals, void* stream);
FO_API fo_status fo_line_solve(fo_mesh m, const double* d_r, double* d_z, void* stream);
/* Krylov helpers on the mesh's device (fixed-order reductions, bitwise
 * reproducible): d_out[j] = V_j . w for j < k (1 <= k <= 64), and
 * w -= sum_j h_j V_j (h: k doubles on the device).  V column-major, column j at
 * d_V + j * ldv, ldv >= n. */
FO_API fo_status fo_krylov_dots(fo_mesh m, int64_t n, int32_t k, const double* d_V, int64_t ldv,
                                const double* d_w, double* d_out, void* stream);
FO_API fo_status fo_krylov_update(fo_mesh m, int64_t n, int32_t k, const double* d_V, int64_t ldv,
                                  const double* d_h, double* d_w, void* stream);

/* NEXT-f1: lateral margin term of the residual on the footprint
 * boundary faces (boundary edges of the GLOBAL footprint x L layers), by
 * DESIGN.md reading L12:  2 mu eps_a . n = [rho g (s - z) - rho_w g max(-z, 0)] n_a,
 * i.e.  R_{a,i} -= int_{Gamma_l} P(z) n_a phi_i dGamma  (quadrature: reading L20).
 * U-independent: the Jacobian values are unchanged.  enable = 0 (default)
 * leaves it out.  Applies to later fo_assemble_* calls on this mesh (one extra
 * kernel, one writer per residual entry: deterministic). */
FO_API fo_status fo_set_lateral(fo_mesh m, int enable);

/* Scatter strategy of fo_assemble_jacobian (ablation; default FO_SCATTER_OWNER):
 * FO_SCATTER_OWNER    column-patch owner-computes kernel: every CSR value of an
 *                     interior column written exactly once with plain stores
 *                     (deterministic); for wedges the warp-specialised kernel
 *                     (element warpgroup with TMEM scratch + scatter warpgroup);
 *                     for hexahedra the quad-patch kernel (KH-patch)
 * FO_SCATTER_ATOMIC   one thread per wedge, fp64 atomics into zeroed outputs;
 *                     hexahedra: one thread per hexahedron, coloured
 *                     read-modify-write into zeroed outputs
 * FO_SCATTER_OWNER_WS the warp-specialised kernel explicitly (wedges, R + J)
 * FO_SCATTER_OWNER_1WG the round-1 single-warpgroup patch kernel (element and
 *                     scatter phases alternate in the same threads). */
typedef enum { FO_SCATTER_OWNER = 0, FO_SCATTER_ATOMIC = 1, FO_SCATTER_OWNER_WS = 2,
               FO_SCATTER_OWNER_1WG = 3 } fo_scatter;
FO_API fo_status fo_set_scatter(fo_mesh m, fo_scatter s);

/* Kernel launches the last assembly call enqueued (for bench accounting). */
FO_API fo_status fo_last_launch_count(fo_mesh m, int32_t* n);

/* Kernel timing (bench): while enabled, every assembly call records a pair of
 * CUDA events around its main assembly kernel on the caller's stream.
 * fo_kernel_time_ms synchronises the recorded events, returns the summed
 * elapsed milliseconds and the number of timed launches, and clears them. */
FO_API fo_status fo_kernel_timing(fo_mesh m, int32_t enable);
FO_API fo_status fo_kernel_time_ms(fo_mesh m, double* total_ms, int32_t* n_launches);

/* ---- multi-GPU halo (P:175 Import, P:185 Export) ----
 * nccl_unique_id: 128-byte ncclUniqueId, identical on all ranks (rank 0
 * creates it with fo_nccl_unique_id and the harness broadcasts it).
 * Collective over n_ranks; rank r must pass the local mesh of part r. */
FO_API fo_status fo_nccl_unique_id(void* id128);
FO_API fo_status fo_halo_create(fo_mesh local, fo_graph local_g, const void* nccl_unique_id,
                         int32_t rank, int32_t n_ranks, fo_halo* out);
/* Loopback transport (one process, one device): creates the n_parts halos of
 * one partition at once, out[p] for parts[p] (the local mesh of part p, made
 * with fo_mesh_create_part, and its graph).  fo_halo_import / fo_halo_sum on
 * these halos run the same plans, staging buffers, gather and unpack-add
 * kernels and sender order as the NCCL halos; only the point-to-point
 * transfers are device-to-device copies on the callers' streams instead of
 * ncclSend / ncclRecv.  Sends are eager; a part's unpack-add is enqueued when
 * the last slice it receives has been sent, which can be inside a later part's
 * call -- so call a phase (import, sum) for every part before enqueueing work
 * that depends on it.  Used to run the halo path on one GPU (tests, bench).
 * Errors: FO_EINVAL (NULL, different devices), FO_ESTATE (parts[p] is not part
 * p of one n_parts partition of one footprint, or graph/mesh mismatch). */
FO_API fo_status fo_halo_create_loopback(const fo_mesh* parts, const fo_graph* graphs, int32_t n_parts,
                                         fo_halo* out);
/* ghost U <- owners' U (owned prefix of d_U is read, ghost part written) */
FO_API fo_status fo_halo_import(fo_halo h, double* d_U, void* stream);
/* owners' rows += ghost-row partial sums of the other ranks; after the call
 * the owned prefix of d_R / d_vals is complete (ghost rows unspecified).
 * Either pointer may be NULL. */
FO_API fo_status fo_halo_sum(fo_halo h, double* d_R, double* d_vals, void* stream);
/* Assembly and Export in one call, overlapped:
 * R = F(U) and, if d_vals != NULL, the Jacobian values of the local (part)
 * mesh, then the ghost-row sum of fo_halo_sum -- with the patches holding the
 * ghost-touching triangles (a part mesh orders them first) computed on the
 * halo's own higher-priority stream, and their rows sent to the owners while
 * the interior patches are still being computed on `stream`.  Same results
 * as fo_assemble_jacobian (or fo_assemble_residual) followed by fo_halo_sum,
 * bit for bit.  The ghost U must be current (fo_halo_import before).  Falls
 * back to that sequential order for one part, the atomic scatter and the
 * lateral term (which adds into ghost rows after every patch).  All work is
 * joined into `stream` on return.  d_U[n_dofs], d_R[n_dofs] (not NULL),
 * d_vals[nnz] or NULL (residual only; g may then be NULL).  With the loopback
 * transport the same phase rule as fo_halo_sum applies.  Errors: FO_EINVAL
 * (NULL mesh / halo / U / R, hexahedral mesh), FO_ESTATE (graph or halo built
 * for another mesh), FO_ECUDA, FO_ENCCL. */
FO_API fo_status fo_assemble_jacobian_halo(fo_mesh m, fo_graph g, fo_halo h, const double* d_U, double* d_R,
                                           double* d_vals, void* stream);
/* halo plan sizes: neighbours, ghost DOFs received, values received */
FO_API fo_status fo_halo_info(fo_halo h, int32_t* n_neighbors, int64_t* recv_rows, int64_t* recv_vals);

/* Host-only local numbering and CSR pattern of part my_part (exactly what
 * fo_mesh_create_part + fo_graph_build produce), without a device.  glob
 * receives local -> global column ids; row_ptr[2*n_cols*(L+1)+1] and
 * col_idx[nnz] the local pattern.  Call with NULL arrays to get the sizes. */
FO_API fo_status fo_part_graph_host(int64_t n_vert, int64_t n_tri, const int32_t* tri,
                                    int32_t n_layers, const int32_t* part_of_tri,
                                    int32_t n_parts, int32_t my_part, int64_t* n_cols,
                                    int64_t* n_owned, int64_t* n_ghost, int64_t* nnz,
                                    int64_t* glob, int64_t* row_ptr, int32_t* col_idx);

/* Host-only halo plan (no device, no NCCL) for part my_part: for every other
 * part q the list of (row, value) positions this part SENDS to q (offsets into
 * the sender's local R / CSR values) and the positions in the owner's local
 * arrays they are added to.  Used by the CPU tests of the plan.
 * Call with NULL arrays to get the sizes; arrays are concatenated over q in
 * ascending order, counts[q] / vcounts[q] give the per-part lengths. */
FO_API fo_status fo_halo_plan_host(int64_t n_vert, int64_t n_tri, const int32_t* tri, int32_t n_layers,
                            const int32_t* part_of_tri, int32_t n_parts, int32_t my_part,
                            int64_t* counts, int64_t* vcounts,
                            int64_t* send_rows, int64_t* dest_rows,
                            int64_t* send_vals, int64_t* dest_vals);

FO_API const char* fo_last_error(void);
FO_API void fo_mesh_destroy(fo_mesh m);
FO_API void fo_graph_destroy(fo_graph g);
FO_API void fo_halo_destroy(fo_halo h);

#ifdef __cplusplus
}
#endif
#endif /* FO_H */
