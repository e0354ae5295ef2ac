// fo_internal.h -- private structures of libfo (host + device side).
// Layout and numbering: DESIGN.md "Layout in HBM"; public contract: include/fo.h.
#pragma once
#include <cstdint>
#include <vector_types.h>
#include <cuda_runtime.h>
#include <functional>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only; ranges cost nothing without a profiler attached

#include "../../include/fo.h"

namespace fo {

// Per-column record, 48 bytes, gathered by the assembly kernels (one per
// extruded column; the paper's "boundary data aligned to its map" lesson,
// every field a wedge needs is in one contiguous record).
struct alignas(16) ColRec {
  double x, y;       // footprint position (m)
  double base, H;    // bed-side base z = s - H, thickness
  double beta;       // basal friction after the floating mask
  int64_t cs_n;      // (CSR value offset of the column's first row) << 8 | list length n_c
};

// Per-triangle record, 24 bytes: local column ids and the 9 structural slots
// slot[i][j] = position of column v[j] in the sorted coupling list of v[i].
struct alignas(8) TriRec {
  int32_t v[3];
  uint8_t slot[9];
  uint8_t pad[3];   // pad[0]: corners sorted by global vertex id, 2 bits each (NEXT-f4)
};

// NEXT-f4 hexahedra: per-quad record, 32 bytes: corner columns and the 16
// slots slot[4 i + j] = position of corner j's column in corner i's list
struct alignas(8) QuadRec {
  int32_t v[4];
  uint8_t slot[16];
};

// Triangles per patch of the owner-computes kernel (one thread per triangle
// column, 99 fp64 of shared memory per triangle).
#ifdef FO_EXPERIMENT_PATCH255
constexpr int kPatchTris = 255;
#else
constexpr int kPatchTris = 128;
#endif
// CTAs resident per SM (2: one CTA's gather phase overlaps the other's
// element phase)
#ifdef FO_EXPERIMENT_PATCH255
constexpr int kPatchCtasPerSm = 1;
#else
constexpr int kPatchCtasPerSm = 2;
#endif
// row stride (doubles) of the [entry][triangle] shared-memory arrays: odd, so
// entries of one triangle fall in different banks
constexpr int kPatchStride = kPatchTris + 1;
// shared-memory budget of one patch's plan (columns, pairs, contributions)
constexpr int kPlanBytes = (233472 - 1024 * kPatchCtasPerSm) / kPatchCtasPerSm - 99 * kPatchStride * 8 - 64;

// Hexahedral patches (NEXT-f4 owner-computes, fo_hex.cu): <= kPatchQuads
// quads per patch, shared memory per quad: D = (bottom,bottom) block of the 8
// bottom dofs (36, 2x2 node-block layout) + 8 residual entries, O = the 8 x 8
// (bottom, top) block
constexpr int kPatchQuads = 96;
constexpr int kPatchStrideQ = kPatchQuads + 1;
constexpr int kHexDE = 44, kHexOE = 64;
constexpr int kHexCtasPerSm = 2;
constexpr int kPlanBytesHex =
    (233472 - 1024 * kHexCtasPerSm) / kHexCtasPerSm - (kHexDE + kHexOE) * kPatchStrideQ * 8 - 64;

// Encoded contribution (fo_plan.cpp contrib_code) of an element with NV
// footprint corners (3: wedge, 4: hexahedron): element slot tl | D base of the
// (j, j2) 2x2 node block | its stride pattern | O base of (row (j,0), column
// (j2,0)) | O base of the transpose | j.  Field widths per NV:
template <int NV>
struct CodeBits {
  static constexpr int kTl = NV == 3 ? 8 : 7;    // bits [0, kTl)
  static constexpr int kDb = 13 - kTl;           // bits [kTl, 13)
  static constexpr int kPat = 13;                // bits 13-14
  static constexpr int kOw = NV == 3 ? 5 : 6;
  static constexpr int kO = 15, kOt = 15 + kOw, kJ = 15 + 2 * kOw;
  static constexpr int kRow = 2 * NV;            // O row stride (dofs of one level)
  static constexpr int kDsym = NV * (2 * NV + 1);  // D entries before the residual
};

// plan records (fo_plan.cpp); copied to shared memory by the kernel
struct PlanCol {            // 24 bytes
  int64_t colstart;         // CSR value offset of the column's first row
  int32_t c;                // local column id
  int32_t info;             // n_c | interior << 8 | self slot << 9 | multi << 30
  uint16_t self_off;        // contributions of the self slot (residual)
  uint16_t self_cnt;
  uint32_t pad;             // multi columns: this patch's partial block
};
// a column touched by >= 3 patches: self-slot and residual partial sums go to
// partial blocks base .. base + cnt - 1 (patch order), summed by the fix-up pass
struct MultiRec {           // 24 bytes
  int64_t colstart;
  int32_t c;
  int32_t nc_self;          // n_c | self slot << 8
  int32_t base;
  int32_t cnt;
};
// doubles per (partial block, level): dg 4, up 4, nx 4, residual 2 (+2 pad)
constexpr int kPartialStride = 16;
struct alignas(16) PlanPair {   // 16 bytes: one (column, slot) of phase B
  uint16_t off;             // contributions 2 .. cnt-1 (patch-relative index)
  uint8_t cnt;              // number of contributions (even, >= 2)
  uint8_t slot;             // slot in the column's coupling list
  uint16_t col;             // patch-local column record
  uint16_t pad;
  uint32_t c0, c1;          // contributions 0 and 1, inline (an edge pair's whole list)
};

// Work decomposition of the owner-computes kernel.
struct PatchPlan {
  int32_t n_patches = 0;
  int64_t max_plan_bytes = 0;
  std::vector<int32_t> t_begin;      // [n_patches+1] triangle range of patch p
  std::vector<int32_t> col_ptr;      // [n_patches+1]
  std::vector<int32_t> pair_ptr;     // [n_patches+1]
  std::vector<int64_t> contrib_ptr;  // [n_patches+1]
  std::vector<PlanCol> cols;
  std::vector<PlanPair> pairs;
  std::vector<uint32_t> contrib;     // encoded contribution (fo_plan.cpp contrib_code)
  std::vector<int32_t> zero_cols;    // boundary columns (zero-filled before the kernel)
  std::vector<MultiRec> multi;       // columns touched by >= 3 patches
  std::vector<int32_t> nedge;        // [n_patches] leading edge pairs (two entries each)
  int32_t n_partials = 0;
  // part meshes: patches [0, n_bnd_patches) hold every triangle touching a
  // ghost column; multi records [0, n_multi_bnd) are touched by those patches only
  int32_t n_bnd_patches = 0;
  int32_t n_multi_bnd = 0;
  // in-kernel zero fill (KA-ws, single launch): the LEAD patch of a boundary
  // column (the first patch touching it) zero-fills it; zl[zl_ptr[p] ..
  // zl_ptr[p+1]) are the columns patch p leads, wl[wl_ptr[p] .. wl_ptr[p+1])
  // the lead patches p waits for before its first boundary RED
  std::vector<int32_t> zl, zl_ptr, wl, wl_ptr;
};

struct DevPatch {
  int32_t* t_begin = nullptr;
  int32_t* col_ptr = nullptr;
  int32_t* pair_ptr = nullptr;
  int64_t* contrib_ptr = nullptr;
  PlanCol* cols = nullptr;
  PlanPair* pairs = nullptr;
  uint32_t* contrib = nullptr;
  int32_t* zero_cols = nullptr;
  uint8_t* blob = nullptr;           // per-patch plan blobs (shared-memory layout)
  int64_t* blob_off = nullptr;       // [n_patches+1] byte offsets, multiples of 16
  int32_t* nedge = nullptr;          // [n_patches]
  MultiRec* multi = nullptr;
  double* partials = nullptr;        // [n_partials][L+1][kPartialStride]
  int32_t* zl = nullptr;
  int32_t* zl_ptr = nullptr;
  int32_t* wl = nullptr;
  int32_t* wl_ptr = nullptr;
  int32_t* flags = nullptr;          // [n_patches + 1]: zero-fill done per patch; [n_patches] = patch ticket
};

}  // namespace fo

struct fo_mesh_s {
  int device = 0;
  fo_params p{};
  int32_t L = 0;
  int64_t n_col = 0, nA = 0, nB = 0, nC = 0;  // local columns by class
  int64_t n_tri = 0;                          // local triangles
  int64_t n_bnd_tri = 0;                      // of which the leading ones touch a ghost column
  int64_t n_node = 0, n_dof = 0, n_elem = 0, n_owned_dof = 0;
  int64_t nnz = 0;
  // host topology (kept for graph / halo construction)
  std::vector<int64_t> glob;       // local column -> global column
  std::vector<int64_t> tri_glob;   // local triangle -> global triangle
  std::vector<int32_t> tri;        // local triangles, local column ids
  std::vector<int64_t> nbr_ptr;    // coupling lists (incl. self), sorted by local id
  std::vector<int32_t> nbr;
  std::vector<int64_t> colstart;   // [n_col+1] CSR value offset of each column block
  std::vector<fo::TriRec> trirec;
  std::vector<fo::QuadRec> quadrec;   // hexahedral meshes (tri then holds 4 corners per quad)
  std::vector<fo::ColRec> colrec;
  std::vector<double> sigma;
  bool has_A_elem = false;
  int32_t part = 0, n_parts = 1;
  // global footprint topology (partitioned meshes only; for the halo plan)
  int64_t global_n_vert = 0;
  std::vector<int32_t> global_tri;
  std::vector<int32_t> global_part;
  // device copies
  fo::ColRec* d_col = nullptr;
  fo::TriRec* d_tri = nullptr;
  double* d_sigma = nullptr;
  double* d_A = nullptr;           // per-wedge A^(-1/n) or nullptr
  double* d_T = nullptr;           // per-wedge T* (NEXT-f3) or nullptr
  double A0fac = 0.0, QnR = 0.0;   // Arrhenius constants folded for the kernels
  int elem_type = FO_ELEM_WEDGE;   // NEXT-f4 (fo_element_tet.cuh)
  bool quad = false;               // NEXT-f4 hexahedral mesh (fo_hex.cu)
  fo::QuadRec* d_quad = nullptr;
  int32_t* d_hex_ids = nullptr;    // quads grouped by colour
  std::vector<int64_t> hex_color_ptr;
  std::vector<int32_t> tri_ccw;    // the caller's (CCW) corner order, kept while
  std::vector<fo::TriRec> trirec_ccw;   // FO_ELEM_TET3 runs on global-id order
  // NEXT-f1 lateral margin term (fo_lateral.cu)
  bool lateral = false;
  int32_t n_lat_cols = 0, n_lat_faces = 0;
  int4* d_lat_cols = nullptr;      // (column, first ref, ref count, 0)
  int2* d_lat_faces = nullptr;     // (c0, c1) CCW edge of a margin face
  int32_t* d_lat_refs = nullptr;   // face * 2 + role
  // NEXT-f2 Newton consumer (fo_solve.cu), allocated on first use
  int64_t* d_nbr_ptr = nullptr;
  int32_t* d_nbr = nullptr;
  int32_t* d_self_slot = nullptr;
  double* d_line_fac = nullptr;    // [n_cols][L+1][8] block Thomas factors
  double* d_kry_work = nullptr;    // dot-product partials
  const double* line_vals = nullptr;   // the values fo_line_factor factored
  fo::PatchPlan plan;
  fo::DevPatch d_plan;
  fo_scatter scatter = FO_SCATTER_OWNER;
  int32_t last_launches = 0;
  bool timing = false;
  std::vector<std::pair<void*, void*>> timed;   // (start, stop) cudaEvent_t pairs
  // host-API staging
  double* d_stage_U = nullptr;
  double* d_stage_R = nullptr;
  double* d_stage_vals = nullptr;
  double* d_scratch_R = nullptr;   // residual scratch when the caller passes no R
  int64_t stage_vals_n = 0;
};

struct fo_graph_s {
  fo_mesh mesh = nullptr;
  int64_t n_rows = 0, nnz = 0;
  int64_t* d_row_ptr = nullptr;
  int32_t* d_col_idx = nullptr;
};

namespace fo {
// NVTX range over one public call (nsys / ncu --nvtx-include):
// fo_assemble_*, fo_halo_import / fo_halo_sum
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
// Local topology of one footprint part (fo_host.cpp build_topology).
struct Topo {
  int64_t nA = 0, nB = 0, nC = 0;
  std::vector<int64_t> glob;      // local -> global column
  std::vector<int64_t> tri_glob;  // local -> global triangle
  std::vector<int32_t> tri;       // local triangles (local ids)
  std::vector<int64_t> nbr_ptr;
  std::vector<int32_t> nbr;
  std::vector<int64_t> colstart;
  std::vector<TriRec> trirec;
  int64_t n_bnd_tri = 0;          // leading local triangles touching a ghost column
};
fo_status build_topology(int64_t n_vert, int64_t n_tri, const int32_t* tri, int32_t L,
                         const int32_t* part, int32_t my_part, Topo& T);
void build_csr(const Topo& T, int32_t L, std::vector<int64_t>* row_ptr,
               std::vector<int32_t>* col_idx, int64_t* nnz_out);
void set_error(const std::string& msg);
fo_status cuda_status(int err, const char* what);   // err: cudaError_t
// kernels (fo_kernels.cu)
fo_status launch_residual(fo_mesh m, const double* d_U, double* d_R, void* stream);
fo_status launch_jacobian(fo_mesh m, const double* d_U, double* d_R, double* d_vals,
                          void* stream);
fo_status build_patch_plan(fo_mesh m, bool upload = true);
// owner-computes assembly pieces (fo_owner.cu)
fo_status launch_owner_prologue(fo_mesh m, double* R, double* vals, cudaStream_t s, int* launches,
                                bool inkz = false);
fo_status launch_owner_fixup(fo_mesh m, double* R, double* vals, cudaStream_t s, int* launches);
fo_status launch_owner_overlap(fo_mesh m, const double* d_U, double* d_R, double* d_vals, cudaStream_t s,
                               cudaStream_t side, cudaEvent_t ev0,
                               const std::function<fo_status(cudaStream_t, const int32_t*)>& wait_ready);
void free_patch_plan(fo_mesh m);
fo_status plan_check(const fo_mesh m, int64_t* stats);
// NEXT-f1 lateral margin term (fo_lateral.cu)
fo_status build_lateral(fo_mesh m, int64_t n_tri_global, const int32_t* tri_global);
fo_status launch_lateral(fo_mesh m, double* d_R, void* stream);
// NEXT-f4 hexahedra (fo_hex.cu)
fo_status launch_hex(fo_mesh m, const double* d_U, double* d_R, double* d_vals, cudaStream_t s);
}  // namespace fo
