// fo_plan.cpp -- host construction of the work decomposition of the
// owner-computes assembly kernel (fo_owner.cu), DESIGN.md "KA-patch".
//
// A patch is a contiguous range of (Hilbert-ordered) local triangles, computed
// by one CTA, one thread per triangle column.  For every column the patch
// touches the plan stores a column record, and for every slot of the column's
// coupling list a (column, slot) PAIR with its list of contributions: the
// (patch-local triangle tl, local vertex j of the column, local vertex j' of
// the slot's neighbour) whose element entries land in that slot.  Phase B of
// the kernel gives one pair to one thread, which sums the 12 values (comp a,
// level group g, comp b) of the slot for the current level.
//
// A column is INTERIOR to a patch when the patch holds its whole triangle
// fan: its rows are written with plain stores (every slot, zeros included).
// Otherwise it is a BOUNDARY column: its rows are zero-filled before the
// kernel and every touching patch adds its partial sums with fp64 RED, for
// the slots it contributes to only.  Two partial sums added onto zero give
// the same double in either order; where three or more patches touch a column
// (its self slot and residual collect all of them), each patch instead stores
// its partial sums to a scratch block of its own and a fix-up pass adds them
// in patch order, so the assembly is bitwise reproducible.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "fo_internal.h"

namespace fo {

namespace {
template <class T>
fo_status upload_vec(T** dst, const std::vector<T>& v) {
  *dst = nullptr;
  if (v.empty()) return FO_OK;
  fo_status st = cuda_status(cudaMalloc(reinterpret_cast<void**>(dst), v.size() * sizeof(T)), "cudaMalloc");
  if (st) return st;
  return cuda_status(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice),
                     "cudaMemcpy H2D");
}

struct PatchBuild {
  std::vector<PlanCol> cols;
  std::vector<PlanPair> pairs;
  std::vector<uint32_t> contrib;
  int32_t nedge = 0;   // pairs [0, nedge) are edge slots with exactly two entries
};

// Contribution of wedge-triangle tl (local vertex j = the row column, j2 = the
// slot's column) encoded with the shared-memory offsets phase B needs:
//   bits  0- 7  tl
//   bits  8-12  D base of the (j, j2) 2x2 node block (fo_owner.cu dmap)
//   bits 13-14  its (row a, column b) strides: 0 -> (1,1) diagonal block,
//               1 -> (2,1) for j < j2, 2 -> (1,2) for j > j2
//   bits 15-19  O index of (row (j,0), column (j2,0)) = 12 j + 2 j2
//   bits 20-24  O index of (row (j2,0), column (j,0)) = 12 j2 + 2 j (transpose)
//   bits 25-26  j (residual entry 21 + 2 j + a)
// The code kPatchTris (tl = kPatchTris, all offsets 0) is the pad entry
// (kPatchQuads for hexahedra).
// Hexahedra (NV = 4, CodeBits<4>): the same fields for the 8 bottom dofs of
// a quad -- off-diagonal node blocks j < j2 at 4 rank(j, j2), diagonal ones
// at 24 + 3 j, O index 16 j + 2 j2, residual entry 36 + 2 j + a.
template <int NV>
uint32_t contrib_code(int tl, int j, int j2) {
  using CB = CodeBits<NV>;
  uint32_t dbase, pat;
  const int lo = j < j2 ? j : j2, hi = j < j2 ? j2 : j;
  if (j == j2) { dbase = uint32_t(4 * NV * (NV - 1) / 2 + 3 * j); pat = 0; }
  else { dbase = uint32_t(4 * (lo * (2 * NV - 1 - lo) / 2 + (hi - lo - 1))); pat = j < j2 ? 1 : 2; }
  return uint32_t(tl) | (dbase << CB::kTl) | (pat << CB::kPat) | (uint32_t(2 * CB::kRow * j + 2 * j2) << CB::kO) |
         (uint32_t(2 * CB::kRow * j2 + 2 * j) << CB::kOt) | (uint32_t(j) << CB::kJ);
}

// the corners of element t and the slot of corner j2's column in corner j's list
template <int NV>
struct ElemView;
template <>
struct ElemView<3> {
  const fo_mesh m;
  int32_t corner(int64_t t, int j) const { return m->tri[size_t(3 * t + j)]; }
  int slot(int64_t t, int j, int j2) const { return m->trirec[size_t(t)].slot[3 * j + j2]; }
};
template <>
struct ElemView<4> {
  const fo_mesh m;
  int32_t corner(int64_t t, int j) const { return m->quadrec[size_t(t)].v[j]; }
  int slot(int64_t t, int j, int j2) const { return m->quadrec[size_t(t)].slot[4 * j + j2]; }
};

// plan of the element range [t0, t1)
template <int NV>
void build_one(const fo_mesh m, const std::vector<int32_t>& fan, int32_t t0, int32_t t1,
               PatchBuild& B, std::vector<char>& boundary) {
  const ElemView<NV> ev{m};
  const uint32_t kPad = uint32_t(NV == 3 ? kPatchTris : kPatchQuads);   // pad entry: the zero element slot
  B.cols.clear();
  B.pairs.clear();
  B.contrib.clear();
  std::vector<PlanPair> self_pairs;   // appended after the edge pairs (see below)
  std::vector<std::pair<int32_t, int32_t>> inc;   // (column, tl*4 + j)
  for (int32_t t = t0; t < t1; ++t)
    for (int j = 0; j < NV; ++j) inc.push_back({ev.corner(t, j), (t - t0) * 4 + j});
  std::sort(inc.begin(), inc.end());
  size_t i = 0;
  while (i < inc.size()) {
    const int32_t c = inc[i].first;
    size_t e = i;
    while (e < inc.size() && inc[e].first == c) ++e;
    const bool interior = int32_t(e - i) == fan[size_t(c)];
    if (!interior) boundary[size_t(c)] = 1;
    const int64_t nc = m->nbr_ptr[size_t(c) + 1] - m->nbr_ptr[size_t(c)];
    const int32_t* lst = m->nbr.data() + m->nbr_ptr[size_t(c)];
    const int32_t self = int32_t(std::lower_bound(lst, lst + nc, c) - lst);
    std::vector<std::vector<uint32_t>> per_slot(static_cast<size_t>(nc));
    for (size_t q = i; q < e; ++q) {
      const int32_t tl = inc[q].second >> 2, j = inc[q].second & 3;
      for (int j2 = 0; j2 < NV; ++j2)
        per_slot[size_t(ev.slot(t0 + tl, j, j2))].push_back(contrib_code<NV>(tl, j, j2));
    }
    PlanCol pc{};
    pc.colstart = m->colstart[size_t(c)];
    pc.c = c;
    pc.info = int32_t(nc) | (interior ? 256 : 0) | (self << 9);
    const int32_t ci = int32_t(B.cols.size());
    for (int64_t s = 0; s < nc; ++s) {
      auto& l = per_slot[size_t(s)];
      // even lengths: phase B gathers two contributions per step; the pad
      // entry reads triangle slot kPatchTris, kept zero by the kernel
      if (l.size() & 1) l.push_back(kPad);
      if (s != self && (interior || !l.empty()))   // edge slots: exactly two entries
        while (l.size() < 2) l.push_back(kPad);   // (interior slots of a part mesh may have none)
      if (l.empty() && !interior) continue;   // boundary: only touched slots
      PlanPair pp{};
      pp.cnt = uint8_t(l.size());
      pp.slot = uint8_t(s);
      pp.col = uint16_t(ci);
      pp.c0 = l[0];   // the first two contributions inline: one 16-byte
      pp.c1 = l[1];   // shared load gives an edge pair's whole list
      if (s == self) {
        // the self list is kept whole for the residual gather (phase_b_r)
        pc.self_off = uint16_t(B.contrib.size());
        pc.self_cnt = uint16_t(l.size());
        pp.off = uint16_t(B.contrib.size() + 2);
        B.contrib.insert(B.contrib.end(), l.begin(), l.end());
        self_pairs.push_back(pp);
      } else {
        pp.off = uint16_t(B.contrib.size());
        B.contrib.insert(B.contrib.end(), l.begin() + 2, l.end());
        B.pairs.push_back(pp);
      }
    }
    B.cols.push_back(pc);
    i = e;
  }
  // Edge slots have 1-2 contributions, self slots one per fan triangle (~6):
  // edge pairs first (column order, coalesced stores), then the self pairs, so
  // the lanes of a warp run loops of nearly equal length.
  B.nedge = int32_t(B.pairs.size());
  B.pairs.insert(B.pairs.end(), self_pairs.begin(), self_pairs.end());
}

size_t plan_bytes(const PatchBuild& B) {
  return B.cols.size() * sizeof(PlanCol) + B.pairs.size() * sizeof(PlanPair) +
         ((B.contrib.size() * sizeof(uint32_t) + 15) / 16) * 16;
}

}  // namespace

void free_patch_plan(fo_mesh m) {
  DevPatch& d = m->d_plan;
  void* ptrs[] = {d.t_begin, d.col_ptr, d.pair_ptr, d.contrib_ptr, d.cols, d.pairs, d.contrib, d.zero_cols,
                  d.blob, d.blob_off, d.nedge, d.multi, d.partials, d.zl, d.zl_ptr, d.wl, d.wl_ptr, d.flags};
  for (void* q : ptrs) cudaFree(q);
  d = DevPatch();
  m->plan = PatchPlan();
}

fo_status build_patch_plan(fo_mesh m, bool upload) {
  PatchPlan& P = m->plan;
  P = PatchPlan();
  const int64_t nt = m->n_tri;
  const int64_t nk = m->nA + m->nB;     // columns with rows
  if (nt == 0) return FO_OK;
  const int nv = m->quad ? 4 : 3;
  std::vector<int32_t> fan(size_t(m->n_col), 0);
  for (int64_t t = 0; t < nt; ++t)
    for (int j = 0; j < nv; ++j) fan[size_t(m->tri[size_t(nv * t + j)])]++;
  std::vector<char> boundary(size_t(nk), 0);
  P.t_begin.assign(1, 0);
  P.col_ptr.assign(1, 0);
  P.pair_ptr.assign(1, 0);
  P.contrib_ptr.assign(1, 0);
  PatchBuild B;
  int64_t t0 = 0;
  // equal-size ranges of at most kPatchTris triangles (kPatchQuads quads); a
  // range whose plan exceeds the shared-memory budget is halved
  const int64_t per_patch = m->quad ? kPatchQuads : kPatchTris;
  const size_t budget = size_t(m->quad ? kPlanBytesHex : kPlanBytes);
  const int64_t np0 = (nt + per_patch - 1) / per_patch;
  std::vector<int64_t> bounds;
  for (int64_t p = 0; p <= np0; ++p) bounds.push_back((p * nt) / np0);
  for (size_t b = 0; b + 1 < bounds.size(); ++b) {
    std::vector<std::pair<int64_t, int64_t>> todo{{bounds[b], bounds[b + 1]}};
    while (!todo.empty()) {
      auto [a0, a1] = todo.back();
      todo.pop_back();
      std::vector<char> bnd_tmp = boundary;
      if (m->quad) build_one<4>(m, fan, int32_t(a0), int32_t(a1), B, bnd_tmp);
      else build_one<3>(m, fan, int32_t(a0), int32_t(a1), B, bnd_tmp);
      if (plan_bytes(B) > budget && a1 - a0 > 1) {
        const int64_t mid = (a0 + a1) / 2;
        todo.push_back({mid, a1});
        todo.push_back({a0, mid});
        continue;
      }
      boundary.swap(bnd_tmp);
      t0 = a1;
      P.t_begin.push_back(int32_t(a1));
      P.cols.insert(P.cols.end(), B.cols.begin(), B.cols.end());
      P.pairs.insert(P.pairs.end(), B.pairs.begin(), B.pairs.end());
      P.contrib.insert(P.contrib.end(), B.contrib.begin(), B.contrib.end());
      for (int32_t q = 0; q < int32_t(B.pairs.size()); ++q)   // an edge joins <= 2 triangles: padded to 2
        if ((q < B.nedge && B.pairs[size_t(q)].cnt != 2) || B.pairs[size_t(q)].cnt < 2 ||
            (B.pairs[size_t(q)].cnt & 1))
          return FO_EINVAL;
      P.nedge.push_back(B.nedge);
      P.col_ptr.push_back(int32_t(P.cols.size()));
      P.pair_ptr.push_back(int32_t(P.pairs.size()));
      P.contrib_ptr.push_back(int64_t(P.contrib.size()));
      P.max_plan_bytes = std::max<int64_t>(P.max_plan_bytes, int64_t(plan_bytes(B)));
    }
  }
  (void)t0;
  P.n_patches = int32_t(P.t_begin.size() - 1);
  for (int64_t c = 0; c < nk; ++c)
    if (boundary[size_t(c)]) P.zero_cols.push_back(int32_t(c));
  {   // lead patch of every boundary column, its zero list and the wait lists
    std::vector<int32_t> lead(size_t(m->n_col), -1);
    for (int32_t p = 0; p < P.n_patches; ++p)
      for (int32_t ci = P.col_ptr[size_t(p)]; ci < P.col_ptr[size_t(p) + 1]; ++ci)
        if (lead[size_t(P.cols[size_t(ci)].c)] < 0) lead[size_t(P.cols[size_t(ci)].c)] = p;
    P.zl_ptr.assign(size_t(P.n_patches) + 1, 0);
    for (int32_t c : P.zero_cols) P.zl_ptr[size_t(lead[size_t(c)]) + 1]++;
    for (int32_t p = 0; p < P.n_patches; ++p) P.zl_ptr[size_t(p) + 1] += P.zl_ptr[size_t(p)];
    P.zl.assign(P.zero_cols.size(), 0);
    std::vector<int32_t> fill(P.zl_ptr.begin(), P.zl_ptr.end() - 1);
    for (int32_t c : P.zero_cols) P.zl[size_t(fill[size_t(lead[size_t(c)])]++)] = c;
    P.wl_ptr.assign(1, 0);
    for (int32_t p = 0; p < P.n_patches; ++p) {
      std::vector<int32_t> w;
      for (int32_t ci = P.col_ptr[size_t(p)]; ci < P.col_ptr[size_t(p) + 1]; ++ci) {
        const int32_t c = P.cols[size_t(ci)].c;
        if (boundary[size_t(c)] && lead[size_t(c)] != p) w.push_back(lead[size_t(c)]);
      }
      std::sort(w.begin(), w.end());
      w.erase(std::unique(w.begin(), w.end()), w.end());
      P.wl.insert(P.wl.end(), w.begin(), w.end());
      P.wl_ptr.push_back(int32_t(P.wl.size()));
    }
  }
  // MULTI columns: touched by >= 3 patches; partial block b = base + rank
  // (rank = order of the patch among the column's patches)
  {
    std::vector<int32_t> touch(size_t(m->n_col), 0), base(size_t(m->n_col), -1), next(size_t(m->n_col), 0);
    for (const PlanCol& pc : P.cols) touch[size_t(pc.c)]++;
    int32_t nb = 0;
    for (const PlanCol& pc : P.cols) {
      const int32_t c = pc.c;
      if (touch[size_t(c)] >= 3 && base[size_t(c)] < 0) {
        base[size_t(c)] = nb;
        nb += touch[size_t(c)];
        MultiRec mr{};
        mr.colstart = pc.colstart;
        mr.c = c;
        mr.nc_self = (pc.info & 255) | (((pc.info >> 9) & 255) << 8);
        mr.base = base[size_t(c)];
        mr.cnt = touch[size_t(c)];
        P.multi.push_back(mr);
      }
    }
    for (PlanCol& pc : P.cols)   // patches in order: ranks ascend with the patch index
      if (base[size_t(pc.c)] >= 0) {
        pc.info |= 1 << 30;
        pc.pad = uint32_t(base[size_t(pc.c)] + next[size_t(pc.c)]++);
      }
    P.n_partials = nb;
  }
  // part meshes: the leading patches holding the ghost-touching triangles, and
  // the multi columns touched by those patches only (their fix-up can run
  // before the interior patches are done), moved to the front of the list
  for (int32_t p = 0; p < P.n_patches; ++p)
    if (P.t_begin[size_t(p)] < m->n_bnd_tri) P.n_bnd_patches = p + 1;
  if (P.n_bnd_patches > 0 && !P.multi.empty()) {
    std::vector<int32_t> last(size_t(m->n_col), -1);
    for (int32_t p = 0; p < P.n_patches; ++p)
      for (int32_t ci = P.col_ptr[size_t(p)]; ci < P.col_ptr[size_t(p) + 1]; ++ci)
        last[size_t(P.cols[size_t(ci)].c)] = p;
    std::stable_partition(P.multi.begin(), P.multi.end(),
                          [&](const MultiRec& r) { return last[size_t(r.c)] < P.n_bnd_patches; });
    for (const MultiRec& r : P.multi)
      if (last[size_t(r.c)] < P.n_bnd_patches) ++P.n_multi_bnd;
  }
  // one 16-byte aligned blob per patch in the shared-memory layout of the
  // kernel (pairs | columns | contributions: the 16-byte pair records first,
  // so they stay 16-byte aligned), copied with one bulk copy
  std::vector<uint8_t> blob;
  std::vector<int64_t> blob_off(1, 0);
  for (int32_t p = 0; p < P.n_patches; ++p) {
    auto put = [&](const void* src, size_t n) {
      const uint8_t* b = static_cast<const uint8_t*>(src);
      blob.insert(blob.end(), b, b + n);
    };
    put(P.pairs.data() + P.pair_ptr[size_t(p)],
        sizeof(PlanPair) * size_t(P.pair_ptr[size_t(p) + 1] - P.pair_ptr[size_t(p)]));
    put(P.cols.data() + P.col_ptr[size_t(p)], sizeof(PlanCol) * size_t(P.col_ptr[size_t(p) + 1] - P.col_ptr[size_t(p)]));
    put(P.contrib.data() + P.contrib_ptr[size_t(p)],
        sizeof(uint32_t) * size_t(P.contrib_ptr[size_t(p) + 1] - P.contrib_ptr[size_t(p)]));
    blob.resize((blob.size() + 15) / 16 * 16, 0);
    blob_off.push_back(int64_t(blob.size()));
  }
  if (!upload) return FO_OK;
  fo_status st = upload_vec(&m->d_plan.t_begin, P.t_begin);
  if (!st) st = upload_vec(&m->d_plan.col_ptr, P.col_ptr);
  if (!st) st = upload_vec(&m->d_plan.pair_ptr, P.pair_ptr);
  if (!st) st = upload_vec(&m->d_plan.blob, blob);
  if (!st) st = upload_vec(&m->d_plan.blob_off, blob_off);
  if (!st) st = upload_vec(&m->d_plan.nedge, P.nedge);
  if (!st) st = upload_vec(&m->d_plan.zero_cols, P.zero_cols);
  if (!st) st = upload_vec(&m->d_plan.multi, P.multi);
  if (!st) st = upload_vec(&m->d_plan.zl, P.zl);
  if (!st) st = upload_vec(&m->d_plan.zl_ptr, P.zl_ptr);
  if (!st) st = upload_vec(&m->d_plan.wl, P.wl);
  if (!st) st = upload_vec(&m->d_plan.wl_ptr, P.wl_ptr);
  if (!st)
    st = cuda_status(cudaMalloc(reinterpret_cast<void**>(&m->d_plan.flags), sizeof(int32_t) * (P.n_patches + 3)),
                     "cudaMalloc");
  if (!st && P.n_partials > 0)
    st = cuda_status(cudaMalloc(reinterpret_cast<void**>(&m->d_plan.partials),
                                sizeof(double) * kPartialStride * size_t(m->L + 1) * size_t(P.n_partials)),
                     "cudaMalloc");
  return st;
}

// Host check of a plan's coverage (fo_plan_check_host): every coupling-list
// slot and residual of a column with rows must be written either by one
// store (an interior column's pair; the fix-up of a multi column's self slot)
// or by RED partial sums onto a zero-filled boundary column -- never both,
// never neither; every element entry (t, j, j2) must be gathered exactly once,
// by the pair of column v_j, slot of v_j2.  stats[8] = {patches, pairs,
// contributions (pads excluded), zero-filled columns, multi columns,
// slot / residual violations, element-entry violations, largest plan bytes}.
fo_status plan_check(const fo_mesh m, int64_t* stats) {
  const PatchPlan& P = m->plan;
  const int64_t nk = m->nA + m->nB;
  std::vector<int32_t> store(m->nbr.size(), 0), red(m->nbr.size(), 0);
  std::vector<int32_t> rstore(size_t(m->n_col), 0), rred(size_t(m->n_col), 0);
  std::vector<char> zeroed(size_t(m->n_col), 0), multi(size_t(m->n_col), 0);
  for (int32_t c : P.zero_cols) zeroed[size_t(c)] = 1;
  for (const MultiRec& r : P.multi) multi[size_t(r.c)] = 1;
  const bool quad = m->quad;
  const int nv = quad ? 4 : 3;
  std::vector<int32_t> seen(size_t(nv * nv * m->n_tri), 0);
  int64_t n_contrib = 0, bad_elem = 0;
  for (int32_t p = 0; p < P.n_patches; ++p) {
    const PlanCol* cols = P.cols.data() + P.col_ptr[size_t(p)];
    const int32_t t0 = P.t_begin[size_t(p)];
    for (int32_t q = P.pair_ptr[size_t(p)]; q < P.pair_ptr[size_t(p) + 1]; ++q) {
      const PlanPair& pp = P.pairs[size_t(q)];
      const PlanCol& pc = cols[pp.col];
      const int64_t e = m->nbr_ptr[size_t(pc.c)] + pp.slot;
      const bool interior = (pc.info >> 8) & 1;
      const bool mself = ((pc.info >> 30) & 1) && pp.slot == ((pc.info >> 9) & 255);
      if (mself) {
        // written by the fix-up: counted once per column below
      } else if (interior) {
        store[size_t(e)]++;
      } else {
        red[size_t(e)]++;
      }
      for (int i = 0; i < pp.cnt; ++i) {
        const uint32_t cb = i == 0 ? pp.c0 : i == 1 ? pp.c1
                                    : P.contrib[size_t(P.contrib_ptr[size_t(p)] + pp.off + i - 2)];
        // decode with the element's field layout (CodeBits<3> / <4>)
        const int tlb = quad ? CodeBits<4>::kTl : CodeBits<3>::kTl;
        const int ob = CodeBits<3>::kO, ow = quad ? CodeBits<4>::kOw : CodeBits<3>::kOw;
        const int jb = quad ? CodeBits<4>::kJ : CodeBits<3>::kJ, row = 2 * nv;
        const int tl = int(cb & ((1u << tlb) - 1));
        if (tl == (quad ? kPatchQuads : kPatchTris)) continue;   // pad
        ++n_contrib;
        const int j = int((cb >> jb) & 3);
        const int o = int((cb >> ob) & ((1u << ow) - 1));   // 2 row j + 2 j2
        const int j2 = (o - 2 * row * j) / 2;
        const int64_t t = t0 + tl;
        const int32_t vj = quad ? m->quadrec[size_t(t)].v[j] : m->trirec[size_t(t)].v[j];
        const int sl = quad ? m->quadrec[size_t(t)].slot[4 * j + j2] : m->trirec[size_t(t)].slot[3 * j + j2];
        if (vj != pc.c || sl != pp.slot) ++bad_elem;
        seen[size_t(nv * nv * t + nv * j + j2)]++;
      }
    }
    for (int32_t ci = P.col_ptr[size_t(p)]; ci < P.col_ptr[size_t(p) + 1]; ++ci) {
      const PlanCol& pc = P.cols[size_t(ci)];
      if ((pc.info >> 30) & 1) continue;   // fix-up
      if ((pc.info >> 8) & 1) rstore[size_t(pc.c)]++; else rred[size_t(pc.c)]++;
    }
  }
  for (int32_t v : seen) if (v != 1) ++bad_elem;
  int64_t bad_slot = 0;
  for (int64_t c = 0; c < nk; ++c) {
    const int64_t nc = m->nbr_ptr[size_t(c) + 1] - m->nbr_ptr[size_t(c)];
    const int64_t self = std::lower_bound(m->nbr.begin() + m->nbr_ptr[size_t(c)],
                                          m->nbr.begin() + m->nbr_ptr[size_t(c) + 1], int32_t(c)) -
                         (m->nbr.begin() + m->nbr_ptr[size_t(c)]);
    for (int64_t s = 0; s < nc; ++s) {
      const int64_t e = m->nbr_ptr[size_t(c)] + s;
      int st = store[size_t(e)], rd = red[size_t(e)];
      if (multi[size_t(c)] && s == self) st += 1;   // the fix-up store
      const bool ok = (st == 1 && rd == 0) || (st == 0 && rd >= 1 && zeroed[size_t(c)]) ||
                      (st == 0 && rd == 0 && false);
      // a slot no local triangle couples (part meshes: foreign coupling) is
      // stored as zero by an interior pair or cleared by the zero fill
      const bool empty_ok = st == 0 && rd == 0 && zeroed[size_t(c)];
      if (!ok && !empty_ok) ++bad_slot;
    }
    int rs = rstore[size_t(c)] + (multi[size_t(c)] ? 1 : 0), rr = rred[size_t(c)];
    if (!((rs == 1 && rr == 0) || (rs == 0 && rr >= 1 && zeroed[size_t(c)]))) ++bad_slot;
  }
  // in-kernel zero fill of KA-ws: every zero-filled column is in the zero list
  // of exactly one patch -- the first patch holding it -- and every later
  // patch holding it waits for that patch
  {
    std::vector<int32_t> lead_of(size_t(m->n_col), -1);
    for (int32_t p = 0; p < P.n_patches; ++p)
      for (int32_t i = P.zl_ptr[size_t(p)]; i < P.zl_ptr[size_t(p) + 1]; ++i) {
        if (lead_of[size_t(P.zl[size_t(i)])] >= 0) ++bad_slot;
        lead_of[size_t(P.zl[size_t(i)])] = p;
      }
    for (int32_t c : P.zero_cols)
      if (lead_of[size_t(c)] < 0) ++bad_slot;
    for (int32_t p = 0; p < P.n_patches; ++p) {
      const int32_t* w0 = P.wl.data() + P.wl_ptr[size_t(p)];
      const int32_t* w1 = P.wl.data() + P.wl_ptr[size_t(p) + 1];
      for (int32_t ci = P.col_ptr[size_t(p)]; ci < P.col_ptr[size_t(p) + 1]; ++ci) {
        const int32_t c = P.cols[size_t(ci)].c, l = lead_of[size_t(c)];
        if (!zeroed[size_t(c)]) continue;
        if (l > p) ++bad_slot;   // the lead is the FIRST patch holding the column
        if (l != p && !std::binary_search(w0, w1, l)) ++bad_slot;
      }
    }
  }
  stats[0] = P.n_patches;
  stats[1] = int64_t(P.pairs.size());
  stats[2] = n_contrib;
  stats[3] = int64_t(P.zero_cols.size());
  stats[4] = int64_t(P.multi.size());
  stats[5] = bad_slot;
  stats[6] = bad_elem;
  stats[7] = P.max_plan_bytes;
  return FO_OK;
}

}  // namespace fo
