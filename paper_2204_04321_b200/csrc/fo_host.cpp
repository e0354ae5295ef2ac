// fo_host.cpp -- host side of libfo: validation, extrusion bookkeeping,
// footprint partition, local numbering, fixed CSR graph, device upload.
//
// Paper context (PAPER.md, P:n = line n): the mesh is the vertical extrusion of
// a triangulated footprint; the Jacobian lives in a fixed CSR
// graph with owned rows first (FeCrsMatrix); the distributed maps
// of Tpetra Import/Export become the local numbering below.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "fo_internal.h"

namespace fo {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

fo_status cuda_status(int err, const char* what) {
  if (err == cudaSuccess) return FO_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(static_cast<cudaError_t>(err)));
  return err == cudaErrorMemoryAllocation ? FO_ENOMEM : FO_ECUDA;
}

namespace {

fo_status fail(fo_status st, const std::string& msg) {
  set_error(msg);
  return st;
}

// levels per row block: m(k) = 2 at the bed and the surface, 3 inside
inline int64_t m_of(int64_t k, int64_t L) { return (k == 0 || k == L) ? 2 : 3; }

fo_status validate(const fo_params* p, int64_t n_vert, const double* xy, int64_t n_tri,
                   const int32_t* tri, int32_t L, const double* sigma,
                   const double* thickness, const double* surface, const double* beta) {
  if (!p) return fail(FO_EINVAL, "params is NULL");
  if (n_vert < 0 || n_tri < 0) return fail(FO_EINVAL, "negative size");
  if (L < 1) return fail(FO_EINVAL, "n_layers must be >= 1");
  if (n_vert > INT32_MAX / 2) return fail(FO_EINVAL, "too many vertices for int32 col_idx");
  if (!(p->glen_n > 0.0) || !(p->A > 0.0) || !(p->eps_reg >= 0.0) || !(p->rho > 0.0))
    return fail(FO_EINVAL, "bad physical parameter (need n > 0, A > 0, eps_reg >= 0, rho > 0)");
  if (sigma) {
    if (sigma[0] != 0.0 || sigma[L] != 1.0)
      return fail(FO_EMESH, "sigma must start at 0 and end at 1");
    for (int32_t k = 0; k < L; ++k)
      if (!(sigma[k + 1] > sigma[k])) return fail(FO_EMESH, "sigma not strictly ascending");
  }
  if (n_vert == 0 && n_tri == 0) return FO_OK;
  if (!xy || !tri || !thickness || !surface || !beta)
    return fail(FO_EINVAL, "NULL mesh array");
  if (2 * (n_vert * int64_t(L + 1)) > int64_t(INT32_MAX))
    return fail(FO_EINVAL, "DOF count exceeds int32 col_idx range");
  std::vector<char> used(size_t(n_vert), 0);
  for (int64_t t = 0; t < n_tri; ++t) {
    const int32_t* v = tri + 3 * t;
    for (int j = 0; j < 3; ++j)
      if (v[j] < 0 || v[j] >= n_vert)
        return fail(FO_EMESH, "triangle " + std::to_string(t) + " vertex index out of range");
    if (v[0] == v[1] || v[1] == v[2] || v[0] == v[2])
      return fail(FO_EMESH, "triangle " + std::to_string(t) + " repeats a vertex");
    const double x0 = xy[2 * v[0]], y0 = xy[2 * v[0] + 1];
    const double x1 = xy[2 * v[1]], y1 = xy[2 * v[1] + 1];
    const double x2 = xy[2 * v[2]], y2 = xy[2 * v[2] + 1];
    const double twoA = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0);
    if (!(twoA > 0.0))
      return fail(FO_EMESH, "triangle " + std::to_string(t) + " is CW or degenerate");
    used[v[0]] = used[v[1]] = used[v[2]] = 1;
  }
  for (int64_t c = 0; c < n_vert; ++c) {
    if (!used[c]) return fail(FO_EMESH, "vertex " + std::to_string(c) + " is in no triangle");
    if (!(thickness[c] >= p->H_min))
      return fail(FO_EMESH, "thickness below H_min at vertex " + std::to_string(c));
    if (!std::isfinite(surface[c]) || !std::isfinite(beta[c]) || beta[c] < 0.0)
      return fail(FO_EMESH, "non-finite surface or negative beta at vertex " + std::to_string(c));
  }
  return FO_OK;
}

// sorted global adjacency (neighbours excluding self) in CSR form
void global_adjacency(int64_t n_vert, int64_t n_tri, const int32_t* tri,
                      std::vector<int64_t>& ptr, std::vector<int32_t>& adj) {
  std::vector<int64_t> cnt(size_t(n_vert) + 1, 0);
  for (int64_t t = 0; t < n_tri; ++t)
    for (int i = 0; i < 3; ++i) cnt[tri[3 * t + i] + 1] += 2;
  for (int64_t c = 0; c < n_vert; ++c) cnt[c + 1] += cnt[c];
  std::vector<int32_t> raw(static_cast<size_t>(cnt[n_vert]));
  std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
  for (int64_t t = 0; t < n_tri; ++t)
    for (int i = 0; i < 3; ++i) {
      const int32_t c = tri[3 * t + i];
      raw[fill[c]++] = tri[3 * t + (i + 1) % 3];
      raw[fill[c]++] = tri[3 * t + (i + 2) % 3];
    }
  ptr.assign(size_t(n_vert) + 1, 0);
  adj.clear();
  adj.reserve(raw.size() / 2 + 16);
  for (int64_t c = 0; c < n_vert; ++c) {
    auto b = raw.begin() + cnt[c], e = raw.begin() + cnt[c + 1];
    std::sort(b, e);
    auto u = std::unique(b, e);
    adj.insert(adj.end(), b, u);
    ptr[c + 1] = int64_t(adj.size());
  }
}



}  // namespace

// Local numbering of part my_part:
// A owned (min incident part == my_part), B ghosts touched by local triangles
// grouped by owner, C column-only couplings of A columns.
fo_status build_topology(int64_t n_vert, int64_t n_tri, const int32_t* tri, int32_t L,
                         const int32_t* part, int32_t my_part, Topo& T) {
  std::vector<int64_t> gptr;
  std::vector<int32_t> gadj;
  global_adjacency(n_vert, n_tri, tri, gptr, gadj);
  std::vector<int32_t> owner(size_t(n_vert), INT32_MAX);
  std::vector<char> touched(size_t(n_vert), 0);
  for (int64_t t = 0; t < n_tri; ++t) {
    const int32_t pt = part ? part[t] : 0;
    for (int i = 0; i < 3; ++i) {
      const int32_t c = tri[3 * t + i];
      owner[c] = std::min(owner[c], pt);
      if (pt == my_part) touched[c] = 1;
    }
  }
  std::vector<int64_t> loc(size_t(n_vert), -1);
  T.glob.clear();
  for (int64_t c = 0; c < n_vert; ++c)
    if (owner[c] == my_part) { loc[c] = int64_t(T.glob.size()); T.glob.push_back(c); }
  T.nA = int64_t(T.glob.size());
  std::vector<std::pair<int32_t, int64_t>> ghosts;
  for (int64_t c = 0; c < n_vert; ++c)
    if (touched[c] && owner[c] != my_part) ghosts.push_back({owner[c], c});
  std::sort(ghosts.begin(), ghosts.end());
  for (auto& g : ghosts) { loc[g.second] = int64_t(T.glob.size()); T.glob.push_back(g.second); }
  T.nB = int64_t(ghosts.size());
  for (int64_t i = 0; i < T.nA; ++i) {
    const int64_t c = T.glob[size_t(i)];
    for (int64_t e = gptr[c]; e < gptr[c + 1]; ++e) {
      const int32_t w = gadj[size_t(e)];
      if (loc[w] < 0) loc[w] = -2;   // mark as column-only candidate
    }
  }
  for (int64_t c = 0; c < n_vert; ++c)
    if (loc[c] == -2) { loc[c] = int64_t(T.glob.size()); T.glob.push_back(c); }
  T.nC = int64_t(T.glob.size()) - T.nA - T.nB;
  const int64_t ncol = int64_t(T.glob.size());
  // local triangles
  T.tri.clear();
  T.tri_glob.clear();
  for (int64_t t = 0; t < n_tri; ++t) {
    if ((part ? part[t] : 0) != my_part) continue;
    T.tri_glob.push_back(t);
    for (int i = 0; i < 3; ++i) T.tri.push_back(int32_t(loc[tri[3 * t + i]]));
  }
  const int64_t nt = int64_t(T.tri_glob.size());
  // part meshes: the local triangles touching a ghost (class B) column lead,
  // each group in its original (Hilbert) order -- the patches holding them
  // come first, so fo_assemble_jacobian_halo can send the ghost rows while
  // the remaining (interior) patches are computed
  T.n_bnd_tri = 0;
  if (part) {
    std::vector<int64_t> bnd, rest;
    for (int64_t t = 0; t < nt; ++t) {
      bool g = false;
      for (int i = 0; i < 3; ++i) g = g || (T.tri[size_t(3 * t + i)] >= T.nA);
      (g ? bnd : rest).push_back(t);
    }
    T.n_bnd_tri = int64_t(bnd.size());
    bnd.insert(bnd.end(), rest.begin(), rest.end());
    std::vector<int32_t> tri2(T.tri.size());
    std::vector<int64_t> glob2(T.tri_glob.size());
    for (int64_t i = 0; i < nt; ++i) {
      const int64_t t = bnd[size_t(i)];
      glob2[size_t(i)] = T.tri_glob[size_t(t)];
      for (int j = 0; j < 3; ++j) tri2[size_t(3 * i + j)] = T.tri[size_t(3 * t + j)];
    }
    T.tri.swap(tri2);
    T.tri_glob.swap(glob2);
  }
  // coupling lists
  std::vector<std::vector<int32_t>> lists(size_t(T.nA + T.nB));
  for (int64_t i = 0; i < T.nA; ++i) {
    const int64_t c = T.glob[size_t(i)];
    auto& l = lists[size_t(i)];
    l.push_back(int32_t(i));
    for (int64_t e = gptr[c]; e < gptr[c + 1]; ++e) l.push_back(int32_t(loc[gadj[size_t(e)]]));
  }
  for (int64_t i = T.nA; i < T.nA + T.nB; ++i) lists[size_t(i)].push_back(int32_t(i));
  for (int64_t t = 0; t < nt; ++t)
    for (int i = 0; i < 3; ++i) {
      const int32_t ci = T.tri[3 * t + i];
      if (ci < T.nA) continue;
      for (int j = 0; j < 3; ++j)
        if (j != i) lists[size_t(ci)].push_back(T.tri[3 * t + j]);
    }
  T.nbr_ptr.assign(size_t(ncol) + 1, 0);
  T.nbr.clear();
  for (int64_t i = 0; i < ncol; ++i) {
    if (i < T.nA + T.nB) {
      auto& l = lists[size_t(i)];
      std::sort(l.begin(), l.end());
      l.erase(std::unique(l.begin(), l.end()), l.end());
      if (l.size() > 255)
        return fail(FO_EMESH, "column " + std::to_string(T.glob[size_t(i)]) +
                                  " couples to more than 254 neighbours");
      T.nbr.insert(T.nbr.end(), l.begin(), l.end());
    }
    T.nbr_ptr[size_t(i) + 1] = int64_t(T.nbr.size());
  }
  // CSR value offset of each column block: 4 n_c (3L+1) values per column
  T.colstart.assign(size_t(ncol) + 1, 0);
  for (int64_t i = 0; i < ncol; ++i) {
    const int64_t nc = T.nbr_ptr[size_t(i) + 1] - T.nbr_ptr[size_t(i)];
    T.colstart[size_t(i) + 1] = T.colstart[size_t(i)] + 4 * nc * (3 * int64_t(L) + 1);
  }
  // per-triangle slot table
  T.trirec.assign(size_t(nt), TriRec{});
  for (int64_t t = 0; t < nt; ++t) {
    TriRec& r = T.trirec[size_t(t)];
    for (int i = 0; i < 3; ++i) r.v[i] = T.tri[3 * t + i];
    {   // NEXT-f4 split order: local corners by GLOBAL vertex id (reading L22)
      const int32_t* g = tri + 3 * T.tri_glob[size_t(t)];
      int o[3] = {0, 1, 2};
      std::sort(o, o + 3, [&](int x, int y) { return g[x] < g[y]; });
      r.pad[0] = uint8_t(o[0] | (o[1] << 2) | (o[2] << 4));
    }
    for (int i = 0; i < 3; ++i) {
      const int32_t ci = r.v[i];
      const int32_t* b = T.nbr.data() + T.nbr_ptr[size_t(ci)];
      const int32_t* e = T.nbr.data() + T.nbr_ptr[size_t(ci) + 1];
      for (int j = 0; j < 3; ++j) {
        const int32_t* it = std::lower_bound(b, e, r.v[j]);
        r.slot[3 * i + j] = uint8_t(it - b);
      }
    }
  }
  return FO_OK;
}

// CSR pattern of a topology: rows for A and B columns, empty rows for C
void build_csr(const Topo& T, int32_t L, std::vector<int64_t>* row_ptr,
               std::vector<int32_t>* col_idx, int64_t* nnz_out) {
  const int64_t ncol = int64_t(T.glob.size());
  const int64_t n_dof = 2 * ncol * (L + 1);
  const int64_t nnz = T.colstart[size_t(ncol)];
  if (nnz_out) *nnz_out = nnz;
  if (row_ptr) {
    row_ptr->assign(size_t(n_dof) + 1, 0);
    int64_t r = 0;
    for (int64_t c = 0; c < ncol; ++c) {
      const int64_t nc = T.nbr_ptr[size_t(c) + 1] - T.nbr_ptr[size_t(c)];
      for (int64_t k = 0; k <= L; ++k)
        for (int a = 0; a < 2; ++a, ++r) (*row_ptr)[size_t(r) + 1] = (*row_ptr)[size_t(r)] + 2 * nc * m_of(k, L);
    }
  }
  if (col_idx) {
    col_idx->resize(size_t(nnz));
    int64_t pos = 0;
    for (int64_t c = 0; c < ncol; ++c) {
      const int64_t b = T.nbr_ptr[size_t(c)], e = T.nbr_ptr[size_t(c) + 1];
      for (int64_t k = 0; k <= L; ++k) {
        const int64_t k0 = std::max<int64_t>(0, k - 1), k1 = std::min<int64_t>(L, k + 1);
        for (int a = 0; a < 2; ++a)
          for (int64_t s = b; s < e; ++s) {
            const int64_t cc = T.nbr[size_t(s)];
            for (int64_t kk = k0; kk <= k1; ++kk)
              for (int bb = 0; bb < 2; ++bb) (*col_idx)[size_t(pos++)] = int32_t(2 * (cc * (L + 1) + kk) + bb);
          }
      }
    }
  }
}

namespace {

template <class T>
fo_status upload(T** dst, const T* src, size_t n) {
  *dst = nullptr;
  if (n == 0) return FO_OK;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), n * sizeof(T));
  if (e != cudaSuccess) return cuda_status(e, "cudaMalloc");
  e = cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice);
  return cuda_status(e, "cudaMemcpy H2D");
}

fo_status mesh_create_impl(const fo_params* p, int64_t n_vert, const double* xy, int64_t n_tri,
                           const int32_t* tri, int32_t L, const double* sigma,
                           const double* thickness, const double* surface, const double* bed,
                           const double* beta, const double* A_elem, const int32_t* part,
                           int32_t my_part, int32_t n_parts, int device, fo_mesh* out,
                           bool host_only = false) {
  if (!out) return fail(FO_EINVAL, "out is NULL");
  *out = nullptr;
  fo_status st = validate(p, n_vert, xy, n_tri, tri, L, sigma, thickness, surface, beta);
  if (st) return st;
  if (part) {
    if (n_parts < 1 || my_part < 0 || my_part >= n_parts) return fail(FO_EINVAL, "bad part ids");
    for (int64_t t = 0; t < n_tri; ++t)
      if (part[t] < 0 || part[t] >= n_parts) return fail(FO_EINVAL, "part_of_tri out of range");
  }
  int ndev = 0;
  if (host_only) goto host_topology;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(FO_ECUDA, "no CUDA device available (libfo has no CPU path)");
  }
  if (device < 0 || device >= ndev) return fail(FO_EINVAL, "bad device ordinal");
  st = cuda_status(cudaSetDevice(device), "cudaSetDevice");
  if (st) return st;
host_topology:
  Topo T;
  st = build_topology(n_vert, n_tri, tri, L, part, my_part, T);
  if (st) return st;

  fo_mesh m = new fo_mesh_s();
  m->device = device;
  m->p = *p;
  m->L = L;
  m->nA = T.nA; m->nB = T.nB; m->nC = T.nC;
  m->n_col = T.nA + T.nB + T.nC;
  m->n_tri = int64_t(T.tri_glob.size());
  m->n_node = m->n_col * (L + 1);
  m->n_dof = 2 * m->n_node;
  m->n_elem = m->n_tri * L;
  m->n_owned_dof = 2 * T.nA * (L + 1);
  m->nnz = T.colstart.back();
  m->part = part ? my_part : 0;
  if (part) {
    m->global_n_vert = n_vert;
    m->global_tri.assign(tri, tri + 3 * n_tri);
    m->global_part.assign(part, part + n_tri);
  }
  m->n_parts = part ? n_parts : 1;
  m->sigma.resize(size_t(L) + 1);
  for (int32_t k = 0; k <= L; ++k) m->sigma[size_t(k)] = sigma ? sigma[k] : double(k) / double(L);
  m->sigma[size_t(L)] = 1.0;
  m->colrec.assign(size_t(m->n_col), ColRec{});
  for (int64_t i = 0; i < m->n_col; ++i) {
    const int64_t c = T.glob[size_t(i)];
    ColRec& r = m->colrec[size_t(i)];
    r.x = xy[2 * c];
    r.y = xy[2 * c + 1];
    r.H = thickness[c];
    r.base = surface[c] - thickness[c];
    const bool floating = bed && (p->rho * thickness[c] < -p->rho_w * bed[c]);
    r.beta = floating ? 0.0 : beta[c];
    const int64_t nc = T.nbr_ptr[size_t(i) + 1] - T.nbr_ptr[size_t(i)];
    r.cs_n = (T.colstart[size_t(i)] << 8) | nc;
  }
  m->glob = std::move(T.glob);
  m->tri_glob = std::move(T.tri_glob);
  m->tri = std::move(T.tri);
  m->nbr_ptr = std::move(T.nbr_ptr);
  m->nbr = std::move(T.nbr);
  m->colstart = std::move(T.colstart);
  m->trirec = std::move(T.trirec);
  m->n_bnd_tri = T.n_bnd_tri;

  if (host_only) {   // the patch plan only, nothing on a device (fo_plan_check_host)
    st = build_patch_plan(m, false);
    if (st) { delete m; return st; }
    *out = m;
    return FO_OK;
  }
  st = upload(&m->d_col, m->colrec.data(), m->colrec.size());
  if (!st) st = upload(&m->d_tri, m->trirec.data(), m->trirec.size());
  if (!st) st = upload(&m->d_sigma, m->sigma.data(), m->sigma.size());
  if (!st && A_elem && m->n_elem > 0) {
    std::vector<double> afac(size_t(m->n_elem));
    for (int64_t t = 0; t < m->n_tri; ++t)
      for (int32_t k = 0; k < L; ++k) {
        const double a = A_elem[m->tri_glob[size_t(t)] * L + k];
        if (!(a > 0.0)) { st = fail(FO_EINVAL, "A_elem must be > 0"); break; }
        afac[size_t(t * L + k)] = std::pow(a, -1.0 / p->glen_n);
      }
    if (!st) st = upload(&m->d_A, afac.data(), afac.size());
    m->has_A_elem = true;
  }
  if (!st) st = build_patch_plan(m);
  if (!st) st = build_lateral(m, n_tri, tri);
  if (st) { fo_mesh_destroy(m); return st; }
  *out = m;
  return FO_OK;
}

}  // namespace
}  // namespace fo

using namespace fo;

extern "C" {

const char* fo_last_error(void) { return g_err.c_str(); }

fo_status fo_plan_check_host(int64_t n_vert, const double* xy, int64_t n_tri, const int32_t* tri, int32_t n_layers,
                             const int32_t* part_of_tri, int32_t my_part, int32_t n_parts, int64_t* stats) {
  if (!stats) return fail(FO_EINVAL, "stats is NULL");
  fo_params p;
  fo_params_default(&p);
  std::vector<double> H(size_t(n_vert), 1000.0), s(size_t(n_vert), 1000.0), beta(size_t(n_vert), 1.0);
  fo_mesh m = nullptr;
  fo_status st = mesh_create_impl(&p, n_vert, xy, n_tri, tri, n_layers, nullptr, H.data(), s.data(), nullptr,
                                  beta.data(), nullptr, part_of_tri, my_part, n_parts, 0, &m, true);
  if (st) return st;
  st = plan_check(m, stats);
  delete m;
  return st;
}

fo_status fo_mesh_set_temperature(fo_mesh m, const double* T_star, double A0, double Q) {
  if (!m) return fail(FO_EINVAL, "mesh is NULL");
  fo_status st = cuda_status(cudaSetDevice(m->device), "cudaSetDevice");
  if (st) return st;
  if (!T_star) {   // revert to the constant-A / A_elem path
    cudaFree(m->d_T);
    m->d_T = nullptr;
    return FO_OK;
  }
  // validate and build the new field first: a rejected call leaves the
  // previous temperature field (and the Arrhenius constants) in place
  if (!(A0 > 0.0)) return fail(FO_EINVAL, "A0 must be > 0");
  constexpr double kGasR = 8.314462618;   // J mol^-1 K^-1 (CODATA 2018)
  const int32_t L = m->L;
  std::vector<double> T(size_t(m->n_elem));
  for (int64_t t = 0; t < m->n_tri; ++t)
    for (int32_t k = 0; k < L; ++k) {
      const double v = T_star[m->tri_glob[size_t(t)] * L + k];
      if (!(v > 0.0)) return fail(FO_EINVAL, "T_star must be > 0 K");
      T[size_t(t * L + k)] = v;
    }
  double* d_new = nullptr;
  if (!T.empty()) {
    st = cuda_status(cudaMalloc(reinterpret_cast<void**>(&d_new), T.size() * sizeof(double)), "cudaMalloc");
    if (!st) st = cuda_status(cudaMemcpy(d_new, T.data(), T.size() * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy");
    if (st) { cudaFree(d_new); return st; }
  }
  cudaFree(m->d_T);
  m->d_T = d_new;
  m->A0fac = std::pow(A0, -1.0 / m->p.glen_n);
  m->QnR = Q / (m->p.glen_n * kGasR);
  return FO_OK;
}

fo_status fo_params_default(fo_params* p) {
  if (!p) return fail(FO_EINVAL, "params is NULL");
  p->rho = 910.0; p->g = 9.81; p->rho_w = 1028.0; p->glen_n = 3.0;
  p->eps_reg = 1e-10; p->A = 1e-16; p->H_min = 1.0;
  return FO_OK;
}

fo_status fo_mesh_create(const fo_params* p, int64_t n_vert, const double* xy, int64_t n_tri,
                         const int32_t* tri, int32_t n_layers, const double* sigma,
                         const double* thickness, const double* surface, const double* bed,
                         const double* beta, const double* A_elem, int device, fo_mesh* out) {
  return mesh_create_impl(p, n_vert, xy, n_tri, tri, n_layers, sigma, thickness, surface, bed,
                          beta, A_elem, nullptr, 0, 1, device, out);
}

fo_status fo_mesh_create_part(const fo_params* p, int64_t n_vert, const double* xy, int64_t n_tri,
                              const int32_t* tri, int32_t n_layers, const double* sigma,
                              const double* thickness, const double* surface, const double* bed,
                              const double* beta, const double* A_elem,
                              const int32_t* part_of_tri, int32_t my_part, int32_t n_parts,
                              int device, fo_mesh* out) {
  if (!part_of_tri) return fail(FO_EINVAL, "part_of_tri is NULL");
  return mesh_create_impl(p, n_vert, xy, n_tri, tri, n_layers, sigma, thickness, surface, bed,
                          beta, A_elem, part_of_tri, my_part, n_parts, device, out);
}

fo_status fo_partition(int64_t n_tri, int32_t n_parts, int32_t* part_of_tri) {
  if (n_parts < 1 || n_tri < 0 || (n_tri > 0 && !part_of_tri))
    return fail(FO_EINVAL, "bad partition arguments");
  for (int64_t t = 0; t < n_tri; ++t)
    part_of_tri[t] = int32_t((t * int64_t(n_parts)) / n_tri);
  return FO_OK;
}

fo_status fo_mesh_info(fo_mesh m, int64_t* n_nodes, int64_t* n_dofs, int64_t* n_elems,
                       int64_t* n_owned_dofs) {
  if (!m) return fail(FO_EINVAL, "mesh is NULL");
  if (n_nodes) *n_nodes = m->n_node;
  if (n_dofs) *n_dofs = m->n_dof;
  if (n_elems) *n_elems = m->n_elem;
  if (n_owned_dofs) *n_owned_dofs = m->n_owned_dof;
  return FO_OK;
}

fo_status fo_mesh_columns(fo_mesh m, int64_t* n_cols, int64_t* n_owned, int64_t* n_ghost,
                          int64_t* n_colonly, int64_t* glob) {
  if (!m) return fail(FO_EINVAL, "mesh is NULL");
  if (n_cols) *n_cols = m->n_col;
  if (n_owned) *n_owned = m->nA;
  if (n_ghost) *n_ghost = m->nB;
  if (n_colonly) *n_colonly = m->nC;
  if (glob) std::copy(m->glob.begin(), m->glob.end(), glob);
  return FO_OK;
}

fo_status fo_graph_host(int64_t n_vert, int64_t n_tri, const int32_t* tri, int32_t n_layers,
                        int64_t* row_ptr, int32_t* col_idx, int64_t* nnz) {
  if (n_layers < 1 || n_vert < 0 || n_tri < 0 || (n_tri > 0 && !tri))
    return fail(FO_EINVAL, "bad graph arguments");
  for (int64_t t = 0; t < 3 * n_tri; ++t)
    if (tri[t] < 0 || tri[t] >= n_vert) return fail(FO_EMESH, "vertex index out of range");
  Topo T;
  fo_status st = build_topology(n_vert, n_tri, tri, n_layers, nullptr, 0, T);
  if (st) return st;
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  int64_t z = 0;
  build_csr(T, n_layers, row_ptr ? &rp : nullptr, col_idx ? &ci : nullptr, &z);
  if (nnz) *nnz = z;
  if (row_ptr) std::copy(rp.begin(), rp.end(), row_ptr);
  if (col_idx) std::copy(ci.begin(), ci.end(), col_idx);
  return FO_OK;
}

fo_status fo_graph_build(fo_mesh m, fo_graph* out) {
  if (!m || !out) return fail(FO_EINVAL, "NULL argument");
  *out = nullptr;
  fo_status st = cuda_status(cudaSetDevice(m->device), "cudaSetDevice");
  if (st) return st;
  Topo T;   // view of the mesh topology
  T.glob = m->glob;
  T.nbr_ptr = m->nbr_ptr;
  T.nbr = m->nbr;
  T.colstart = m->colstart;
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  int64_t nnz = 0;
  build_csr(T, m->L, &rp, &ci, &nnz);
  fo_graph g = new fo_graph_s();
  g->mesh = m;
  g->n_rows = m->n_dof;
  g->nnz = nnz;
  st = upload(&g->d_row_ptr, rp.data(), rp.size());
  if (!st) st = upload(&g->d_col_idx, ci.data(), ci.size());
  if (st) { fo_graph_destroy(g); return st; }
  *out = g;
  return FO_OK;
}

fo_status fo_graph_info(fo_graph g, int64_t* n_rows, int64_t* nnz) {
  if (!g) return fail(FO_EINVAL, "graph is NULL");
  if (n_rows) *n_rows = g->n_rows;
  if (nnz) *nnz = g->nnz;
  return FO_OK;
}

fo_status fo_graph_arrays(fo_graph g, const int64_t** d_row_ptr, const int32_t** d_col_idx) {
  if (!g) return fail(FO_EINVAL, "graph is NULL");
  if (d_row_ptr) *d_row_ptr = g->d_row_ptr;
  if (d_col_idx) *d_col_idx = g->d_col_idx;
  return FO_OK;
}

fo_status fo_graph_to_host(fo_graph g, int64_t* row_ptr, int32_t* col_idx) {
  if (!g) return fail(FO_EINVAL, "graph is NULL");
  fo_status st = cuda_status(cudaSetDevice(g->mesh->device), "cudaSetDevice");
  if (st) return st;
  if (row_ptr && g->d_row_ptr)
    st = cuda_status(cudaMemcpy(row_ptr, g->d_row_ptr, sizeof(int64_t) * (g->n_rows + 1),
                                cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
  else if (row_ptr)
    row_ptr[0] = 0;
  if (!st && col_idx && g->nnz > 0)
    st = cuda_status(cudaMemcpy(col_idx, g->d_col_idx, sizeof(int32_t) * g->nnz,
                                cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
  return st;
}

fo_status fo_assemble_residual(fo_mesh m, const double* d_U, double* d_R, void* stream) {
  NvtxRange nvtx("fo_assemble_residual");
  if (!m) return fail(FO_EINVAL, "mesh is NULL");
  if (m->n_dof > 0 && (!d_U || !d_R)) return fail(FO_EINVAL, "NULL device buffer");
  return launch_residual(m, d_U, d_R, stream);
}

fo_status fo_assemble_jacobian(fo_mesh m, fo_graph g, const double* d_U, double* d_R,
                               double* d_vals, void* stream) {
  NvtxRange nvtx("fo_assemble_jacobian");
  if (!m || !g) return fail(FO_EINVAL, "mesh or graph is NULL");
  if (g->mesh != m) return fail(FO_ESTATE, "graph was built for another mesh");
  if (m->n_dof > 0 && (!d_U || !d_vals)) return fail(FO_EINVAL, "NULL device buffer");
  return launch_jacobian(m, d_U, d_R, d_vals, stream);
}

fo_status fo_assemble_jacobian_host(fo_mesh m, fo_graph g, const double* h_U, double* h_R,
                                    double* h_vals, void* stream) {
  NvtxRange nvtx("fo_assemble_jacobian_host");
  if (!m || !g) return fail(FO_EINVAL, "mesh or graph is NULL");
  if (g->mesh != m) return fail(FO_ESTATE, "graph was built for another mesh");
  if (m->n_dof > 0 && (!h_U || !h_vals)) return fail(FO_EINVAL, "NULL host buffer");
  fo_status st = cuda_status(cudaSetDevice(m->device), "cudaSetDevice");
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!m->d_stage_R && m->n_dof > 0) {   // keyed on the last allocation
    cudaFree(m->d_stage_U);
    m->d_stage_U = nullptr;
    st = cuda_status(cudaMalloc(&m->d_stage_U, sizeof(double) * m->n_dof), "cudaMalloc");
    if (!st) st = cuda_status(cudaMalloc(&m->d_stage_R, sizeof(double) * m->n_dof), "cudaMalloc");
    if (st) return st;
  }
  if (m->stage_vals_n < g->nnz) {
    cudaFree(m->d_stage_vals);
    m->d_stage_vals = nullptr;
    st = cuda_status(cudaMalloc(&m->d_stage_vals, sizeof(double) * g->nnz), "cudaMalloc");
    if (st) return st;
    m->stage_vals_n = g->nnz;
  }
  if (m->n_dof == 0) return FO_OK;
  st = cuda_status(cudaMemcpyAsync(m->d_stage_U, h_U, sizeof(double) * m->n_dof,
                                   cudaMemcpyHostToDevice, s), "cudaMemcpyAsync H2D");
  if (!st) st = launch_jacobian(m, m->d_stage_U, h_R ? m->d_stage_R : nullptr, m->d_stage_vals, stream);
  if (!st && h_R)
    st = cuda_status(cudaMemcpyAsync(h_R, m->d_stage_R, sizeof(double) * m->n_dof,
                                     cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync D2H");
  if (!st)
    st = cuda_status(cudaMemcpyAsync(h_vals, m->d_stage_vals, sizeof(double) * g->nnz,
                                     cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync D2H");
  if (!st) st = cuda_status(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  return st;
}

fo_status fo_set_lateral(fo_mesh m, int enable) {
  if (!m) return fail(FO_EINVAL, "mesh is NULL");
  if (enable && m->quad) return fail(FO_EINVAL, "the lateral term is defined on wedge faces only");
  if (enable && m->elem_type != FO_ELEM_WEDGE)
    return fail(FO_EINVAL, "the lateral term is defined on wedge faces (FO_ELEM_WEDGE only)");
  m->lateral = enable != 0;
  return FO_OK;
}

fo_status fo_set_element(fo_mesh m, fo_element type) {
  if (!m) return fail(FO_EINVAL, "mesh is NULL");
  if (m->quad) return fail(FO_EINVAL, "a quadrilateral mesh always uses hexahedra");
  if (type != FO_ELEM_WEDGE && type != FO_ELEM_TET3) return fail(FO_EINVAL, "unknown element type");
  if (type == FO_ELEM_TET3 && (m->lateral || (m->scatter != FO_SCATTER_OWNER && m->scatter != FO_SCATTER_OWNER_1WG)))
    return fail(FO_EINVAL, "FO_ELEM_TET3 needs the owner scatter and no lateral term");
  if (type == m->elem_type) return FO_OK;
  // The tetrahedral element runs with every triangle's corners in global-id
  // order (its split rule, reading L22, then has compile-time nodes); the
  // wedge needs the caller's CCW order back.  Either way the patch plan is
  // rebuilt for the new corner order.
  fo_status st = cuda_status(cudaSetDevice(m->device), "cudaSetDevice");
  if (st) return st;
  if (type == FO_ELEM_TET3) {
    m->tri_ccw = m->tri;
    m->trirec_ccw = m->trirec;
    for (int64_t t = 0; t < m->n_tri; ++t) {
      const TriRec o = m->trirec_ccw[size_t(t)];
      const int ord[3] = {o.pad[0] & 3, (o.pad[0] >> 2) & 3, (o.pad[0] >> 4) & 3};
      TriRec& r = m->trirec[size_t(t)];
      for (int k = 0; k < 3; ++k) {
        r.v[k] = o.v[ord[k]];
        m->tri[size_t(3 * t + k)] = m->tri_ccw[size_t(3 * t + ord[k])];
        for (int l = 0; l < 3; ++l) r.slot[3 * k + l] = o.slot[3 * ord[k] + ord[l]];
      }
      r.pad[0] = uint8_t(0 | (1 << 2) | (2 << 4));
    }
  } else {
    m->tri.swap(m->tri_ccw);
    m->trirec.swap(m->trirec_ccw);
    m->tri_ccw.clear();
    m->trirec_ccw.clear();
  }
  if (!m->trirec.empty())
    st = cuda_status(cudaMemcpy(m->d_tri, m->trirec.data(), m->trirec.size() * sizeof(TriRec), cudaMemcpyHostToDevice),
                     "cudaMemcpy H2D");
  free_patch_plan(m);
  if (!st) st = build_patch_plan(m);
  if (!st) m->elem_type = type;
  return st;
}

fo_status fo_set_scatter(fo_mesh m, fo_scatter s) {
  if (!m) return fail(FO_EINVAL, "mesh is NULL");
  if (s != FO_SCATTER_OWNER && s != FO_SCATTER_ATOMIC && s != FO_SCATTER_OWNER_WS && s != FO_SCATTER_OWNER_1WG)
    return fail(FO_EINVAL, "bad scatter");
  if (m->quad && s != FO_SCATTER_OWNER && s != FO_SCATTER_ATOMIC)
    return fail(FO_EINVAL, "hexahedra: FO_SCATTER_OWNER (patches) or FO_SCATTER_ATOMIC (coloured ablation)");
  if (s != FO_SCATTER_OWNER && s != FO_SCATTER_OWNER_1WG && m->elem_type != FO_ELEM_WEDGE)
    return fail(FO_EINVAL, "this scatter supports FO_ELEM_WEDGE only");
  m->scatter = s;
  return FO_OK;
}

fo_status fo_kernel_timing(fo_mesh m, int32_t enable) {
  if (!m) return fail(FO_EINVAL, "mesh is NULL");
  m->timing = enable != 0;
  return FO_OK;
}

fo_status fo_kernel_time_ms(fo_mesh m, double* total_ms, int32_t* n_launches) {
  if (!m || !total_ms) return fail(FO_EINVAL, "NULL argument");
  double tot = 0.0;
  fo_status st = FO_OK;
  for (auto& pr : m->timed) {
    cudaEvent_t a = static_cast<cudaEvent_t>(pr.first), b = static_cast<cudaEvent_t>(pr.second);
    float ms = 0.0f;
    if (!st) st = cuda_status(cudaEventSynchronize(b), "cudaEventSynchronize");
    if (!st) st = cuda_status(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
    tot += ms;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  if (n_launches) *n_launches = int32_t(m->timed.size());
  m->timed.clear();
  *total_ms = tot;
  return st;
}

fo_status fo_last_launch_count(fo_mesh m, int32_t* n) {
  if (!m || !n) return fail(FO_EINVAL, "NULL argument");
  *n = m->last_launches;
  return FO_OK;
}

void fo_mesh_destroy(fo_mesh m) {
  if (!m) return;
  cudaSetDevice(m->device);
  cudaFree(m->d_col);
  cudaFree(m->d_tri);
  cudaFree(m->d_sigma);
  cudaFree(m->d_A);
  cudaFree(m->d_T);
  cudaFree(m->d_lat_cols);
  cudaFree(m->d_lat_faces);
  cudaFree(m->d_lat_refs);
  cudaFree(m->d_quad);
  cudaFree(m->d_hex_ids);
  cudaFree(m->d_nbr_ptr);
  cudaFree(m->d_nbr);
  cudaFree(m->d_self_slot);
  cudaFree(m->d_line_fac);
  cudaFree(m->d_kry_work);
  free_patch_plan(m);
  cudaFree(m->d_stage_U);
  cudaFree(m->d_stage_R);
  cudaFree(m->d_stage_vals);
  cudaFree(m->d_scratch_R);
  for (auto& pr : m->timed) {
    cudaEventDestroy(static_cast<cudaEvent_t>(pr.first));
    cudaEventDestroy(static_cast<cudaEvent_t>(pr.second));
  }
  delete m;
}

void fo_graph_destroy(fo_graph g) {
  if (!g) return;
  cudaSetDevice(g->mesh->device);
  cudaFree(g->d_row_ptr);
  cudaFree(g->d_col_idx);
  delete g;
}

}  // extern "C"
