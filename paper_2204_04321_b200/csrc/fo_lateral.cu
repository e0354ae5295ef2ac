// fo_lateral.cu -- NEXT-f1: the lateral margin term of the residual
// (ocean back-pressure; readings L12, L20).
//
// On a lateral face Gamma_l (a footprint boundary edge extruded through one
// layer) the boundary condition reads, by reading L12,
//     2 mu eps_a . n = P(z) n_a,   P(z) = rho g (s - z) - rho_w g max(-z, 0),
// so the weak form gains  R_{a,i} -= int_{face} P(z) n_a phi_i dGamma.  The
// term does not depend on U: the Jacobian is unchanged.
//
// Quadrature (reading L20): 2-point Gauss along the edge; in zeta 2-point
// Gauss on [-1, 1], or on each side of the sea-level crossing z = 0.
//
// Kernel: one thread per (margin column, level).  It walks the column's margin
// faces in a fixed order, integrates P against its own node's basis function
// on the faces below and above the level, and adds the sum to its two
// residual entries: one writer per entry, so the result is deterministic.  It
// runs after the assembly kernel(s), on the same stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <utility>
#include <vector>

#include "fo_internal.h"

namespace fo {

namespace {

// integral of P phi over one face: edge c0 -> c1 (length len), node heights
// zb/zt (bottom/top level of the layer) and surface S of both columns; phi the
// basis function of the node of column c_role on the top (top = 1) or bottom
// level of the layer
__device__ __forceinline__ double face_integral(double zb0, double zt0, double zb1, double zt1,
                                                double S0, double S1, double len, int role, int top,
                                                double rg, double rwg) {
  constexpr double kG = 0.57735026918962576451;   // 1/sqrt(3)
  double I = 0.0;
#pragma unroll
  for (int sp = 0; sp < 2; ++sp) {
    const double sc = sp == 0 ? 0.5 - 0.5 * kG : 0.5 + 0.5 * kG;
    const double zb = (1.0 - sc) * zb0 + sc * zb1;
    const double zt = (1.0 - sc) * zt0 + sc * zt1;
    const double S = (1.0 - sc) * S0 + sc * S1;
    const double ps = role == 0 ? 1.0 - sc : sc;
    double cut0 = -1.0, cut1 = 1.0, cut2 = 1.0;
    int nint = 1;
    if (zb < 0.0 && zt > 0.0) {
      cut1 = -1.0 + 2.0 * (0.0 - zb) / (zt - zb);
      nint = 2;
    }
    for (int iv = 0; iv < nint; ++iv) {
      const double lo = iv == 0 ? cut0 : cut1, hi = iv == 0 ? cut1 : cut2;
#pragma unroll
      for (int zq = 0; zq < 2; ++zq) {
        const double zeta = 0.5 * (lo + hi) + (zq == 0 ? -0.5 : 0.5) * (hi - lo) * kG;
        const double wz = 0.5 * (hi - lo);
        const double z = zb + 0.5 * (1.0 + zeta) * (zt - zb);
        const double P = rg * (S - z) - rwg * fmax(-z, 0.0);
        const double W = len * 0.5 * wz * 0.5 * (zt - zb);
        const double phi = ps * (top ? 0.5 * (1.0 + zeta) : 0.5 * (1.0 - zeta));
        I = fma(W * P, phi, I);
      }
    }
  }
  return I;
}

__global__ void lateral_kernel(const ColRec* __restrict__ col, const double* __restrict__ sigma,
                               const int4* __restrict__ lcols, int n_lcols,
                               const int2* __restrict__ faces, const int32_t* __restrict__ refs,
                               int L, double rg, double rwg, double* __restrict__ R) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_lcols * (L + 1)) return;
  const int lc = i / (L + 1), k = i - lc * (L + 1);
  const int4 lr = __ldg(lcols + lc);   // (column, first ref, ref count, 0)
  double ru = 0.0, rv = 0.0;
  for (int e = lr.y; e < lr.y + lr.z; ++e) {
    const int ref = __ldg(refs + e);
    const int2 f = __ldg(faces + (ref >> 1));
    const int role = ref & 1;
    const ColRec ca = col[f.x], cb = col[f.y];
    const double dx = cb.x - ca.x, dy = cb.y - ca.y;
    const double len = sqrt(dx * dx + dy * dy);
    const double nx = dy / len, ny = -dx / len;   // outward (CCW triangle on the left)
    double I = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {   // h = 0: layer below the level (node on top), 1: above
      const int layer = h == 0 ? k - 1 : k;
      if (layer < 0 || layer >= L) continue;
      const double s0 = __ldg(sigma + layer), s1 = __ldg(sigma + layer + 1);
      I += face_integral(fma(s0, ca.H, ca.base), fma(s1, ca.H, ca.base), fma(s0, cb.H, cb.base),
                         fma(s1, cb.H, cb.base), ca.base + ca.H, cb.base + cb.H, len, role,
                         h == 0 ? 1 : 0, rg, rwg);
    }
    ru = fma(-nx, I, ru);
    rv = fma(-ny, I, rv);
  }
  double2* r = reinterpret_cast<double2*>(R) + int64_t(lr.x) * (L + 1) + k;
  const double2 old = *r;
  *r = make_double2(old.x + ru, old.y + rv);
}

}  // namespace

// Host: margin faces of the local mesh = edges of local triangles that belong
// to exactly one triangle of the GLOBAL footprint (tri[n_tri][3]); per margin
// column the list of its faces with its role (0: first vertex of the CCW edge).
fo_status build_lateral(fo_mesh m, int64_t n_tri_global, const int32_t* tri_global) {
  std::vector<uint64_t> keys;
  keys.reserve(size_t(3 * n_tri_global));
  auto key = [](int64_t a, int64_t b) {
    return (uint64_t(std::min(a, b)) << 32) | uint64_t(std::max(a, b));
  };
  for (int64_t t = 0; t < n_tri_global; ++t)
    for (int j = 0; j < 3; ++j) keys.push_back(key(tri_global[3 * t + j], tri_global[3 * t + (j + 1) % 3]));
  std::sort(keys.begin(), keys.end());
  auto boundary = [&](uint64_t k) {
    auto r = std::equal_range(keys.begin(), keys.end(), k);
    return r.second - r.first == 1;
  };
  std::vector<int2> faces;
  std::vector<std::pair<int32_t, int32_t>> inc;   // (local column, face*2 + role)
  for (int64_t t = 0; t < m->n_tri; ++t) {
    const int64_t g = m->tri_glob[size_t(t)];
    for (int j = 0; j < 3; ++j) {
      const int j1 = (j + 1) % 3;
      if (!boundary(key(tri_global[3 * g + j], tri_global[3 * g + j1]))) continue;
      const int32_t f = int32_t(faces.size());
      faces.push_back(make_int2(m->tri[size_t(3 * t + j)], m->tri[size_t(3 * t + j1)]));
      inc.push_back({m->tri[size_t(3 * t + j)], 2 * f});
      inc.push_back({m->tri[size_t(3 * t + j1)], 2 * f + 1});
    }
  }
  std::sort(inc.begin(), inc.end());
  std::vector<int4> lcols;
  std::vector<int32_t> refs;
  for (size_t i = 0; i < inc.size();) {
    size_t e = i;
    while (e < inc.size() && inc[e].first == inc[i].first) ++e;
    lcols.push_back(make_int4(inc[i].first, int32_t(refs.size()), int32_t(e - i), 0));
    for (size_t q = i; q < e; ++q) refs.push_back(inc[q].second);
    i = e;
  }
  m->n_lat_cols = int32_t(lcols.size());
  m->n_lat_faces = int32_t(faces.size());
  if (lcols.empty()) return FO_OK;
  auto up = [](void** dst, const void* src, size_t bytes) {
    fo_status st = cuda_status(cudaMalloc(dst, bytes), "cudaMalloc");
    if (!st) st = cuda_status(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    return st;
  };
  fo_status st = up(reinterpret_cast<void**>(&m->d_lat_cols), lcols.data(), lcols.size() * sizeof(int4));
  if (!st) st = up(reinterpret_cast<void**>(&m->d_lat_faces), faces.data(), faces.size() * sizeof(int2));
  if (!st) st = up(reinterpret_cast<void**>(&m->d_lat_refs), refs.data(), refs.size() * sizeof(int32_t));
  return st;
}

fo_status launch_lateral(fo_mesh m, double* d_R, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!m->lateral || !d_R || m->n_lat_cols == 0) return FO_OK;
  const int n = m->n_lat_cols * (m->L + 1);
  lateral_kernel<<<(n + 127) / 128, 128, 0, s>>>(m->d_col, m->d_sigma, m->d_lat_cols, m->n_lat_cols,
                                                  m->d_lat_faces, m->d_lat_refs, m->L, m->p.rho * m->p.g,
                                                  m->p.rho_w * m->p.g, d_R);
  fo_status st = cuda_status(cudaGetLastError(), "lateral_kernel launch");
  if (!st) m->last_launches += 1;
  return st;
}

}  // namespace fo
