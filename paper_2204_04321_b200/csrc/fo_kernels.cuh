// fo_kernels.cuh -- shared device helpers of the assembly kernels: kernel
// parameters and the per-wedge gather (a2 of SURVEY.md 8(a)).
#pragma once
#include <cuda_runtime.h>

#include "fo_element.cuh"
#include "fo_internal.h"

namespace fo {

struct KParams {
  int64_t n_elem;     // local wedges
  int L;              // layers
  double rg;          // rho * g
  double eps;         // eps_reg
  double glen_n;      // n
  double Afac;        // A^(-1/n) when no per-wedge field
  int go;             // 1 (opaque to the compiler)
  // NEXT-f3: per-wedge T* -> A^(-1/n) = A0^(-1/n) exp(Q / (n R T*))
  const double* Tw;   // [n_elem] or nullptr
  double A0fac;       // A0^(-1/n)
  double QnR;         // Q / (n R)
};

inline KParams make_kparams(fo_mesh m) {
  KParams kp;
  kp.n_elem = m->n_elem;
  kp.L = m->L;
  kp.rg = m->p.rho * m->p.g;
  kp.eps = m->p.eps_reg;
  kp.glen_n = m->p.glen_n;
  kp.Afac = pow(m->p.A, -1.0 / m->p.glen_n);
  kp.go = 1;
  kp.Tw = m->d_T;
  kp.A0fac = m->A0fac;
  kp.QnR = m->QnR;
  return kp;
}

// A^(-1/n) of wedge (t, k): Arrhenius from T* (NEXT-f3), else the per-wedge
// field, else the scalar (fused into the viscosity step a5)
__device__ __forceinline__ double wedge_afac(const KParams& kp, const double* __restrict__ Aw,
                                             int64_t t, int k) {
  const int64_t w = t * kp.L + k;
  if (kp.Tw) return kp.A0fac * exp(kp.QnR / __ldg(kp.Tw + w));
  return Aw ? __ldg(Aw + w) : kp.Afac;
}

// Per-triangle geometry (layer independent): barycentric gradients, 2|T|,
// edges, the P1 surface gradient (reading L10), the column bases/thicknesses.
struct TriGeo {
  double a[3], b[3], D, e1x, e1y, e2x, e2y, sx, sy;
  double base[3], H[3], beta[3];
  int64_t cs[3];       // CSR value offset of each vertex column
  int nc[3];           // coupling-list length of each vertex column
};

__device__ __forceinline__ void load_tri_geo(const ColRec* __restrict__ col, const TriRec& tr,
                                             TriGeo& g) {
  double x[3], y[3], s[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const ColRec* c = col + tr.v[j];
    const double2 xy = __ldg(reinterpret_cast<const double2*>(c));
    const double2 bh = __ldg(reinterpret_cast<const double2*>(c) + 1);
    const double2 bc = __ldg(reinterpret_cast<const double2*>(c) + 2);
    x[j] = xy.x; y[j] = xy.y;
    g.base[j] = bh.x; g.H[j] = bh.y;
    s[j] = bh.x + bh.y;
    g.beta[j] = bc.x;
    const long long csn = __double_as_longlong(bc.y);
    g.cs[j] = csn >> 8;
    g.nc[j] = int(csn & 255);
  }
  g.e1x = x[1] - x[0]; g.e1y = y[1] - y[0];
  g.e2x = x[2] - x[0]; g.e2y = y[2] - y[0];
  g.D = g.e1x * g.e2y - g.e2x * g.e1y;
  const double iD = rcp_geo(g.D);
  g.a[0] = (g.e1y - g.e2y) * iD; g.a[1] = g.e2y * iD; g.a[2] = -g.e1y * iD;
  g.b[0] = (g.e2x - g.e1x) * iD; g.b[1] = -g.e2x * iD; g.b[2] = g.e1x * iD;
  g.sx = g.a[0] * s[0] + g.a[1] * s[1] + g.a[2] * s[2];
  g.sy = g.b[0] * s[0] + g.b[1] * s[1] + g.b[2] * s[2];
}

__device__ __forceinline__ TriRec load_tri(const TriRec* __restrict__ tris, int64_t t) {
  TriRec tr;
  const int2* p = reinterpret_cast<const int2*>(tris + t);
  int2 q0 = __ldg(p), q1 = __ldg(p + 1), q2 = __ldg(p + 2);
  int* o = reinterpret_cast<int*>(&tr);
  o[0] = q0.x; o[1] = q0.y; o[2] = q1.x; o[3] = q1.y; o[4] = q2.x; o[5] = q2.y;
  return tr;
}

// Fill the per-wedge input for layer k from the triangle geometry and U.
__device__ __forceinline__ void wedge_input(const TriGeo& g, const TriRec& tr,
                                            const double* __restrict__ sigma, double Afac,
                                            const double* __restrict__ U, int L, int k,
                                            WedgeIn& w, bool go = true) {
  const double sk = __ldg(sigma + k), sk1 = __ldg(sigma + k + 1);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    w.a[j] = g.a[j]; w.b[j] = g.b[j];
    w.zb[j] = fma(sk, g.H[j], g.base[j]);
    w.zt[j] = fma(sk1, g.H[j], g.base[j]);
    w.beta[j] = g.beta[j];
    const int64_t node = int64_t(tr.v[j]) * (L + 1) + k;
    const double2 ub = __ldg(reinterpret_cast<const double2*>(U) + node);
    const double2 ut = __ldg(reinterpret_cast<const double2*>(U) + node + 1);
    w.ub[j] = ub.x; w.vb[j] = ub.y; w.ut[j] = ut.x; w.vt[j] = ut.y;
  }
  w.D = g.D; w.e1x = g.e1x; w.e1y = g.e1y; w.e2x = g.e2x; w.e2y = g.e2y;
  w.sx = g.sx; w.sy = g.sy;
  w.Afac = Afac;
  w.basal = (k == 0);
  w.go = go;
}

// wedge_input with the velocities already in registers (bottom / top level)
__device__ __forceinline__ void wedge_input_u(const TriGeo& g, const double* __restrict__ sigma, double Afac,
                                              const double2 (&ub)[3], const double2 (&ut)[3], int k, WedgeIn& w,
                                              bool go = true) {
  const double sk = __ldg(sigma + k), sk1 = __ldg(sigma + k + 1);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    w.a[j] = g.a[j]; w.b[j] = g.b[j];
    w.zb[j] = fma(sk, g.H[j], g.base[j]);
    w.zt[j] = fma(sk1, g.H[j], g.base[j]);
    w.beta[j] = g.beta[j];
    w.ub[j] = ub[j].x; w.vb[j] = ub[j].y; w.ut[j] = ut[j].x; w.vt[j] = ut[j].y;
  }
  w.D = g.D; w.e1x = g.e1x; w.e1y = g.e1y; w.e2x = g.e2x; w.e2y = g.e2y;
  w.sx = g.sx; w.sy = g.sy;
  w.Afac = Afac;
  w.basal = (k == 0);
  w.go = go;
}

// convenience for the one-thread-per-wedge kernels
__device__ __forceinline__ void load_wedge(const ColRec* __restrict__ col,
                                           const TriRec* __restrict__ tris,
                                           const double* __restrict__ sigma,
                                           const double* __restrict__ Aw, const KParams& kp,
                                           const double* __restrict__ U, int64_t t, int k,
                                           WedgeIn& w, TriRec& tr, ColRec* cr) {
  tr = load_tri(tris, t);
  TriGeo g;
  load_tri_geo(col, tr, g);
#pragma unroll
  for (int j = 0; j < 3; ++j) cr[j].cs_n = (g.cs[j] << 8) | g.nc[j];
  const double Afac = wedge_afac(kp, Aw, t, k);
  wedge_input(g, tr, sigma, Afac, U, kp.L, k, w);
}

fo_status launch_owner(fo_mesh m, const double* d_U, double* d_R, double* d_vals,
                       cudaStream_t s);

}  // namespace fo
