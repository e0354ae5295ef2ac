// fo_hex.cu -- NEXT-f4: quadrilateral footprints with 8-node trilinear
// hexahedra (the Antarctic hex meshes; reading L23).
//
// Same weak form, residual and exact Jacobian as the wedge path,
// per hexahedron: 2 x 2 x 2 Gauss points, trilinear basis N_i = Q_c(xi, eta)
// f_l(zeta) with the physical gradients from the generic 3x3 inverse of the
// isoparametric map (the footprint map is bilinear, so nothing separates as for
// the wedge), J = sum_q w_q [2 mu_q H_q - d_q g_q g_q^T] accumulated in the
// thread's registers in three passes (bottom-bottom with the residual, bottom-
// top, top-top) that re-evaluate the point data.
// Basal term: 2 x 2 Gauss on the bilinear bottom face, true 3D area element.
//
// R + J (default): KH-patch, the wedge path's owner-computes patch scheme on
// quad patches (kh_patch_kernel below).
// The residual alone and the FO_SCATTER_ATOMIC ablation: COLOURED.  Quads are
// greedily coloured so that no two quads of a colour share a corner; colour c,
// layer parity l launches touch disjoint node sets, so each thread adds its
// block into the (zeroed) CSR values and residual with plain read-modify-write,
// in a fixed launch order: deterministic.  CSR positions come from the column
// structure (QuadRec slots), col_idx is not read.  The graph, SpMV and line
// preconditioner of the wedge path apply unchanged (they only see columns and
// coupling lists).  Single-domain meshes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "fo_internal.h"
#include "fo_kernels.cuh"
#include "fo_patch.cuh"
#include "fo_tmem.cuh"

namespace fo {

namespace {

constexpr int kHexThreads = 128;


// Geometry and velocities of one hexahedron (registers)
struct HexIn {
  double X[4], Y[4], Zb[4], Zt[4], S[4], Uu[8], Uv[8], B[4];
  double Afac;
};

// basis, physical gradients G and weight W = det J at Gauss point qp, using
// the column structure of the extruded hexahedron: x, y depend on (xi, eta)
// only, so J = [[A, 0], [c^T, z_zeta]] with A the 2 x 2 footprint Jacobian and
// c = (z_xi, z_eta); det J = det A z_zeta and, with N_(j,l) = Q_j(xi, eta)
// f_l(zeta), f_l' = s_l = -1/2, +1/2:
//   grad_xy N_(j,l) = f_l P_j + s_l Q_j K,  P_j = A^-T grad_(xi,eta) Q_j,
//   K = -A^-T c / z_zeta,   d/dz N_(j,l) = s_l Q_j / z_zeta
// (exactly the isoparametric gradient; no general 3 x 3 inverse)
// pk (if not null): the point's column-structure data for the TMEM cache of
// KH-patch: P_j (x, y) for j = 0..3, 1 / z_zeta, K (x, y)
__device__ __forceinline__ double hex_point(const HexIn& h, int qp, double N[8], double G[8][3],
                                            double* pk = nullptr) {
  constexpr double gz = 0.57735026918962576451;
  const double xi = (qp & 1) ? gz : -gz, eta = (qp & 2) ? gz : -gz, zeta = (qp & 4) ? gz : -gz;
  const double cxi[4] = {-1.0, 1.0, 1.0, -1.0}, ceta[4] = {-1.0, -1.0, 1.0, 1.0};
  const double f0 = 0.5 * (1.0 - zeta), f1 = 0.5 * (1.0 + zeta);
  double Q[4], Qx[4], Qe[4];
  double xx = 0, xe = 0, yx = 0, ye = 0, zx = 0, ze = 0, zz = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double ax = 1.0 + cxi[j] * xi, ae = 1.0 + ceta[j] * eta;
    Q[j] = 0.25 * ax * ae;
    Qx[j] = 0.25 * cxi[j] * ae;
    Qe[j] = 0.25 * ceta[j] * ax;
    const double zm = fma(f0, h.Zb[j], f1 * h.Zt[j]);
    xx = fma(h.X[j], Qx[j], xx); xe = fma(h.X[j], Qe[j], xe);
    yx = fma(h.Y[j], Qx[j], yx); ye = fma(h.Y[j], Qe[j], ye);
    zx = fma(zm, Qx[j], zx); ze = fma(zm, Qe[j], ze);
    zz = fma(Q[j], 0.5 * (h.Zt[j] - h.Zb[j]), zz);
  }
  const double detA = xx * ye - xe * yx;
  const double ia = 1.0 / detA, iz = 1.0 / zz;
  // A^-T = ia [[ye, -yx], [-xe, xx]]
  const double kx = -(ye * zx - yx * ze) * ia * iz, ky = -(xx * ze - xe * zx) * ia * iz;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double px = (ye * Qx[j] - yx * Qe[j]) * ia, py = (xx * Qe[j] - xe * Qx[j]) * ia;
    const double hq = 0.5 * Q[j];
    N[j] = Q[j] * f0;
    N[j + 4] = Q[j] * f1;
    G[j][0] = fma(f0, px, -hq * kx);
    G[j][1] = fma(f0, py, -hq * ky);
    G[j][2] = -hq * iz;
    G[j + 4][0] = fma(f1, px, hq * kx);
    G[j + 4][1] = fma(f1, py, hq * ky);
    G[j + 4][2] = hq * iz;
    if (pk) { pk[2 * j] = px; pk[2 * j + 1] = py; }
  }
  if (pk) { pk[8] = iz; pk[9] = kx; pk[10] = ky; }
  return detA * zz;   // Gauss weights 1
}

// KH-patch TMEM row of an element thread (doubles take 2 columns): per point
// qp the 7-double record [e1x, exy, exz, e2y, eyz, c, d], K (x, y) and
// c / (2 z_zeta^2) at 20 qp; per footprint point m = qp & 3 (P_j and
// 1 / z_zeta depend on (xi, eta) only) P_j (x, y), j = 0..3, and 1 / z_zeta at
// kHexTmGeo + 18 m; the vertical-derivative sums T (hex_zz) at kHexTmT
constexpr uint32_t kHexTmRec = 20;
constexpr uint32_t kHexTmGeo = 160;
constexpr uint32_t kHexTmT = 232;
constexpr uint32_t kHexTmCols = 256;   // allocation per CTA (252 used; 2 CTAs per SM)

// passes 2 and 3: the gradients of point qp rebuilt from the cache,
//   grad N_(j,0) = f_0 (P_j, 0) - Q_j / 2 (K, 1 / z_zeta),
//   grad N_(j,1) = f_1 (P_j, 0) + Q_j / 2 (K, 1 / z_zeta)
// (hex_point's formula), and the point's record
__device__ __forceinline__ void hex_grad_tm(uint32_t tm, int qp, double G[8][3], double rec[7]) {
  constexpr double gz = 0.57735026918962576451;
  const double xi = (qp & 1) ? gz : -gz, eta = (qp & 2) ? gz : -gz, zeta = (qp & 4) ? gz : -gz;
  const double cxi[4] = {-1.0, 1.0, 1.0, -1.0}, ceta[4] = {-1.0, -1.0, 1.0, 1.0};
  const double f0 = 0.5 * (1.0 - zeta), f1 = 0.5 * (1.0 + zeta);
  double rk[9], pz[9];
  tmem::ld<9>(tm + kHexTmRec * qp, rk);
  tmem::ld<9>(tm + kHexTmGeo + 18 * (qp & 3), pz);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double hq = 0.125 * (1.0 + cxi[j] * xi) * (1.0 + ceta[j] * eta);
    const double hx = hq * rk[7], hy = hq * rk[8], hz = hq * pz[8];
    G[j][0] = fma(f0, pz[2 * j], -hx);
    G[j][1] = fma(f0, pz[2 * j + 1], -hy);
    G[j][2] = -hz;
    G[j + 4][0] = fma(f1, pz[2 * j], hx);
    G[j + 4][1] = fma(f1, pz[2 * j + 1], hy);
    G[j + 4][2] = hz;
  }
#pragma unroll
  for (int i = 0; i < 7; ++i) rec[i] = rk[i];
}

// viscosity factors and the strain-rate gradients g_{a,i} = eps_a . grad phi_i
template <bool N3>
__device__ __forceinline__ void hex_visc(const HexIn& h, const double G[8][3], double W, const KParams& kp,
                                         double g[16], double& c, double& d) {
  double ux = 0, uy = 0, uz = 0, vx = 0, vy = 0, vz = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    ux = fma(h.Uu[i], G[i][0], ux); uy = fma(h.Uu[i], G[i][1], uy); uz = fma(h.Uu[i], G[i][2], uz);
    vx = fma(h.Uv[i], G[i][0], vx); vy = fma(h.Uv[i], G[i][1], vy); vz = fma(h.Uv[i], G[i][2], vz);
  }
  const double exy = 0.5 * (uy + vx), exz = 0.5 * uz, eyz = 0.5 * vz;
  const double qq = fma(ux, ux, fma(vy, vy, fma(ux, vy, fma(exy, exy, fma(exz, exz, eyz * eyz)))));
  const double qe = qq + kp.eps;
  if (N3) {
    const double y = rcbrt_n3(qe);
    c = W * h.Afac * y;
    d = c * (y * y * y) * (1.0 / 3.0);
  } else {
    c = W * h.Afac * pow(qe, (1.0 - kp.glen_n) / (2.0 * kp.glen_n));
    d = c * ((kp.glen_n - 1.0) / (2.0 * kp.glen_n)) / qe;
  }
  const double e1x = 2.0 * ux + vy, e2y = ux + 2.0 * vy;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    g[2 * i] = fma(e1x, G[i][0], fma(exy, G[i][1], exz * G[i][2]));
    g[2 * i + 1] = fma(exy, G[i][0], fma(e2y, G[i][1], eyz * G[i][2]));
  }
}

// basal Robin term on the bilinear bottom face (readings L6-L8):
// 2 x 2 Gauss points with the true 3D area element; adds into the bottom
// residual r[0..8) and, NEED_J, the (bottom, bottom) block bb (packed p <= p2)
template <bool NEED_J>
__device__ __forceinline__ void hex_basal(const HexIn& h, double (&r)[16], double (&bb)[36]) {
  constexpr double gz = 0.57735026918962576451;
  const double cxi[4] = {-1.0, 1.0, 1.0, -1.0}, ceta[4] = {-1.0, -1.0, 1.0, 1.0};
#pragma unroll
  for (int qp = 0; qp < 4; ++qp) {
    const double xi = (qp & 1) ? gz : -gz, eta = (qp & 2) ? gz : -gz;
    double Q[4], tx0 = 0, tx1 = 0, tx2 = 0, ty0 = 0, ty1 = 0, ty2 = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      Q[j] = 0.25 * (1.0 + cxi[j] * xi) * (1.0 + ceta[j] * eta);
      const double dxi = 0.25 * cxi[j] * (1.0 + ceta[j] * eta), deta = 0.25 * ceta[j] * (1.0 + cxi[j] * xi);
      tx0 = fma(dxi, h.X[j], tx0); tx1 = fma(dxi, h.Y[j], tx1); tx2 = fma(dxi, h.Zb[j], tx2);
      ty0 = fma(deta, h.X[j], ty0); ty1 = fma(deta, h.Y[j], ty1); ty2 = fma(deta, h.Zb[j], ty2);
    }
    const double cx = tx1 * ty2 - tx2 * ty1, cy = tx2 * ty0 - tx0 * ty2, cz = tx0 * ty1 - tx1 * ty0;
    const double w = sqrt(cx * cx + cy * cy + cz * cz);
    const double bq = w * (Q[0] * h.B[0] + Q[1] * h.B[1] + Q[2] * h.B[2] + Q[3] * h.B[3]);
    const double u = Q[0] * h.Uu[0] + Q[1] * h.Uu[1] + Q[2] * h.Uu[2] + Q[3] * h.Uu[3];
    const double v = Q[0] * h.Uv[0] + Q[1] * h.Uv[1] + Q[2] * h.Uv[2] + Q[3] * h.Uv[3];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      r[2 * j] += bq * Q[j] * u;
      r[2 * j + 1] += bq * Q[j] * v;
    }
    if (NEED_J) {
      int e = 0;
#pragma unroll
      for (int p = 0; p < 8; ++p)
#pragma unroll
        for (int p2 = p; p2 < 8; ++p2) {
          if ((p & 1) == (p2 & 1)) bb[e] += bq * Q[p >> 1] * Q[p2 >> 1];
          ++e;
        }
    }
  }
}

// the point's strain-rate vectors and viscosity factors as a 7-double record
// [e1x, exy, exz, e2y, eyz, c, d] (KH-patch keeps it in TMEM for passes 2, 3)
template <bool N3>
__device__ __forceinline__ void hex_visc_rec(const HexIn& h, const double G[8][3], double W, const KParams& kp,
                                             double g[16], double& c, double& d, double rec[7]) {
  double ux = 0, uy = 0, uz = 0, vx = 0, vy = 0, vz = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    ux = fma(h.Uu[i], G[i][0], ux); uy = fma(h.Uu[i], G[i][1], uy); uz = fma(h.Uu[i], G[i][2], uz);
    vx = fma(h.Uv[i], G[i][0], vx); vy = fma(h.Uv[i], G[i][1], vy); vz = fma(h.Uv[i], G[i][2], vz);
  }
  const double exy = 0.5 * (uy + vx), exz = 0.5 * uz, eyz = 0.5 * vz;
  const double qq = fma(ux, ux, fma(vy, vy, fma(ux, vy, fma(exy, exy, fma(exz, exz, eyz * eyz)))));
  const double qe = qq + kp.eps;
  if (N3) {
    const double y = rcbrt_n3(qe);
    c = W * h.Afac * y;
    d = c * (y * y * y) * (1.0 / 3.0);
  } else {
    c = W * h.Afac * pow(qe, (1.0 - kp.glen_n) / (2.0 * kp.glen_n));
    d = c * ((kp.glen_n - 1.0) / (2.0 * kp.glen_n)) / qe;
  }
  const double e1x = 2.0 * ux + vy, e2y = ux + 2.0 * vy;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    g[2 * i] = fma(e1x, G[i][0], fma(exy, G[i][1], exz * G[i][2]));
    g[2 * i + 1] = fma(exy, G[i][0], fma(e2y, G[i][1], eyz * G[i][2]));
  }
  rec[0] = e1x; rec[1] = exy; rec[2] = exz; rec[3] = e2y; rec[4] = eyz; rec[5] = c; rec[6] = d;
}
// g, c, d from a stored record and the point's gradients
__device__ __forceinline__ void hex_g_rec(const double G[8][3], const double rec[7], double g[16], double& c,
                                          double& d) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    g[2 * i] = fma(rec[0], G[i][0], fma(rec[1], G[i][1], rec[2] * G[i][2]));
    g[2 * i + 1] = fma(rec[1], G[i][0], fma(rec[3], G[i][1], rec[4] * G[i][2]));
  }
  c = rec[5];
  d = rec[6];
}

// J entry (row dof p, column dof p2) at one point: c H - d g g^T
__device__ __forceinline__ double hex_jentry(const double G[8][3], const double g[16], double c, double d, int p,
                                             int p2) {
  const int i = p >> 1, a = p & 1, i2 = p2 >> 1, b = p2 & 1;
  const double xx = G[i][0] * G[i2][0], yy = G[i][1] * G[i2][1], zz = G[i][2] * G[i2][2];
  const double xy = G[i][0] * G[i2][1], yx = G[i][1] * G[i2][0];
  double hh;
  if (a == 0 && b == 0) hh = fma(2.0, xx, 0.5 * (yy + zz));
  else if (a == 1 && b == 1) hh = fma(2.0, yy, 0.5 * (xx + zz));
  else if (a == 0) hh = fma(0.5, yx, xy);
  else hh = fma(0.5, xy, yx);
  return fma(c, hh, -d * g[p] * g[p2]);
}

// position of the (column comps 0, 1) pair of row (node i, comp a) at column node i2
__device__ __forceinline__ double2* hex_ptr(double* __restrict__ vals, const QuadRec& qr, const int64_t cs[4],
                                            const int nc[4], int L, int k, int i, int a, int i2) {
  const int j = i & 3, ki = k + (i >> 2), j2 = i2 & 3, ki2 = k + (i2 >> 2);
  const int m = (ki == 0 || ki == L) ? 2 : 3;
  const int P = ki == 0 ? 0 : 3 * ki - 1;
  const int kmin = ki == 0 ? 0 : ki - 1;
  return reinterpret_cast<double2*>(vals + cs[j] + int64_t(4 * nc[j]) * P + int64_t(a) * 2 * nc[j] * m +
                                    int(qr.slot[4 * j + j2]) * 2 * m + 2 * (ki2 - kmin));
}

// read-modify-write of N double2 targets with every load issued before the
// first store: the targets are distinct (colouring), but the compiler cannot
// prove it, and one RMW at a time waits a DRAM latency per target.
// f(n, p, v0, v1) names target n and the values to add.
constexpr int kRmw = 8;   // block RMWs in flight per thread (4 / 16: 19.5 / 18.9 ms vs 18.5)

template <int N, class F>
__device__ __forceinline__ void rmw_batch(F f) {
  double2* p[N];
  double v0[N], v1[N];
  double2 o[N];
#pragma unroll
  for (int n = 0; n < N; ++n) f(n, p[n], v0[n], v1[n]);
#pragma unroll
  for (int n = 0; n < N; ++n) o[n] = *p[n];
#pragma unroll
  for (int n = 0; n < N; ++n) {
    *p[n] = make_double2(o[n].x + v0[n], o[n].y + v1[n]);
  }
}

// One thread per hexahedron; the 16 x 16 block is accumulated in registers in
// three passes over the 8 points -- (bottom, bottom) with the residual and the
// basal term, (bottom, top), (top, top) -- re-evaluating the point data in
// each pass rather than keeping 136 accumulators live; after each pass the
// block is added into the CSR values (both orientations, J symmetric), eight
// read-modify-writes in flight at a time (rmw_batch).
template <bool NEED_J, bool N3>
__global__ void __launch_bounds__(kHexThreads)
hex_kernel(const ColRec* __restrict__ col, const QuadRec* __restrict__ quads, const int32_t* __restrict__ ids,
           int n_ids, int kpar, const double* __restrict__ sigma, const double* __restrict__ Aw, KParams kp,
           const double* __restrict__ U, double* __restrict__ R, double* __restrict__ vals) {
  const int L = kp.L;
  const int nk = (L - kpar + 1) / 2;   // layers k = kpar, kpar + 2, ...
  const int64_t item = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (item >= int64_t(n_ids) * nk) return;
  const int qi = __ldg(ids + item / nk);
  const int k = kpar + 2 * int(item % nk);
  const QuadRec qr = quads[qi];
  HexIn h;
  int64_t cs[4];
  int nc[4];
  const double s0 = __ldg(sigma + k), s1 = __ldg(sigma + k + 1);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const ColRec c = col[qr.v[j]];
    cs[j] = c.cs_n >> 8;
    nc[j] = int(c.cs_n & 255);
    h.X[j] = c.x;
    h.Y[j] = c.y;
    h.Zb[j] = fma(s0, c.H, c.base);
    h.Zt[j] = fma(s1, c.H, c.base);
    h.S[j] = c.base + c.H;
    h.B[j] = c.beta;
    const int64_t node = int64_t(qr.v[j]) * (L + 1) + k;
    const double2 ub = __ldg(reinterpret_cast<const double2*>(U) + node);
    const double2 ut = __ldg(reinterpret_cast<const double2*>(U) + node + 1);
    h.Uu[j] = ub.x; h.Uv[j] = ub.y; h.Uu[j + 4] = ut.x; h.Uv[j + 4] = ut.y;
  }
  h.Afac = wedge_afac(kp, Aw, qi, k);
  // ---- pass 1: residual, (bottom, bottom) block, basal term
  double r[16], bb[36];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 36; ++i) bb[i] = 0.0;
#pragma unroll 1
  for (int qp = 0; qp < 8; ++qp) {
    double N[8], G[8][3], g[16], c, d;
    const double W = hex_point(h, qp, N, G);
    hex_visc<N3>(h, G, W, kp, g, c, d);
    double sx = 0, sy = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { sx = fma(h.S[i & 3], G[i][0], sx); sy = fma(h.S[i & 3], G[i][1], sy); }
    const double bw = W * kp.rg;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      r[2 * i] += fma(c, g[2 * i], bw * sx * N[i]);
      r[2 * i + 1] += fma(c, g[2 * i + 1], bw * sy * N[i]);
    }
    if (NEED_J) {
      int e = 0;
#pragma unroll
      for (int p = 0; p < 8; ++p)
#pragma unroll
        for (int p2 = p; p2 < 8; ++p2) bb[e++] += hex_jentry(G, g, c, d, p, p2);
    }
  }
  if (k == 0) hex_basal<NEED_J>(h, r, bb);
  rmw_batch<8>([&](int i, double2*& p, double& v0, double& v1) {
    p = reinterpret_cast<double2*>(R) + int64_t(qr.v[i & 3]) * (L + 1) + k + (i >> 2);
    v0 = r[2 * i];
    v1 = r[2 * i + 1];
  });
  if (!NEED_J) return;
  // (bottom, bottom): rows of bottom node i, columns of bottom node i2
  auto sym = [](const double* blk, int p, int p2) {
    const int lo = p < p2 ? p : p2, hi = p < p2 ? p2 : p;
    return blk[lo * 8 - (lo * (lo - 1)) / 2 + (hi - lo)];
  };
#pragma unroll
  for (int c0 = 0; c0 < 32; c0 += kRmw)
    rmw_batch<kRmw>([&](int n, double2*& p, double& v0, double& v1) {
      const int e = c0 + n, i = e >> 3, i2 = (e >> 1) & 3, a = e & 1;
      p = hex_ptr(vals, qr, cs, nc, L, k, i, a, i2);
      v0 = sym(bb, 2 * i + a, 2 * i2);
      v1 = sym(bb, 2 * i + a, 2 * i2 + 1);
    });
  // ---- pass 2: (bottom, top) block; written for both orientations
  {
    double bt[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) bt[i] = 0.0;
#pragma unroll 1
    for (int qp = 0; qp < 8; ++qp) {
      double N[8], G[8][3], g[16], c, d;
      const double W = hex_point(h, qp, N, G);
      hex_visc<N3>(h, G, W, kp, g, c, d);
#pragma unroll
      for (int p = 0; p < 8; ++p)
#pragma unroll
        for (int p2 = 0; p2 < 8; ++p2) bt[8 * p + p2] += hex_jentry(G, g, c, d, p, 8 + p2);
    }
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += kRmw)
      rmw_batch<kRmw>([&](int n, double2*& p, double& v0, double& v1) {
        const int e = c0 + n, i = e >> 4, i2 = (e >> 2) & 3, a = (e >> 1) & 1;
        if ((e & 1) == 0) {   // row bottom node i, column top node 4 + i2
          p = hex_ptr(vals, qr, cs, nc, L, k, i, a, 4 + i2);
          v0 = bt[8 * (2 * i + a) + 2 * i2];
          v1 = bt[8 * (2 * i + a) + 2 * i2 + 1];
        } else {              // row top node 4 + i2, column bottom node i (transpose)
          p = hex_ptr(vals, qr, cs, nc, L, k, 4 + i2, a, i);
          v0 = bt[8 * (2 * i) + 2 * i2 + a];
          v1 = bt[8 * (2 * i + 1) + 2 * i2 + a];
        }
      });
  }
  // ---- pass 3: (top, top) block
  {
    double tt[36];
#pragma unroll
    for (int i = 0; i < 36; ++i) tt[i] = 0.0;
#pragma unroll 1
    for (int qp = 0; qp < 8; ++qp) {
      double N[8], G[8][3], g[16], c, d;
      const double W = hex_point(h, qp, N, G);
      hex_visc<N3>(h, G, W, kp, g, c, d);
      int e = 0;
#pragma unroll
      for (int p = 0; p < 8; ++p)
#pragma unroll
        for (int p2 = p; p2 < 8; ++p2) tt[e++] += hex_jentry(G, g, c, d, 8 + p, 8 + p2);
    }
#pragma unroll
    for (int c0 = 0; c0 < 32; c0 += kRmw)
      rmw_batch<kRmw>([&](int n, double2*& p, double& v0, double& v1) {
        const int e = c0 + n, i = e >> 3, i2 = (e >> 1) & 3, a = e & 1;
        p = hex_ptr(vals, qr, cs, nc, L, k, 4 + i, a, 4 + i2);
        v0 = sym(tt, 2 * i + a, 2 * i2);
        v1 = sym(tt, 2 * i + a, 2 * i2 + 1);
      });
  }
}

// One point's contribution c H - d g g^T to a block of the 16 x 16 element
// matrix, with the row node's gradient prescaled once by the viscosity factor
// (uu: (2 c Gx, c Gy / 2, c Gz / 2) . G', vv: (c Gx / 2, 2 c Gy, c Gz / 2) . G',
// uv: c Gx Gy' + (c Gy / 2) Gx', vu: (c Gx / 2) Gy' + c Gy Gx', H of SURVEY.md
// App. A.3): 3-4 FMA per entry instead of hex_jentry's products per entry.
// BLK 0: (bottom, bottom) packed p <= p2 (36); 1: (bottom, top) [8 p + p2] (64);
// 2: (top, top) packed (36).  The (c / 2) G_z G_z' part of the uu and vv
// entries is left out here and added once per block by hex_zz.
//
// hex_zz: G_z of node (j, l) is -/+ Q_j / (2 z_zeta) (l = 0 / 1) and Q_j, z_zeta
// depend on the footprint point m only, so over the 8 points
//   sum_q (c_q / 2) G_z(j,l) G_z(j2,l2) = s(l) s(l2) T(j, j2),
//   T(j, j2) = sum_m (Q_j Q_j2 / 4)(m) sum_zeta c / (2 z_zeta^2),
// s(0) = -1, s(1) = +1: 10 numbers per hexahedron instead of two FMA per
// entry and point.  T is built after pass 1 and added with sign +
// ((bottom, bottom), (top, top)) or - ((bottom, top)).
__device__ __forceinline__ void hex_zz_build(uint32_t tm) {
  constexpr double gz = 0.57735026918962576451;
  const double cxi[4] = {-1.0, 1.0, 1.0, -1.0}, ceta[4] = {-1.0, -1.0, 1.0, 1.0};
  double w[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    double a, b;
    tmem::ld1(tm + kHexTmRec * m + 18, &a);
    tmem::ld1(tm + kHexTmRec * (m + 4) + 18, &b);
    w[m] = a + b;
  }
  double T[10];
  int e = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int j2 = j; j2 < 4; ++j2) {
      double t = 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const double xi = (m & 1) ? gz : -gz, eta = (m & 2) ? gz : -gz;
        const double hq = 0.125 * (1.0 + cxi[j] * xi) * (1.0 + ceta[j] * eta);
        const double hq2 = 0.125 * (1.0 + cxi[j2] * xi) * (1.0 + ceta[j2] * eta);
        t = fma(hq * hq2, w[m], t);   // (Q_j / 2)(Q_j2 / 2): compile-time constants
      }
      T[e++] = t;
    }
  tmem::st<10>(tm + kHexTmT, T);
}
__host__ __device__ constexpr int tidx4(int j, int j2) {
  return j <= j2 ? j * 4 - (j * (j - 1)) / 2 + (j2 - j) : j2 * 4 - (j2 * (j2 - 1)) / 2 + (j - j2);
}
// add +/- T to the uu / vv entries of a block in hex_accum's layout
template <int BLK>
__device__ __forceinline__ void hex_zz_add(uint32_t tm, double* acc) {
  double T[10];
  tmem::ld<10>(tm + kHexTmT, T);
  auto sym = [](int a, int b) { return a * 8 - (a * (a - 1)) / 2 + (b - a); };
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int j2 = 0; j2 < 4; ++j2) {
      if (BLK != 1 && j2 < j) continue;
      const double t = T[tidx4(j, j2)];
      if (BLK == 1) {
        acc[8 * (2 * j) + 2 * j2] -= t;
        acc[8 * (2 * j + 1) + 2 * j2 + 1] -= t;
      } else {
        acc[sym(2 * j, 2 * j2)] += t;
        acc[sym(2 * j + 1, 2 * j2 + 1)] += t;
      }
    }
}
template <int BLK>
__device__ __forceinline__ void hex_accum(const double G[8][3], const double g[16], double c, double d,
                                          double* acc) {
  constexpr int r0 = BLK == 2 ? 4 : 0, c0 = BLK == 0 ? 0 : 4;
#pragma unroll
  for (int i = r0; i < r0 + 4; ++i) {
    const double cx = c * G[i][0], cy = c * G[i][1];
    const double ax = 2.0 * cx, ay = 0.5 * cy, bx = 0.5 * cx, by = 2.0 * cy;
    const double du = -d * g[2 * i], dv = -d * g[2 * i + 1];
#pragma unroll
    for (int i2 = c0; i2 < c0 + 4; ++i2) {
      if (BLK != 1 && i2 < i) continue;
      const double gx = G[i2][0], gy = G[i2][1];
      const int p = 2 * (i - r0), p2 = 2 * (i2 - c0);
      auto sym = [](int a, int b) { return a * 8 - (a * (a - 1)) / 2 + (b - a); };
      double& euu = BLK == 1 ? acc[8 * p + p2] : acc[sym(p, p2)];
      double& euv = BLK == 1 ? acc[8 * p + p2 + 1] : acc[sym(p, p2 + 1)];
      double& evv = BLK == 1 ? acc[8 * (p + 1) + p2 + 1] : acc[sym(p + 1, p2 + 1)];
      euu = fma(du, g[2 * i2], fma(ay, gy, fma(ax, gx, euu)));
      euv = fma(du, g[2 * i2 + 1], fma(ay, gx, fma(cx, gy, euv)));
      evv = fma(dv, g[2 * i2 + 1], fma(by, gy, fma(bx, gx, evv)));
      if (BLK == 1 || i2 != i) {
        double& evu = BLK == 1 ? acc[8 * (p + 1) + p2] : acc[sym(p + 1, p2)];
        evu = fma(dv, g[2 * i2], fma(cy, gx, fma(bx, gy, evu)));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// KH-patch: owner-computes hexahedral assembly (DESIGN.md "Hexahedral
// variant").  The wedge path's patch scheme on a quadrilateral footprint: one
// CTA = <= kPatchQuads consecutive (Hilbert-ordered) quads, one thread per quad
// column, layers k = 0..L-1.  Per layer the thread evaluates hexahedron (q, k)
// in the three passes of hex_kernel and publishes into shared memory: the
// (bottom, bottom) block and the bottom residual are ADDED to D (which holds
// the (top, top) block + top residual of hexahedron (q, k-1): the vertical
// merge of level k), the (bottom, top) block is STORED to O, the (top, top)
// block + top residual stay in registers (held) and become D after phase B.
// Phase B: one thread per (column, slot) pair of the patch gathers its
// contributions (plan contribution lists, CodeBits<4>) and writes the CSR
// values and R exactly like the wedge scatter (interior columns: plain stores;
// boundary: RED onto the zero fill; multi columns: partial blocks + fix-up).
constexpr int TPQ = kPatchStrideQ;   // SoA row stride of D / O (odd)
using CBQ = CodeBits<4>;
// D entry of (bottom dof p, bottom dof p2), p <= p2: 2x2 node blocks
__host__ __device__ constexpr int dmap4(int p, int p2) {
  return (p >> 1) == (p2 >> 1)
             ? 24 + 3 * (p >> 1) + (p & 1) + (p2 & 1)
             : 4 * ((p >> 1) * (7 - (p >> 1)) / 2 + ((p2 >> 1) - (p >> 1) - 1)) + 2 * (p & 1) + (p2 & 1);
}
constexpr int kHexDR = 36;   // residual entries of D: 36 + 2 j + a
constexpr int kPlanOffsetQ = (kHexDE + kHexOE) * TPQ * 8 / 16 * 16 + 16;
constexpr int kPlanOffsetQR = kHexDE * TPQ * 8 / 16 * 16 + 16;

template <bool UP, bool FIRST>
__device__ __forceinline__ void gather2q(uint2 c2, const double* D, const double* O, PairSums& s) {
  constexpr unsigned mt = (1u << CBQ::kTl) - 1, md = (1u << CBQ::kDb) - 1, mo = (1u << CBQ::kOw) - 1;
  const int tla = int(c2.x & mt), tlb = int(c2.y & mt);
  const int pata = int((c2.x >> CBQ::kPat) & 3), patb = int((c2.y >> CBQ::kPat) & 3);
  const int saa = pata == 1 ? 2 * TPQ : TPQ, sba = pata == 2 ? 2 * TPQ : TPQ;
  const int sab = patb == 1 ? 2 * TPQ : TPQ, sbb = patb == 2 ? 2 * TPQ : TPQ;
  const double* Da = D + int((c2.x >> CBQ::kTl) & md) * TPQ + tla;
  const double* Db = D + int((c2.y >> CBQ::kTl) & md) * TPQ + tlb;
  if (FIRST) {
    s.dg[0] = Da[0] + Db[0];
    s.dg[1] = Da[sba] + Db[sbb];
    s.dg[2] = Da[saa] + Db[sab];
    s.dg[3] = Da[saa + sba] + Db[sab + sbb];
  } else {
    s.dg[0] = (s.dg[0] + Da[0]) + Db[0];
    s.dg[1] = (s.dg[1] + Da[sba]) + Db[sbb];
    s.dg[2] = (s.dg[2] + Da[saa]) + Db[sab];
    s.dg[3] = (s.dg[3] + Da[saa + sba]) + Db[sab + sbb];
  }
  if (UP) {
    const double* Oua = O + int((c2.x >> CBQ::kO) & mo) * TPQ + tla;
    const double* Ona = O + int((c2.x >> CBQ::kOt) & mo) * TPQ + tla;
    const double* Oub = O + int((c2.y >> CBQ::kO) & mo) * TPQ + tlb;
    const double* Onb = O + int((c2.y >> CBQ::kOt) & mo) * TPQ + tlb;
    constexpr int ou[4] = {0, TPQ, 8 * TPQ, 9 * TPQ}, on[4] = {0, 8 * TPQ, TPQ, 9 * TPQ};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (FIRST) {
        s.up[i] = Oua[ou[i]] + Oub[ou[i]];
        s.nx[i] = Ona[on[i]] + Onb[on[i]];
      } else {
        s.up[i] = (s.up[i] + Oua[ou[i]]) + Oub[ou[i]];
        s.nx[i] = (s.nx[i] + Ona[on[i]]) + Onb[on[i]];
      }
    }
  }
}

template <bool UP>
__device__ __forceinline__ void phase_bq_j(const SmemPlan& sp, int kk, int L, const double* D, const double* O,
                                           double* __restrict__ vals, double* __restrict__ partials, int tid,
                                           int nthr) {
  for (int pi = tid; pi < sp.npairs; pi += nthr) {
    const PlanPair pp = sp.pairs[pi];
    PairSums s;
    const uint32_t* cp = sp.contrib + pp.off - 2;
    gather2q<UP, true>(make_uint2(pp.c0, pp.c1), D, O, s);
    for (int e = 2; e < pp.cnt; e += 2) gather2q<UP, false>(*reinterpret_cast<const uint2*>(cp + e), D, O, s);
    emit<UP>(pp, sp.cols[pp.col], s, kk, L, vals, partials);
  }
}

__device__ __forceinline__ void phase_bq_r(const SmemPlan& sp, int kk, int L, const double* Dr,
                                           double* __restrict__ R, double* __restrict__ partials, int tid,
                                           int nthr) {
  constexpr unsigned mt = (1u << CBQ::kTl) - 1;
  for (int ci = tid; ci < sp.ncols; ci += nthr) {
    const PlanCol& pc = sp.cols[ci];
    double r0 = 0.0, r1 = 0.0;
    for (int e = pc.self_off; e < pc.self_off + pc.self_cnt; e += 2) {
      const uint2 c2 = *reinterpret_cast<const uint2*>(sp.contrib + e);
      const double* Da = Dr + 2 * int((c2.x >> CBQ::kJ) & 3) * TPQ + int(c2.x & mt);
      const double* Db = Dr + 2 * int((c2.y >> CBQ::kJ) & 3) * TPQ + int(c2.y & mt);
      r0 += Da[0];
      r1 += Da[TPQ];
      r0 += Db[0];
      r1 += Db[TPQ];
    }
    if ((pc.info >> 30) & 1)
      *reinterpret_cast<double2*>(partials + (int64_t(pc.pad) * (L + 1) + kk) * kPartialStride + 12) =
          make_double2(r0, r1);
    else
      put2(R + 2 * (int64_t(pc.c) * (L + 1) + kk), r0, r1, (pc.info >> 8) & 1);
  }
}

// threads per CTA: one per quad of a patch (kPatchQuads = 3 warps) plus a
// fourth warp (the register file holds 2 CTAs x 128 x 255 registers) that
// zero-fills the patch's lead boundary columns in-kernel while the element
// warps compute layer 0 and then joins phase B (700 x 700 x 10 R + J 5.86 ->
// 5.61 ms; FO_HEX_BLOCK=96: three warps and the zero kernel)
#ifndef FO_HEX_BLOCK
#define FO_HEX_BLOCK 128
#endif
constexpr int kHexBlock = FO_HEX_BLOCK;
// unroll factors of the point loops (pass 1, the (bottom,bottom) / (top,top)
// passes, the (bottom,top) pass): 1 / 2 / 2 -- 5.38 -> 5.31 ms; pass 1 x2
// spills (5.50 ms), profiles/r02ah_ab_hex_unroll.txt
#ifndef FO_HEX_U_P1
#define FO_HEX_U_P1 1
#endif
#ifndef FO_HEX_U_BB
#define FO_HEX_U_BB 2
#endif
#ifndef FO_HEX_U_BT
#define FO_HEX_U_BT 2
#endif
constexpr int kHexUP1 = FO_HEX_U_P1, kHexUBB = FO_HEX_U_BB, kHexUBT = FO_HEX_U_BT;
static_assert(kHexBlock >= kPatchQuads && kHexBlock % 32 == 0, "hex block");

template <bool NEED_J, bool N3>
__global__ void __launch_bounds__(kHexBlock, kHexCtasPerSm)
kh_patch_kernel(const ColRec* __restrict__ col, const QuadRec* __restrict__ quads,
                const double* __restrict__ sigma, const double* __restrict__ Aw, KParams kp, PlanView pv,
                const double* __restrict__ U, double* __restrict__ R, double* __restrict__ vals) {
  extern __shared__ __align__(16) double smem[];
  double* const D = smem;                  // [kHexDE][TPQ]
  double* const O = smem + kHexDE * TPQ;   // [kHexOE][TPQ] (R + J)
  __shared__ uint64_t plan_bar;
  __shared__ uint32_t tmem_base;
  __shared__ int ticket;
  // in-kernel zero fill (pv.inkz, kHexBlock > kPatchQuads): patches in ticket
  // order, so a lead patch (lower ticket) is already running when waited for
  if (pv.inkz && threadIdx.x == 0) ticket = atomicAdd(pv.flags + pv.n_patches, 1);
  if (pv.inkz) __syncthreads();
  const int p = pv.inkz ? ticket : int(blockIdx.x);
  const int t0 = __ldg(pv.t_begin + p), nt = __ldg(pv.t_begin + p + 1) - t0;
  SmemPlan sp;
  {
    const int c0 = __ldg(pv.col_ptr + p), c1 = __ldg(pv.col_ptr + p + 1);
    const int q0 = __ldg(pv.pair_ptr + p), q1 = __ldg(pv.pair_ptr + p + 1);
    const int64_t b0 = __ldg(pv.blob_off + p), b1 = __ldg(pv.blob_off + p + 1);
    char* base = reinterpret_cast<char*>(smem) + (NEED_J ? kPlanOffsetQ : kPlanOffsetQR);
    sp.pairs = reinterpret_cast<const PlanPair*>(base);
    sp.cols = reinterpret_cast<const PlanCol*>(base + (q1 - q0) * sizeof(PlanPair));
    sp.contrib = reinterpret_cast<const uint32_t*>(base + (c1 - c0) * sizeof(PlanCol) + (q1 - q0) * sizeof(PlanPair));
    sp.ncols = c1 - c0; sp.npairs = q1 - q0;
    sp.nedge = __ldg(pv.nedge + p);
    if (threadIdx.x == 0) bulk_init(&plan_bar);
    if (NEED_J && threadIdx.x < 32) tmem::alloc(&tmem_base, kHexTmCols);   // warp 0 owns the TMEM
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    if (threadIdx.x == 0) bulk_load(base, pv.blob + b0, unsigned(b1 - b0), &plan_bar);
  }
  const int L = kp.L;
  const int tl = threadIdx.x;
  const bool active = tl < nt;
  // tcgen05.ld / st are warp-collective: lanes without a quad evaluate a copy
  // of the patch's last one and publish nothing
  const bool run = tl < kPatchQuads && (NEED_J ? true : active);
  const int qi = t0 + (active ? tl : nt - 1);
  const uint32_t tm = tmem_base + (uint32_t(tl & ~31) << 16);   // this warp's lane quarter
  const QuadRec qr = quads[run ? qi : t0];
  if (active) {
#pragma unroll
    for (int i = 0; i < kHexDE; ++i) D[i * TPQ + tl] = 0.0;
  }
  // quad slot kPatchQuads: the zero column the plan's pad entries read
  for (int i = threadIdx.x; i < kHexDE; i += blockDim.x) D[i * TPQ + kPatchQuads] = 0.0;
  if (NEED_J)
    for (int i = threadIdx.x; i < kHexOE; i += blockDim.x) O[i * TPQ + kPatchQuads] = 0.0;
  if (kHexBlock > kPatchQuads && pv.inkz && threadIdx.x >= kPatchQuads && threadIdx.x < kPatchQuads + 32) {
    // the phase-B warp, while the element warps compute layer 0: zero-fill the
    // boundary columns this patch leads, raise its flag, then wait for the
    // leads of its other boundary columns (the first RED follows the CTA
    // barrier before phase B of level 0)
    const int lane = threadIdx.x & 31;
    const int z0 = __ldg(pv.zl_ptr + p), z1 = __ldg(pv.zl_ptr + p + 1);
    for (int i = z0; i < z1; ++i) {
      const int c = __ldg(pv.zl + i);
      for (int j = lane; j < L + 1; j += 32)
        *reinterpret_cast<double2*>(R + 2 * (int64_t(c) * (L + 1) + j)) = make_double2(0.0, 0.0);
      if (NEED_J) {
        const long long csn = __double_as_longlong(__ldg(reinterpret_cast<const double*>(col + c) + 5));
        double2* v = reinterpret_cast<double2*>(vals + (csn >> 8));
        const int64_t len2 = int64_t(2 * (csn & 255)) * (3 * L + 1);
        for (int64_t j = lane; j < len2; j += 32) v[j] = make_double2(0.0, 0.0);   // no L2 hint (slower here)
      }
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();   // the warp's zero stores (ordered by __syncwarp) before the flag
      asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(pv.flags + p), "r"(1) : "memory");
    }
    const int w0 = __ldg(pv.wl_ptr + p), w1 = __ldg(pv.wl_ptr + p + 1);
    for (int i = w0 + lane; i < w1; i += 32) {
      const int32_t* f = pv.flags + __ldg(pv.wl + i);
      int v = 0;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v) break;
        __nanosleep(64);
      }
    }
    __syncwarp();
  }
  double held[kHexDE];
  for (int k = 0; k < L; ++k) {
    if (run) {
      HexIn h;
      const double s0 = __ldg(sigma + k), s1 = __ldg(sigma + k + 1);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const ColRec c = col[qr.v[j]];
        h.X[j] = c.x;
        h.Y[j] = c.y;
        h.Zb[j] = fma(s0, c.H, c.base);
        h.Zt[j] = fma(s1, c.H, c.base);
        h.S[j] = c.base + c.H;
        h.B[j] = c.beta;
        const int64_t node = int64_t(qr.v[j]) * (L + 1) + k;
        const double2 ub = __ldg(reinterpret_cast<const double2*>(U) + node);
        const double2 ut = __ldg(reinterpret_cast<const double2*>(U) + node + 1);
        h.Uu[j] = ub.x; h.Uv[j] = ub.y; h.Uu[j + 4] = ut.x; h.Uv[j + 4] = ut.y;
      }
      h.Afac = wedge_afac(kp, Aw, qi, k);
      // ---- pass 1: residual, (bottom, bottom) block, basal term -> D (+=), top residual -> held
      {
        double r[16], bb[36];
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = 0.0;
#pragma unroll
        for (int i = 0; i < 36; ++i) bb[i] = 0.0;
#pragma unroll kHexUP1
        for (int qp = 0; qp < 8; ++qp) {
          double N[8], G[8][3], g[16], c, d, pk[11];
          const double W = hex_point(h, qp, N, G, NEED_J ? pk : nullptr);
          if (NEED_J) {
            double rec[10];
            hex_visc_rec<N3>(h, G, W, kp, g, c, d, rec);
            rec[7] = pk[9];
            rec[8] = pk[10];
            rec[9] = 0.5 * c * pk[8] * pk[8];   // hex_zz
            tmem::st<10>(tm + kHexTmRec * qp, rec);
            if (qp < 4) tmem::st<9>(tm + kHexTmGeo + 18 * qp, pk);
          } else {
            hex_visc<N3>(h, G, W, kp, g, c, d);
          }
          double sx = 0, sy = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) { sx = fma(h.S[i & 3], G[i][0], sx); sy = fma(h.S[i & 3], G[i][1], sy); }
          const double bw = W * kp.rg;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            r[2 * i] += fma(c, g[2 * i], bw * sx * N[i]);
            r[2 * i + 1] += fma(c, g[2 * i + 1], bw * sy * N[i]);
          }
        }
        // (bottom, bottom) block in a pass of its own from the TMEM cache: pass 1
        // then holds only the residual (no spills in its point loop; with the
        // block accumulated in pass 1: 400 B of spills, 6.91 vs 5.83 ms)
        if (NEED_J) {
          tmem::wait_st();
          hex_zz_build(tm);
#pragma unroll kHexUBB
          for (int qp = 0; qp < 8; ++qp) {
            double G[8][3], g[16], c, d, rec[7];
            hex_grad_tm(tm, qp, G, rec);
            hex_g_rec(G, rec, g, c, d);
            hex_accum<0>(G, g, c, d, bb);
          }
          tmem::wait_st();
          hex_zz_add<0>(tm, bb);
        }
        if (k == 0) hex_basal<NEED_J>(h, r, bb);
        if (active) {
#pragma unroll
          for (int i = 0; i < 8; ++i) D[(kHexDR + i) * TPQ + tl] += r[i];
          if (NEED_J) {
            int e = 0;
#pragma unroll
            for (int pp = 0; pp < 8; ++pp)
#pragma unroll
              for (int p2 = pp; p2 < 8; ++p2) { D[dmap4(pp, p2) * TPQ + tl] += bb[e]; ++e; }
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) held[kHexDR + i] = r[8 + i];
      }
      if (NEED_J) tmem::wait_st();   // the point records are in TMEM
      if (NEED_J) {
        // ---- pass 2: (bottom, top) block -> O
        double bt[64];
#pragma unroll
        for (int i = 0; i < 64; ++i) bt[i] = 0.0;
#pragma unroll kHexUBT
        for (int qp = 0; qp < 8; ++qp) {
          double G[8][3], g[16], c, d, rec[7];
          hex_grad_tm(tm, qp, G, rec);
          hex_g_rec(G, rec, g, c, d);
          hex_accum<1>(G, g, c, d, bt);
        }
        hex_zz_add<1>(tm, bt);
        if (active) {
#pragma unroll
          for (int i = 0; i < 64; ++i) O[i * TPQ + tl] = bt[i];
        }
        // ---- pass 3: (top, top) block -> held
        double tt[36];
#pragma unroll
        for (int i = 0; i < 36; ++i) tt[i] = 0.0;
#pragma unroll kHexUBB
        for (int qp = 0; qp < 8; ++qp) {
          double G[8][3], g[16], c, d, rec[7];
          hex_grad_tm(tm, qp, G, rec);
          hex_g_rec(G, rec, g, c, d);
          hex_accum<2>(G, g, c, d, tt);
        }
        hex_zz_add<2>(tm, tt);
        int e = 0;
#pragma unroll
        for (int pp = 0; pp < 8; ++pp)
#pragma unroll
          for (int p2 = pp; p2 < 8; ++p2) { held[dmap4(pp, p2)] = tt[e]; ++e; }
      }
    }
    if (k == 0) bulk_wait(&plan_bar);
    __syncthreads();
#ifndef FO_PROBE_HEX_NO_B   // timing probe only: the element alone (wrong values)
    if (NEED_J) {
      if (k < L) phase_bq_j<true>(sp, k, L, D, O, vals, pv.partials, threadIdx.x, blockDim.x);
    }
#endif
    phase_bq_r(sp, k, L, D + kHexDR * TPQ, R, pv.partials, threadIdx.x, blockDim.x);
    __syncthreads();
    if (active) {   // the held top block becomes level k+1's diagonal block
      if (NEED_J) {
#pragma unroll
        for (int i = 0; i < kHexDE; ++i) D[i * TPQ + tl] = held[i];
      } else {
#pragma unroll
        for (int i = kHexDR; i < kHexDE; ++i) D[i * TPQ + tl] = held[i];
      }
    }
  }
  if (L == 0) bulk_wait(&plan_bar);
  __syncthreads();
  if (NEED_J) phase_bq_j<false>(sp, L, L, D, O, vals, pv.partials, threadIdx.x, blockDim.x);
  phase_bq_r(sp, L, L, D + kHexDR * TPQ, R, pv.partials, threadIdx.x, blockDim.x);
  if (NEED_J) {
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    if (threadIdx.x < 32) tmem::dealloc(tmem_base, kHexTmCols);
  }
}

}  // namespace

// ------------------------------------------------------------------ host

fo_status hex_create_impl(const fo_params* p, int64_t n_vert, const double* xy, int64_t n_quad,
                          const int32_t* quad, int32_t L, const double* sigma, const double* thickness,
                          const double* surface, const double* bed, const double* beta, const double* A_elem,
                          int device, fo_mesh* out, bool host_only = false) {
  auto bad = [](fo_status st, const std::string& msg) { set_error(msg); return st; };
  if (!out || !p) return bad(FO_EINVAL, "NULL argument");
  *out = nullptr;
  if (n_vert < 0 || n_quad < 0 || L < 1) return bad(FO_EINVAL, "bad sizes");
  if (n_vert > 0 && (!xy || !quad || !thickness || !surface || !beta)) return bad(FO_EINVAL, "NULL array");
  if (!(p->glen_n > 0.0) || !(p->A > 0.0) || p->eps_reg < 0.0) return bad(FO_EINVAL, "bad parameters");
  if (sigma) {
    if (sigma[0] != 0.0 || sigma[L] != 1.0) return bad(FO_EMESH, "sigma must run 0 .. 1");
    for (int32_t k = 0; k < L; ++k)
      if (!(sigma[k + 1] > sigma[k])) return bad(FO_EMESH, "sigma not strictly ascending");
  }
  std::vector<char> used(size_t(n_vert), 0);
  for (int64_t t = 0; t < n_quad; ++t) {
    const int32_t* v = quad + 4 * t;
    for (int j = 0; j < 4; ++j)
      if (v[j] < 0 || v[j] >= n_vert) return bad(FO_EMESH, "quad corner out of range");
    for (int j = 0; j < 4; ++j) {   // convex and CCW: every corner turns left
      const int32_t a = v[(j + 3) % 4], b = v[j], c = v[(j + 1) % 4];
      const double cr = (xy[2 * b] - xy[2 * a]) * (xy[2 * c + 1] - xy[2 * b + 1]) -
                        (xy[2 * b + 1] - xy[2 * a + 1]) * (xy[2 * c] - xy[2 * b]);
      if (!(cr > 0.0)) return bad(FO_EMESH, "quad " + std::to_string(t) + " is not convex CCW");
      used[size_t(b)] = 1;
    }
  }
  for (int64_t c = 0; c < n_vert; ++c) {
    if (!used[size_t(c)]) return bad(FO_EMESH, "vertex in no quad");
    if (!(thickness[c] >= p->H_min)) return bad(FO_EMESH, "thickness below H_min");
  }
  fo_status st = FO_OK;
  if (!host_only) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      return bad(FO_ECUDA, "no CUDA device available (libfo has no CPU path)");
    }
    if (device < 0 || device >= ndev) return bad(FO_EINVAL, "bad device ordinal");
    st = cuda_status(cudaSetDevice(device), "cudaSetDevice");
    if (st) return st;
  }

  // quads in Hilbert order of their centroids (the patch kernel's patches are
  // runs of consecutive quads, so they come out compact); `order[t]` = the
  // caller's index of local quad t
  std::vector<int32_t> order(static_cast<size_t>(n_quad));
  {
    double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
    for (int64_t c = 0; c < n_vert; ++c) {
      x0 = std::min(x0, xy[2 * c]); x1 = std::max(x1, xy[2 * c]);
      y0 = std::min(y0, xy[2 * c + 1]); y1 = std::max(y1, xy[2 * c + 1]);
    }
    const double span = std::max(std::max(x1 - x0, y1 - y0), 1e-300);
    std::vector<uint64_t> key(static_cast<size_t>(n_quad));
    for (int64_t t = 0; t < n_quad; ++t) {
      double cx = 0.0, cy = 0.0;
      for (int j = 0; j < 4; ++j) { cx += xy[2 * quad[4 * t + j]]; cy += xy[2 * quad[4 * t + j] + 1]; }
      const uint32_t n = 1u << 16;
      uint32_t ix = uint32_t(std::min(double(n - 1), (0.25 * cx - x0) / span * double(n)));
      uint32_t iy = uint32_t(std::min(double(n - 1), (0.25 * cy - y0) / span * double(n)));
      uint64_t d = 0;   // Hilbert index (xy -> d)
      for (uint32_t sq = n / 2; sq > 0; sq /= 2) {
        const uint32_t rx = (ix & sq) > 0, ry = (iy & sq) > 0;
        d += uint64_t(sq) * sq * ((3 * rx) ^ ry);
        if (ry == 0) {
          if (rx == 1) { ix = n - 1 - ix; iy = n - 1 - iy; }
          std::swap(ix, iy);
        }
      }
      key[size_t(t)] = d;
      order[size_t(t)] = int32_t(t);
    }
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return key[size_t(a)] < key[size_t(b)]; });
  }

  fo_mesh m = new fo_mesh_s();
  m->device = device;
  m->p = *p;
  m->L = L;
  m->quad = true;
  m->n_col = n_vert;
  m->nA = n_vert;
  m->n_tri = n_quad;
  m->n_node = n_vert * (L + 1);
  m->n_dof = 2 * m->n_node;
  m->n_elem = n_quad * L;
  m->n_owned_dof = m->n_dof;
  m->glob.resize(size_t(n_vert));
  for (int64_t c = 0; c < n_vert; ++c) m->glob[size_t(c)] = c;
  m->tri_glob.resize(size_t(n_quad));
  for (int64_t t = 0; t < n_quad; ++t) m->tri_glob[size_t(t)] = order[size_t(t)];
  // coupling lists: every corner of every quad around the column, sorted
  std::vector<std::vector<int32_t>> lists(static_cast<size_t>(n_vert));
  for (int64_t c = 0; c < n_vert; ++c) lists[size_t(c)].push_back(int32_t(c));
  for (int64_t t = 0; t < n_quad; ++t)
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) lists[size_t(quad[4 * t + i])].push_back(quad[4 * t + j]);
  m->nbr_ptr.assign(size_t(n_vert) + 1, 0);
  for (int64_t c = 0; c < n_vert; ++c) {
    auto& l = lists[size_t(c)];
    std::sort(l.begin(), l.end());
    l.erase(std::unique(l.begin(), l.end()), l.end());
    if (l.size() > 255) { fo_mesh_destroy(m); return bad(FO_EMESH, "column couples to more than 254 neighbours"); }
    m->nbr.insert(m->nbr.end(), l.begin(), l.end());
    m->nbr_ptr[size_t(c) + 1] = int64_t(m->nbr.size());
  }
  m->colstart.assign(size_t(n_vert) + 1, 0);
  for (int64_t c = 0; c < n_vert; ++c)
    m->colstart[size_t(c) + 1] = m->colstart[size_t(c)] +
                                 4 * (m->nbr_ptr[size_t(c) + 1] - m->nbr_ptr[size_t(c)]) * (3 * int64_t(L) + 1);
  m->nnz = m->colstart.back();
  m->sigma.resize(size_t(L) + 1);
  for (int32_t k = 0; k <= L; ++k) m->sigma[size_t(k)] = sigma ? sigma[k] : double(k) / double(L);
  m->sigma[size_t(L)] = 1.0;
  m->colrec.assign(size_t(n_vert), ColRec{});
  for (int64_t c = 0; c < n_vert; ++c) {
    ColRec& r = m->colrec[size_t(c)];
    r.x = xy[2 * c];
    r.y = xy[2 * c + 1];
    r.H = thickness[c];
    r.base = surface[c] - thickness[c];
    const bool floating = bed && (p->rho * thickness[c] < -p->rho_w * bed[c]);
    r.beta = floating ? 0.0 : beta[c];
    r.cs_n = (m->colstart[size_t(c)] << 8) | (m->nbr_ptr[size_t(c) + 1] - m->nbr_ptr[size_t(c)]);
  }
  std::vector<QuadRec>& qrec = m->quadrec;
  qrec.assign(static_cast<size_t>(n_quad), QuadRec{});
  m->tri.resize(size_t(4 * n_quad));
  for (int64_t t = 0; t < n_quad; ++t) {
    QuadRec& q = qrec[size_t(t)];
    for (int i = 0; i < 4; ++i) q.v[i] = quad[4 * int64_t(order[size_t(t)]) + i];
    for (int i = 0; i < 4; ++i) m->tri[size_t(4 * t + i)] = q.v[i];
    for (int i = 0; i < 4; ++i) {
      const int32_t* b = m->nbr.data() + m->nbr_ptr[size_t(q.v[i])];
      const int32_t* e = m->nbr.data() + m->nbr_ptr[size_t(q.v[i]) + 1];
      for (int j = 0; j < 4; ++j) q.slot[4 * i + j] = uint8_t(std::lower_bound(b, e, q.v[j]) - b);
    }
  }
  // greedy colouring: quads sharing a corner get different colours
  std::vector<std::vector<int32_t>> vq(static_cast<size_t>(n_vert));
  for (int64_t t = 0; t < n_quad; ++t)
    for (int i = 0; i < 4; ++i) vq[size_t(qrec[size_t(t)].v[i])].push_back(int32_t(t));
  std::vector<int32_t> color(size_t(n_quad), -1);
  int ncol = 0;
  for (int64_t t = 0; t < n_quad; ++t) {
    uint64_t taken = 0;
    for (int i = 0; i < 4; ++i)
      for (int32_t o : vq[size_t(qrec[size_t(t)].v[i])])
        if (color[size_t(o)] >= 0 && color[size_t(o)] < 64) taken |= 1ull << color[size_t(o)];
    int c = 0;
    while (c < 64 && ((taken >> c) & 1)) ++c;
    if (c == 64) { fo_mesh_destroy(m); return bad(FO_EMESH, "quad colouring needs more than 64 colours"); }
    color[size_t(t)] = c;
    ncol = std::max(ncol, c + 1);
  }
  m->hex_color_ptr.assign(size_t(ncol) + 1, 0);
  for (int64_t t = 0; t < n_quad; ++t) m->hex_color_ptr[size_t(color[size_t(t)]) + 1]++;
  for (int c = 0; c < ncol; ++c) m->hex_color_ptr[size_t(c) + 1] += m->hex_color_ptr[size_t(c)];
  std::vector<int32_t> ids(static_cast<size_t>(n_quad));
  {
    std::vector<int64_t> pos(m->hex_color_ptr.begin(), m->hex_color_ptr.end() - 1);
    for (int64_t t = 0; t < n_quad; ++t) ids[size_t(pos[size_t(color[size_t(t)])]++)] = int32_t(t);
  }
  if (host_only) {   // the patch plan only, nothing on a device (fo_plan_check_quad_host)
    st = build_patch_plan(m, false);
    if (st) { delete m; return st; }
    *out = m;
    return FO_OK;
  }
  auto up = [](void** dst, const void* src, size_t bytes) {
    if (bytes == 0) return FO_OK;
    fo_status s = cuda_status(cudaMalloc(dst, bytes), "cudaMalloc");
    if (!s) s = cuda_status(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    return s;
  };
  st = up(reinterpret_cast<void**>(&m->d_col), m->colrec.data(), m->colrec.size() * sizeof(ColRec));
  if (!st) st = up(reinterpret_cast<void**>(&m->d_sigma), m->sigma.data(), m->sigma.size() * sizeof(double));
  if (!st) st = up(reinterpret_cast<void**>(&m->d_quad), qrec.data(), qrec.size() * sizeof(QuadRec));
  if (!st) st = up(reinterpret_cast<void**>(&m->d_hex_ids), ids.data(), ids.size() * sizeof(int32_t));
  if (!st && A_elem && m->n_elem > 0) {
    std::vector<double> afac(static_cast<size_t>(m->n_elem));
    for (int64_t i = 0; i < m->n_elem; ++i) {   // local order: quad t, layer k
      const double a = A_elem[int64_t(order[size_t(i / L)]) * L + i % L];
      if (!(a > 0.0)) { st = bad(FO_EINVAL, "A_elem must be > 0"); break; }
      afac[size_t(i)] = std::pow(a, -1.0 / p->glen_n);
    }
    if (!st) st = up(reinterpret_cast<void**>(&m->d_A), afac.data(), afac.size() * sizeof(double));
    m->has_A_elem = true;
  }
  if (!st) st = build_patch_plan(m);   // owner-computes patches (KH-patch)
  if (st) { fo_mesh_destroy(m); return st; }
  *out = m;
  return FO_OK;
}

// KH-patch: zero fill of boundary columns, the patch kernel, the multi fix-up
static fo_status launch_hex_owner(fo_mesh m, const double* d_U, double* R, double* d_vals, cudaStream_t s) {
  int launches = 0;
  // a phase-B warp beside the element warps zero-fills in-kernel (no zero kernel)
  constexpr bool inkz = kHexBlock > kPatchQuads;
  fo_status st = launch_owner_prologue(m, R, d_vals, s, &launches, inkz);
  if (st) return st;
  const bool n3 = m->p.glen_n == 3.0;
  const KParams kp = make_kparams(m);
  PlanView pv{m->d_plan.t_begin, m->d_plan.col_ptr, m->d_plan.pair_ptr, m->d_plan.nedge, m->d_plan.blob,
              m->d_plan.blob_off, m->d_plan.partials, 0, m->d_plan.zl, m->d_plan.zl_ptr, m->d_plan.wl,
              m->d_plan.wl_ptr, m->d_plan.flags, inkz ? 1 : 0, m->plan.n_patches, m->d_plan.multi, 0, 0, 0};
  const size_t sm = size_t(d_vals ? kPlanOffsetQ : kPlanOffsetQR) + kPlanBytesHex;
  auto go = [&](auto kern) -> fo_status {
    fo_status e = cuda_status(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)),
                              "cudaFuncSetAttribute");
    if (e) return e;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (m->timing) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
    }
    kern<<<m->plan.n_patches, kHexBlock, sm, s>>>(m->d_col, m->d_quad, m->d_sigma, m->d_A, kp, pv, d_U, R, d_vals);
    if (m->timing) {
      cudaEventRecord(e1, s);
      m->timed.push_back({e0, e1});
    }
    return cuda_status(cudaGetLastError(), "kh_patch_kernel launch");
  };
  if (d_vals) st = n3 ? go(kh_patch_kernel<true, true>) : go(kh_patch_kernel<true, false>);
  else st = n3 ? go(kh_patch_kernel<false, true>) : go(kh_patch_kernel<false, false>);
  if (st) return st;
  ++launches;
  st = launch_owner_fixup(m, R, d_vals, s, &launches);
  if (st) return st;
  m->last_launches = launches;
  return FO_OK;
}

fo_status launch_hex(fo_mesh m, const double* d_U, double* d_R, double* d_vals, cudaStream_t s) {
  const bool need_j = d_vals != nullptr;
  double* R = d_R;
  if (!R) {
    if (!m->d_scratch_R) {
      fo_status st = cuda_status(cudaMalloc(&m->d_scratch_R, sizeof(double) * m->n_dof), "cudaMalloc");
      if (st) return st;
    }
    R = m->d_scratch_R;
  }
  // R + J: the quad-patch kernel; the residual alone (16 values per
  // hexahedron) is faster with the coloured read-modify-write, which is also
  // the R + J ablation (FO_SCATTER_ATOMIC): both deterministic
  if (need_j && m->scatter != FO_SCATTER_ATOMIC && m->plan.n_patches > 0)
    return launch_hex_owner(m, d_U, R, d_vals, s);
  fo_status st = cuda_status(cudaMemsetAsync(R, 0, sizeof(double) * m->n_dof, s), "cudaMemsetAsync");
  if (!st && need_j) st = cuda_status(cudaMemsetAsync(d_vals, 0, sizeof(double) * m->nnz, s), "cudaMemsetAsync");
  if (st) return st;
  const size_t smem = 0;
  const KParams kp = make_kparams(m);
  const bool n3 = m->p.glen_n == 3.0;
  int launches = 0;
  const int ncol = int(m->hex_color_ptr.size()) - 1;
  for (int kpar = 0; kpar < 2 && kpar < m->L; ++kpar)
    for (int c = 0; c < ncol; ++c) {
      const int n = int(m->hex_color_ptr[size_t(c) + 1] - m->hex_color_ptr[size_t(c)]);
      const int nk = (m->L - kpar + 1) / 2;
      const int64_t items = int64_t(n) * nk;
      if (items == 0) continue;
      const unsigned blocks = unsigned((items + kHexThreads - 1) / kHexThreads);
      const int32_t* ids = m->d_hex_ids + m->hex_color_ptr[size_t(c)];
      if (need_j) {
        if (n3) hex_kernel<true, true><<<blocks, kHexThreads, smem, s>>>(m->d_col, m->d_quad, ids, n, kpar, m->d_sigma, m->d_A, kp, d_U, R, d_vals);
        else hex_kernel<true, false><<<blocks, kHexThreads, smem, s>>>(m->d_col, m->d_quad, ids, n, kpar, m->d_sigma, m->d_A, kp, d_U, R, d_vals);
      } else {
        if (n3) hex_kernel<false, true><<<blocks, kHexThreads, smem, s>>>(m->d_col, m->d_quad, ids, n, kpar, m->d_sigma, m->d_A, kp, d_U, R, nullptr);
        else hex_kernel<false, false><<<blocks, kHexThreads, smem, s>>>(m->d_col, m->d_quad, ids, n, kpar, m->d_sigma, m->d_A, kp, d_U, R, nullptr);
      }
      st = cuda_status(cudaGetLastError(), "hex_kernel launch");
      if (st) return st;
      ++launches;
    }
  m->last_launches = launches;
  return FO_OK;
}

}  // namespace fo

using namespace fo;

extern "C" {

fo_status fo_plan_check_quad_host(int64_t n_vert, const double* xy, int64_t n_quad, const int32_t* quad,
                                  int32_t n_layers, int64_t* stats) {
  if (!stats) { set_error("stats is NULL"); return FO_EINVAL; }
  fo_params p;
  fo_params_default(&p);
  std::vector<double> H(size_t(n_vert), 1000.0), srf(size_t(n_vert), 1000.0), beta(size_t(n_vert), 1.0);
  fo_mesh m = nullptr;
  fo_status st = hex_create_impl(&p, n_vert, xy, n_quad, quad, n_layers, nullptr, H.data(), srf.data(), nullptr,
                                 beta.data(), nullptr, 0, &m, true);
  if (st) return st;
  st = plan_check(m, stats);
  delete m;
  return st;
}

fo_status fo_mesh_create_quad(const fo_params* p, int64_t n_vert, const double* xy, int64_t n_quad,
                              const int32_t* quad, int32_t n_layers, const double* sigma,
                              const double* thickness, const double* surface, const double* bed,
                              const double* beta, const double* A_elem, int device, fo_mesh* out) {
  return hex_create_impl(p, n_vert, xy, n_quad, quad, n_layers, sigma, thickness, surface, bed, beta, A_elem,
                         device, out);
}

}  // extern "C"
