// fo_element.cuh -- per-wedge element math of the FO-Stokes residual and
// exact Jacobian, column-structured.
//
// PAPER.md (P:n = line n): first-order momentum balance eq:FOStokes,
// strain-rate vectors eps_1, eps_2 and components, Glen viscosity
// eq:effvisc with the effective strain rate eq:effeps,
// basal Robin sliding, extruded prismatic elements,
// residual eq:residual and Jacobian eq:linearsystem.
//
// The wedge (t,k) has bottom nodes (j, l=0) and top nodes (j, l=1), j = 0..2
// the footprint vertices.  Vertical columns make the map x,y depend on the
// footprint barycentrics L_j only and z = sum_j L_j (m_j + zeta h_j), so
//   z_zeta = sum_j L_j h_j              (per triangle quadrature point),
//   z_x    = sum_j a_j (m_j + zeta h_j) (per Gauss level zeta),
//   phi_z(j,l) = sigma_l L_j / (2 z_zeta),  phi_x = a_j f_l - z_x phi_z,
// with a_j, b_j the constant footprint gradients of L_j and f_0 = (1-zeta)/2,
// f_1 = (1+zeta)/2, sigma_0 = -1, sigma_1 = +1.  This is an exact rewrite of
// the isoparametric gradient (it is NOT the oracle's generic 3x3 inverse).
// Quadrature: 3-point triangle rule (barycentric 2/3,1/6,1/6; weight 1/6) x
// 2-point Gauss in zeta (reading L4); basal: same 3 points on the planar 3D
// bottom triangle (readings L6-L8).
//
// Local DOF p = 2*i + comp, node i = j + 3*l.  Outputs: r[12] and the upper
// triangle J[78] (packed row-major, p <= q) of the symmetric 12x12 block:
//   J = sum_q c_q [H_q - ((n-1)/(2n)) g_q g_q^T / (q_q + eps)] + basal mass,
//   c_q = w_q 2mu_q, g_{a,i} = eps_a . grad phi_i.
#pragma once

namespace fo {

__host__ __device__ constexpr int jidx(int p, int q) { return p * 12 - (p * (p - 1)) / 2 + (q - p); }

// (x)^(-1/3) for the n = 3 viscosity: an fp32 seed from the SFU
// (log2 / exp2, relative error ~1e-6) and two Newton steps y <- y (4 - x y^3) / 3
// in fp64 (error ~2 e^2 per step: 1e-6 -> 2e-12 -> 1e-23, i.e. correctly
// rounded up to an ulp); x = q + eps_reg >= eps_reg > 0 lies in the fp32
// normal range.  Fewer issue slots than the libdevice rcbrt.
__device__ __forceinline__ double rcbrt_n3(double x) {
  const float xf = __double2float_rn(x);
  float l2, yf;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(xf));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"(-0.333333343f * l2));
  double y = double(yf);
  constexpr double k43 = 4.0 / 3.0, k13 = 1.0 / 3.0;
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const double t = x * y * y * y;
    y = y * fma(-k13, t, k43);
  }
  return y;
}

// 1/x for the geometry's reciprocals (x != 0, |x| in the fp32 normal range: a
// layer's vertical half-height in metres, twice a footprint triangle's area in
// m^2): fp32 SFU seed (relative error ~1e-7) and two Newton steps
// y <- y + y (1 - x y) (1e-7 -> 1e-14 -> 1e-28), no slow-path branches.
__device__ __forceinline__ double rcp_geo(double x) {
  float yf;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"(__double2float_rn(x)));
  double y = double(yf);
#pragma unroll
  for (int it = 0; it < 2; ++it) y = fma(y, fma(-x, y, 1.0), y);
  return y;
}

struct WedgeIn {
  double a[3], b[3];   // footprint gradients of the barycentrics
  double D;            // 2 |T|
  double e1x, e1y, e2x, e2y;  // footprint edges P1-P0, P2-P0 (3D basal area)
  double sx, sy;       // P1 surface gradient (reading L10)
  double zb[3], zt[3]; // bottom / top node heights
  double ub[3], vb[3], ut[3], vt[3];
  double beta[3];      // basal friction (k == 0 only)
  double Afac;         // A^(-1/n)
  bool basal;
  bool go;             // always true at run time (scheduling boundaries)
};

template <bool NEED_J, bool N3>
__device__ __forceinline__ void wedge_element(const WedgeIn& w, double rg, double eps,
                                              double glen_n, double* __restrict__ r,
                                              double* __restrict__ J) {
  constexpr double kZeta = 0.57735026918962576451;   // 1/sqrt(3)
  constexpr double kTwoThirds = 2.0 / 3.0, kSixth = 1.0 / 6.0;
#pragma unroll
  for (int p = 0; p < 12; ++p) r[p] = 0.0;
  if (NEED_J) {
#pragma unroll
    for (int p = 0; p < 78; ++p) J[p] = 0.0;
  }
  double h[3], zz[3], izz[3], uzt[3], vzt[3];
  double Zx0 = 0.0, Zx1 = 0.0, Zy0 = 0.0, Zy1 = 0.0;
  double Ux0 = 0.0, Ux1 = 0.0, Uy0 = 0.0, Uy1 = 0.0;
  double Vx0 = 0.0, Vx1 = 0.0, Vy0 = 0.0, Vy1 = 0.0;
  double du[3], dv[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    h[j] = 0.5 * (w.zt[j] - w.zb[j]);
    const double m = 0.5 * (w.zt[j] + w.zb[j]);
    Zx0 = fma(w.a[j], m, Zx0); Zx1 = fma(w.a[j], h[j], Zx1);
    Zy0 = fma(w.b[j], m, Zy0); Zy1 = fma(w.b[j], h[j], Zy1);
    const double ubar = 0.5 * (w.ut[j] + w.ub[j]), vbar = 0.5 * (w.vt[j] + w.vb[j]);
    du[j] = 0.5 * (w.ut[j] - w.ub[j]);
    dv[j] = 0.5 * (w.vt[j] - w.vb[j]);
    Ux0 = fma(w.a[j], ubar, Ux0); Ux1 = fma(w.a[j], du[j], Ux1);
    Uy0 = fma(w.b[j], ubar, Uy0); Uy1 = fma(w.b[j], du[j], Uy1);
    Vx0 = fma(w.a[j], vbar, Vx0); Vx1 = fma(w.a[j], dv[j], Vx1);
    Vy0 = fma(w.b[j], vbar, Vy0); Vy1 = fma(w.b[j], dv[j], Vy1);
  }
  const double hs = h[0] + h[1] + h[2];
  const double dus = du[0] + du[1] + du[2], dvs = dv[0] + dv[1] + dv[2];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    zz[a] = (3.0 * h[a] + hs) * kSixth;       // z_zeta at triangle point a
    izz[a] = 1.0 / zz[a];
    uzt[a] = (3.0 * du[a] + dus) * kSixth;    // u_zeta at point a
    vzt[a] = (3.0 * dv[a] + dvs) * kSixth;
  }
  const double W0 = w.D * kSixth;             // weight 1/6 x det = D z_zeta
  // body force: rho g grad s . int phi_(j,l) = rho g (D/6) sum_a z_zeta(a) L_j(a)
  {
    const double zs = zz[0] + zz[1] + zz[2];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double bj = rg * W0 * (3.0 * zz[j] + zs) * kSixth;
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        r[2 * (j + 3 * l)] = w.sx * bj;
        r[2 * (j + 3 * l) + 1] = w.sy * bj;
      }
    }
  }
  const double ex1 = (1.0 - glen_n) / (2.0 * glen_n);
  const double kap = (glen_n - 1.0) / (2.0 * glen_n);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const double zeta = s == 0 ? -kZeta : kZeta;
      const double f[2] = {0.5 - 0.5 * zeta, 0.5 + 0.5 * zeta};
      const double zx = fma(zeta, Zx1, Zx0), zy = fma(zeta, Zy1, Zy0);
      const double uz = uzt[a] * izz[a], vz = vzt[a] * izz[a];
      const double ux = fma(zeta, Ux1, Ux0) - zx * uz;
      const double uy = fma(zeta, Uy1, Uy0) - zy * uz;
      const double vx = fma(zeta, Vx1, Vx0) - zx * vz;
      const double vy = fma(zeta, Vy1, Vy0) - zy * vz;
      const double exy = 0.5 * (uy + vx), exz = 0.5 * uz, eyz = 0.5 * vz;
      // effective strain rate squared, eq:effeps
      double q = fma(ux, ux, fma(vy, vy, fma(ux, vy, fma(exy, exy, fma(exz, exz, eyz * eyz)))));
      const double qe = q + eps;
      const double W = W0 * zz[a];
      double c, d;
      if (N3) {
        const double y = rcbrt(qe);            // (q+eps)^(-1/3)
        c = W * w.Afac * y;                     // w * 2mu
        d = c * (y * y * y) * (1.0 / 3.0);      // c (n-1)/(2n) / (q+eps)
      } else {
        c = W * w.Afac * pow(qe, ex1);
        d = c * kap / qe;
      }
      // strain-rate vectors
      const double e1x = 2.0 * ux + vy, e1y = exy, e1z = exz;
      const double e2x = exy, e2y = ux + 2.0 * vy, e2z = eyz;
      const double Qu = e1z - e1x * zx - e1y * zy;
      const double Qv = e2z - e2x * zx - e2y * zy;
      double g[12], phx[6], phy[6], phz[6];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const double rj = (j == a ? kTwoThirds : kSixth) * 0.5 * izz[a];
        const double Pu = fma(e1x, w.a[j], e1y * w.b[j]);
        const double Pv = fma(e2x, w.a[j], e2y * w.b[j]);
#pragma unroll
        for (int l = 0; l < 2; ++l) {
          const double sg = l == 0 ? -1.0 : 1.0;
          const int i = j + 3 * l;
          g[2 * i] = fma(f[l], Pu, sg * rj * Qu);
          g[2 * i + 1] = fma(f[l], Pv, sg * rj * Qv);
          phz[i] = sg * rj;
          phx[i] = fma(w.a[j], f[l], -zx * phz[i]);
          phy[i] = fma(w.b[j], f[l], -zy * phz[i]);
        }
      }
#pragma unroll
      for (int p = 0; p < 12; ++p) r[p] = fma(c, g[p], r[p]);
      if (NEED_J) {
#pragma unroll
        for (int p = 0; p < 12; ++p) {
          const int i = p >> 1, ca = p & 1;
          const double dg = d * g[p];
          const double cx = c * phx[i], cy = c * phy[i], cz = 0.5 * c * phz[i];
#pragma unroll
          for (int qq = p; qq < 12; ++qq) {
            const int i2 = qq >> 1, cb = qq & 1;
            double hv;
            if (ca == 0 && cb == 0)
              hv = fma(2.0 * cx, phx[i2], fma(0.5 * cy, phy[i2], cz * phz[i2]));
            else if (ca == 1 && cb == 1)
              hv = fma(0.5 * cx, phx[i2], fma(2.0 * cy, phy[i2], cz * phz[i2]));
            else if (ca == 0 && cb == 1)
              hv = fma(cx, phy[i2], 0.5 * cy * phx[i2]);
            else
              hv = fma(cy, phx[i2], 0.5 * cx * phy[i2]);
            J[jidx(p, qq)] += fma(-dg, g[qq], hv);
          }
        }
      }
    }
  }
  if (w.basal) {
    // planar 3D bottom triangle, true area (reading L7)
    const double dz1 = w.zb[1] - w.zb[0], dz2 = w.zb[2] - w.zb[0];
    const double cxp = w.e1y * dz2 - dz1 * w.e2y;
    const double cyp = dz1 * w.e2x - w.e1x * dz2;
    const double area = 0.5 * sqrt(cxp * cxp + cyp * cyp + w.D * w.D);
    const double wb = area * (1.0 / 3.0);
    double M[3][3];
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int j2 = 0; j2 < 3; ++j2) M[j][j2] = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double La[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) La[j] = j == a ? kTwoThirds : kSixth;
      const double bq = wb * (La[0] * w.beta[0] + La[1] * w.beta[1] + La[2] * w.beta[2]);
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int j2 = 0; j2 < 3; ++j2) M[j][j2] = fma(bq * La[j], La[j2], M[j][j2]);
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      r[2 * j] = fma(M[j][0], w.ub[0], fma(M[j][1], w.ub[1], fma(M[j][2], w.ub[2], r[2 * j])));
      r[2 * j + 1] = fma(M[j][0], w.vb[0], fma(M[j][1], w.vb[1], fma(M[j][2], w.vb[2], r[2 * j + 1])));
      if (NEED_J) {
#pragma unroll
        for (int j2 = j; j2 < 3; ++j2) {
          J[jidx(2 * j, 2 * j2)] += M[j][j2];
          J[jidx(2 * j + 1, 2 * j2 + 1)] += M[j][j2];
        }
      }
    }
  }
}

}  // namespace fo
