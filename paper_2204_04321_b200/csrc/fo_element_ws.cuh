// fo_element_ws.cuh -- the wedge element of the warp-specialised patch kernel
// (KA-ws): the same mathematics as fo_element_v4.cuh
// (PAPER.md eq:FOStokes P:83-89, strain rates P:90-100, Glen's law
// eq:effvisc / eq:effeps P:102-108 regularised by reading L1, driving stress
// P:85-86 with reading L10, basal sliding P:128-132 with readings L6-L8, the
// residual eq:residual P:155-158 and its exact Jacobian eq:linearsystem
// P:160-164; derivation DESIGN.md section 6), with every intermediate block
// kept in the thread's private TMEM row instead of the shared D / O arrays --
// those belong to the scatter warpgroup, which gathers the previous level
// from them while this element is computed.
//
// Order (one accumulator set live at a time):
//   1. per-point compact data (d, e1x, e1y, Qu, e2y, Qv)         -> TMEM C
//   2. frozen-viscosity part in closed form (v4's hpart4): the
//      (bottom, bottom) entries -> TMEM BB, the (bottom, top) block -> TMEM O,
//      the (top, top) entries stay in registers (at)
//   3. basal mass and driving stress; rank-1 (bottom,bottom) + (top,top) pass
//      with both residual halves; then the level-k diagonal block
//      D(k) = HELD (top block of wedge k-1) + bottom block        -> TMEM BB,
//      HELD <- top block + top residual of this wedge
//   4. rank-1 (bottom, top) pass onto TMEM O                      -> acc[36]
// The caller copies acc (O) and TMEM BB (D) into shared memory once the
// scatter warps have released them.
#pragma once

#include "fo_element.cuh"
#include "fo_element_v4.cuh"
#include "fo_tmem.cuh"

namespace fo {

// TMEM column offsets of the per-thread row (doubles take 2 columns)
constexpr uint32_t kTmC = 0;      // 6 points x 6 doubles
constexpr uint32_t kTmO = 72;     // 36 doubles, node-pair order (oidx)
constexpr uint32_t kTmBB = 144;   // 21 frozen (bottom,bottom) entries (bidx), then D(k) (dmap, 27)
constexpr uint32_t kTmHeld = 198; // 27 doubles (dmap): top block + top residual of the last wedge
constexpr uint32_t kTmCols = 256; // allocation per CTA (252 used)

// node pairs (j <= j2) in the order (0,0) (0,1) (0,2) (1,1) (1,2) (2,2)
__host__ __device__ constexpr int npair(int j, int j2) { return j == 0 ? j2 : (j == 1 ? 2 + j2 : 5); }
// O stash: diagonal node pairs 4 entries [ca][cb], off-diagonal 8: O(2j+ca, 2j2+cb)
// at [ca][cb], then O(2j2+cb, 2j+ca) at 4 + [cb][ca]
__host__ __device__ constexpr int onp_off(int np) {
  return np == 0 ? 0 : np == 1 ? 4 : np == 2 ? 12 : np == 3 ? 20 : np == 4 ? 24 : 32;
}
__host__ __device__ constexpr int oidx(int p, int p2) {
  return (p >> 1) == (p2 >> 1) ? onp_off(npair(p >> 1, p >> 1)) + 2 * (p & 1) + (p2 & 1)
         : (p >> 1) < (p2 >> 1) ? onp_off(npair(p >> 1, p2 >> 1)) + 2 * (p & 1) + (p2 & 1)
                                : onp_off(npair(p2 >> 1, p >> 1)) + 4 + 2 * (p & 1) + (p2 & 1);
}
// BB stash (p <= p2): diagonal node pairs 3 entries, off-diagonal 4
__host__ __device__ constexpr int bnp_off(int np) {
  return np == 0 ? 0 : np == 1 ? 3 : np == 2 ? 7 : np == 3 ? 11 : np == 4 ? 14 : 18;
}
__host__ __device__ constexpr int bidx(int p, int p2) {
  return (p >> 1) == (p2 >> 1) ? bnp_off(npair(p >> 1, p >> 1)) + (p & 1) + (p2 & 1)
                               : bnp_off(npair(p >> 1, p2 >> 1)) + 2 * (p & 1) + (p2 & 1);
}

template <bool N3>
__device__ __forceinline__ void wedge_element_ws(const WedgeIn& w, double rg, double eps, double glen_n,
                                                 uint32_t tm, double (&acc)[36]) {
  constexpr double kZeta = 0.57735026918962576451;   // 1/sqrt(3)
  constexpr double kTwoThirds = 2.0 / 3.0, kSixth = 1.0 / 6.0;
  // ---- per-wedge setup (column-structured geometry)
  double zz[3], rho[3], uz[3], vz[3];
  double Zx0 = 0.0, Zx1 = 0.0, Zy0 = 0.0, Zy1 = 0.0;
  double Ux0 = 0.0, Ux1 = 0.0, Uy0 = 0.0, Uy1 = 0.0;
  double Vx0 = 0.0, Vx1 = 0.0, Vy0 = 0.0, Vy1 = 0.0;
  {
    double h[3], du[3], dv[3];
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
      zz[a] = (3.0 * h[a] + hs) * kSixth;           // z_zeta at triangle point a
      const double izz = rcp_geo(zz[a]);
      rho[a] = 0.5 * izz;                           // r_j(a) = L_j(a) rho_a
      uz[a] = (3.0 * du[a] + dus) * kSixth * izz;   // u_z at point a
      vz[a] = (3.0 * dv[a] + dvs) * kSixth * izz;
    }
  }
  const double W0 = w.D * kSixth;   // quadrature weight 1/6 x det, det = 2|T| z_zeta
  // ---- 1. per-point compact data -> TMEM C: [d, e1x, e1y(=e2x), Qu, e2y, Qv]
  //      (Qu, Qv stored as rho_a Q / 6: r_j Q = (j == a ? 4 : 1) x the stored value)
  double cq[6];
  {
    const double ex1 = (1.0 - glen_n) / (2.0 * glen_n);
    const double kap = (glen_n - 1.0) / (2.0 * glen_n);
    double qe[6];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int q = 2 * a + s;
        const double zeta = s == 0 ? -kZeta : kZeta;
        const double zx = fma(zeta, Zx1, Zx0), zy = fma(zeta, Zy1, Zy0);
        const double ux = fma(zeta, Ux1, Ux0) - zx * uz[a];
        const double uy = fma(zeta, Uy1, Uy0) - zy * uz[a];
        const double vx = fma(zeta, Vx1, Vx0) - zx * vz[a];
        const double vy = fma(zeta, Vy1, Vy0) - zy * vz[a];
        const double exy = 0.5 * (uy + vx), exz = 0.5 * uz[a], eyz = 0.5 * vz[a];
        // effective strain rate squared, eq:effeps
        const double qq = fma(ux, ux, fma(vy, vy, fma(ux, vy, fma(exy, exy, fma(exz, exz, eyz * eyz)))));
        qe[q] = qq + eps;
        // strain-rate vectors
        const double e1x = 2.0 * ux + vy, e1y = exy, e1z = exz;
        const double e2x = exy, e2y = ux + 2.0 * vy, e2z = eyz;
        const double r6 = rho[a] * kSixth;
        const double v5[5] = {e1x, e1y, (e1z - e1x * zx - e1y * zy) * r6, e2y, (e2z - e2x * zx - e2y * zy) * r6};
        tmem::st<4>(tm + kTmC + 12 * q + 2, v5);
        tmem::st<1>(tm + kTmC + 12 * q + 10, v5 + 4);
      }
    }
    // the six viscosities together: independent rcbrt chains interleave
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const int a = q >> 1;
      const double W = W0 * (a == 0 ? zz[0] : (a == 1 ? zz[1] : zz[2]));
      double c, d;
      if (N3) {
        const double y = rcbrt_n3(qe[q]);            // (q + eps)^(-1/3)
        c = W * w.Afac * y;                           // w_q 2 mu_q
        d = c * (y * y * y) * (1.0 / 3.0);            // c (n-1)/(2n) / (q+eps)
      } else {
        c = W * w.Afac * pow(qe[q], ex1);
        d = c * kap / qe[q];
      }
      cq[q] = c;
      tmem::st<1>(tm + kTmC + 12 * q, &d);
    }
  }
  // ---- 2. frozen-viscosity part in closed form from the six c_q (v4)
  double at[21];   // (top, top), pk6 order
  {
    double F[3];
    double T2x[2][3], T2y[2][3];
    double KKuu[6], KKvv[6], KKuv[6];
    {
      double S[3], Dd[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        S[a] = cq[2 * a] + cq[2 * a + 1];
        Dd[a] = kZeta * (cq[2 * a + 1] - cq[2 * a]);
      }
      const double St = S[0] + S[1] + S[2], Dt = Dd[0] + Dd[1] + Dd[2];
      F[0] = St * (1.0 / 3.0) - 0.5 * Dt;
      F[1] = St * kSixth;
      F[2] = St * (1.0 / 3.0) + 0.5 * Dt;
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        const double sg = l == 0 ? -1.0 : 1.0;
        double Yx[3], Yy[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double s3 = S[a] * (1.0 / 3.0);
          Yx[a] = rho[a] * 0.5 * fma(Zx0, S[a], fma(Zx1 + sg * Zx0, Dd[a], sg * Zx1 * s3));
          Yy[a] = rho[a] * 0.5 * fma(Zy0, S[a], fma(Zy1 + sg * Zy0, Dd[a], sg * Zy1 * s3));
        }
        const double sx6 = (Yx[0] + Yx[1] + Yx[2]) * kSixth, sy6 = (Yy[0] + Yy[1] + Yy[2]) * kSixth;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          T2x[l][j] = fma(0.5, Yx[j], sx6);
          T2y[l][j] = fma(0.5, Yy[j], sy6);
        }
      }
      double ku[3], kv[3], kuv[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double s3 = S[a] * (1.0 / 3.0);
        const double XXx = fma(Zx0 * Zx0, S[a], fma(2.0 * Zx0 * Zx1, Dd[a], Zx1 * Zx1 * s3));
        const double XXy = fma(Zy0 * Zy0, S[a], fma(2.0 * Zy0 * Zy1, Dd[a], Zy1 * Zy1 * s3));
        const double XXxy = fma(Zx0 * Zy0, S[a], fma(fma(Zx0, Zy1, Zx1 * Zy0), Dd[a], Zx1 * Zy1 * s3));
        const double r2 = rho[a] * rho[a];
        ku[a] = r2 * fma(2.0, XXx, 0.5 * (XXy + S[a]));
        kv[a] = r2 * fma(2.0, XXy, 0.5 * (XXx + S[a]));
        kuv[a] = r2 * 1.5 * XXxy;
      }
      const double su = (ku[0] + ku[1] + ku[2]) * (1.0 / 36.0);
      const double sv = (kv[0] + kv[1] + kv[2]) * (1.0 / 36.0);
      const double suv = (kuv[0] + kuv[1] + kuv[2]) * (1.0 / 36.0);
      int i = 0;
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int j2 = j; j2 < 3; ++j2) {
          const double wj = j == j2 ? 15.0 / 36.0 : 3.0 / 36.0;
          const double pu = j == j2 ? ku[j] : ku[j] + ku[j2];
          const double pv = j == j2 ? kv[j] : kv[j] + kv[j2];
          const double puv = j == j2 ? kuv[j] : kuv[j] + kuv[j2];
          KKuu[i] = fma(wj, pu, su);
          KKvv[i] = fma(wj, pv, sv);
          KKuv[i] = fma(wj, puv, suv);
          ++i;
        }
    }
    double a2[3], ah[3], b2[3], bh[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      a2[j] = 2.0 * w.a[j]; ah[j] = 0.5 * w.a[j];
      b2[j] = 2.0 * w.b[j]; bh[j] = 0.5 * w.b[j];
    }
    // the four level blocks of one (row comp ca, node j; column comp cb, node
    // j2) entry: entry(l, l2) = F_{l+l2} AA - s(l2) Rt(l) - s(l) Ct(l2) + s(l) s(l2) KK
    auto hpart4 = [&](int ca, int j, int cb, int j2, double& e00, double& e01, double& e10, double& e11) {
      const int kk = j <= j2 ? (j * 3 - (j * (j - 1)) / 2 + (j2 - j)) : (j2 * 3 - (j2 * (j2 - 1)) / 2 + (j - j2));
      const double aj = w.a[j], bj = w.b[j], aj2 = w.a[j2], bj2 = w.b[j2];
      double AA, KK, Rt[2], Ct[2];
      if (ca == 0 && cb == 0) {
        AA = fma(a2[j], aj2, bh[j] * bj2);
        KK = KKuu[kk];
#pragma unroll
        for (int l = 0; l < 2; ++l) {
          Rt[l] = fma(a2[j], T2x[l][j2], bh[j] * T2y[l][j2]);
          Ct[l] = fma(a2[j2], T2x[l][j], bh[j2] * T2y[l][j]);
        }
      } else if (ca == 1 && cb == 1) {
        AA = fma(ah[j], aj2, b2[j] * bj2);
        KK = KKvv[kk];
#pragma unroll
        for (int l = 0; l < 2; ++l) {
          Rt[l] = fma(ah[j], T2x[l][j2], b2[j] * T2y[l][j2]);
          Ct[l] = fma(ah[j2], T2x[l][j], b2[j2] * T2y[l][j]);
        }
      } else if (ca == 0) {
        AA = fma(aj, bj2, ah[j2] * bj);
        KK = KKuv[kk];
#pragma unroll
        for (int l = 0; l < 2; ++l) {
          Rt[l] = fma(aj, T2y[l][j2], bh[j] * T2x[l][j2]);
          Ct[l] = fma(bj2, T2x[l][j], ah[j2] * T2y[l][j]);
        }
      } else {
        AA = fma(aj2, bj, ah[j] * bj2);
        KK = KKuv[kk];
#pragma unroll
        for (int l = 0; l < 2; ++l) {
          Rt[l] = fma(bj, T2x[l][j2], ah[j] * T2y[l][j2]);
          Ct[l] = fma(aj2, T2y[l][j], bh[j2] * T2x[l][j]);
        }
      }
      const double X = fma(F[1], AA, -KK);
      e01 = (X - Rt[0]) + Ct[1];
      e10 = (X + Rt[1]) - Ct[0];
      e00 = fma(F[0], AA, KK + (Rt[0] + Ct[0]));
      e11 = fma(F[2], AA, KK - (Rt[1] + Ct[1]));
    };
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int j2 = j; j2 < 3; ++j2) {
        double ob[8], bb[4];
#pragma unroll
        for (int ca = 0; ca < 2; ++ca)
#pragma unroll
          for (int cb = 0; cb < 2; ++cb) {
            const int p = 2 * j + ca, p2 = 2 * j2 + cb;
            double e00, e01, e10, e11;
            hpart4(ca, j, cb, j2, e00, e01, e10, e11);
            if (p <= p2) {
              at[pk6(p, p2)] = e11;
              bb[bidx(p, p2) - bnp_off(npair(j, j2))] = e00;
            }
            ob[2 * ca + cb] = e01;
            if (j != j2) ob[4 + 2 * cb + ca] = e10;
          }
        const uint32_t oo = tm + kTmO + 2 * onp_off(npair(j, j2));
        const uint32_t bo = tm + kTmBB + 2 * bnp_off(npair(j, j2));
        if (j != j2) {
          tmem::st<8>(oo, ob);
          tmem::st<4>(bo, bb);
        } else {
          tmem::st<4>(oo, ob);
          tmem::st<3>(bo, bb);
        }
      }
  }
  // ---- 3. basal mass, driving stress, rank-1 (bottom,bottom) + (top,top) pass
  double rb[6], rt[6];
  double Mb[6];   // basal P1 mass block (j <= j2), layer 0 only
  {
    const double zs = zz[0] + zz[1] + zz[2];
#pragma unroll
    for (int j = 0; j < 3; ++j) {   // driving stress rho g grad s . int phi (reading L10)
      const double bj = rg * W0 * (3.0 * zz[j] + zs) * kSixth;
      rb[2 * j] = w.sx * bj;
      rb[2 * j + 1] = w.sy * bj;
      rt[2 * j] = w.sx * bj;
      rt[2 * j + 1] = w.sy * bj;
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) Mb[i] = 0.0;
    if (w.basal) {   // P:128-131, readings L6-L8: 3-point rule on the 3D bottom triangle
      const double dz1 = w.zb[1] - w.zb[0], dz2 = w.zb[2] - w.zb[0];
      const double cxp = w.e1y * dz2 - dz1 * w.e2y;
      const double cyp = dz1 * w.e2x - w.e1x * dz2;
      const double wb = (1.0 / 6.0) * sqrt(cxp * cxp + cyp * cyp + w.D * w.D);   // |T3D| / 3
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double La[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) La[j] = j == a ? kTwoThirds : kSixth;
        const double bq = wb * (La[0] * w.beta[0] + La[1] * w.beta[1] + La[2] * w.beta[2]);
        int i = 0;
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
          for (int j2 = j; j2 < 3; ++j2) Mb[i] = fma(bq * La[j], La[j2], Mb[i]), ++i;
      }
      auto mb = [&](int j, int j2) { return Mb[j <= j2 ? (j * 3 - (j * (j - 1)) / 2 + (j2 - j)) : (j2 * 3 - (j2 * (j2 - 1)) / 2 + (j - j2))]; };
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        rb[2 * j] = fma(mb(j, 0), w.ub[0], fma(mb(j, 1), w.ub[1], fma(mb(j, 2), w.ub[2], rb[2 * j])));
        rb[2 * j + 1] = fma(mb(j, 0), w.vb[0], fma(mb(j, 1), w.vb[1], fma(mb(j, 2), w.vb[2], rb[2 * j + 1])));
      }
    }
  }
  tmem::wait_st();   // C and the frozen stashes are in TMEM
  {
    double ab[21];   // bidx order
    tmem::ld<21>(tm + kTmBB, ab);
    if (w.basal) {
      int i = 0;
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int j2 = j; j2 < 3; ++j2) {
          ab[bidx(2 * j, 2 * j2)] += Mb[i];
          ab[bidx(2 * j + 1, 2 * j2 + 1)] += Mb[i];
          ++i;
        }
    }
#pragma unroll 2
    for (int q = 0; q < 6; ++q) {
      const int a = q >> 1;
      const double zeta = (q & 1) ? kZeta : -kZeta;
      const double f0 = 0.5 - 0.5 * zeta, f1 = 0.5 + 0.5 * zeta;
      const double cc = q == 0 ? cq[0] : q == 1 ? cq[1] : q == 2 ? cq[2] : q == 3 ? cq[3] : q == 4 ? cq[4] : cq[5];
      double pt[6];
      tmem::ld<6>(tm + kTmC + 12 * q, pt);
      const double dd = pt[0];
      const double qu6 = pt[3], qv6 = pt[5], qu4 = 4.0 * qu6, qv4 = 4.0 * qv6;
      double gb[6], gt[6], dgb[6], dgt[6];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const double qu = j == a ? qu4 : qu6, qv = j == a ? qv4 : qv6;
        const double pu = fma(pt[1], w.a[j], pt[2] * w.b[j]);
        const double pv = fma(pt[2], w.a[j], pt[4] * w.b[j]);
        gb[2 * j] = fma(f0, pu, -qu);
        gb[2 * j + 1] = fma(f0, pv, -qv);
        gt[2 * j] = fma(f1, pu, qu);
        gt[2 * j + 1] = fma(f1, pv, qv);
      }
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        dgb[p] = dd * gb[p];
        dgt[p] = dd * gt[p];
        rb[p] = fma(cc, gb[p], rb[p]);   // R_{a,(j,0)} += c_q g
        rt[p] = fma(cc, gt[p], rt[p]);   // R_{a,(j,1)} += c_q g
      }
#pragma unroll
      for (int p = 0; p < 6; ++p)
#pragma unroll
        for (int p2 = p; p2 < 6; ++p2) {
          ab[bidx(p, p2)] = fma(-dgb[p], gb[p2], ab[bidx(p, p2)]);
          at[pk6(p, p2)] = fma(-dgt[p], gt[p2], at[pk6(p, p2)]);
        }
    }
    // D(k) = HELD (top block of wedge k-1) + this bottom block; HELD <- top block
    double hd[27];
    tmem::ld<27>(tm + kTmHeld, hd);
#pragma unroll
    for (int p = 0; p < 6; ++p)
#pragma unroll
      for (int p2 = p; p2 < 6; ++p2) hd[dmap(p, p2)] += ab[bidx(p, p2)];
#pragma unroll
    for (int p = 0; p < 6; ++p) hd[21 + p] += rb[p];
    tmem::st<27>(tm + kTmBB, hd);
#pragma unroll
    for (int p = 0; p < 6; ++p)
#pragma unroll
      for (int p2 = p; p2 < 6; ++p2) hd[dmap(p, p2)] = at[pk6(p, p2)];
#pragma unroll
    for (int p = 0; p < 6; ++p) hd[21 + p] = rt[p];
    tmem::st<27>(tm + kTmHeld, hd);
  }
  // ---- 4. rank-1 (bottom, top) pass onto the frozen O block
  tmem::ld<36>(tm + kTmO, acc);
#pragma unroll 2
  for (int q = 0; q < 6; ++q) {
    const int a = q >> 1;
    const double zeta = (q & 1) ? kZeta : -kZeta;
    const double f0 = 0.5 - 0.5 * zeta, f1 = 0.5 + 0.5 * zeta;
    double pt[6];
    tmem::ld<6>(tm + kTmC + 12 * q, pt);
    const double dg = pt[0];
    const double qu6 = pt[3], qv6 = pt[5], qu4 = 4.0 * qu6, qv4 = 4.0 * qv6;
    double gb[6], gt[6];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double qu = j == a ? qu4 : qu6, qv = j == a ? qv4 : qv6;
      const double pu = fma(pt[1], w.a[j], pt[2] * w.b[j]);
      const double pv = fma(pt[2], w.a[j], pt[4] * w.b[j]);
      gb[2 * j] = dg * fma(f0, pu, -qu);
      gb[2 * j + 1] = dg * fma(f0, pv, -qv);
      gt[2 * j] = fma(f1, pu, qu);
      gt[2 * j + 1] = fma(f1, pv, qv);
    }
#pragma unroll
    for (int p = 0; p < 6; ++p)
#pragma unroll
      for (int p2 = 0; p2 < 6; ++p2) acc[oidx(p, p2)] = fma(-gb[p], gt[p2], acc[oidx(p, p2)]);
  }
}

}  // namespace fo
