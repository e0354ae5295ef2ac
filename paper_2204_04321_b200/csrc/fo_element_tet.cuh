// fo_element_tet.cuh -- NEXT-f4: the prism layer as three P1 tetrahedra
// (the Greenland 1-7 km mesh has 3 tets per prism layer).
//
// Split (reading L22): with the triangle's corners a < b < c by
// GLOBAL vertex id (TriRec.pad[0]) and their top nodes a', b', c',
//     {a, b, c, c'},  {a, b, b', c'},  {a, a', b', c'};
// every vertical quad face (x < y) gets the diagonal x-bottom -- y-top, so
// neighbouring prisms split their shared faces alike.  The tets tile the
// prism exactly (vertical, hence planar, side faces), so the prism-column
// graph of the wedge path holds every coupling (3 of its 15 node pairs per
// prism are structural zeros).
//
// Per tetrahedron (same weak form as the wedge): constant gradients
// of the barycentrics from the inverse edge matrix, one quadrature point
// (exact: the viscous integrand is constant, int phi_i = vol/4), 2 mu and
// d = 2 mu (n-1)/(2n)/(q+eps) at that point, and the exact Jacobian
//     J = vol [2 mu H - d g g^T],  g_{a,i} = eps_a . grad phi_i,
// with H the second derivative of q:
//     H_uu = 2 px px' + py py'/2 + pz pz'/2     H_uv = px py' + py px'/2
//     H_vv = px px'/2 + 2 py py' + pz pz'/2      H_vu = H_uv^T.
// The basal Robin term is the wedge's (same bottom triangle, reading L7/L8).
// Output through the wedge sink of fo_owner.cu (level blocks + residual).
#pragma once

#include "fo_element.cuh"
#include "fo_element_v4.cuh"   // pk6
#include "fo_element_ws.cuh"   // TMEM layout, oidx (tet3_element_ws)

namespace fo {

// top residual add with a run-time index: compare-select over the six entries
// keeps the sink's register-held block out of local memory
template <class Sink>
__device__ __forceinline__ void r_top_add_rt(Sink& sink, int p, double v) {
#pragma unroll
  for (int q = 0; q < 6; ++q)
    if (q == p) sink.r_top_add(q, v);
}

// SORTED: the corners already are in global-id order (fo_set_element permutes
// the triangle records), so every node index below is a compile-time constant
template <bool N3, bool SORTED, class Sink>
__device__ __forceinline__ void tet3_element(const WedgeIn& w, int order, double rg, double eps, double glen_n,
                                             Sink& sink) {
  // fresh top block, bottom-top block and top residual (the sink adds below)
#pragma unroll
  for (int i = 0; i < 21; ++i) sink.top(i, 0.0);
#pragma unroll
  for (int p = 0; p < 6; ++p) {
    sink.r_top(p, 0.0);
#pragma unroll
    for (int p2 = 0; p2 < 6; ++p2) sink.off(p, p2, 0.0);
  }
  // node positions relative to corner 0 (vertical columns: x, y per corner)
  const double X[3] = {0.0, w.e1x, w.e2x}, Y[3] = {0.0, w.e1y, w.e2y};
  const int ca = SORTED ? 0 : order & 3, cb = SORTED ? 1 : (order >> 2) & 3, cc = SORTED ? 2 : (order >> 4) & 3;
  const double ex1 = (1.0 - glen_n) / (2.0 * glen_n), kap = (glen_n - 1.0) / (2.0 * glen_n);
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    // wedge-local nodes (corner + 3 * level) of tet t
    int nd[4];
    nd[0] = ca;
    nd[1] = t == 2 ? ca + 3 : cb;
    nd[2] = t == 0 ? cc : cb + 3;
    nd[3] = cc + 3;
    double px[4], py[4], pz[4], uu[4], vv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = nd[q] % 3, top = nd[q] / 3;
      px[q] = j == 0 ? X[0] : (j == 1 ? X[1] : X[2]);
      py[q] = j == 0 ? Y[0] : (j == 1 ? Y[1] : Y[2]);
      const double zb = j == 0 ? w.zb[0] : (j == 1 ? w.zb[1] : w.zb[2]);
      const double zt = j == 0 ? w.zt[0] : (j == 1 ? w.zt[1] : w.zt[2]);
      const double ub = j == 0 ? w.ub[0] : (j == 1 ? w.ub[1] : w.ub[2]);
      const double ut = j == 0 ? w.ut[0] : (j == 1 ? w.ut[1] : w.ut[2]);
      const double vb = j == 0 ? w.vb[0] : (j == 1 ? w.vb[1] : w.vb[2]);
      const double vt = j == 0 ? w.vt[0] : (j == 1 ? w.vt[1] : w.vt[2]);
      pz[q] = top ? zt : zb;
      uu[q] = top ? ut : ub;
      vv[q] = top ? vt : vb;
    }
    // edge matrix M (columns: node q - node 0), gradients = rows of M^-1
    const double m00 = px[1] - px[0], m01 = px[2] - px[0], m02 = px[3] - px[0];
    const double m10 = py[1] - py[0], m11 = py[2] - py[0], m12 = py[3] - py[0];
    const double m20 = pz[1] - pz[0], m21 = pz[2] - pz[0], m22 = pz[3] - pz[0];
    const double c00 = m11 * m22 - m12 * m21, c01 = m12 * m20 - m10 * m22, c02 = m10 * m21 - m11 * m20;
    const double det = m00 * c00 + m01 * c01 + m02 * c02;
    const double id = 1.0 / det;
    double G[4][3];
    G[1][0] = c00 * id;
    G[1][1] = (m02 * m21 - m01 * m22) * id;
    G[1][2] = (m01 * m12 - m02 * m11) * id;
    G[2][0] = c01 * id;
    G[2][1] = (m00 * m22 - m02 * m20) * id;
    G[2][2] = (m02 * m10 - m00 * m12) * id;
    G[3][0] = c02 * id;
    G[3][1] = (m01 * m20 - m00 * m21) * id;
    G[3][2] = (m00 * m11 - m01 * m10) * id;
#pragma unroll
    for (int r = 0; r < 3; ++r) G[0][r] = -(G[1][r] + G[2][r] + G[3][r]);
    const double vol = fabs(det) * (1.0 / 6.0);
    double ux = 0, uy = 0, uz = 0, vx = 0, vy = 0, vz = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ux = fma(uu[q], G[q][0], ux); uy = fma(uu[q], G[q][1], uy); uz = fma(uu[q], G[q][2], uz);
      vx = fma(vv[q], G[q][0], vx); vy = fma(vv[q], G[q][1], vy); vz = fma(vv[q], G[q][2], vz);
    }
    const double exy = 0.5 * (uy + vx), exz = 0.5 * uz, eyz = 0.5 * vz;
    const double qq = fma(ux, ux, fma(vy, vy, fma(ux, vy, fma(exy, exy, fma(exz, exz, eyz * eyz)))));
    const double qe = qq + eps;
    double c, d;
    if (N3) {
      const double y = rcbrt_n3(qe);
      c = vol * w.Afac * y;
      d = c * (y * y * y) * (1.0 / 3.0);
    } else {
      c = vol * w.Afac * pow(qe, ex1);
      d = c * kap / qe;
    }
    const double e1x = 2.0 * ux + vy, e2y = ux + 2.0 * vy;
    double g[4][2];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      g[q][0] = fma(e1x, G[q][0], fma(exy, G[q][1], exz * G[q][2]));
      g[q][1] = fma(exy, G[q][0], fma(e2y, G[q][1], eyz * G[q][2]));
    }
    const double bq = rg * vol * 0.25;   // rho g int phi_i = rho g vol / 4
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = nd[q] % 3, top = nd[q] / 3;
      const double r0 = fma(c, g[q][0], bq * w.sx), r1 = fma(c, g[q][1], bq * w.sy);
      if (top) { r_top_add_rt(sink, 2 * j, r0); r_top_add_rt(sink, 2 * j + 1, r1); }
      else { sink.r_bot_add(2 * j, r0); sink.r_bot_add(2 * j + 1, r1); }
    }
    // Jacobian entries of node pair (q, q2), comps (a, b)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) {
        const int j = nd[q] % 3, tq = nd[q] / 3, j2 = nd[q2] % 3, tq2 = nd[q2] / 3;
        if (tq > tq2) continue;   // (top, bottom) = transpose of (bottom, top)
        const double xx = G[q][0] * G[q2][0], yy = G[q][1] * G[q2][1], zz = G[q][2] * G[q2][2];
        const double xy = G[q][0] * G[q2][1], yx = G[q][1] * G[q2][0];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            double h;
            if (a == 0 && b == 0) h = fma(2.0, xx, 0.5 * (yy + zz));
            else if (a == 1 && b == 1) h = fma(2.0, yy, 0.5 * (xx + zz));
            else if (a == 0) h = fma(0.5, yx, xy);    // row u_q, column v_q2
            else h = fma(0.5, xy, yx);                // row v_q, column u_q2
            const double v = fma(c, h, -d * g[q][a] * g[q2][b]);
            const int p = 2 * j + a, p2 = 2 * j2 + b;
            if (tq == 0 && tq2 == 0) {
              if (p <= p2) sink.bot_add(p, p2, v);
            } else if (tq == 1 && tq2 == 1) {
              if (p <= p2) sink.top_add(pk6(p, p2), v);
            } else {
              sink.off_add(p, p2, v);
            }
          }
      }
  }
  // basal Robin term on layer 0 (readings L6-L8): the wedge's
  if (w.basal) {
    constexpr double kTwoThirds = 2.0 / 3.0, kSixth = 1.0 / 6.0;
    const double dz1 = w.zb[1] - w.zb[0], dz2 = w.zb[2] - w.zb[0];
    const double cxp = w.e1y * dz2 - dz1 * w.e2y;
    const double cyp = dz1 * w.e2x - w.e1x * dz2;
    const double wb = (1.0 / 6.0) * sqrt(cxp * cxp + cyp * cyp + w.D * w.D);
    double Mb[3][3];
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int j2 = 0; j2 < 3; ++j2) Mb[j][j2] = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double La[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) La[j] = j == a ? kTwoThirds : kSixth;
      const double bq = wb * (La[0] * w.beta[0] + La[1] * w.beta[1] + La[2] * w.beta[2]);
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int j2 = 0; j2 < 3; ++j2) Mb[j][j2] = fma(bq * La[j], La[j2], Mb[j][j2]);
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      sink.r_bot_add(2 * j, Mb[j][0] * w.ub[0] + Mb[j][1] * w.ub[1] + Mb[j][2] * w.ub[2]);
      sink.r_bot_add(2 * j + 1, Mb[j][0] * w.vb[0] + Mb[j][1] * w.vb[1] + Mb[j][2] * w.vb[2]);
#pragma unroll
      for (int j2 = j; j2 < 3; ++j2) {
        sink.bot_add(2 * j, 2 * j2, Mb[j][j2]);
        sink.bot_add(2 * j + 1, 2 * j2 + 1, Mb[j][j2]);
      }
    }
  }
}


// ---------------------------------------------------------------------------
// The tetrahedral prism for the warp-specialised kernel (KA-ws, DESIGN.md
// section 7): same mathematics as tet3_element (SORTED corners), same output
// contract as wedge_element_ws -- TMEM BB <- D(k) = HELD (top block of the
// wedge below) + this prism's (bottom, bottom) block and bottom residual,
// TMEM HELD <- its (top, top) block and top residual (dmap layout, residual at
// 21 + p), acc <- the (bottom, top) block (oidx layout).  The three tets'
// gradients, strain-rate vectors and viscosity factors are computed once and
// stashed in the thread's TMEM row (cols 0 .. 131, the wedge's C / O stash
// region), then each block is accumulated in registers in its own pass.
namespace tetws {
constexpr uint32_t kTet = 44;   // TMEM columns per tet record: G[4][3], g[4][2], c, d (22 doubles)
}

template <bool N3>
__device__ __forceinline__ void tet3_element_ws(const WedgeIn& w, double rg, double eps, double glen_n, uint32_t tm,
                                                double (&acc)[36]) {
  // SORTED corners: a = 0, b = 1, c = 2; tets {a,b,c,c'}, {a,b,b',c'}, {a,a',b',c'}
  constexpr int ND[3][4] = {{0, 1, 2, 5}, {0, 1, 4, 5}, {0, 3, 4, 5}};
  const double X[3] = {0.0, w.e1x, w.e2x}, Y[3] = {0.0, w.e1y, w.e2y};
  const double ex1 = (1.0 - glen_n) / (2.0 * glen_n), kap = (glen_n - 1.0) / (2.0 * glen_n);
  double rb[6], rt[6];
#pragma unroll
  for (int p = 0; p < 6; ++p) rb[p] = rt[p] = 0.0;
  // ---- 1. per tet: gradients, viscosity, residual; record -> TMEM
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    double px[4], py[4], pz[4], uu[4], vv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = ND[t][q] % 3, top = ND[t][q] / 3;
      px[q] = X[j];
      py[q] = Y[j];
      pz[q] = top ? w.zt[j] : w.zb[j];
      uu[q] = top ? w.ut[j] : w.ub[j];
      vv[q] = top ? w.vt[j] : w.vb[j];
    }
    const double m00 = px[1] - px[0], m01 = px[2] - px[0], m02 = px[3] - px[0];
    const double m10 = py[1] - py[0], m11 = py[2] - py[0], m12 = py[3] - py[0];
    const double m20 = pz[1] - pz[0], m21 = pz[2] - pz[0], m22 = pz[3] - pz[0];
    const double c00 = m11 * m22 - m12 * m21, c01 = m12 * m20 - m10 * m22, c02 = m10 * m21 - m11 * m20;
    const double det = m00 * c00 + m01 * c01 + m02 * c02;
    const double id = 1.0 / det;
    double rec[22];   // G[4][3], g[4][2], c, d
    double (*G)[3] = reinterpret_cast<double (*)[3]>(rec);
    G[1][0] = c00 * id;
    G[1][1] = (m02 * m21 - m01 * m22) * id;
    G[1][2] = (m01 * m12 - m02 * m11) * id;
    G[2][0] = c01 * id;
    G[2][1] = (m00 * m22 - m02 * m20) * id;
    G[2][2] = (m02 * m10 - m00 * m12) * id;
    G[3][0] = c02 * id;
    G[3][1] = (m01 * m20 - m00 * m21) * id;
    G[3][2] = (m00 * m11 - m01 * m10) * id;
#pragma unroll
    for (int r = 0; r < 3; ++r) G[0][r] = -(G[1][r] + G[2][r] + G[3][r]);
    const double vol = fabs(det) * (1.0 / 6.0);
    double ux = 0, uy = 0, uz = 0, vx = 0, vy = 0, vz = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ux = fma(uu[q], G[q][0], ux); uy = fma(uu[q], G[q][1], uy); uz = fma(uu[q], G[q][2], uz);
      vx = fma(vv[q], G[q][0], vx); vy = fma(vv[q], G[q][1], vy); vz = fma(vv[q], G[q][2], vz);
    }
    const double exy = 0.5 * (uy + vx), exz = 0.5 * uz, eyz = 0.5 * vz;
    const double qq = fma(ux, ux, fma(vy, vy, fma(ux, vy, fma(exy, exy, fma(exz, exz, eyz * eyz)))));
    const double qe = qq + eps;
    double c, d;
    if (N3) {
      const double y = rcbrt_n3(qe);
      c = vol * w.Afac * y;
      d = c * (y * y * y) * (1.0 / 3.0);
    } else {
      c = vol * w.Afac * pow(qe, ex1);
      d = c * kap / qe;
    }
    const double e1x = 2.0 * ux + vy, e2y = ux + 2.0 * vy;
    const double bq = rg * vol * 0.25;   // rho g int phi_i = rho g vol / 4
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double g0 = fma(e1x, G[q][0], fma(exy, G[q][1], exz * G[q][2]));
      const double g1 = fma(exy, G[q][0], fma(e2y, G[q][1], eyz * G[q][2]));
      rec[12 + 2 * q] = g0;
      rec[13 + 2 * q] = g1;
      const int j = ND[t][q] % 3;
      const double r0 = fma(c, g0, bq * w.sx), r1 = fma(c, g1, bq * w.sy);
      if (ND[t][q] / 3) { rt[2 * j] += r0; rt[2 * j + 1] += r1; }
      else { rb[2 * j] += r0; rb[2 * j + 1] += r1; }
    }
    rec[20] = c;
    rec[21] = d;
    tmem::st<22>(tm + tetws::kTet * t, rec);
  }
  // entry (node q, comp a; node q2, comp b) of one tet's c H - d g g^T
  auto entry = [](const double* r, int q, int a, int q2, int b) {
    const double* G = r;
    const double xx = G[3 * q] * G[3 * q2], yy = G[3 * q + 1] * G[3 * q2 + 1], zz = G[3 * q + 2] * G[3 * q2 + 2];
    const double xy = G[3 * q] * G[3 * q2 + 1], yx = G[3 * q + 1] * G[3 * q2];
    double h;
    if (a == 0 && b == 0) h = fma(2.0, xx, 0.5 * (yy + zz));
    else if (a == 1 && b == 1) h = fma(2.0, yy, 0.5 * (xx + zz));
    else if (a == 0) h = fma(0.5, yx, xy);
    else h = fma(0.5, xy, yx);
    return fma(r[20], h, -r[21] * r[12 + 2 * q + a] * r[12 + 2 * q2 + b]);
  };
  tmem::wait_st();
  // ---- 2. D(k) = HELD + (bottom, bottom) blocks + bottom residual (+ basal) -> TMEM BB
  {
    double hd[27];
    tmem::ld<27>(tm + kTmHeld, hd);
#pragma unroll
    for (int p = 0; p < 6; ++p) hd[21 + p] += rb[p];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      double r[22];
      tmem::ld<22>(tm + tetws::kTet * t, r);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int q2 = 0; q2 < 4; ++q2) {
          if (ND[t][q] / 3 || ND[t][q2] / 3) continue;
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const int p = 2 * (ND[t][q] % 3) + a, p2 = 2 * (ND[t][q2] % 3) + b;
              if (p <= p2) hd[dmap(p, p2)] += entry(r, q, a, q2, b);
            }
        }
    }
    if (w.basal) {   // the wedge's basal Robin term (readings L6-L8)
      constexpr double kTwoThirds = 2.0 / 3.0, kSixth = 1.0 / 6.0;
      const double dz1 = w.zb[1] - w.zb[0], dz2 = w.zb[2] - w.zb[0];
      const double cxp = w.e1y * dz2 - dz1 * w.e2y;
      const double cyp = dz1 * w.e2x - w.e1x * dz2;
      const double wb = (1.0 / 6.0) * sqrt(cxp * cxp + cyp * cyp + w.D * w.D);
      double Mb[3][3];
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int j2 = 0; j2 < 3; ++j2) Mb[j][j2] = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double La[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) La[j] = j == a ? kTwoThirds : kSixth;
        const double bq = wb * (La[0] * w.beta[0] + La[1] * w.beta[1] + La[2] * w.beta[2]);
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
          for (int j2 = 0; j2 < 3; ++j2) Mb[j][j2] = fma(bq * La[j], La[j2], Mb[j][j2]);
      }
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        hd[21 + 2 * j] += Mb[j][0] * w.ub[0] + Mb[j][1] * w.ub[1] + Mb[j][2] * w.ub[2];
        hd[22 + 2 * j] += Mb[j][0] * w.vb[0] + Mb[j][1] * w.vb[1] + Mb[j][2] * w.vb[2];
#pragma unroll
        for (int j2 = j; j2 < 3; ++j2) {
          hd[dmap(2 * j, 2 * j2)] += Mb[j][j2];
          hd[dmap(2 * j + 1, 2 * j2 + 1)] += Mb[j][j2];
        }
      }
    }
    tmem::st<27>(tm + kTmBB, hd);
  }
  // ---- 3. HELD <- (top, top) blocks + top residual
  {
    double ht[27];
#pragma unroll
    for (int i = 0; i < 21; ++i) ht[i] = 0.0;
#pragma unroll
    for (int p = 0; p < 6; ++p) ht[21 + p] = rt[p];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      double r[22];
      tmem::ld<22>(tm + tetws::kTet * t, r);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int q2 = 0; q2 < 4; ++q2) {
          if (!(ND[t][q] / 3) || !(ND[t][q2] / 3)) continue;
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const int p = 2 * (ND[t][q] % 3) + a, p2 = 2 * (ND[t][q2] % 3) + b;
              if (p <= p2) ht[dmap(p, p2)] += entry(r, q, a, q2, b);
            }
        }
    }
    tmem::st<27>(tm + kTmHeld, ht);   // HELD was read in step 2 (ld + wait::ld)
  }
  // ---- 4. the (bottom, top) block -> acc
#pragma unroll
  for (int i = 0; i < 36; ++i) acc[i] = 0.0;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    double r[22];
    tmem::ld<22>(tm + tetws::kTet * t, r);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) {
        if (ND[t][q] / 3 || !(ND[t][q2] / 3)) continue;
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int p = 2 * (ND[t][q] % 3) + a, p2 = 2 * (ND[t][q2] % 3) + b;
            acc[oidx(p, p2)] += entry(r, q, a, q2, b);
          }
      }
  }
}

}  // namespace fo
