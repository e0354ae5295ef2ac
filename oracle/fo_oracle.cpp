/*
 * fo_oracle.cpp -- plain, slow, serial CPU oracle for the FO-Stokes residual and
 * Newton Jacobian on extruded wedge meshes.
 *
 * TEST INFRASTRUCTURE ONLY (see fo_oracle.h).  Shares no code with the CUDA path.
 * Compiled -O2, no fast-math, no threads, no atomics.
 *
 * Every step follows PAPER.md (/root/reference/PAPER.md, "P:n" = line n) and the
 * readings listed in DESIGN.md ("Readings of the paper"); the step-by-step order
 * is SURVEY.md section 8(c) c2:
 *   1. validate the footprint (reading L16/L17),
 *   2. extrude: node = c*(L+1)+k, z = (s-H) + sigma_k*H,
 *      floating mask beta = 0 where rho*H < -rho_w*b (reading L9),
 *   3. brute-force graph (every element-coupled DOF pair, sorted, reading L16),
 *   4. per wedge, per quadrature point (3-point triangle rule x 2-point Gauss,
 *      reading L4) a GENERIC isoparametric 3x3 Jacobian, its determinant and
 *      cofactor inverse, grad(phi) = J^-T grad_ref(phi);
 *      strain rates, effective strain rate, Glen viscosity
 *      2mu = A^(-1/n) (q + eps_reg)^((1-n)/(2n)) (P:103-105 + reading L1),
 *      residual R_{a,i} += w detJ [2mu eps_a . grad(phi_i) + rho g ds/dx_a phi_i]
 *      (weak form of eq:FOStokes P:85-86, surface BC P:124-126 contributes nothing),
 *   5. basal Robin term on layer-0 wedges (readings L6-L8):
 *      + int_{Gamma_beta} beta u_a phi_i dGamma, 3-point rule on the planar 3D
 *      bottom triangle,
 *   6. scatter with plain += (no atomics), J entries located by binary search,
 *   Jacobian: the same residual code instantiated on Dual<12> (forward AD seeded
 *   on the wedge's 12 DOFs), the analogue of the paper's Sacado SFad.
 *   NEXT-f1 (term ORA_LATERAL): lateral margin faces, P:133-140 / reading L12;
 *   NEXT-f3 (T_star): A = A0 exp(-Q / (R T*)) per wedge.
 */
#include "fo_oracle.h"

#include <map>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

namespace {

/* ---------------- forward-mode dual number with 12 partials ---------------- */
struct Dual {
  double v;
  double d[12];
};
inline Dual dconst(double x) { Dual r; r.v = x; for (int i = 0; i < 12; ++i) r.d[i] = 0.0; return r; }
inline Dual operator+(const Dual& a, const Dual& b) { Dual r; r.v = a.v + b.v; for (int i = 0; i < 12; ++i) r.d[i] = a.d[i] + b.d[i]; return r; }
inline Dual operator-(const Dual& a, const Dual& b) { Dual r; r.v = a.v - b.v; for (int i = 0; i < 12; ++i) r.d[i] = a.d[i] - b.d[i]; return r; }
inline Dual operator*(const Dual& a, const Dual& b) { Dual r; r.v = a.v * b.v; for (int i = 0; i < 12; ++i) r.d[i] = a.d[i] * b.v + a.v * b.d[i]; return r; }
inline Dual operator*(double a, const Dual& b) { Dual r; r.v = a * b.v; for (int i = 0; i < 12; ++i) r.d[i] = a * b.d[i]; return r; }
inline Dual operator*(const Dual& b, double a) { return a * b; }
inline Dual operator+(const Dual& a, double b) { Dual r = a; r.v += b; return r; }
inline Dual& operator+=(Dual& a, const Dual& b) { a = a + b; return a; }
inline Dual pow(const Dual& a, double p) {
  Dual r; r.v = std::pow(a.v, p);
  double dp = p * std::pow(a.v, p - 1.0);
  for (int i = 0; i < 12; ++i) r.d[i] = dp * a.d[i];
  return r;
}
inline double pow(double a, double p) { return std::pow(a, p); }
template <class T> inline T zero();
template <> inline double zero<double>() { return 0.0; }
template <> inline Dual zero<Dual>() { return dconst(0.0); }
/* a U-independent double promoted to the scalar type T */
template <class T> inline T promote(double x);
template <> inline double promote<double>(double x) { return x; }
template <> inline Dual promote<Dual>(double x) { return dconst(x); }

/* ---------------- quadrature (reading L4) ---------------- */
/* triangle points a = 0..2: barycentrics (L0, L1, L2) = (2/3,1/6,1/6) cyclic,
 * i.e. reference (xi, eta) = (1/6,1/6), (2/3,1/6), (1/6,2/3); weight 1/6 each on
 * the reference triangle of area 1/2.  Gauss points zeta = -1/sqrt(3), +1/sqrt(3),
 * weight 1.  Loop order: triangle point outer, zeta inner. */
const double kTriXi[3] = {1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0};
const double kTriEta[3] = {1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0};
const double kTriW = 1.0 / 6.0;

const double kGasR = 8.314462618;   /* J mol^-1 K^-1 (CODATA 2018) */

struct Geo {           /* one wedge's data */
  double X[6][3];      /* nodal coordinates, local node i = t + 3*level */
  double s[6];         /* nodal surface elevation (of the node's column) */
  double beta[3];      /* basal friction at the 3 columns (after floating mask) */
  double A;            /* flow factor of this wedge */
  bool basal;          /* k == 0 */
  int lateral;         /* bit jj: edge (jj, jj+1 mod 3) lies on the footprint boundary */
  int tet;             /* NEXT-f4: 1 = three P1 tetrahedra instead of the wedge */
  int ord[3];          /* local bottom nodes sorted by global vertex id (tet split) */
  int64_t gdof[12];    /* global DOFs, local dof = 2*i + a */
};

/* reference basis N_i = L_t(xi,eta) f_l(zeta), i = t + 3l */
void ref_basis(double xi, double eta, double zeta, double N[6], double dN[6][3]) {
  const double Lt[3] = {1.0 - xi - eta, xi, eta};
  const double dLxi[3] = {-1.0, 1.0, 0.0};
  const double dLeta[3] = {-1.0, 0.0, 1.0};
  const double f[2] = {0.5 * (1.0 - zeta), 0.5 * (1.0 + zeta)};
  const double df[2] = {-0.5, 0.5};
  for (int l = 0; l < 2; ++l)
    for (int t = 0; t < 3; ++t) {
      int i = t + 3 * l;
      N[i] = Lt[t] * f[l];
      dN[i][0] = dLxi[t] * f[l];
      dN[i][1] = dLeta[t] * f[l];
      dN[i][2] = Lt[t] * df[l];
    }
}

/* generic 3x3 isoparametric map: Jm[r][c] = dX_r/dxi_c; returns det, fills
 * physical gradients G[i][r] = dN_i/dx_r = sum_c inv(Jm)[c][r] dN_i/dxi_c */
double phys_grad(const double X[6][3], const double dN[6][3], double G[6][3]) {
  double Jm[3][3] = {{0}};
  for (int i = 0; i < 6; ++i)
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) Jm[r][c] += X[i][r] * dN[i][c];
  double det = Jm[0][0] * (Jm[1][1] * Jm[2][2] - Jm[1][2] * Jm[2][1]) -
               Jm[0][1] * (Jm[1][0] * Jm[2][2] - Jm[1][2] * Jm[2][0]) +
               Jm[0][2] * (Jm[1][0] * Jm[2][1] - Jm[1][1] * Jm[2][0]);
  double inv[3][3];
  inv[0][0] = (Jm[1][1] * Jm[2][2] - Jm[1][2] * Jm[2][1]) / det;
  inv[0][1] = (Jm[0][2] * Jm[2][1] - Jm[0][1] * Jm[2][2]) / det;
  inv[0][2] = (Jm[0][1] * Jm[1][2] - Jm[0][2] * Jm[1][1]) / det;
  inv[1][0] = (Jm[1][2] * Jm[2][0] - Jm[1][0] * Jm[2][2]) / det;
  inv[1][1] = (Jm[0][0] * Jm[2][2] - Jm[0][2] * Jm[2][0]) / det;
  inv[1][2] = (Jm[0][2] * Jm[1][0] - Jm[0][0] * Jm[1][2]) / det;
  inv[2][0] = (Jm[1][0] * Jm[2][1] - Jm[1][1] * Jm[2][0]) / det;
  inv[2][1] = (Jm[0][1] * Jm[2][0] - Jm[0][0] * Jm[2][1]) / det;
  inv[2][2] = (Jm[0][0] * Jm[1][1] - Jm[0][1] * Jm[1][0]) / det;
  for (int i = 0; i < 6; ++i)
    for (int r = 0; r < 3; ++r) {
      double acc = 0.0;
      for (int c = 0; c < 3; ++c) acc += inv[c][r] * dN[i][c];
      G[i][r] = acc;
    }
  return det;
}

/* NEXT-f4: P1 tetrahedron `which` (0..2) of the wedge split by global vertex
 * id (reading L22): with bottom nodes a < b < c (global ids) and tops a', b', c',
 *   {a, b, c, c'}, {a, b, b', c'}, {a, a', b', c'};
 * every quad side face (x < y) gets the diagonal x-bottom -- y-top, so
 * neighbouring prisms split their shared face alike.  Returns, over the
 * wedge's 6 local nodes, the centroid values N (1/4 on the tet's nodes, 0
 * elsewhere), the constant physical gradients G (generic 3x3 inverse of the
 * edge matrix) and the weight W = volume. */
void tet_basis(const Geo& e, int which, double N[6], double G[6][3], double* W) {
  const int a = e.ord[0], b = e.ord[1], c = e.ord[2];
  const int nodes[3][4] = {{a, b, c, c + 3}, {a, b, b + 3, c + 3}, {a, a + 3, b + 3, c + 3}};
  const int* nd = nodes[which];
  double Xt[6][3] = {{0}};
  double dN[6][3] = {{0}};
  /* reference tet: N0 = 1 - xi - eta - zeta, N1 = xi, N2 = eta, N3 = zeta,
   * evaluated through the 6-node interface (unused nodes: zero) */
  const double dref[4][3] = {{-1, -1, -1}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int i = 0; i < 6; ++i) { N[i] = 0.0; for (int r = 0; r < 3; ++r) G[i][r] = 0.0; }
  for (int q = 0; q < 4; ++q)
    for (int r = 0; r < 3; ++r) { Xt[nd[q]][r] = e.X[nd[q]][r]; dN[nd[q]][r] = dref[q][r]; }
  double det = phys_grad(Xt, dN, G);
  for (int q = 0; q < 4; ++q) N[nd[q]] = 0.25;
  *W = std::fabs(det) / 6.0;
}

/* Element residual r[12] (local dof 2i+a) and energy, templated on the scalar
 * type of U (double -> residual; Dual -> residual + Jacobian rows). */
template <class T>
void element(const Geo& e, const ora_params& p, int terms, const T Ul[12], T r[12], T* pi) {
  for (int j = 0; j < 12; ++j) r[j] = zero<T>();
  T energy = zero<T>();
  const double n = p.glen_n;
  const double Afac = std::pow(e.A, -1.0 / n);      /* A^(-1/n) */
  const double rg = p.rho * p.g;
  const double gz = 1.0 / std::sqrt(3.0);
  const double zq[2] = {-gz, gz};
  /* volume quadrature points: the wedge's 3 x 2 rule (reading L4), or for
   * NEXT-f4 one centroid point per P1 tetrahedron (exact: constant gradients) */
  const int n_pts = e.tet ? 3 : 6;
  for (int pt = 0; pt < n_pts; ++pt) {
    {
      double N[6], dN[6][3], G[6][3];
      double W;
      if (e.tet) {
        tet_basis(e, pt, N, G, &W);
      } else {
        const int a = pt / 2, sq = pt % 2;
        ref_basis(kTriXi[a], kTriEta[a], zq[sq], N, dN);
        double det = phys_grad(e.X, dN, G);
        W = kTriW * 1.0 * det;                    /* weights 1/6 (triangle) x 1 (Gauss) */
      }
      /* velocity gradient */
      T ux = zero<T>(), uy = zero<T>(), uz = zero<T>(), vx = zero<T>(), vy = zero<T>(), vz = zero<T>();
      T u = zero<T>(), v = zero<T>();
      for (int i = 0; i < 6; ++i) {
        ux += Ul[2 * i] * G[i][0]; uy += Ul[2 * i] * G[i][1]; uz += Ul[2 * i] * G[i][2];
        vx += Ul[2 * i + 1] * G[i][0]; vy += Ul[2 * i + 1] * G[i][1]; vz += Ul[2 * i + 1] * G[i][2];
        u += Ul[2 * i] * N[i]; v += Ul[2 * i + 1] * N[i];
      }
      if (terms & ORA_VISC) {
        /* strain-rate components */
        T exx = ux, eyy = vy;
        T exy = 0.5 * (uy + vx);
        T exz = 0.5 * uz, eyz = 0.5 * vz;
        /* effective strain rate squared */
        T q = exx * exx + eyy * eyy + exx * eyy + exy * exy + exz * exz + eyz * eyz;
        T qe = q + p.eps_reg;
        /* 2 mu_e = A^(-1/n) (q + eps)^((1-n)/(2n))  (reading L1) */
        T two_mu = Afac * pow(qe, (1.0 - n) / (2.0 * n));
        /* strain-rate vectors */
        T e1[3] = {2.0 * exx + eyy, exy, exz};
        T e2[3] = {exy, exx + 2.0 * eyy, eyz};
        for (int i = 0; i < 6; ++i) {
          T g1 = e1[0] * G[i][0] + e1[1] * G[i][1] + e1[2] * G[i][2];
          T g2 = e2[0] * G[i][0] + e2[1] * G[i][1] + e2[2] * G[i][2];
          r[2 * i] += (W * two_mu) * g1;
          r[2 * i + 1] += (W * two_mu) * g2;
        }
        /* energy density (2n/(n+1)) A^(-1/n) (q+eps)^((n+1)/(2n)) */
        energy += (W * (2.0 * n / (n + 1.0)) * Afac) * pow(qe, (n + 1.0) / (2.0 * n));
      }
      if (terms & ORA_BODY) {
        /* grad s = 3D basis gradient of nodal s (reading L10) */
        double sx = 0.0, sy = 0.0;
        for (int i = 0; i < 6; ++i) { sx += e.s[i] * G[i][0]; sy += e.s[i] * G[i][1]; }
        for (int i = 0; i < 6; ++i) {
          r[2 * i] += promote<T>(W * rg * sx * N[i]);
          r[2 * i + 1] += promote<T>(W * rg * sy * N[i]);
        }
        energy += (W * rg * sx) * u + (W * rg * sy) * v;
      }
    }
  }
  if ((terms & ORA_BASAL) && e.basal) {
    /* planar 3D bottom triangle (nodes 0,1,2), true area (reading L7) */
    double e1[3], e2[3], cr[3];
    for (int r3 = 0; r3 < 3; ++r3) { e1[r3] = e.X[1][r3] - e.X[0][r3]; e2[r3] = e.X[2][r3] - e.X[0][r3]; }
    cr[0] = e1[1] * e2[2] - e1[2] * e2[1];
    cr[1] = e1[2] * e2[0] - e1[0] * e2[2];
    cr[2] = e1[0] * e2[1] - e1[1] * e2[0];
    double area = 0.5 * std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
    for (int a = 0; a < 3; ++a) {
      const double Lt[3] = {1.0 - kTriXi[a] - kTriEta[a], kTriXi[a], kTriEta[a]};
      double w = kTriW * 2.0 * area;             /* 3-point rule, weights sum to area */
      double b = Lt[0] * e.beta[0] + Lt[1] * e.beta[1] + Lt[2] * e.beta[2];  /* P1 beta (L8) */
      T u = Lt[0] * Ul[0] + Lt[1] * Ul[2] + Lt[2] * Ul[4];
      T v = Lt[0] * Ul[1] + Lt[1] * Ul[3] + Lt[2] * Ul[5];
      for (int t = 0; t < 3; ++t) {
        r[2 * t] += (w * b * Lt[t]) * u;
        r[2 * t + 1] += (w * b * Lt[t]) * v;
      }
      energy += (0.5 * w * b) * (u * u + v * v);
    }
  }
  if (terms & ORA_LATERAL) {
    /* NEXT-f1: lateral margin faces, reading L12:
     *   2 mu eps_a . n = [rho g (s - z) - rho_w g max(-z, 0)] n_a  on Gamma_l,
     * so the weak form gains  - int_{Gamma_l} P(z) n_a phi_i dGamma.
     * Quadrature (reading L20): 2-point Gauss along the edge; in zeta 2-point
     * Gauss on [-1, 1], or on each side of the sea-level crossing z = 0. */
    const double gz = 1.0 / std::sqrt(3.0);
    for (int jj = 0; jj < 3; ++jj) {
      if (!((e.lateral >> jj) & 1)) continue;
      const int j0 = jj, j1 = (jj + 1) % 3;
      const double dx = e.X[j1][0] - e.X[j0][0], dy = e.X[j1][1] - e.X[j0][1];
      const double len = std::sqrt(dx * dx + dy * dy);
      const double nx = dy / len, ny = -dx / len;     /* outward for a CCW triangle */
      for (int sp = 0; sp < 2; ++sp) {
        const double sc = 0.5 + (sp == 0 ? -0.5 : 0.5) * gz;   /* edge coordinate */
        const double zb = (1.0 - sc) * e.X[j0][2] + sc * e.X[j1][2];
        const double zt = (1.0 - sc) * e.X[j0 + 3][2] + sc * e.X[j1 + 3][2];
        const double S = (1.0 - sc) * e.s[j0] + sc * e.s[j1];
        double cut[3] = {-1.0, 1.0, 1.0};
        int nint = 1;
        if (zb < 0.0 && zt > 0.0) {
          cut[1] = -1.0 + 2.0 * (0.0 - zb) / (zt - zb);
          nint = 2;
        }
        for (int iv = 0; iv < nint; ++iv) {
          const double lo = cut[iv], hi = cut[iv + 1];
          for (int zq2 = 0; zq2 < 2; ++zq2) {
            const double zeta = 0.5 * (lo + hi) + (zq2 == 0 ? -0.5 : 0.5) * (hi - lo) * gz;
            const double wz = 0.5 * (hi - lo);
            const double z = zb + 0.5 * (1.0 + zeta) * (zt - zb);
            const double P = p.rho * p.g * (S - z) - p.rho_w * p.g * std::max(-z, 0.0);
            const double W = len * 0.5 * wz * 0.5 * (zt - zb);
            const double phi[4] = {(1.0 - sc) * 0.5 * (1.0 - zeta), sc * 0.5 * (1.0 - zeta),
                                   (1.0 - sc) * 0.5 * (1.0 + zeta), sc * 0.5 * (1.0 + zeta)};
            const int node[4] = {j0, j1, j0 + 3, j1 + 3};
            T un = zero<T>();
            for (int q = 0; q < 4; ++q) {
              r[2 * node[q]] += promote<T>(-W * P * nx * phi[q]);
              r[2 * node[q] + 1] += promote<T>(-W * P * ny * phi[q]);
              un += (nx * phi[q]) * Ul[2 * node[q]] + (ny * phi[q]) * Ul[2 * node[q] + 1];
            }
            energy += (-W * P) * un;
          }
        }
      }
    }
  }
  if (pi) *pi = energy;
}

struct Mesh {
  const ora_mesh* m;
  int64_t n_col, n_node, n_dof, n_elem;
  int L;
  std::vector<double> z;      /* [n_node] */
  std::vector<double> beta;   /* masked */
  std::vector<uint8_t> lateral;   /* [n_tri] boundary-edge bits (NEXT-f1) */
};

int validate_quads(const ora_mesh* m);

int validate(const ora_mesh* m) {
  if (!m) return -1;
  if (m->n_vert < 0 || m->n_tri < 0 || m->n_layers < 1) return -1;
  if (m->n_vert == 0 && m->n_tri == 0) return 0;       /* empty footprint is valid */
  if (!m->xy || !m->tri || !m->thickness || !m->surface || !m->beta) return -1;
  if (m->p.glen_n <= 0.0 || m->p.A <= 0.0 || m->p.eps_reg < 0.0) return -1;
  if (m->T_star && !(m->A0 > 0.0)) return -1;
  if (m->elem_type != 0 && m->elem_type != 1 && m->elem_type != 2) return -1;
  if (m->elem_type == 2) return validate_quads(m);
  const int L = m->n_layers;
  if (m->sigma) {
    if (m->sigma[0] != 0.0 || m->sigma[L] != 1.0) return -2;
    for (int k = 0; k < L; ++k) if (!(m->sigma[k + 1] > m->sigma[k])) return -2;
  }
  std::vector<char> used(m->n_vert, 0);
  for (int64_t t = 0; t < m->n_tri; ++t) {
    const int32_t* v = m->tri + 3 * t;
    for (int j = 0; j < 3; ++j) if (v[j] < 0 || v[j] >= m->n_vert) return -2;
    if (v[0] == v[1] || v[1] == v[2] || v[0] == v[2]) return -2;
    double x0 = m->xy[2 * v[0]], y0 = m->xy[2 * v[0] + 1];
    double x1 = m->xy[2 * v[1]], y1 = m->xy[2 * v[1] + 1];
    double x2 = m->xy[2 * v[2]], y2 = m->xy[2 * v[2] + 1];
    double twoA = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0);
    if (!(twoA > 0.0)) return -2;                      /* CW or degenerate */
    used[v[0]] = used[v[1]] = used[v[2]] = 1;
  }
  for (int64_t c = 0; c < m->n_vert; ++c) {
    if (!used[c]) return -2;                           /* isolated vertex */
    if (!(m->thickness[c] >= m->p.H_min)) return -2;
  }
  return 0;
}

void extrude(const ora_mesh* m, Mesh& M) {
  M.m = m;
  M.L = m->n_layers;
  M.n_col = m->n_vert;
  M.n_node = m->n_vert * (M.L + 1);
  M.n_dof = 2 * M.n_node;
  M.n_elem = m->n_tri * M.L;
  M.z.assign(M.n_node, 0.0);
  for (int64_t c = 0; c < M.n_col; ++c)
    for (int k = 0; k <= M.L; ++k) {
      double sig = m->sigma ? m->sigma[k] : double(k) / double(M.L);
      double base = m->surface[c] - m->thickness[c];
      M.z[c * (M.L + 1) + k] = base + sig * m->thickness[c];
    }
  M.beta.assign(M.n_col, 0.0);
  for (int64_t c = 0; c < M.n_col; ++c) {
    bool floating = m->bed && (m->p.rho * m->thickness[c] < -m->p.rho_w * m->bed[c]);
    M.beta[c] = floating ? 0.0 : m->beta[c];
  }
}

void wedge_geo(const Mesh& M, int64_t t, int k, Geo& e) {
  const ora_mesh* m = M.m;
  const int32_t* v = m->tri + 3 * t;
  for (int l = 0; l < 2; ++l)
    for (int j = 0; j < 3; ++j) {
      int i = j + 3 * l;
      int64_t node = int64_t(v[j]) * (M.L + 1) + k + l;
      e.X[i][0] = m->xy[2 * v[j]];
      e.X[i][1] = m->xy[2 * v[j] + 1];
      e.X[i][2] = M.z[node];
      e.s[i] = m->surface[v[j]];
      e.gdof[2 * i] = 2 * node;
      e.gdof[2 * i + 1] = 2 * node + 1;
    }
  for (int j = 0; j < 3; ++j) e.beta[j] = M.beta[v[j]];
  if (m->T_star)   /* Arrhenius relation */
    e.A = m->A0 * std::exp(-m->Q_act / (kGasR * m->T_star[t * M.L + k]));
  else
    e.A = m->A_elem ? m->A_elem[t * M.L + k] : m->p.A;
  e.basal = (k == 0);
  e.lateral = M.lateral.empty() ? 0 : M.lateral[t];
  e.tet = m->elem_type == 1;
  {   /* bottom local nodes by global vertex id (NEXT-f4 split) */
    int o[3] = {0, 1, 2};
    std::sort(o, o + 3, [&](int x, int y) { return v[x] < v[y]; });
    for (int j = 0; j < 3; ++j) e.ord[j] = o[j];
  }
}

/* footprint boundary edges: undirected edges used by exactly one triangle */
void find_lateral(const ora_mesh* m, Mesh& M) {
  std::map<std::pair<int32_t, int32_t>, int> cnt;
  for (int64_t t = 0; t < m->n_tri; ++t)
    for (int jj = 0; jj < 3; ++jj) {
      int32_t a = m->tri[3 * t + jj], b = m->tri[3 * t + (jj + 1) % 3];
      cnt[{std::min(a, b), std::max(a, b)}]++;
    }
  M.lateral.assign(m->n_tri, 0);
  for (int64_t t = 0; t < m->n_tri; ++t)
    for (int jj = 0; jj < 3; ++jj) {
      int32_t a = m->tri[3 * t + jj], b = m->tri[3 * t + (jj + 1) % 3];
      if (cnt[{std::min(a, b), std::max(a, b)}] == 1) M.lateral[t] |= uint8_t(1 << jj);
    }
}

int prepare(const ora_mesh* m, Mesh& M, int terms = 0) {
  int st = validate(m);
  if (st) return st;
  extrude(m, M);
  if ((terms & ORA_LATERAL) && m->elem_type != 2) find_lateral(m, M);
  return 0;
}


/* =================== NEXT-f4: 8-node trilinear hexahedra =================== */
/* reading L23: quadrilateral footprint (CCW corners 0..3), element = the
 * column segment between two levels, nodes 0..3 bottom (corner order), 4..7
 * top; N_i = Q_c(xi, eta) f_l(zeta) with the bilinear Q_c at reference corners
 * (-1,-1), (1,-1), (1,1), (-1,1); 2 x 2 x 2 Gauss points (+-1/sqrt 3, weight
 * 1) with the generic 3x3 inverse; driving stress with the 3D basis gradient
 * of nodal s; basal term with 2 x 2 Gauss on the bilinear bottom face, true 3D
 * area element |X_xi x X_eta|, beta bilinear.  Jacobian by a 16-partial dual. */
struct Dual16 {
  double v;
  double d[16];
};
inline Dual16 d16(double x) { Dual16 r; r.v = x; for (int i = 0; i < 16; ++i) r.d[i] = 0.0; return r; }
inline Dual16 operator+(const Dual16& a, const Dual16& b) { Dual16 r; r.v = a.v + b.v; for (int i = 0; i < 16; ++i) r.d[i] = a.d[i] + b.d[i]; return r; }
inline Dual16 operator*(const Dual16& a, const Dual16& b) { Dual16 r; r.v = a.v * b.v; for (int i = 0; i < 16; ++i) r.d[i] = a.d[i] * b.v + a.v * b.d[i]; return r; }
inline Dual16 operator*(double a, const Dual16& b) { Dual16 r; r.v = a * b.v; for (int i = 0; i < 16; ++i) r.d[i] = a * b.d[i]; return r; }
inline Dual16 operator*(const Dual16& b, double a) { return a * b; }
inline Dual16 operator+(const Dual16& a, double b) { Dual16 r = a; r.v += b; return r; }
inline Dual16& operator+=(Dual16& a, const Dual16& b) { a = a + b; return a; }
inline Dual16 pow(const Dual16& a, double p) {
  Dual16 r; r.v = std::pow(a.v, p);
  double dp = p * std::pow(a.v, p - 1.0);
  for (int i = 0; i < 16; ++i) r.d[i] = dp * a.d[i];
  return r;
}
template <> inline Dual16 zero<Dual16>() { return d16(0.0); }
template <> inline Dual16 promote<Dual16>(double x) { return d16(x); }

const double kQxi[4] = {-1.0, 1.0, 1.0, -1.0}, kQeta[4] = {-1.0, -1.0, 1.0, 1.0};

struct Geo8 {
  double X[8][3];
  double s[8];
  double beta[4];
  double A;
  bool basal;
  int64_t gdof[16];
};

int validate_quads(const ora_mesh* m) {
  const int L = m->n_layers;
  if (m->sigma) {
    if (m->sigma[0] != 0.0 || m->sigma[L] != 1.0) return -2;
    for (int k = 0; k < L; ++k) if (!(m->sigma[k + 1] > m->sigma[k])) return -2;
  }
  std::vector<char> used(m->n_vert, 0);
  for (int64_t t = 0; t < m->n_tri; ++t) {
    const int32_t* v = m->tri + 4 * t;
    for (int j = 0; j < 4; ++j) if (v[j] < 0 || v[j] >= m->n_vert) return -2;
    for (int j = 0; j < 4; ++j) {   /* convex, CCW: every corner turns left */
      const int32_t a = v[(j + 3) % 4], b = v[j], c = v[(j + 1) % 4];
      const double cr = (m->xy[2 * b] - m->xy[2 * a]) * (m->xy[2 * c + 1] - m->xy[2 * b + 1]) -
                        (m->xy[2 * b + 1] - m->xy[2 * a + 1]) * (m->xy[2 * c] - m->xy[2 * b]);
      if (!(cr > 0.0)) return -2;
      used[b] = 1;
    }
  }
  for (int64_t c = 0; c < m->n_vert; ++c) {
    if (!used[c]) return -2;
    if (!(m->thickness[c] >= m->p.H_min)) return -2;
  }
  return 0;
}

void hex_geo(const Mesh& M, int64_t t, int k, Geo8& e) {
  const ora_mesh* m = M.m;
  const int32_t* v = m->tri + 4 * t;
  for (int l = 0; l < 2; ++l)
    for (int j = 0; j < 4; ++j) {
      const int i = j + 4 * l;
      const int64_t node = int64_t(v[j]) * (M.L + 1) + k + l;
      e.X[i][0] = m->xy[2 * v[j]];
      e.X[i][1] = m->xy[2 * v[j] + 1];
      e.X[i][2] = M.z[node];
      e.s[i] = m->surface[v[j]];
      e.gdof[2 * i] = 2 * node;
      e.gdof[2 * i + 1] = 2 * node + 1;
    }
  for (int j = 0; j < 4; ++j) e.beta[j] = M.beta[v[j]];
  if (m->T_star)
    e.A = m->A0 * std::exp(-m->Q_act / (kGasR * m->T_star[t * M.L + k]));
  else
    e.A = m->A_elem ? m->A_elem[t * M.L + k] : m->p.A;
  e.basal = (k == 0);
}

/* N, dN/d(xi,eta,zeta) of the 8 nodes; physical gradients by the generic inverse */
double hex_basis(const Geo8& e, double xi, double eta, double zeta, double N[8], double G[8][3]) {
  double dN[8][3];
  for (int l = 0; l < 2; ++l)
    for (int j = 0; j < 4; ++j) {
      const int i = j + 4 * l;
      const double fq = 0.25 * (1.0 + kQxi[j] * xi) * (1.0 + kQeta[j] * eta);
      const double fz = l == 0 ? 0.5 * (1.0 - zeta) : 0.5 * (1.0 + zeta);
      N[i] = fq * fz;
      dN[i][0] = 0.25 * kQxi[j] * (1.0 + kQeta[j] * eta) * fz;
      dN[i][1] = 0.25 * kQeta[j] * (1.0 + kQxi[j] * xi) * fz;
      dN[i][2] = fq * (l == 0 ? -0.5 : 0.5);
    }
  double Jm[3][3] = {{0}};
  for (int i = 0; i < 8; ++i)
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) Jm[r][c] += e.X[i][r] * dN[i][c];
  const double det = Jm[0][0] * (Jm[1][1] * Jm[2][2] - Jm[1][2] * Jm[2][1]) -
                     Jm[0][1] * (Jm[1][0] * Jm[2][2] - Jm[1][2] * Jm[2][0]) +
                     Jm[0][2] * (Jm[1][0] * Jm[2][1] - Jm[1][1] * Jm[2][0]);
  double inv[3][3];
  inv[0][0] = (Jm[1][1] * Jm[2][2] - Jm[1][2] * Jm[2][1]) / det;
  inv[0][1] = (Jm[0][2] * Jm[2][1] - Jm[0][1] * Jm[2][2]) / det;
  inv[0][2] = (Jm[0][1] * Jm[1][2] - Jm[0][2] * Jm[1][1]) / det;
  inv[1][0] = (Jm[1][2] * Jm[2][0] - Jm[1][0] * Jm[2][2]) / det;
  inv[1][1] = (Jm[0][0] * Jm[2][2] - Jm[0][2] * Jm[2][0]) / det;
  inv[1][2] = (Jm[0][2] * Jm[1][0] - Jm[0][0] * Jm[1][2]) / det;
  inv[2][0] = (Jm[1][0] * Jm[2][1] - Jm[1][1] * Jm[2][0]) / det;
  inv[2][1] = (Jm[0][1] * Jm[2][0] - Jm[0][0] * Jm[2][1]) / det;
  inv[2][2] = (Jm[0][0] * Jm[1][1] - Jm[0][1] * Jm[1][0]) / det;
  for (int i = 0; i < 8; ++i)
    for (int r = 0; r < 3; ++r) {
      double acc = 0.0;
      for (int c = 0; c < 3; ++c) acc += inv[c][r] * dN[i][c];
      G[i][r] = acc;
    }
  return det;
}

template <class T>
void element_hex(const Geo8& e, const ora_params& p, int terms, const T Ul[16], T r[16], T* pi) {
  for (int j = 0; j < 16; ++j) r[j] = zero<T>();
  T energy = zero<T>();
  const double n = p.glen_n;
  const double Afac = std::pow(e.A, -1.0 / n);
  const double rg = p.rho * p.g;
  const double gz = 1.0 / std::sqrt(3.0);
  for (int qx = 0; qx < 2; ++qx)
    for (int qy = 0; qy < 2; ++qy)
      for (int qz = 0; qz < 2; ++qz) {
        double N[8], G[8][3];
        const double det = hex_basis(e, qx ? gz : -gz, qy ? gz : -gz, qz ? gz : -gz, N, G);
        const double W = det;   /* Gauss weights 1 x 1 x 1 */
        T ux = zero<T>(), uy = zero<T>(), uz = zero<T>(), vx = zero<T>(), vy = zero<T>(), vz = zero<T>();
        T u = zero<T>(), v = zero<T>();
        for (int i = 0; i < 8; ++i) {
          ux += Ul[2 * i] * G[i][0]; uy += Ul[2 * i] * G[i][1]; uz += Ul[2 * i] * G[i][2];
          vx += Ul[2 * i + 1] * G[i][0]; vy += Ul[2 * i + 1] * G[i][1]; vz += Ul[2 * i + 1] * G[i][2];
          u += Ul[2 * i] * N[i]; v += Ul[2 * i + 1] * N[i];
        }
        if (terms & ORA_VISC) {
          T exx = ux, eyy = vy, exy = 0.5 * (uy + vx), exz = 0.5 * uz, eyz = 0.5 * vz;
          T q = exx * exx + eyy * eyy + exx * eyy + exy * exy + exz * exz + eyz * eyz;
          T qe = q + p.eps_reg;
          T two_mu = Afac * pow(qe, (1.0 - n) / (2.0 * n));
          T e1[3] = {2.0 * exx + eyy, exy, exz};
          T e2[3] = {exy, exx + 2.0 * eyy, eyz};
          for (int i = 0; i < 8; ++i) {
            T g1 = e1[0] * G[i][0] + e1[1] * G[i][1] + e1[2] * G[i][2];
            T g2 = e2[0] * G[i][0] + e2[1] * G[i][1] + e2[2] * G[i][2];
            r[2 * i] += (W * two_mu) * g1;
            r[2 * i + 1] += (W * two_mu) * g2;
          }
          energy += (W * (2.0 * n / (n + 1.0)) * Afac) * pow(qe, (n + 1.0) / (2.0 * n));
        }
        if (terms & ORA_BODY) {
          double sx = 0.0, sy = 0.0;
          for (int i = 0; i < 8; ++i) { sx += e.s[i] * G[i][0]; sy += e.s[i] * G[i][1]; }
          for (int i = 0; i < 8; ++i) {
            r[2 * i] += promote<T>(W * rg * sx * N[i]);
            r[2 * i + 1] += promote<T>(W * rg * sy * N[i]);
          }
          energy += (W * rg * sx) * u + (W * rg * sy) * v;
        }
      }
  if ((terms & ORA_BASAL) && e.basal) {
    for (int qx = 0; qx < 2; ++qx)
      for (int qy = 0; qy < 2; ++qy) {
        const double xi = qx ? gz : -gz, eta = qy ? gz : -gz;
        double Q[4], tx[3] = {0, 0, 0}, ty[3] = {0, 0, 0};
        for (int j = 0; j < 4; ++j) {
          Q[j] = 0.25 * (1.0 + kQxi[j] * xi) * (1.0 + kQeta[j] * eta);
          const double dxi = 0.25 * kQxi[j] * (1.0 + kQeta[j] * eta);
          const double deta = 0.25 * kQeta[j] * (1.0 + kQxi[j] * xi);
          for (int r3 = 0; r3 < 3; ++r3) { tx[r3] += dxi * e.X[j][r3]; ty[r3] += deta * e.X[j][r3]; }
        }
        const double cx = tx[1] * ty[2] - tx[2] * ty[1], cy = tx[2] * ty[0] - tx[0] * ty[2],
                     cz = tx[0] * ty[1] - tx[1] * ty[0];
        const double w = std::sqrt(cx * cx + cy * cy + cz * cz);   /* weight 1 x 1 */
        double b = 0.0;
        for (int j = 0; j < 4; ++j) b += Q[j] * e.beta[j];
        T u = zero<T>(), v = zero<T>();
        for (int j = 0; j < 4; ++j) { u += Q[j] * Ul[2 * j]; v += Q[j] * Ul[2 * j + 1]; }
        for (int j = 0; j < 4; ++j) {
          r[2 * j] += (w * b * Q[j]) * u;
          r[2 * j + 1] += (w * b * Q[j]) * v;
        }
        energy += (0.5 * w * b) * (u * u + v * v);
      }
  }
  if (pi) *pi = energy;
}

/* hexahedral versions of the drivers (elem_type 2) */
int graph_hex(const ora_mesh* m, const Mesh& M, int64_t* row_ptr, int32_t* col_idx, int64_t* nnz) {
  std::vector<std::vector<int64_t>> rows(M.n_dof);
  for (int64_t t = 0; t < m->n_tri; ++t)
    for (int k = 0; k < M.L; ++k) {
      Geo8 e;
      hex_geo(M, t, k, e);
      for (int p = 0; p < 16; ++p)
        for (int q = 0; q < 16; ++q) rows[e.gdof[p]].push_back(e.gdof[q]);
    }
  int64_t total = 0;
  for (int64_t r = 0; r < M.n_dof; ++r) {
    std::sort(rows[r].begin(), rows[r].end());
    rows[r].erase(std::unique(rows[r].begin(), rows[r].end()), rows[r].end());
    total += int64_t(rows[r].size());
  }
  if (nnz) *nnz = total;
  if (row_ptr) {
    row_ptr[0] = 0;
    for (int64_t r = 0; r < M.n_dof; ++r) row_ptr[r + 1] = row_ptr[r] + int64_t(rows[r].size());
  }
  if (col_idx) {
    int64_t pos = 0;
    for (int64_t r = 0; r < M.n_dof; ++r)
      for (int64_t c : rows[r]) col_idx[pos++] = int32_t(c);
  }
  return 0;
}

int residual_hex(const ora_mesh* m, const Mesh& M, int terms, const double* U, double* R, double* Mabs,
                 double* Pi, int64_t dof) {
  double pi_total = 0.0;
  for (int64_t t = 0; t < m->n_tri; ++t)
    for (int k = 0; k < M.L; ++k) {
      Geo8 e;
      hex_geo(M, t, k, e);
      if (dof >= 0) {
        bool touches = false;
        for (int j = 0; j < 16 && !touches; ++j) touches = (e.gdof[j] == dof);
        if (!touches) continue;
      }
      double Ul[16], r[16], pi;
      for (int j = 0; j < 16; ++j) Ul[j] = U[e.gdof[j]];
      element_hex<double>(e, m->p, terms, Ul, r, &pi);
      for (int j = 0; j < 16; ++j) {
        if (R) R[e.gdof[j]] += r[j];
        if (Mabs) Mabs[e.gdof[j]] += std::fabs(r[j]);
      }
      pi_total += pi;
    }
  if (Pi) *Pi = pi_total;
  return 0;
}

int jacobian_hex(const ora_mesh* m, const Mesh& M, int terms, const double* U, const int64_t* row_ptr,
                 const int32_t* col_idx, double* R, double* vals) {
  for (int64_t t = 0; t < m->n_tri; ++t)
    for (int k = 0; k < M.L; ++k) {
      Geo8 e;
      hex_geo(M, t, k, e);
      Dual16 Ul[16], r[16];
      for (int j = 0; j < 16; ++j) {
        Ul[j] = d16(U[e.gdof[j]]);
        Ul[j].d[j] = 1.0;
      }
      element_hex<Dual16>(e, m->p, terms, Ul, r, nullptr);
      for (int p = 0; p < 16; ++p) {
        const int64_t row = e.gdof[p];
        if (R) R[row] += r[p].v;
        const int32_t* b = col_idx + row_ptr[row];
        const int32_t* end = col_idx + row_ptr[row + 1];
        for (int q = 0; q < 16; ++q) {
          const int32_t* it = std::lower_bound(b, end, int32_t(e.gdof[q]));
          if (it == end || *it != e.gdof[q]) return -3;
          vals[it - col_idx] += r[p].d[q];
        }
      }
    }
  return 0;
}

}  // namespace

extern "C" {

int ora_validate(const ora_mesh* m) { return validate(m); }

int ora_graph(const ora_mesh* m, int64_t* row_ptr, int32_t* col_idx, int64_t* nnz) {
  Mesh M;
  int st = prepare(m, M);
  if (st) return st;
  if (m->elem_type == 2) return graph_hex(m, M, row_ptr, col_idx, nnz);
  /* brute force: every DOF pair of every wedge, then sort + unique per row */
  std::vector<std::vector<int64_t>> rows(M.n_dof);
  for (int64_t t = 0; t < m->n_tri; ++t)
    for (int k = 0; k < M.L; ++k) {
      Geo e;
      wedge_geo(M, t, k, e);
      for (int p = 0; p < 12; ++p)
        for (int q = 0; q < 12; ++q) rows[e.gdof[p]].push_back(e.gdof[q]);
    }
  int64_t total = 0;
  for (int64_t r = 0; r < M.n_dof; ++r) {
    std::sort(rows[r].begin(), rows[r].end());
    rows[r].erase(std::unique(rows[r].begin(), rows[r].end()), rows[r].end());
    total += int64_t(rows[r].size());
  }
  if (nnz) *nnz = total;
  if (row_ptr) {
    row_ptr[0] = 0;
    for (int64_t r = 0; r < M.n_dof; ++r) row_ptr[r + 1] = row_ptr[r] + int64_t(rows[r].size());
  }
  if (col_idx) {
    int64_t pos = 0;
    for (int64_t r = 0; r < M.n_dof; ++r)
      for (int64_t c : rows[r]) col_idx[pos++] = int32_t(c);
  }
  return 0;
}

int ora_residual(const ora_mesh* m, int terms, const double* U, double* R, double* Mabs, double* Pi) {
  Mesh M;
  int st = prepare(m, M, terms);
  if (st) return st;
  if (R) std::memset(R, 0, sizeof(double) * M.n_dof);
  if (Mabs) std::memset(Mabs, 0, sizeof(double) * M.n_dof);
  if (m->elem_type == 2) return residual_hex(m, M, terms, U, R, Mabs, Pi, -1);
  double pi_total = 0.0;
  for (int64_t t = 0; t < m->n_tri; ++t)
    for (int k = 0; k < M.L; ++k) {
      Geo e;
      wedge_geo(M, t, k, e);
      double Ul[12], r[12], pi;
      for (int j = 0; j < 12; ++j) Ul[j] = U[e.gdof[j]];
      element<double>(e, m->p, terms, Ul, r, &pi);
      for (int j = 0; j < 12; ++j) {
        if (R) R[e.gdof[j]] += r[j];
        if (Mabs) Mabs[e.gdof[j]] += std::fabs(r[j]);
      }
      pi_total += pi;
    }
  if (Pi) *Pi = pi_total;
  return 0;
}

int ora_jacobian(const ora_mesh* m, int terms, const double* U, const int64_t* row_ptr,
                 const int32_t* col_idx, double* R, double* vals) {
  Mesh M;
  int st = prepare(m, M, terms);
  if (st) return st;
  if (!row_ptr || !col_idx || !vals) return -1;
  if (R) std::memset(R, 0, sizeof(double) * M.n_dof);
  std::memset(vals, 0, sizeof(double) * row_ptr[M.n_dof]);
  if (m->elem_type == 2) return jacobian_hex(m, M, terms, U, row_ptr, col_idx, R, vals);
  for (int64_t t = 0; t < m->n_tri; ++t)
    for (int k = 0; k < M.L; ++k) {
      Geo e;
      wedge_geo(M, t, k, e);
      Dual Ul[12], r[12];
      for (int j = 0; j < 12; ++j) {
        Ul[j] = dconst(U[e.gdof[j]]);
        Ul[j].d[j] = 1.0;                                /* seed */
      }
      element<Dual>(e, m->p, terms, Ul, r, nullptr);
      for (int p = 0; p < 12; ++p) {
        int64_t row = e.gdof[p];
        if (R) R[row] += r[p].v;
        const int32_t* b = col_idx + row_ptr[row];
        const int32_t* end = col_idx + row_ptr[row + 1];
        for (int q = 0; q < 12; ++q) {
          const int32_t* it = std::lower_bound(b, end, int32_t(e.gdof[q]));
          if (it == end || *it != e.gdof[q]) return -3;  /* graph does not cover the pair */
          vals[it - col_idx] += r[p].d[q];
        }
      }
    }
  return 0;
}

int ora_energy(const ora_mesh* m, int terms, const double* U, int64_t dof, double* Pi) {
  Mesh M;
  int st = prepare(m, M, terms);
  if (st) return st;
  if (m->elem_type == 2) return residual_hex(m, M, terms, U, nullptr, nullptr, Pi, dof);
  double total = 0.0;
  for (int64_t t = 0; t < m->n_tri; ++t)
    for (int k = 0; k < M.L; ++k) {
      Geo e;
      wedge_geo(M, t, k, e);
      bool touches = dof < 0;
      for (int j = 0; j < 12 && !touches; ++j) touches = (e.gdof[j] == dof);
      if (!touches) continue;
      double Ul[12], r[12], pi;
      for (int j = 0; j < 12; ++j) Ul[j] = U[e.gdof[j]];
      element<double>(e, m->p, terms, Ul, r, &pi);
      total += pi;
    }
  *Pi = total;
  return 0;
}

int ora_element(const ora_mesh* m, int terms, const double* U, int64_t t, int32_t k,
                double* r, double* Je, int64_t* gdof) {
  Mesh M;
  int st = prepare(m, M, terms);
  if (st) return st;
  if (t < 0 || t >= m->n_tri || k < 0 || k >= M.L || m->elem_type == 2) return -1;
  Geo e;
  wedge_geo(M, t, k, e);
  Dual Ul[12], rr[12];
  for (int j = 0; j < 12; ++j) { Ul[j] = dconst(U[e.gdof[j]]); Ul[j].d[j] = 1.0; }
  element<Dual>(e, m->p, terms, Ul, rr, nullptr);
  for (int p = 0; p < 12; ++p) {
    if (r) r[p] = rr[p].v;
    if (Je) for (int q = 0; q < 12; ++q) Je[12 * p + q] = rr[p].d[q];
    if (gdof) gdof[p] = e.gdof[p];
  }
  return 0;
}

}  // extern "C"
