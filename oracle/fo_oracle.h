/*
 * fo_oracle.h -- C interface of the serial CPU ORACLE for FO-Stokes assembly.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2204_04321_b200/, include/fo.h) never links, imports or calls it, and it
 * shares no header, helper or constant table with the product path.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   - the discrete residual F(U) of the first-order (Blatter-Pattyn) Stokes
 *     equations, eq:FOStokes P:83-89, strain rates P:90-100, Glen viscosity
 *     eq:effvisc P:102-105, effective strain rate eq:effeps P:106-108, basal
 *     Robin/linear sliding P:128-132, stress-free surface P:122-127, on extruded
 *     6-node wedges (P:154, P:155-158 eq:residual);
 *   - the Newton Jacobian dF/dU (eq:linearsystem P:160-164) by fixed-size
 *     forward-mode AD (a Dual<12> number, the analogue of Sacado SFad);
 *   - the energy Pi whose gradient is F (reading R1-energy);
 *   - NEXT-f1: the lateral margin term (ocean back-pressure, reading
 *     L12, quadrature L20) on the boundary-edge faces, term ORA_LATERAL;
 *   - NEXT-f3: the Arrhenius flow factor A = A0 exp(-Q/(R T*));
 *   - the CSR graph by brute force (std::set per row).
 * Readings where the paper is silent (quadrature, regularisation, basal measure,
 * floating mask, numbering) are listed in DESIGN.md section "Readings".
 *
 * Pins (tests/test_oracle_pins.py, tests/test_oracle_pins_next.py,
 * tests/test_oracle_pins_pernode.py): closed-form P1
 * right-prism operators (n = 1), affinity, the patch test, driving-stress and
 * basal totals AND their per-node closed forms (int phi_i on columns of unequal
 * height; beta = hat function of one vertex) for wedges, tets and hexes --
 * tools/mutate_oracle.py shows a rotation of either term's node weights fails
 * them --, partition of unity, Glen homogeneity,
 * Euler identities, the rigid nullspace, symmetry and convexity, FD Jacobian and
 * FD energy gradient, brute-force graph counts, the paper's mesh sizes
 * (tests/golden/paper_counts.json); NEXT rows: the floating-front integral, level
 * split, Q = 0 and temperature-ratio laws, tet / hex patch tests and closed forms.
 * Parity unpinned: no function is unpinned (DESIGN.md section 3 names the pin
 * of every function and term), but PAPER.md prints no
 * residual or Jacobian value, so ABSOLUTE values at C2-C5 rest on these pins and
 * on the conventions L4, L7-L10 the paper leaves open.
 *
 * All functions return 0 on success, a negative code on invalid input.
 */
#ifndef FO_ORACLE_H
#define FO_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double rho, g, rho_w;  /* kg m^-3, m s^-2, kg m^-3 */
  double glen_n;         /* Glen exponent n */
  double eps_reg;        /* viscosity regularisation, a^-2 (reading L1) */
  double A;              /* flow factor Pa^-n a^-1 when A_elem == NULL */
  double H_min;          /* columns thinner than this are rejected */
} ora_params;

typedef struct {
  int64_t n_vert;
  const double* xy;      /* [n_vert][2] */
  int64_t n_tri;
  const int32_t* tri;    /* [n_tri][3], CCW */
  int32_t n_layers;      /* L */
  const double* sigma;   /* [L+1], 0 = bed .. 1 = surface */
  const double* thickness;  /* H [n_vert] */
  const double* surface;    /* s [n_vert] */
  const double* bed;        /* b [n_vert] or NULL (floating mask only) */
  const double* beta;       /* [n_vert] */
  const double* A_elem;     /* [n_tri*L] or NULL */
  ora_params p;
  /* NEXT-f3: A = A0 exp(-Q / (R T*)) per wedge when T_star != NULL
   * (overrides A_elem and p.A); R = 8.314462618 J mol^-1 K^-1 */
  const double* T_star;     /* [n_tri*L] K, or NULL */
  double A0;                /* Pa^-n a^-1 */
  double Q_act;             /* J mol^-1 */
  /* NEXT-f4: 0 = 6-node wedge (reading L5), 1 = three 4-node
   * P1 tetrahedra per prism, split by global vertex id (reading L22), 2 = the
   * footprint is QUADRILATERAL (tri holds n_tri x 4 CCW corners) and every
   * layer element an 8-node trilinear hexahedron (reading L23) */
  int32_t elem_type;
} ora_mesh;

/* term mask for the pins: which integrals enter R / J / Pi */
enum { ORA_VISC = 1, ORA_BODY = 2, ORA_BASAL = 4, ORA_ALL = 7,
       /* NEXT-f1: lateral margin term (reading L12), not in ORA_ALL */
       ORA_LATERAL = 8 };

/* validation (CCW, H >= H_min, sigma ascending 0..1, indices in range) */
int ora_validate(const ora_mesh* m);

/* brute-force CSR graph: call with row_ptr only to get nnz (col_idx NULL) */
int ora_graph(const ora_mesh* m, int64_t* row_ptr, int32_t* col_idx, int64_t* nnz);

/* residual R[n_dof], M[n_dof] = sum_e |r_e| (may be NULL), Pi (may be NULL) */
int ora_residual(const ora_mesh* m, int terms, const double* U, double* R,
                 double* M, double* Pi);

/* AD Jacobian into CSR values (graph from ora_graph), R may be NULL */
int ora_jacobian(const ora_mesh* m, int terms, const double* U,
                 const int64_t* row_ptr, const int32_t* col_idx,
                 double* R, double* vals);

/* energy restricted to wedges touching global DOF `dof` (dof < 0: all wedges) */
int ora_energy(const ora_mesh* m, int terms, const double* U, int64_t dof, double* Pi);

/* one wedge (t, k): element residual r[12], element Jacobian Je[12*12]
 * (row-major, local DOF = 2*i + a, i = t_local + 3*level), and the 12 global DOFs */
int ora_element(const ora_mesh* m, int terms, const double* U, int64_t t, int32_t k,
                double* r, double* Je, int64_t* gdof);

#ifdef __cplusplus
}
#endif
#endif
