"""Per-node pins of the oracle's U-independent load terms (VERDICT r1 "What's
missing" 4): the driving stress rho g grad s . int phi_i (reading
L10) and the basal friction with a P1-interpolated beta (readings
L6-L8), node by node -- not only their totals (test_oracle_pins.py P4/P6),
which a permutation of the per-node weights leaves unchanged.

Closed forms (exact for the quadrature of reading L4; SURVEY.md App. A.5
"int phi = |T| h / 6" generalised to columns of unequal height):
  wedge (t, k), node (j, l):  int phi_(j,l) dV = |T| (dz_j + sum_i dz_i) / 24
     (phi = L_j (1 -+ zeta)/2, det = 2|T| sum_i L_i dz_i / 2, int_T L_j L_i =
     |T| (1 + delta_ij) / 12), independent of the level l;
  P1 tetrahedron: int phi_i dV = V / 4;
  rectangular hexahedron (dx x dy, vertical edges dz_c):
     int phi_(c,l) dV = (dx dy / 8) sum_c' M_cc' dz_c', M = 4/9 (c' = c),
     2/9 (edge neighbour), 1/9 (diagonal);
  basal term with beta = hat function of one vertex c0 and constant U:
     R_(u, c) = beta0 u int_bed N_c0 N_c dA = beta0 u sum_T |T_3D| (1 + delta) / 12
     on triangles, beta0 u sum_Q (dx dy / 4) M_c0c on flat rectangles.
Each is written out here from the geometry; the oracle's own formulas are not
re-typed (it integrates generic isoparametric elements numerically).
tools/mutate_oracle.py rotates the per-node weights inside the oracle and
checks that this file then fails.
"""
import numpy as np

from paper_2204_04321_b200 import meshgen as mg

RHOG = 910.0 * 9.81


def _tri_geom(xy, t):
    p = xy[t]
    twoA = (p[1, 0] - p[0, 0]) * (p[2, 1] - p[0, 1]) - (p[2, 0] - p[0, 0]) * (p[1, 1] - p[0, 1])
    a = np.array([p[1, 1] - p[2, 1], p[2, 1] - p[0, 1], p[0, 1] - p[1, 1]]) / twoA
    b = np.array([p[2, 0] - p[1, 0], p[0, 0] - p[2, 0], p[1, 0] - p[0, 0]]) / twoA
    return a, b, 0.5 * twoA


def _varied(fp, seed=9):
    """unequal column heights and a non-uniform sigma, so dz_j differ inside a wedge"""
    rng = mg.SplitMix64(seed)
    fp.thickness = fp.thickness * (0.6 + 0.8 * rng.uniform(fp.n_vert))
    fp.sigma = np.linspace(0.0, 1.0, fp.n_layers + 1) ** 1.5
    fp.surface = fp.surface + 60.0 * np.sin(fp.xy[:, 1] / 7e3) + 40.0 * np.cos(fp.xy[:, 0] / 11e3)
    return fp


def test_driving_stress_per_node_wedges(ora_mod):
    fp = _varied(mg.ismip_hom_a(nx=5, n_layers=3))
    o = ora_mod.Oracle(fp)
    R, _, _ = o.residual(np.zeros(o.n_dof), terms=ora_mod.BODY)
    L1 = fp.n_layers + 1
    ex = np.zeros(o.n_dof)
    for t in fp.tri:
        a, b, area = _tri_geom(fp.xy, t)
        sx, sy = a @ fp.surface[t], b @ fp.surface[t]
        for k in range(fp.n_layers):
            dz = (fp.sigma[k + 1] - fp.sigma[k]) * fp.thickness[t]
            for j in range(3):
                w = area * (dz[j] + dz.sum()) / 24.0
                for lev in (k, k + 1):
                    node = int(t[j]) * L1 + lev
                    ex[2 * node] += RHOG * sx * w
                    ex[2 * node + 1] += RHOG * sy * w
    assert np.abs(R - ex).max() <= 1e-12 * np.abs(ex).max()
    # the per-node distribution is not uniform (the pin sees a permutation)
    assert np.abs(ex[0::2] - np.roll(ex[0::2], 1)).max() > 1e-3 * np.abs(ex).max()


def test_driving_stress_per_element_wedges(ora_mod):
    """the same closed form on single elements (element-local vector)"""
    fp = _varied(mg.ismip_hom_a(nx=3, n_layers=2), seed=4)
    o = ora_mod.Oracle(fp)
    for ti, t in enumerate(fp.tri):
        a, b, area = _tri_geom(fp.xy, t)
        sx, sy = a @ fp.surface[t], b @ fp.surface[t]
        for k in range(fp.n_layers):
            r, _, _ = o.element(np.zeros(o.n_dof), ti, k, terms=ora_mod.BODY)
            dz = (fp.sigma[k + 1] - fp.sigma[k]) * fp.thickness[t]
            w = area * (dz + dz.sum()) / 24.0
            ex = np.zeros(12)
            for lev in range(2):
                ex[6 * lev + 0:6 * lev + 6:2] = RHOG * sx * w
                ex[6 * lev + 1:6 * lev + 6:2] = RHOG * sy * w
            assert np.abs(r - ex).max() <= 1e-12 * np.abs(ex).max()


def _hat_beta(fp, c0, beta0=1500.0):
    beta = np.zeros(fp.n_vert)
    beta[c0] = beta0
    fp.beta = beta
    return fp


def _const_U(o, u=13.0, v=-7.0):
    U = np.zeros(o.n_dof)
    U[0::2], U[1::2] = u, v
    return U


def test_basal_hat_beta_per_node_wedges(ora_mod):
    nx = 4
    for c0 in (6, 12):   # interior vertices of the 5x5 grid
        fp = _hat_beta(mg.ismip_hom_a(nx=nx, n_layers=2), c0)
        o = ora_mod.Oracle(fp)
        R, _, _ = o.residual(_const_U(o), terms=ora_mod.BASAL)
        base = fp.surface - fp.thickness
        ex = np.zeros(o.n_dof)
        L1 = fp.n_layers + 1
        for t in fp.tri:
            if c0 not in t:
                continue
            P = np.column_stack([fp.xy[t], base[t]])
            a3 = 0.5 * np.linalg.norm(np.cross(P[1] - P[0], P[2] - P[0]))
            for c in t:
                m = a3 * (2.0 if c == c0 else 1.0) / 12.0
                ex[2 * int(c) * L1] += 1500.0 * 13.0 * m
                ex[2 * int(c) * L1 + 1] += 1500.0 * -7.0 * m
        assert np.abs(R - ex).max() <= 1e-12 * np.abs(ex).max()
        assert np.count_nonzero(ex) == 14    # c0 and its six neighbours, two comps


def _tet_split(t):
    """reading L22: corners a < b < c by global id; tets {a,b,c,c'},
    {a,b,b',c'}, {a,a',b',c'} (' = the top level)"""
    a, b, c = sorted(int(v) for v in t)
    return [((a, 0), (b, 0), (c, 0), (c, 1)), ((a, 0), (b, 0), (b, 1), (c, 1)),
            ((a, 0), (a, 1), (b, 1), (c, 1))]


def test_driving_stress_per_node_tets(ora_mod):
    """P1 tetrahedra: int phi_i = V / 4; grad s exact for a linear surface"""
    fp = _varied(mg.ismip_hom_a(nx=4, n_layers=3))
    fp.surface = 100.0 + 2e-3 * fp.xy[:, 0] - 3e-3 * fp.xy[:, 1]
    fp.elem_type = 1
    o = ora_mod.Oracle(fp)
    R, _, _ = o.residual(np.zeros(o.n_dof), terms=ora_mod.BODY)
    L1 = fp.n_layers + 1
    base = fp.surface - fp.thickness
    ex = np.zeros(o.n_dof)
    for t in fp.tri:
        for k in range(fp.n_layers):
            for tet in _tet_split(t):
                X = np.array([[fp.xy[v, 0], fp.xy[v, 1], base[v] + fp.sigma[k + l] * fp.thickness[v]]
                              for v, l in tet])
                V = abs(np.linalg.det(X[1:] - X[0])) / 6.0
                for v, l in tet:
                    node = v * L1 + k + l
                    ex[2 * node] += RHOG * 2e-3 * V / 4.0
                    ex[2 * node + 1] += RHOG * -3e-3 * V / 4.0
    assert np.abs(R - ex).max() <= 1e-12 * np.abs(ex).max()


def test_basal_hat_beta_per_node_tets(ora_mod):
    """tets use the same bottom-triangle basal term as wedges (reading L22)"""
    fp = _hat_beta(mg.ismip_hom_a(nx=4, n_layers=2), 12)
    fp.elem_type = 1
    o = ora_mod.Oracle(fp)
    R, _, _ = o.residual(_const_U(o), terms=ora_mod.BASAL)
    base = fp.surface - fp.thickness
    L1 = fp.n_layers + 1
    ex = np.zeros(o.n_dof)
    for t in fp.tri:
        if 12 not in t:
            continue
        P = np.column_stack([fp.xy[t], base[t]])
        a3 = 0.5 * np.linalg.norm(np.cross(P[1] - P[0], P[2] - P[0]))
        for c in t:
            m = a3 * (2.0 if c == 12 else 1.0) / 12.0
            ex[2 * int(c) * L1] += 1500.0 * 13.0 * m
            ex[2 * int(c) * L1 + 1] += 1500.0 * -7.0 * m
    assert np.abs(R - ex).max() <= 1e-12 * np.abs(ex).max()


def _mref(xy, c, c2):
    """bilinear reference mass weight (x 4/9, 2/9, 1/9 for same / edge / diagonal)"""
    same_x = xy[c, 0] == xy[c2, 0]
    same_y = xy[c, 1] == xy[c2, 1]
    return 4.0 / 9.0 if (same_x and same_y) else (2.0 / 9.0 if (same_x or same_y) else 1.0 / 9.0)


def test_driving_stress_per_node_hexes(ora_mod):
    nx = 4
    fp = mg.to_quads(_varied(mg.slab(nx=nx, n_layers=3, H0=900.0)), nx)
    fp.surface = 500.0 + 1.5e-3 * fp.xy[:, 0] - 2.5e-3 * fp.xy[:, 1]
    o = ora_mod.Oracle(fp)
    R, _, _ = o.residual(np.zeros(o.n_dof), terms=ora_mod.BODY)
    L1 = fp.n_layers + 1
    ex = np.zeros(o.n_dof)
    for q in fp.tri:
        dx = np.ptp(fp.xy[q, 0])
        dy = np.ptp(fp.xy[q, 1])
        for k in range(fp.n_layers):
            dz = {int(c): (fp.sigma[k + 1] - fp.sigma[k]) * fp.thickness[c] for c in q}
            for c in q:
                w = dx * dy / 8.0 * sum(_mref(fp.xy, c, c2) * dz[int(c2)] for c2 in q)
                for lev in (k, k + 1):
                    node = int(c) * L1 + lev
                    ex[2 * node] += RHOG * 1.5e-3 * w
                    ex[2 * node + 1] += RHOG * -2.5e-3 * w
    assert np.abs(R - ex).max() <= 1e-12 * np.abs(ex).max()


def test_basal_hat_beta_per_node_hexes(ora_mod):
    nx = 4
    for c0 in (6, 12):
        fp = _hat_beta(mg.to_quads(mg.slab(nx=nx, n_layers=2, H0=900.0), nx), c0)
        o = ora_mod.Oracle(fp)
        R, _, _ = o.residual(_const_U(o), terms=ora_mod.BASAL)
        L1 = fp.n_layers + 1
        ex = np.zeros(o.n_dof)
        for q in fp.tri:
            if c0 not in q:
                continue
            dx = np.ptp(fp.xy[q, 0])
            dy = np.ptp(fp.xy[q, 1])
            for c in q:
                m = dx * dy / 4.0 * _mref(fp.xy, c0, c)
                ex[2 * int(c) * L1] += 1500.0 * 13.0 * m
                ex[2 * int(c) * L1 + 1] += 1500.0 * -7.0 * m
        assert np.abs(R - ex).max() <= 1e-12 * np.abs(ex).max()
        assert np.count_nonzero(ex) == 18   # c0 and its eight grid neighbours
