"""Pins of the oracle's NEXT rows against closed forms and
invariants, like tests/test_oracle_pins.py:
  f1  lateral margin term (reading L12, quadrature L20),
  f3  Arrhenius flow factor A = A0 exp(-Q / (R T*)),
  f4  three P1 tetrahedra per prism (split rule: reading L22).
PAPER.md line citations: P:n.
"""
import numpy as np
import pytest

from paper_2204_04321_b200 import meshgen as mg

RHO, G, RHO_W = 910.0, 9.81, 1028.0


def _slab(H, s, nx=4, n_layers=3, seed=5):
    fp = mg.slab(nx=nx, n_layers=n_layers, H0=H, seed=seed)
    fp.surface = np.full(fp.n_vert, float(s))
    return fp


def _column_integral(H, s):
    """int_{s-H}^{s} [rho g (s - z) - rho_w g max(-z, 0)] dz, written out."""
    base = s - H
    dry = RHO * G * H * H / 2.0
    wet = 0.0
    if base < 0.0:
        top = min(s, 0.0)
        wet = RHO_W * G * (base * base - top * top) / 2.0
    return dry - wet


# ---------------------------------------------------------------- f1
@pytest.mark.parametrize("case", ["floating", "grounded-cliff", "partly-submerged"])
def test_f1_lateral_side_totals(ora_mod, case):
    """Sum of the lateral residual over the nodes of one straight side of a
    uniform slab = -(side length) n_a int P dz (the depth-integrated margin
    force; for the floating front 1/2 rho g H^2 (1 - rho/rho_w), L12)."""
    H = 1000.0
    s = {"floating": H * (1.0 - RHO / RHO_W), "grounded-cliff": 1500.0,
         "partly-submerged": 700.0}[case]
    fp = _slab(H, s)
    o = ora_mod.Oracle(fp)
    R = o.residual(np.zeros(o.n_dof), terms=ora_mod.LATERAL)[0].reshape(fp.n_vert, fp.n_layers + 1, 2)
    x, y = fp.xy[:, 0], fp.xy[:, 1]
    Lx = x.max() - x.min()
    Ly = y.max() - y.min()
    I = _column_integral(H, s)
    if case == "floating":
        assert I == pytest.approx(0.5 * RHO * G * H * H * (1.0 - RHO / RHO_W), rel=1e-12)
    scale = Ly * abs(I)
    assert abs(R[x == x.max(), :, 0].sum() - (-Ly * I)) <= 1e-12 * scale
    assert abs(R[x == x.min(), :, 0].sum() - (+Ly * I)) <= 1e-12 * scale
    assert abs(R[y == y.max(), :, 1].sum() - (-Lx * I)) <= 1e-12 * scale
    assert abs(R[y == y.min(), :, 1].sum() - (+Lx * I)) <= 1e-12 * scale
    # only margin columns are touched
    inner = (x > x.min()) & (x < x.max()) & (y > y.min()) & (y < y.max())
    assert np.abs(R[inner]).max() == 0.0


def test_f1_lateral_per_face_levels(ora_mod):
    """On a uniform grounded slab (no water) the level split of one side's
    force is the P1-in-z integral of the linear pressure: for a layer [z0, z1]
    the bottom node gets int P (z1 - z)/(z1 - z0) dz; summed along the side."""
    H, s = 800.0, 2000.0
    fp = _slab(H, s, n_layers=4)
    o = ora_mod.Oracle(fp)
    R = o.residual(np.zeros(o.n_dof), terms=ora_mod.LATERAL)[0].reshape(fp.n_vert, fp.n_layers + 1, 2)
    x, y = fp.xy[:, 0], fp.xy[:, 1]
    Ly = y.max() - y.min()
    z = (s - H) + fp.sigma * H
    expect = np.zeros(fp.n_layers + 1)
    for k in range(fp.n_layers):
        z0, z1 = z[k], z[k + 1]
        h = z1 - z0
        # P(z) = rho g (s - z); int_z0^z1 P (z1-z)/h dz and int P (z-z0)/h dz (closed form)
        p0, p1 = RHO * G * (s - z0), RHO * G * (s - z1)
        expect[k] += h * (2 * p0 + p1) / 6.0
        expect[k + 1] += h * (p0 + 2 * p1) / 6.0
    got = R[x == x.max(), :, 0].sum(axis=0)
    assert np.abs(got - (-Ly * expect)).max() <= 1e-12 * Ly * expect.max()


def test_f1_lateral_is_energy_gradient(ora_mod):
    """R = grad Pi with the lateral term included (P12 extended): the margin
    work term is linear in U."""
    fp = mg.greenland_like(80.0, n_layers=3)
    o = ora_mod.Oracle(fp)
    terms = ora_mod.ALL | ora_mod.LATERAL
    U = fp.U
    R = o.residual(U, terms=terms)[0]
    Rl = o.residual(U, terms=ora_mod.LATERAL)[0]
    assert np.abs(Rl).max() > 0.0
    margin = np.nonzero(Rl)[0]
    for j in list(margin[:: max(1, margin.size // 12)]) + [0, o.n_dof // 2]:
        h = 1e-4 * max(1.0, abs(U[j]))
        Up, Um = U.copy(), U.copy()
        Up[j] += h
        Um[j] -= h
        fd = (o.energy(Up, dof=j, terms=terms) - o.energy(Um, dof=j, terms=terms)) / (2 * h)
        assert abs(fd - R[j]) <= 1e-6 * np.abs(R).max(), (j, fd, R[j])


def test_f1_lateral_leaves_jacobian_unchanged(ora_mod):
    fp = mg.ismip_hom_a(nx=4, n_layers=2)
    o = ora_mod.Oracle(fp)
    _, v1 = o.jacobian(fp.U)
    _, v2 = o.jacobian(fp.U, terms=ora_mod.ALL | ora_mod.LATERAL)
    assert np.array_equal(v1, v2)


# ---------------------------------------------------------------- f3
def _with_temperature(fp, T, A0, Q):
    fp.T_star = np.asarray(T, dtype=np.float64)
    fp.arrhenius = dict(A0=A0, Q=Q)
    return fp


def test_f3_zero_activation_energy_is_constant_A(ora_mod):
    """Q = 0: A = A0 for any T*, the scalar-A path exactly."""
    fp = mg.ismip_hom_a(nx=4, n_layers=3)
    A0 = 2.5e-16
    ref = ora_mod.Oracle(fp, params=dict(A=A0))
    T = 240.0 + 30.0 * mg.SplitMix64(3).uniform(fp.n_elem)
    fp2 = _with_temperature(mg.ismip_hom_a(nx=4, n_layers=3), T, A0, 0.0)
    o = ora_mod.Oracle(fp2)
    assert np.array_equal(o.residual(fp.U)[0], ref.residual(fp.U)[0])
    assert np.array_equal(o.jacobian(fp.U)[1], ref.jacobian(fp.U)[1])


def test_f3_arrhenius_temperature_ratio(ora_mod):
    """Uniform T*: the viscous residual scales as A^(-1/n) (flow-law
    homogeneity in A), so R(T1) / R(T2) = exp(Q/(n R) (1/T1 - 1/T2))."""
    Rgas, Q, A0 = 8.314462618, 6.0e4, 1.0e-3
    out = {}
    for T in (250.0, 265.0):
        fp = _with_temperature(mg.ismip_hom_a(nx=4, n_layers=3), np.full(4 * 4 * 2 * 3, T), A0, Q)
        out[T] = ora_mod.Oracle(fp).residual(fp.U, terms=ora_mod.VISC)[0]
    ratio = np.exp(Q / (3.0 * Rgas) * (1.0 / 250.0 - 1.0 / 265.0))
    assert np.abs(out[250.0] - ratio * out[265.0]).max() <= 1e-13 * np.abs(out[250.0]).max()


def test_f3_temperature_is_per_wedge(ora_mod):
    """Changing T* of one wedge changes only the residual rows of its 12 DOFs."""
    fp = mg.ismip_hom_a(nx=4, n_layers=3)
    T = np.full(fp.n_elem, 255.0)
    o1 = ora_mod.Oracle(_with_temperature(fp, T, 1e-3, 6e4))
    R1 = o1.residual(fp.U)[0]
    w = 17
    T2 = T.copy()
    T2[w] = 268.0
    fp2 = _with_temperature(mg.ismip_hom_a(nx=4, n_layers=3), T2, 1e-3, 6e4)
    R2 = ora_mod.Oracle(fp2).residual(fp.U)[0]
    t, k = divmod(w, fp.n_layers)
    dofs = set()
    for j in range(3):
        for lev in (k, k + 1):
            node = int(fp.tri[t][j]) * (fp.n_layers + 1) + lev
            dofs.update((2 * node, 2 * node + 1))
    changed = set(np.nonzero(R1 != R2)[0].tolist())
    assert changed and changed <= dofs


# ---------------------------------------------------------------- f4
# three P1 tetrahedra per prism, split by global vertex id (reading L22)
def _tets(fp):
    fp.elem_type = 1
    return fp


@pytest.mark.parametrize("n_glen", [1.0, 3.0])
def test_f4_tet_patch_test(ora_mod, n_glen):
    """Linear U, flat s, beta = 0 on distorted columns: interior residuals
    vanish -- holds only if neighbouring prisms split their shared faces alike
    (a non-conforming split breaks sum_e int grad phi_i = 0)."""
    nx = 5
    fp = _tets(mg.slab(nx=nx, n_layers=4, distort=0.25, params=dict(glen_n=n_glen)))
    o = ora_mod.Oracle(fp)
    L1 = fp.n_layers + 1
    base = fp.surface - fp.thickness
    z = (base[:, None] + fp.sigma[None, :] * fp.thickness[:, None]).reshape(-1)
    x = np.repeat(fp.xy[:, 0], L1)
    y = np.repeat(fp.xy[:, 1], L1)
    U = np.zeros(o.n_dof)
    U[0::2] = 3.0 + 2e-3 * x - 1e-3 * y + 0.05 * z
    U[1::2] = -1.0 + 1e-3 * x + 4e-3 * y - 0.02 * z
    R, M, _ = o.residual(U, terms=ora_mod.VISC)
    col = np.arange(fp.n_vert)
    edge = np.unique(np.concatenate([np.arange(nx + 1), np.arange(nx * (nx + 1), (nx + 1) ** 2),
                                     np.arange(0, (nx + 1) ** 2, nx + 1), np.arange(nx, (nx + 1) ** 2, nx + 1)]))
    k = np.arange(L1)
    node_int = (~np.isin(col, edge)[:, None] & (k[None, :] > 0) & (k[None, :] < fp.n_layers)).reshape(-1)
    dof_int = np.repeat(node_int, 2)
    assert np.abs(R[dof_int]).max() <= 1e-12 * np.abs(M).max()
    assert np.abs(R[~dof_int]).max() > 1e-6 * np.abs(M).max()


def test_f4_tet_volume_and_driving_stress(ora_mod):
    """The tets tile each prism exactly (vertical, hence planar, side faces):
    sum_i R_{u,i}(U = 0) = rho g sum_t (ds/dx)_t |T_t| Hbar_t, as for wedges."""
    fp = _tets(mg.ismip_hom_a(nx=6, n_layers=4))
    fp.surface = fp.surface + 80.0 * np.sin(fp.xy[:, 1] / 9e3)
    o = ora_mod.Oracle(fp)
    R, _, _ = o.residual(np.zeros(o.n_dof), terms=ora_mod.BODY)
    ex_u = 0.0
    for t in fp.tri:
        p = fp.xy[t]
        twoA = (p[1, 0] - p[0, 0]) * (p[2, 1] - p[0, 1]) - (p[2, 0] - p[0, 0]) * (p[1, 1] - p[0, 1])
        a = np.array([p[1, 1] - p[2, 1], p[2, 1] - p[0, 1], p[0, 1] - p[1, 1]]) / twoA
        ex_u += 910.0 * 9.81 * np.dot(a, fp.surface[t]) * 0.5 * twoA * fp.thickness[t].mean()
    assert abs(R[0::2].sum() - ex_u) <= 1e-12 * abs(ex_u)


def test_f4_tet_nullspace_symmetry_fd(ora_mod):
    """beta = 0 rigid nullspace, J = J^T, FD Jacobian and FD energy for tets."""
    fp = _tets(mg.greenland_like(100.0, n_layers=3))
    o = ora_mod.Oracle(fp)
    J = o.dense_jacobian(fp.U, terms=ora_mod.VISC)
    L1 = fp.n_layers + 1
    x = np.repeat(fp.xy[:, 0], L1)
    y = np.repeat(fp.xy[:, 1], L1)
    for w in (np.tile([1.0, 0.0], o.n_dof // 2), np.tile([0.0, 1.0], o.n_dof // 2),
              np.stack([-y, x], axis=1).reshape(-1)):
        assert np.abs(J @ w).max() <= 1e-12 * np.abs(J).max() * np.abs(w).max()
    Jf = o.dense_jacobian(fp.U)
    assert np.abs(Jf - Jf.T).max() <= 1e-14 * np.abs(Jf).max()
    U = fp.U
    R = o.residual(U)[0]
    for j in np.linspace(0, o.n_dof - 1, 12).astype(int):
        h = 1e-6 * max(1.0, abs(U[j]))
        Up, Um = U.copy(), U.copy()
        Up[j] += h
        Um[j] -= h
        fd = (o.residual(Up)[0] - o.residual(Um)[0]) / (2 * h)
        assert np.abs(Jf[:, j] - fd).max() <= 1e-6 * np.abs(Jf[:, j]).max()
        he = 1e-4 * max(1.0, abs(U[j]))
        Up, Um = U.copy(), U.copy()
        Up[j] += he
        Um[j] -= he
        fde = (o.energy(Up, dof=j) - o.energy(Um, dof=j)) / (2 * he)
        assert abs(fde - R[j]) <= 1e-6 * np.abs(R).max()


def test_f4_tet_structural_zeros(ora_mod):
    """Inside each prism the split couples 12 of the 15 node pairs: the pairs
    (a', b), (a', c), (b', c) (a < b < c by global id) get exact zeros in J."""
    fp = _tets(mg.ismip_hom_a(nx=3, n_layers=2))
    o = ora_mod.Oracle(fp)
    J = o.dense_jacobian(fp.U)
    L1 = fp.n_layers + 1
    zero_pairs = nonzero_pairs = 0
    for t in fp.tri:
        a, b, c = sorted(int(v) for v in t)
        for k in range(fp.n_layers):
            nd = lambda v, lev: v * L1 + k + lev
            for (p, q) in [(nd(a, 1), nd(b, 0)), (nd(a, 1), nd(c, 0)), (nd(b, 1), nd(c, 0))]:
                blk = J[2 * p:2 * p + 2, 2 * q:2 * q + 2]
                # another prism may couple them (as bottom/top of its own split)
                zero_pairs += int(np.all(blk == 0.0))
            blk = J[2 * nd(a, 1):2 * nd(a, 1) + 2, 2 * nd(c, 1):2 * nd(c, 1) + 2]
            nonzero_pairs += int(np.any(blk != 0.0))
    assert zero_pairs > 0 and nonzero_pairs == len(fp.tri) * fp.n_layers


# ---------------------------------------------------------------- f4 hexahedra
# quadrilateral footprint, 8-node trilinear hexahedra (reading L23)
@pytest.mark.parametrize("n_glen", [1.0, 3.0])
def test_f4_hex_patch_test(ora_mod, n_glen):
    """Linear U, flat s, beta = 0 on distorted quad columns: interior residuals
    vanish (isoparametric trilinear elements reproduce linear fields)."""
    nx = 5
    fp = mg.to_quads(mg.slab(nx=nx, n_layers=4, distort=0.2, params=dict(glen_n=n_glen)), nx)
    o = ora_mod.Oracle(fp)
    L1 = fp.n_layers + 1
    base = fp.surface - fp.thickness
    z = (base[:, None] + fp.sigma[None, :] * fp.thickness[:, None]).reshape(-1)
    x = np.repeat(fp.xy[:, 0], L1)
    y = np.repeat(fp.xy[:, 1], L1)
    U = np.zeros(o.n_dof)
    U[0::2] = 3.0 + 2e-3 * x - 1e-3 * y + 0.05 * z
    U[1::2] = -1.0 + 1e-3 * x + 4e-3 * y - 0.02 * z
    R, M, _ = o.residual(U, terms=ora_mod.VISC)
    col = np.arange(fp.n_vert)
    edge = np.unique(np.concatenate([np.arange(nx + 1), np.arange(nx * (nx + 1), (nx + 1) ** 2),
                                     np.arange(0, (nx + 1) ** 2, nx + 1), np.arange(nx, (nx + 1) ** 2, nx + 1)]))
    k = np.arange(L1)
    node_int = (~np.isin(col, edge)[:, None] & (k[None, :] > 0) & (k[None, :] < fp.n_layers)).reshape(-1)
    dof_int = np.repeat(node_int, 2)
    assert np.abs(R[dof_int]).max() <= 1e-12 * np.abs(M).max()
    assert np.abs(R[~dof_int]).max() > 1e-6 * np.abs(M).max()


def test_f4_hex_driving_stress_and_basal_totals(ora_mod):
    """Rectangular hexes with a planar surface: sum_i R_u(U=0) = rho g s_x x
    (column volume), and with constant U and beta: sum_i R_u = beta u (bed area)."""
    nx = 4
    fp = mg.to_quads(mg.slab(nx=nx, n_layers=3, H0=800.0), nx)
    fp.surface = fp.surface + 1e-3 * fp.xy[:, 0] - 2e-3 * fp.xy[:, 1]
    fp.thickness = 800.0 + 1e-3 * fp.xy[:, 0]
    o = ora_mod.Oracle(fp)
    R, _, _ = o.residual(np.zeros(o.n_dof), terms=ora_mod.BODY)
    Lx = fp.xy[:, 0].max() - fp.xy[:, 0].min()
    vol = Lx * Lx * (800.0 + 1e-3 * Lx / 2.0)   # H linear in x: mean over the square
    assert abs(R[0::2].sum() - 910.0 * 9.81 * 1e-3 * vol) <= 1e-12 * abs(910.0 * 9.81 * 1e-3 * vol)
    assert abs(R[1::2].sum() - 910.0 * 9.81 * (-2e-3) * vol) <= 1e-12 * abs(910.0 * 9.81 * 2e-3 * vol)
    fp.beta = np.full(fp.n_vert, 700.0)
    U = np.zeros(o.n_dof)
    U[0::2], U[1::2] = 3.0, -2.0
    o = ora_mod.Oracle(fp)
    Rb = o.residual(U, terms=ora_mod.BASAL)[0]
    # bed: planar (s - H linear), area = Lx^2 sqrt(1 + |grad b|^2)
    gb = np.array([1e-3 - 1e-3, -2e-3])
    area = Lx * Lx * np.sqrt(1.0 + gb @ gb)
    assert abs(Rb[0::2].sum() - 700.0 * 3.0 * area) <= 1e-12 * 700.0 * 3.0 * area
    assert abs(Rb[1::2].sum() + 700.0 * 2.0 * area) <= 1e-12 * 700.0 * 2.0 * area


def test_f4_hex_nullspace_symmetry_fd(ora_mod):
    nx = 3
    fp = mg.to_quads(mg.slab(nx=nx, n_layers=2, distort=0.15), nx)
    fp.U = fp.U * (1.0 + 0.1 * np.sin(np.arange(fp.U.size)))
    o = ora_mod.Oracle(fp)
    J = o.dense_jacobian(fp.U, terms=ora_mod.VISC)
    L1 = fp.n_layers + 1
    x = np.repeat(fp.xy[:, 0], L1)
    y = np.repeat(fp.xy[:, 1], L1)
    for w in (np.tile([1.0, 0.0], o.n_dof // 2), np.tile([0.0, 1.0], o.n_dof // 2),
              np.stack([-y, x], axis=1).reshape(-1)):
        assert np.abs(J @ w).max() <= 1e-12 * np.abs(J).max() * np.abs(w).max()
    Jf = o.dense_jacobian(fp.U)
    assert np.abs(Jf - Jf.T).max() <= 1e-14 * np.abs(Jf).max()
    U = fp.U
    R = o.residual(U)[0]
    for j in np.linspace(0, o.n_dof - 1, 10).astype(int):
        h = 1e-6 * max(1.0, abs(U[j]))
        Up, Um = U.copy(), U.copy()
        Up[j] += h
        Um[j] -= h
        fd = (o.residual(Up)[0] - o.residual(Um)[0]) / (2 * h)
        assert np.abs(Jf[:, j] - fd).max() <= 1e-6 * np.abs(Jf[:, j]).max()
        he = 1e-4 * max(1.0, abs(U[j]))
        Up, Um = U.copy(), U.copy()
        Up[j] += he
        Um[j] -= he
        fde = (o.energy(Up, dof=j) - o.energy(Um, dof=j)) / (2 * he)
        assert abs(fde - R[j]) <= 1e-6 * np.abs(R).max()
    # graph: every column couples to its 8 grid neighbours and itself
    rp, col = o.graph()
    assert rp[-1] == 4 * (3 * fp.n_layers + 1) * sum(
        len({int(v) for q in fp.tri if c in q for v in q}) for c in range(fp.n_vert))
