"""GPU parity: libfo's CUDA kernels (through the C ABI) against the CPU oracle,
element by element on the same seeded inputs:
  residual  |R_gpu - R_ora|_inf <= 1e-12 ||M||_inf, M = sum_e |r_e| (oracle)
  Jacobian  |dJ_ij| <= 1e-11 max_k |J_ora_ik|   (row-scaled)
  graph     row_ptr / col_idx byte-identical.
"""
import numpy as np
import pytest

from paper_2204_04321_b200 import meshgen as mg

pytestmark = pytest.mark.gpu

R_TOL, J_TOL = 1e-12, 1e-11


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2204_04321_b200 import _build
    _build.build()
    return torch


def gpu_assemble(torch, fp, params=None, scatter=None, lateral=False):
    from paper_2204_04321_b200 import fo
    mesh = fo.Mesh.from_footprint(fp, params=params)
    if getattr(fp, "elem_type", 0) == 1:
        mesh.set_element(fp.elem_type)
    if lateral:
        mesh.set_lateral(True)
    if scatter is not None:
        mesh.set_scatter(scatter)
    if getattr(fp, "T_star", None) is not None:
        mesh.set_temperature(fp.T_star, fp.arrhenius["A0"], fp.arrhenius["Q"])
    U = torch.tensor(fp.U, dtype=torch.float64, device="cuda")
    R = mesh.residual(U)
    RJ, vals = mesh.jacobian(U)
    torch.cuda.synchronize()
    rp, col = mesh.graph().to_host()
    out = dict(R=R.cpu().numpy(), RJ=RJ.cpu().numpy(), vals=vals.cpu().numpy(), row_ptr=rp, col=col,
               mesh=mesh)
    return out


def check_parity(o, g, params=None, fp=None, terms=None):
    kw = {} if terms is None else dict(terms=terms)
    R, M, _ = o.residual(fp.U, **kw)
    rp, col = o.graph()
    assert g["row_ptr"].tobytes() == rp.tobytes()
    assert g["col"].tobytes() == col.tobytes()
    _, vals = o.jacobian(fp.U, **kw)
    scale = np.abs(M).max() if M.size else 1.0
    assert np.abs(g["R"] - R).max(initial=0.0) <= R_TOL * scale
    assert np.abs(g["RJ"] - R).max(initial=0.0) <= R_TOL * scale
    rows = np.repeat(np.arange(rp.size - 1), np.diff(rp))
    rowmax = np.zeros(rp.size - 1)
    np.maximum.at(rowmax, rows, np.abs(vals))
    err = np.abs(g["vals"] - vals)
    bad = err > J_TOL * rowmax[rows]
    assert not bad.any(), (err[bad][:5], rowmax[rows][bad][:5], np.nonzero(bad)[0][:5])
    return err.max(initial=0) / max(np.abs(vals).max(initial=1.0), 1e-300)


SCATTERS = [0, 1, 2, 3]   # owner (default), atomic, warp-specialised owner, round-1 owner


@pytest.mark.parametrize("scatter", SCATTERS)
@pytest.mark.parametrize("case", ["C1", "gris-40km", "slab-distorted", "C5-small"])
def test_parity_workloads(torch_cuda, ora_mod, case, scatter):
    fp = {"C1": mg.ismip_hom_a,
          "gris-40km": lambda: mg.greenland_like(40.0),
          "slab-distorted": lambda: mg.slab(nx=7, n_layers=4, distort=0.25),
          "C5-small": lambda: mg.antarctica_like(D_km=150.0, n_layers=3)}[case]()
    if case == "C5-small":
        fp = mg.sub_footprint(fp, 0, min(fp.n_tri, 6000))
    g = gpu_assemble(torch_cuda, fp, scatter=scatter)
    check_parity(ora_mod.Oracle(fp), g, fp=fp)


def test_parity_c2_full(torch_cuda, ora_mod):
    """C2 (Greenland-like 16 km, 10 layers) at its full size."""
    fp = mg.greenland_like(16.0)
    g = gpu_assemble(torch_cuda, fp)
    check_parity(ora_mod.Oracle(fp), g, fp=fp)


@pytest.mark.parametrize("params", [dict(glen_n=1.0), dict(eps_reg=0.0), dict(glen_n=2.0),
                                    dict(A=3e-17, eps_reg=1e-6)])
def test_parity_parameters(torch_cuda, ora_mod, params):
    fp = mg.ismip_hom_a(nx=9, n_layers=4)
    fp.params.update(params)
    g = gpu_assemble(torch_cuda, fp)
    check_parity(ora_mod.Oracle(fp), g, fp=fp)


def test_parity_A_elem_and_floating(torch_cuda, ora_mod):
    fp = mg.greenland_like(60.0, n_layers=6)
    rng = mg.SplitMix64(9)
    fp.A_elem = 1e-16 * (0.2 + 2.0 * rng.uniform(fp.n_elem))
    assert (fp.params["rho"] * fp.thickness < -fp.params["rho_w"] * fp.bed).any()
    g = gpu_assemble(torch_cuda, fp)
    check_parity(ora_mod.Oracle(fp), g, fp=fp)


@pytest.mark.parametrize("scatter", SCATTERS)
def test_parity_temperature_flow_factor(torch_cuda, ora_mod, scatter):
    """NEXT-f3: A = A0 exp(-Q/(R T*)) per wedge inside the kernels."""
    fp = mg.with_temperature(mg.greenland_like(60.0, n_layers=6))
    g = gpu_assemble(torch_cuda, fp, scatter=scatter)
    check_parity(ora_mod.Oracle(fp), g, fp=fp)
    # reverting restores the scalar-A assembly
    fp0 = mg.greenland_like(60.0, n_layers=6)
    g0 = gpu_assemble(torch_cuda, fp0, scatter=scatter)
    g["mesh"].set_temperature(None)
    import torch
    R = g["mesh"].residual(torch.tensor(fp.U, device="cuda")).cpu().numpy()
    if scatter == 0:   # owner-computes: bitwise reproducible
        assert np.array_equal(R, g0["R"])
    else:              # atomic ablation: summation order varies
        assert np.abs(R - g0["R"]).max() <= 1e-13 * np.abs(g0["R"]).max()


@pytest.mark.parametrize("scatter", SCATTERS)
@pytest.mark.parametrize("case", ["gris-60km", "C5-small"])
def test_parity_lateral_margin_term(torch_cuda, ora_mod, case, scatter):
    """NEXT-f1: lateral margin term (readings L12/L20); C5-small has
    floating fronts (water pressure below sea level)."""
    if case == "C5-small":
        fp = mg.antarctica_like(D_km=150.0, n_layers=3)
        fp = mg.sub_footprint(fp, 0, min(fp.n_tri, 6000))
    else:
        fp = mg.greenland_like(60.0, n_layers=6)
    g = gpu_assemble(torch_cuda, fp, scatter=scatter, lateral=True)
    o = ora_mod.Oracle(fp)
    check_parity(o, g, fp=fp, terms=ora_mod.ALL | ora_mod.LATERAL)
    # the lateral term alone, at a scale where it is not hidden by the viscous
    # part: at U = 0 only the driving stress and the margin term remain
    import torch
    U0 = torch.zeros(fp.n_dof, dtype=torch.float64, device="cuda")
    R_on = g["mesh"].residual(U0).cpu().numpy()
    g["mesh"].set_lateral(False)
    R_off = g["mesh"].residual(U0).cpu().numpy()
    Rl = o.residual(np.zeros(fp.n_dof), terms=ora_mod.LATERAL)[0]
    Rb, Mb, _ = o.residual(np.zeros(fp.n_dof), terms=ora_mod.BODY | ora_mod.LATERAL)
    assert np.abs(Rl).max() > 0.0
    assert np.abs((R_on - R_off) - Rl).max() <= R_TOL * np.abs(Mb).max()


@pytest.mark.parametrize("case", ["C1", "gris-40km", "slab-distorted", "C5-small", "C2"])
def test_parity_tetrahedra(torch_cuda, ora_mod, case):
    """NEXT-f4: three P1 tetrahedra per prism (reading L22)."""
    fp = {"C1": mg.ismip_hom_a,
          "gris-40km": lambda: mg.greenland_like(40.0),
          "slab-distorted": lambda: mg.slab(nx=7, n_layers=4, distort=0.25),
          "C5-small": lambda: mg.antarctica_like(D_km=150.0, n_layers=3),
          "C2": lambda: mg.greenland_like(16.0)}[case]()
    if case == "C5-small":
        fp = mg.sub_footprint(fp, 0, min(fp.n_tri, 6000))
    fp.elem_type = 1
    g = gpu_assemble(torch_cuda, fp)
    check_parity(ora_mod.Oracle(fp), g, fp=fp)


@pytest.mark.parametrize("scatter", [0, 1])
@pytest.mark.parametrize("case", ["C1-quads", "slab-quads-distorted", "quads-temperature", "quads-40x40",
                                  "quads-33x33-distorted", "quads-1-layer"])
def test_parity_hexahedra(torch_cuda, ora_mod, case, scatter):
    """NEXT-f4: quadrilateral footprint, 8-node trilinear hexahedra (P:478,
    reading L23): the quad-patch owner-computes kernel (scatter 0; the 40 x 40
    and 33 x 33 footprints span 17 / 12 patches, so boundary, multi and pad
    handling are exercised; one layer: levels 0 and L only) and the coloured
    read-modify-write ablation (1)."""
    if case == "C1-quads":
        fp = mg.to_quads(mg.ismip_hom_a(nx=10, n_layers=5), 10)
    elif case == "slab-quads-distorted":
        fp = mg.to_quads(mg.slab(nx=7, n_layers=4, distort=0.2), 7)
    elif case == "quads-40x40":
        fp = mg.to_quads(mg.ismip_hom_a(nx=40, n_layers=3), 40)
    elif case == "quads-33x33-distorted":
        fp = mg.to_quads(mg.slab(nx=33, n_layers=2, distort=0.2), 33)
    elif case == "quads-1-layer":   # L = 1: the basal and surface levels only, 7 patches
        fp = mg.to_quads(mg.ismip_hom_a(nx=26, n_layers=1), 26)
    else:
        fp = mg.with_temperature(mg.to_quads(mg.ismip_hom_a(nx=6, n_layers=3), 6))
    g = gpu_assemble(torch_cuda, fp, scatter=scatter)
    check_parity(ora_mod.Oracle(fp), g, fp=fp)
    import torch
    R2, V2 = g["mesh"].jacobian(torch.tensor(fp.U, device="cuda"))
    torch.cuda.synchronize()
    assert np.array_equal(R2.cpu().numpy(), g["RJ"]) and np.array_equal(V2.cpu().numpy(), g["vals"])


def test_tetrahedra_partitioned_and_rejections(torch_cuda, ora_mod):
    """f4 on a 2-part partition (owned rows after the halo plan's sums equal
    the single-domain tet assembly); unsupported combinations are rejected."""
    import torch
    from paper_2204_04321_b200 import fo
    fp = mg.greenland_like(40.0, n_layers=4)
    fp.elem_type = 1
    L, P = fp.n_layers, 2
    full = fo.Mesh.from_footprint(fp)
    full.set_element(1)
    Rf, Vf = full.jacobian(torch.tensor(fp.U, device="cuda"))
    Rf = Rf.cpu().numpy()
    part = fo.partition(fp.n_tri, P)
    outs, meshes = [], []
    for p in range(P):
        m = fo.Mesh.from_footprint(fp, part=part, my_part=p, n_parts=P)
        m.set_element(1)
        glob, nA, nB, nC = m.columns()
        Ul = fp.U.reshape(fp.n_vert, L + 1, 2)[glob].reshape(-1)
        outs.append(list(m.jacobian(torch.tensor(Ul, device="cuda"))))
        meshes.append((m, glob))
    plans = [fo.halo_plan_host(fp.n_vert, fp.tri, L, part, P, p) for p in range(P)]
    for p in range(P):
        for q, (sr, dr, sv, dv) in plans[p].items():
            outs[q][0].index_add_(0, torch.tensor(dr, device="cuda"), outs[p][0][torch.tensor(sr, device="cuda")])
    torch.cuda.synchronize()
    for p in range(P):
        m, glob = meshes[p]
        L1 = L + 1
        gd = np.stack([2 * (glob[:, None] * L1 + np.arange(L1)), 2 * (glob[:, None] * L1 + np.arange(L1)) + 1],
                      axis=2).reshape(-1)
        R = outs[p][0].cpu().numpy()
        n = m.n_owned_dofs
        assert np.abs(R[:n] - Rf[gd[:n]]).max() <= 1e-12 * np.abs(Rf).max()
    with pytest.raises(fo.FoError):
        full.set_lateral(True)
    with pytest.raises(fo.FoError):
        full.set_scatter(1)
    # back to wedges: the caller's corner order and plan are restored (bitwise)
    full.set_element(0)
    fresh = fo.Mesh.from_footprint(fp)
    Uw = torch.tensor(fp.U, device="cuda")
    Rw, Vw = full.jacobian(Uw)
    Rw2, Vw2 = fresh.jacobian(Uw)
    torch.cuda.synchronize()
    assert torch.equal(Rw, Rw2) and torch.equal(Vw, Vw2)


@pytest.mark.parametrize("L", [1, 2, 17])
def test_parity_layer_counts(torch_cuda, ora_mod, L):
    fp = mg.ismip_hom_a(nx=6, n_layers=L)
    g = gpu_assemble(torch_cuda, fp)
    check_parity(ora_mod.Oracle(fp), g, fp=fp)


def test_single_triangle(torch_cuda, ora_mod):
    fp = mg.slab(nx=1, n_layers=3, distort=0.0)
    fp = mg.sub_footprint(fp, 1, 2)
    g = gpu_assemble(torch_cuda, fp)
    check_parity(ora_mod.Oracle(fp), g, fp=fp)


@pytest.mark.parametrize("spokes", [80, 200])
def test_high_degree_vertex(torch_cuda, ora_mod, spokes):
    """A wheel: one column coupled to `spokes` neighbours (row nnz 6 (spokes+1),
    one or two patches around it), the maximum-degree case of the plan."""
    rng = mg.SplitMix64(21)
    th = 2 * np.pi * np.arange(spokes) / spokes
    xy = np.vstack([[0.0, 0.0], np.stack([2e4 * np.cos(th), 2e4 * np.sin(th)], axis=1)])
    tri = np.array([[0, 1 + i, 1 + (i + 1) % spokes] for i in range(spokes)], dtype=np.int32)
    nv, L = xy.shape[0], 4
    H = 900.0 + 200.0 * rng.uniform(nv)
    s_ = 1200.0 + 1e-2 * xy[:, 0]
    beta = 100.0 + 900.0 * rng.uniform(nv)
    U = 20.0 * rng.normal(2 * nv * (L + 1)) + 40.0
    fp = mg.Footprint("wheel", xy, tri, np.linspace(0.0, 1.0, L + 1), H, s_, None, beta, U,
                      dict(mg.DEFAULT_PARAMS))
    g = gpu_assemble(torch_cuda, fp)
    check_parity(ora_mod.Oracle(fp), g, fp=fp)


def test_empty_mesh(torch_cuda):
    from paper_2204_04321_b200 import fo
    fp = mg.ismip_hom_a(nx=2, n_layers=2)
    fp.xy = np.zeros((0, 2)); fp.tri = np.zeros((0, 3), np.int32)
    for a in ("thickness", "surface", "beta"):
        setattr(fp, a, np.zeros(0))
    fp.U = np.zeros(0)
    mesh = fo.Mesh.from_footprint(fp)
    assert mesh.n_dofs == 0 and mesh.n_elems == 0
    assert mesh.graph().nnz == 0


def test_symmetry_and_overwrite(torch_cuda):
    """J symmetric to roundoff; outputs are overwritten, not accumulated."""
    import torch
    from paper_2204_04321_b200 import fo
    fp = mg.greenland_like(50.0, n_layers=5)
    mesh = fo.Mesh.from_footprint(fp)
    U = torch.tensor(fp.U, device="cuda")
    g = mesh.graph()
    R = torch.full((mesh.n_dofs,), 7.0, dtype=torch.float64, device="cuda")
    vals = torch.full((g.nnz,), -3.0, dtype=torch.float64, device="cuda")
    mesh.jacobian(U, R=R, vals=vals)
    R2, vals2 = mesh.jacobian(U)
    torch.cuda.synchronize()
    Rh, Rh2 = R.cpu().numpy(), R2.cpu().numpy()
    sc = np.abs(Rh).max()
    assert np.abs(Rh - Rh2).max() <= 1e-13 * sc
    assert np.abs(vals.cpu().numpy() - vals2.cpu().numpy()).max() <= 1e-13 * np.abs(vals2.cpu().numpy()).max()
    rp, col = g.to_host()
    import scipy.sparse as sp
    J = sp.csr_matrix((vals2.cpu().numpy(), col, rp), shape=(mesh.n_dofs, mesh.n_dofs))
    assert abs(J - J.T).max() <= 1e-14 * abs(J).max()


def test_host_buffer_entry_point(torch_cuda):
    import torch
    from paper_2204_04321_b200 import fo
    fp = mg.greenland_like(50.0, n_layers=5)
    mesh = fo.Mesh.from_footprint(fp)
    g = mesh.graph()
    Uh = torch.tensor(fp.U).pin_memory()
    Rh = torch.zeros(mesh.n_dofs, dtype=torch.float64).pin_memory()
    Vh = torch.zeros(g.nnz, dtype=torch.float64).pin_memory()
    mesh.jacobian_host(Uh, Rh, Vh, g)
    Rd, Vd = mesh.jacobian(torch.tensor(fp.U, device="cuda"))
    torch.cuda.synchronize()
    assert np.abs(Rh.numpy() - Rd.cpu().numpy()).max() <= 1e-13 * np.abs(Rh.numpy()).max()
    assert np.abs(Vh.numpy() - Vd.cpu().numpy()).max() <= 1e-13 * np.abs(Vh.numpy()).max()


@pytest.mark.parametrize("cfg", ["C3", "C5", "C3-tet"])
def test_c3_full_size_sampled(torch_cuda, ora_mod, cfg):
    """C3 (and C5, with its floating shelves) at full size in the bench's launch
    configuration: complete rows of sampled columns vs the oracle on the
    sub-footprint of their triangle fans (R + J kernel and residual-only kernel)."""
    import torch
    from paper_2204_04321_b200 import fo
    fp = mg.antarctica_like() if cfg == "C5" else mg.greenland_like_1_10()
    if cfg == "C3-tet":   # NEXT-f4 at full size: three tetrahedra per prism
        fp.elem_type = 1
    mesh = fo.Mesh.from_footprint(fp)
    if cfg == "C3-tet":
        mesh.set_element(1)
    U = torch.tensor(fp.U, device="cuda")
    g = mesh.graph()
    R, vals = mesh.jacobian(U)
    Rr = mesh.residual(U)   # the residual-only kernel (KR, compact shared layout)
    torch.cuda.synchronize()
    R = R.cpu().numpy()
    Rr = Rr.cpu().numpy()
    rp = np.empty(g.n_rows + 1, np.int64)
    rp, _ = g.to_host()
    vals = vals.cpu().numpy()
    rng = mg.SplitMix64(77)
    cols = np.unique((rng.uniform(48) * fp.n_vert).astype(np.int64))
    _check_full_size_columns(ora_mod, fp, cols, rp, vals, (R, Rr))


def _check_full_size_columns(ora_mod, fp, cols, rp, vals, Rs):
    """complete rows of the columns `cols` of a full-size assembly against the
    oracle on the sub-footprint of their triangle fans"""
    fan = np.nonzero(np.isin(fp.tri, cols).any(axis=1))[0]
    sub = mg.sub_footprint_tris(fp, fan)
    o = ora_mod.Oracle(sub)
    Ro, Mo, _ = o.residual(sub.U)
    orp, _ = o.graph()
    _, ov = o.jacobian(sub.U)
    L1 = fp.n_layers + 1
    loc = {int(v): i for i, v in enumerate(sub.vertex_ids)}
    for c in cols:
        lc = loc[int(c)]
        for k in range(L1):
            for a in range(2):
                r_g = 2 * (c * L1 + k) + a
                r_o = 2 * (lc * L1 + k) + a
                for Rx in Rs:
                    assert abs(Rx[r_g] - Ro[r_o]) <= R_TOL * np.abs(Mo).max()
                seg_g = vals[rp[r_g]:rp[r_g + 1]]
                seg_o = ov[orp[r_o]:orp[r_o + 1]]
                assert seg_g.size == seg_o.size
                assert np.abs(seg_g - seg_o).max() <= J_TOL * np.abs(seg_o).max()


def _patch_classes(fp, patch_tris=128):
    """per column: the number of patches of the owner-computes plan whose
    triangles touch it (1 interior, 2 boundary, >= 3 multi), from the plan's
    equal-size ranges of <= patch_tris consecutive triangles (fo_plan.cpp)"""
    nt = fp.n_tri
    np0 = (nt + patch_tris - 1) // patch_tris
    bounds = (np.arange(np0 + 1, dtype=np.int64) * nt) // np0
    patch = np.searchsorted(bounds, np.arange(nt), side="right") - 1
    pairs = np.unique(np.stack([fp.tri.reshape(-1).astype(np.int64), np.repeat(patch, 3)], axis=1), axis=0)
    return np.bincount(pairs[:, 0], minlength=fp.n_vert)


@pytest.mark.parametrize("cfg", ["C3", "C5"])
def test_full_size_targeted_columns(torch_cuda, ora_mod, cfg):
    """at full size in the bench's launch configuration,
    deliberately sample the scatter's hard cases -- columns touched by >= 3
    patches (the multi fix-up path), patch-boundary columns (zero fill + RED),
    the highest-degree column and its neighbours, and interior columns -- with
    complete rows (R + J kernel and residual-only kernel) against the oracle."""
    import torch
    from paper_2204_04321_b200 import fo
    fp = mg.antarctica_like() if cfg == "C5" else mg.greenland_like_1_10()
    mesh = fo.Mesh.from_footprint(fp)
    U = torch.tensor(fp.U, device="cuda")
    g = mesh.graph()
    R, vals = mesh.jacobian(U)
    Rr = mesh.residual(U)
    torch.cuda.synchronize()
    rp, _ = g.to_host()
    npatch = _patch_classes(fp)
    deg = np.bincount(fp.tri.reshape(-1), minlength=fp.n_vert)
    rng = mg.SplitMix64(91)
    pick = lambda ids, n: ids[(rng.uniform(n) * ids.size).astype(np.int64)] if ids.size else ids
    top = int(np.argmax(deg))
    nbr = np.unique(fp.tri[(fp.tri == top).any(axis=1)])
    multi, bnd, inner = (np.nonzero(npatch >= 3)[0], np.nonzero(npatch == 2)[0], np.nonzero(npatch == 1)[0])
    assert multi.size and bnd.size and inner.size
    cols = np.unique(np.concatenate([pick(multi, 12), pick(bnd, 12), pick(inner, 6), nbr]))
    _check_full_size_columns(ora_mod, fp, cols, rp, vals.cpu().numpy(), (R.cpu().numpy(), Rr.cpu().numpy()))


@pytest.mark.parametrize("lateral", [False, True])
@pytest.mark.parametrize("P", [2, 3])
def test_partitioned_assembly_with_halo_plan(torch_cuda, ora_mod, P, lateral):
    """local meshes of a P-way footprint partition (fo_mesh_create_part) on one
    GPU, ghost-row partial sums added into the owners with the library's host
    halo plan (fo_halo_plan_host) applied here by index_add_: owned rows equal
    the single-domain assembly, with and without the lateral term.  Ghost U is
    copied from the global array here; the library's own fo_halo_import /
    fo_halo_sum are tested in tests/test_gpu_halo.py."""
    import torch
    from paper_2204_04321_b200 import fo
    fp = mg.greenland_like(40.0, n_layers=5)
    L = fp.n_layers
    part = fo.partition(fp.n_tri, P)
    full = fo.Mesh.from_footprint(fp)
    full.set_lateral(lateral)
    Rf, Vf = full.jacobian(torch.tensor(fp.U, device="cuda"))
    grp, gcol = full.graph().to_host()
    Rf, Vf = Rf.cpu().numpy(), Vf.cpu().numpy()
    meshes, outs = [], []
    for p in range(P):
        m = fo.Mesh.from_footprint(fp, part=part, my_part=p, n_parts=P)
        m.set_lateral(lateral)
        glob, nA, nB, nC = m.columns()
        Ul = fp.U.reshape(fp.n_vert, L + 1, 2)[glob].reshape(-1)
        R, V = m.jacobian(torch.tensor(Ul, device="cuda"))
        meshes.append((m, glob, nA))
        outs.append([R, V])
    torch.cuda.synchronize()
    plans = [fo.halo_plan_host(fp.n_vert, fp.tri, L, part, P, p) for p in range(P)]
    for p in range(P):
        for q, (sr, dr, sv, dv) in plans[p].items():
            Rq, Vq = outs[q]
            Rq.index_add_(0, torch.tensor(dr, device="cuda"), outs[p][0][torch.tensor(sr, device="cuda")])
            Vq.index_add_(0, torch.tensor(dv, device="cuda"), outs[p][1][torch.tensor(sv, device="cuda")])
    torch.cuda.synchronize()
    for p in range(P):
        m, glob, nA = meshes[p]
        rp, col = m.graph().to_host()
        L1 = L + 1
        g = (np.stack([2 * (glob[:, None] * L1 + np.arange(L1)), 2 * (glob[:, None] * L1 + np.arange(L1)) + 1],
                      axis=2)).reshape(-1)
        R = outs[p][0].cpu().numpy()
        V = outs[p][1].cpu().numpy()
        n_owned = m.n_owned_dofs
        assert np.abs(R[:n_owned] - Rf[g[:n_owned]]).max() <= 1e-12 * np.abs(Rf).max()
        for r in range(0, n_owned, 3):
            gr = g[r]
            seg = Vf[grp[gr]:grp[gr + 1]]
            loc = V[rp[r]:rp[r + 1]]
            order = np.argsort(g[col[rp[r]:rp[r + 1]]])
            assert np.abs(loc[order] - seg).max() <= 1e-11 * np.abs(seg).max()


def test_c3_bitwise_reproducible_and_overwritten(torch_cuda):
    """the owner-computes scatter is bitwise run-to-run
    stable (interior stores; at most two RED partial sums per boundary entry;
    sums of three or more patches added in patch order), and every output
    entry is overwritten (NaN-filled buffers come back NaN-free)."""
    import torch
    from paper_2204_04321_b200 import fo
    fp = mg.greenland_like_1_10()
    mesh = fo.Mesh.from_footprint(fp)
    U = torch.tensor(fp.U, device="cuda")
    g = mesh.graph()
    outs = []
    for rep in range(3):
        R = torch.full((mesh.n_dofs,), float("nan"), dtype=torch.float64, device="cuda")
        vals = torch.full((g.nnz,), float("nan"), dtype=torch.float64, device="cuda")
        mesh.jacobian(U, R=R, vals=vals)
        assert 1 <= mesh.last_launch_count() <= 3
        Rr = torch.full((mesh.n_dofs,), float("nan"), dtype=torch.float64, device="cuda")
        mesh.residual(U, R=Rr)
        torch.cuda.synchronize()
        assert not torch.isnan(R).any() and not torch.isnan(vals).any() and not torch.isnan(Rr).any()
        outs.append((R.cpu().numpy().tobytes(), vals.cpu().numpy().tobytes(), Rr.cpu().numpy().tobytes()))
    assert outs[0] == outs[1] == outs[2]


def test_assembly_captures_into_a_cuda_graph(torch_cuda):
    """No host synchronisation inside fo_assemble_jacobian: the whole call
    (zero-fill, patch kernel, fix-up) captures into a CUDA graph whose replay
    equals the eager assembly bit for bit, also after U changes in place."""
    import torch
    from paper_2204_04321_b200 import fo
    fp = mg.greenland_like(30.0, n_layers=6)
    mesh = fo.Mesh.from_footprint(fp)
    g = mesh.graph()
    U = torch.tensor(fp.U, device="cuda")
    R, V = mesh.jacobian(U)                       # eager (also first-call setup)
    Rg = torch.empty_like(R)
    Vg = torch.empty_like(V)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        mesh.jacobian(U, R=Rg, vals=Vg)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        mesh.jacobian(U, R=Rg, vals=Vg)
    Rg.fill_(float("nan"))
    Vg.fill_(float("nan"))
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(Rg, R) and torch.equal(Vg, V)
    U.mul_(1.5)
    R2, V2 = mesh.jacobian(U)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(Rg, R2) and torch.equal(Vg, V2)
    assert not torch.equal(R2, R)


def test_hexahedra_full_size_sampled(torch_cuda, ora_mod):
    """NEXT-f4 at the timed size: 700 x 700 quads x 10 layers (4.9 M
    hexahedra, ~5 100 quad patches) through the quad-patch kernel; complete rows
    of 40 random columns (about 40 % of all columns are patch-boundary columns)
    and of the domain's corner / edge columns vs the oracle on the
    sub-footprint of their quad fans."""
    import torch
    from paper_2204_04321_b200 import fo
    nx = 700
    fp = mg.to_quads(mg.ismip_hom_a(nx=nx, n_layers=10), nx)
    mesh = fo.Mesh.from_footprint(fp)
    U = torch.tensor(fp.U, device="cuda")
    g = mesh.graph()
    R, vals = mesh.jacobian(U)
    torch.cuda.synchronize()
    rp, _ = g.to_host()
    rng = mg.SplitMix64(123)
    n1 = nx + 1
    special = np.array([0, nx, nx * n1, n1 * n1 - 1, n1 // 2, (nx // 2) * n1 + nx // 2])
    cols = np.unique(np.concatenate([(rng.uniform(40) * fp.n_vert).astype(np.int64), special]))
    _check_full_size_columns(ora_mod, fp, cols, rp, vals.cpu().numpy(), (R.cpu().numpy(),))


def test_c3_repeated_assemblies_bitwise_on_device(torch_cuda):
    """Stress of the in-kernel zero fill (atomic patch tickets, lead flags,
    waits) and of the boundary REDs: 50 back-to-back C3 R + J assemblies into
    the same buffers, each compared bit for bit with the first on the device;
    the values are poisoned with NaN between calls, so a slot the zero fill or
    the stores missed would show."""
    import torch
    from paper_2204_04321_b200 import fo
    fp = mg.greenland_like_1_10()
    mesh = fo.Mesh.from_footprint(fp)
    g = mesh.graph()
    U = torch.tensor(fp.U, device="cuda")
    R = torch.empty(mesh.n_dofs, dtype=torch.float64, device="cuda")
    V = torch.empty(g.nnz, dtype=torch.float64, device="cuda")
    mesh.jacobian(U, g, R, V)
    R0, V0 = R.clone(), V.clone()
    assert not torch.isnan(V0).any() and not torch.isnan(R0).any()
    bad = 0
    for _ in range(50):
        R.fill_(float("nan"))
        V.fill_(float("nan"))
        mesh.jacobian(U, g, R, V)
        bad += int(not torch.equal(V, V0)) + int(not torch.equal(R, R0))
    torch.cuda.synchronize()
    assert bad == 0


def test_hexahedra_repeated_assemblies_bitwise_on_device(torch_cuda):
    """Stress of the quad-patch kernel's in-kernel zero fill (the fourth warp
    of each CTA: atomic patch tickets, lead flags, waits) and of its boundary
    REDs: 30 back-to-back R + J assemblies of 250 x 250 quads x 6 layers (~650
    patches, several waves of two CTAs per SM) into NaN-poisoned buffers, each
    equal bit for bit to the first, which is NaN-free; the residual-only path
    (zero kernel) likewise."""
    import torch
    from paper_2204_04321_b200 import fo
    fp = mg.to_quads(mg.ismip_hom_a(nx=250, n_layers=6), 250)
    mesh = fo.Mesh.from_footprint(fp)
    g = mesh.graph()
    U = torch.tensor(fp.U, device="cuda")
    R = torch.full((mesh.n_dofs,), float("nan"), dtype=torch.float64, device="cuda")
    V = torch.full((g.nnz,), float("nan"), dtype=torch.float64, device="cuda")
    mesh.jacobian(U, g, R, V)
    R0, V0 = R.clone(), V.clone()
    assert not torch.isnan(V0).any() and not torch.isnan(R0).any()
    Rr = torch.full((mesh.n_dofs,), float("nan"), dtype=torch.float64, device="cuda")
    mesh.residual(U, Rr)
    assert not torch.isnan(Rr).any()
    assert torch.allclose(Rr, R0, rtol=0.0, atol=1e-12 * float(R0.abs().max()))
    bad = 0
    for _ in range(30):
        R.fill_(float("nan"))
        V.fill_(float("nan"))
        mesh.jacobian(U, g, R, V)
        bad += int(not torch.equal(V, V0)) + int(not torch.equal(R, R0))
    torch.cuda.synchronize()
    assert bad == 0
