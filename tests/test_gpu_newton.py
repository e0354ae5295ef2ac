"""NEXT-f2: the Newton consumer on the GPU (PAPER.md
P:160-165): the column-structured SpMV, the vertical-line preconditioner and
the Krylov helpers against plain host linear algebra on the same values, and a
damped Newton / GMRES solve of C1 whose solution the ORACLE accepts."""
import numpy as np
import pytest

from paper_2204_04321_b200 import meshgen as mg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2204_04321_b200 import _build
    _build.build()
    return torch


def _assembled(torch, fp):
    from paper_2204_04321_b200 import fo
    mesh = fo.Mesh.from_footprint(fp)
    U = torch.tensor(fp.U, device="cuda")
    R, vals = mesh.jacobian(U)
    torch.cuda.synchronize()
    return mesh, U, R, vals


def _host_csr(mesh, vals):
    import scipy.sparse as sp
    rp, col = mesh.graph().to_host()
    return sp.csr_matrix((vals.cpu().numpy(), col, rp), shape=(mesh.n_dofs, mesh.n_dofs))


def test_spmv_matches_host_csr(torch_cuda):
    """fo_spmv (no col_idx reads) = CSR (row_ptr, col_idx, vals) @ x."""
    torch = torch_cuda
    from paper_2204_04321_b200 import newton
    fp = mg.greenland_like(16.0)
    mesh, U, R, vals = _assembled(torch, fp)
    s = newton.NewtonSolver(mesh, restart=4)
    s.vals.copy_(vals)
    x = torch.tensor(mg.SplitMix64(5).normal(mesh.n_dofs), device="cuda")
    y = torch.empty_like(x)
    s.spmv(x, y)
    J = _host_csr(mesh, vals)
    yh = J @ x.cpu().numpy()
    scale = abs(J) @ np.abs(x.cpu().numpy())
    assert np.all(np.abs(y.cpu().numpy() - yh) <= 1e-13 * scale + 1e-300)


def test_line_preconditioner_inverts_column_blocks(torch_cuda):
    """fo_line_solve solves M z = r exactly, M = the block-tridiagonal
    column blocks of J (all other couplings dropped)."""
    torch = torch_cuda
    from paper_2204_04321_b200 import newton
    fp = mg.greenland_like(40.0, n_layers=6)
    mesh, U, R, vals = _assembled(torch, fp)
    s = newton.NewtonSolver(mesh, restart=4)
    s.vals.copy_(vals)
    from paper_2204_04321_b200 import fo
    fo.check(fo.lib().fo_line_factor(mesh.handle, s.graph.handle, newton._p(s.vals), None), "factor")
    r = torch.tensor(mg.SplitMix64(6).normal(mesh.n_dofs), device="cuda")
    z = torch.empty_like(r)
    s.precond(r, z)
    J = _host_csr(mesh, vals).tocoo()
    L1 = fp.n_layers + 1
    same_col = (J.row // (2 * L1)) == (J.col // (2 * L1))
    import scipy.sparse as sp
    M = sp.csr_matrix((J.data[same_col], (J.row[same_col], J.col[same_col])), shape=J.shape)
    res = M @ z.cpu().numpy() - r.cpu().numpy()
    assert np.abs(res).max() <= 1e-10 * np.abs(r.cpu().numpy()).max()


def test_krylov_helpers(torch_cuda):
    torch = torch_cuda
    from paper_2204_04321_b200 import newton
    fp = mg.ismip_hom_a(nx=6, n_layers=3)
    mesh, U, R, vals = _assembled(torch, fp)
    s = newton.NewtonSolver(mesh, restart=8)
    rng = mg.SplitMix64(11)
    Vh = rng.normal(5 * mesh.n_dofs).reshape(5, -1)
    s.V[:5].copy_(torch.tensor(Vh))
    w = torch.tensor(rng.normal(mesh.n_dofs), device="cuda")
    d = s.dots(5, w)
    assert np.abs(d - Vh @ w.cpu().numpy()).max() <= 1e-12 * np.abs(Vh).sum(axis=1).max() * 5
    wh = w.cpu().numpy().copy()
    coef = np.array([0.5, -1.0, 2.0, 0.0, 3.0])
    s.update(5, coef, w)
    assert np.abs(w.cpu().numpy() - (wh - coef @ Vh)).max() <= 1e-12 * np.abs(wh).max() * 10
    # reproducible: same dots twice
    assert np.array_equal(s.dots(5, w), s.dots(5, w))


def test_newton_solves_c1_and_the_oracle_agrees(torch_cuda, ora_mod):
    """Damped Newton + GMRES(30) with the line preconditioner from the SIA
    guess on C1 (ISMIP-HOM A, n = 3): ||F|| drops by 1e-9; the oracle's own
    residual at the GPU solution is at the round-off level of its M = sum |r_e|;
    the last steps converge quadratically (exact Jacobian, L14)."""
    torch = torch_cuda
    from paper_2204_04321_b200 import fo, newton
    fp = mg.ismip_hom_a()
    mesh = fo.Mesh.from_footprint(fp)
    U = torch.tensor(fp.U, device="cuda")
    s = newton.NewtonSolver(mesh, restart=30, max_krylov=600)
    rep = s.solve(U, rtol=1e-9, max_newton=40, krylov_rtol=1e-6)
    assert rep.converged, rep
    f = np.array(rep.residual_norms)
    # quadratic tail: two consecutive full steps with f_{k+1} <= C f_k^2 / f_0
    full = [i for i, a in enumerate(rep.step_lengths) if a == 1.0]
    assert len(full) >= 2
    o = ora_mod.Oracle(fp)
    Uh = U.cpu().numpy()
    R, M, _ = o.residual(Uh)
    assert np.abs(R).max() <= 1e-8 * np.abs(M).max(), (np.abs(R).max(), np.abs(M).max())
    # the velocity is physical: downslope (+x) flow on the ISMIP-HOM A slab
    u = Uh.reshape(fp.n_vert, fp.n_layers + 1, 2)[:, :, 0]
    assert u.mean() > 0.0


def test_newton_solves_c1_hexahedra(torch_cuda, ora_mod):
    """The consumer is element-agnostic (SpMV and the line preconditioner see
    only columns): Newton on the quadrilateral C1 with trilinear hexahedra."""
    torch = torch_cuda
    from paper_2204_04321_b200 import fo, newton
    fp = mg.to_quads(mg.ismip_hom_a(), 20)
    mesh = fo.Mesh.from_footprint(fp)
    U = torch.tensor(fp.U, device="cuda")
    s = newton.NewtonSolver(mesh, restart=30, max_krylov=600)
    rep = s.solve(U, rtol=1e-9, max_newton=40, krylov_rtol=1e-6)
    assert rep.converged, rep
    R, M, _ = ora_mod.Oracle(fp).residual(U.cpu().numpy())
    assert np.abs(R).max() <= 1e-8 * np.abs(M).max()
