"""GPU tests of the halo data path (a1 import, a9 ghost-row sum; P:175, P:185,
P:250-255) through libfo's own fo_halo_import / fo_halo_sum.

On one GPU the P part meshes of a footprint partition live in one process and
use the loopback transport (fo_halo_create_loopback): the same plans, staging
buffers, gather / unpack-add kernels and sender order as the NCCL halos, with
device copies in place of ncclSend / ncclRecv.  The NCCL transport itself runs
in test_nccl_halo_two_ranks (torchrun, two GPUs; skipped on a one-GPU box).

Checked after import -> fo_assemble_jacobian -> fo_halo_sum on every part:
  * imported ghost U is bit-identical to the global U (ghost slices start NaN;
    column-only (class C) U stays NaN and nothing reads it);
  * owned rows equal the single-domain GPU assembly (R <= 1e-12 max|R|,
    J <= 1e-11 row-scaled) and, on sampled columns (random, next to ghosts,
    next to column-only couplings), the oracle;
  * ghost (class B) rows hold exactly the part's own partial sums (oracle on
    the part's triangles of the fan).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2204_04321_b200 import meshgen as mg

pytestmark = pytest.mark.gpu

R_TOL, J_TOL = 1e-12, 1e-11
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2204_04321_b200 import _build
    _build.build()
    return torch


def _global_dofs(glob, L1):
    n = glob[:, None] * L1 + np.arange(L1)
    return np.stack([2 * n, 2 * n + 1], axis=2).reshape(-1)


def _oracle_rows(ora_mod, fp, tri_ids, col):
    """oracle R, M and CSR rows of global column `col` on the sub-footprint of
    tri_ids (all of col's fan: its complete rows; a part's share: partial rows)"""
    sub = mg.sub_footprint_tris(fp, tri_ids)
    o = ora_mod.Oracle(sub)
    R, M, _ = o.residual(sub.U)
    rp, _ = o.graph()
    _, v = o.jacobian(sub.U)
    lc = int(np.nonzero(sub.vertex_ids == col)[0][0])
    return R, M, rp, v, lc


def _run_loopback(torch, fp, P, poison=True):
    from paper_2204_04321_b200 import fo
    L1 = fp.n_layers + 1
    part = fo.partition(fp.n_tri, P)
    meshes = [fo.Mesh.from_footprint(fp, part=part, my_part=p, n_parts=P) for p in range(P)]
    halos = fo.Halo.loopback(meshes)
    Ug = fp.U.reshape(fp.n_vert, L1, 2)
    st = []
    for p, m in enumerate(meshes):
        glob, nA, nB, nC = m.columns()
        Ul = Ug[glob].reshape(-1).copy()
        if poison:
            Ul[2 * nA * L1:] = np.nan        # ghost (B) and column-only (C) U unknown
        st.append(dict(m=m, glob=glob, nA=nA, nB=nB, nC=nC, U=torch.tensor(Ul, device="cuda")))
    for p in range(P):                       # a1: import, every part
        halos[p].import_(st[p]["U"])
    for p in range(P):
        st[p]["R"], st[p]["V"] = st[p]["m"].jacobian(st[p]["U"])
    for p in range(P):                       # a9: ghost-row sum, every part
        halos[p].sum(st[p]["R"], st[p]["V"])
    torch.cuda.synchronize()
    for p in range(P):
        s = st[p]
        s["U"], s["R"], s["V"] = s["U"].cpu().numpy(), s["R"].cpu().numpy(), s["V"].cpu().numpy()
        s["rp"], s["col"] = s["m"].graph().to_host()
    return part, st, halos


def _check_import(fp, st):
    L1 = fp.n_layers + 1
    Ug = fp.U.reshape(fp.n_vert, L1, 2)
    for s in st:
        nA, nB = s["nA"], s["nB"]
        ghost = s["U"][2 * nA * L1:2 * (nA + nB) * L1]
        want = Ug[s["glob"][nA:nA + nB]].reshape(-1)
        assert ghost.tobytes() == want.tobytes()                      # bit-identical
        assert np.array_equal(s["U"][:2 * nA * L1], Ug[s["glob"][:nA]].reshape(-1))
        assert np.isnan(s["U"][2 * (nA + nB) * L1:]).all()            # class C never imported
        assert not np.isnan(s["R"]).any() and not np.isnan(s["V"]).any()


def _check_owned_vs_full(torch, fp, st):
    """every owned row of every part against the single-domain assembly: the
    part's entries sorted by (global row, global column) must hit the global
    CSR's positions one for one (same pattern) with row-scaled parity"""
    from paper_2204_04321_b200 import fo
    full = fo.Mesh.from_footprint(fp)
    Rf, Vf = full.jacobian(torch.tensor(fp.U, device="cuda"))
    grp, gcol_full = full.graph().to_host()
    dev = "cuda"
    grp_t = torch.tensor(grp, device=dev)
    gcol_full_t = torch.tensor(gcol_full.astype(np.int64), device=dev)
    absV = Vf.abs()
    rowmax = torch.zeros(grp.size - 1, dtype=torch.float64, device=dev)
    rows_full = torch.repeat_interleave(torch.arange(grp.size - 1, device=dev), grp_t[1:] - grp_t[:-1])
    rowmax.scatter_reduce_(0, rows_full, absV, reduce="amax")
    Rf = Rf.cpu().numpy()
    L1 = fp.n_layers + 1
    rmax = np.abs(Rf).max()
    n_glob = 2 * fp.n_vert * L1
    for s in st:
        g = _global_dofs(s["glob"], L1)
        no = 2 * s["nA"] * L1
        assert np.abs(s["R"][:no] - Rf[g[:no]]).max(initial=0.0) <= R_TOL * rmax
        rp, col = s["rp"], s["col"]
        ne = int(rp[no])
        g_t = torch.tensor(g, device=dev)
        rows = torch.repeat_interleave(torch.arange(no, device=dev), torch.tensor(np.diff(rp[:no + 1]), device=dev))
        gr = g_t[rows]
        gc = g_t[torch.tensor(col[:ne].astype(np.int64), device=dev)]
        key, order = torch.sort(gr * n_glob + gc)
        gr_s = key // n_glob
        first = torch.searchsorted(key, gr_s * n_glob)          # first entry of each row
        pos = grp_t[gr_s] + (torch.arange(ne, device=dev) - first)
        assert torch.equal(gcol_full_t[pos], key % n_glob)         # identical global pattern
        assert torch.equal(grp_t[gr_s + 1] - grp_t[gr_s],
                           torch.tensor(np.diff(rp[:no + 1]), device=dev)[rows[order]])
        got = torch.tensor(s["V"][:ne], device=dev)[order]
        err = (got - Vf[pos]).abs()
        assert bool((err <= J_TOL * rowmax[gr_s]).all())


def _sample_columns(s, L1, rng, n_rand=6):
    """owned columns: random, next to a ghost (B), next to a column-only (C)
    coupling; and ghost (B) columns"""
    nA, nB = s["nA"], s["nB"]
    rp, col = s["rp"], s["col"]
    near_b, near_c = [], []
    for c in range(nA):
        r = 2 * c * L1 + 2   # level-1 u row: couples every neighbour column
        nb = np.unique(col[rp[r]:rp[r + 1]] // (2 * L1))
        if (nb >= nA + nB).any():
            near_c.append(c)
        elif (nb >= nA).any():
            near_b.append(c)
    pick = lambda lst, n: [lst[int(i)] for i in (rng.uniform(n) * len(lst)).astype(int)] if lst else []
    owned = sorted(set(pick(list(range(nA)), n_rand) + pick(near_b, 3) + pick(near_c, 3)))
    ghosts = sorted(set(int(nA + i) for i in (rng.uniform(3) * nB).astype(int))) if nB else []
    return owned, ghosts, len(near_b), len(near_c)


def _check_sampled_vs_oracle(ora_mod, fp, part, st, seed=5):
    L1 = fp.n_layers + 1
    rng = mg.SplitMix64(seed)
    n_c = 0
    for p, s in enumerate(st):
        owned, ghosts, _, nc = _sample_columns(s, L1, rng)
        n_c += nc
        g = _global_dofs(s["glob"], L1)
        for c in owned + ghosts:
            gc = int(s["glob"][c])
            fan = np.nonzero((fp.tri == gc).any(axis=1))[0]
            if c >= s["nA"]:   # ghost column: the part's own triangles of the fan only
                fan = fan[part[fan] == p]
            Ro, Mo, orp, ov, lc = _oracle_rows(ora_mod, fp, fan, gc)
            for k in range(L1):
                for a in range(2):
                    r = 2 * (c * L1 + k) + a
                    ro = 2 * (lc * L1 + k) + a
                    assert abs(s["R"][r] - Ro[ro]) <= R_TOL * np.abs(Mo).max()
                    seg_o = ov[orp[ro]:orp[ro + 1]]
                    loc = s["V"][s["rp"][r]:s["rp"][r + 1]]
                    order = np.argsort(g[s["col"][s["rp"][r]:s["rp"][r + 1]]], kind="stable")
                    assert loc.size == seg_o.size
                    assert np.abs(loc[order] - seg_o).max() <= J_TOL * np.abs(seg_o).max()
    return n_c


@pytest.mark.parametrize("P", [2, 3, 8])
def test_loopback_halo_c2(torch_cuda, ora_mod, P):
    """C2 (Greenland-like 16 km, 10 layers) in P parts on one GPU."""
    fp = mg.greenland_like(16.0)
    part, st, halos = _run_loopback(torch_cuda, fp, P)
    nn, rr, rv = halos[0].info()
    assert nn >= 1 and rr > 0 and rv > 0
    _check_import(fp, st)
    _check_owned_vs_full(torch_cuda, fp, st)
    assert _check_sampled_vs_oracle(ora_mod, fp, part, st) > 0   # class-C couplings were sampled


def test_loopback_halo_c4x2(torch_cuda, ora_mod):
    """C4 x 2 (the weak-scaling mesh of 2 GPUs, 9.6 M wedges) in 2 parts on one
    GPU: import bit-exact, owned rows vs the single-domain assembly, sampled
    owned (random / next to ghosts / next to column-only couplings) and ghost
    rows vs the oracle."""
    fp = mg.greenland_like_1_10(2.0)
    part, st, halos = _run_loopback(torch_cuda, fp, 2)
    _check_import(fp, st)
    _check_owned_vs_full(torch_cuda, fp, st)
    _check_sampled_vs_oracle(ora_mod, fp, part, st, seed=9)


def test_loopback_halo_residual_only_and_repeat(torch_cuda):
    """fo_halo_sum with d_vals = NULL (residual only): owned R equals the R + J
    path's; both run twice are bitwise equal (deterministic unpack order)."""
    import torch
    from paper_2204_04321_b200 import fo
    fp = mg.greenland_like(40.0, n_layers=5)
    P, L1 = 3, 6
    part = fo.partition(fp.n_tri, P)
    meshes = [fo.Mesh.from_footprint(fp, part=part, my_part=p, n_parts=P) for p in range(P)]
    halos = fo.Halo.loopback(meshes)
    Ug = fp.U.reshape(fp.n_vert, L1, 2)
    outs = []
    for rep in range(2):
        Us = [torch.tensor(Ug[m.columns()[0]].reshape(-1), device="cuda") for m in meshes]
        Rs = [m.residual(U) for m, U in zip(meshes, Us)]
        for h, R in zip(halos, Rs):
            h.sum(R, None)
        RV = [m.jacobian(U) for m, U in zip(meshes, Us)]
        for h, (R, V) in zip(halos, RV):
            h.sum(R, V)
        torch.cuda.synchronize()
        out = []
        for m, R, (Rj, V) in zip(meshes, Rs, RV):
            no = m.n_owned_dofs
            a, b = R.cpu().numpy()[:no], Rj.cpu().numpy()[:no]
            assert np.abs(a - b).max() <= R_TOL * np.abs(b).max()
            out.append((a.tobytes(), b.tobytes(), V.cpu().numpy().tobytes()))
        outs.append(out)
    assert outs[0] == outs[1]


@pytest.mark.parametrize("case,P", [("C2", 2), ("C2", 3), ("C2", 8), ("C4x2", 2)])
def test_fused_halo_assembly_matches_sequential(torch_cuda, case, P):
    """fo_assemble_jacobian_halo (boundary patches on the halo's side stream,
    ghost rows sent while the interior patches run, unpack-add joined back)
    gives, bit for bit, what fo_assemble_jacobian + fo_halo_sum give -- for
    R + J and residual only, on every part; a part mesh orders its
    ghost-touching triangles first (the boundary patches lead)."""
    import torch
    from paper_2204_04321_b200 import fo
    fp = mg.greenland_like(16.0) if case == "C2" else mg.greenland_like_1_10(2.0)
    L1 = fp.n_layers + 1
    part = fo.partition(fp.n_tri, P)
    meshes = [fo.Mesh.from_footprint(fp, part=part, my_part=p, n_parts=P) for p in range(P)]
    halos = fo.Halo.loopback(meshes)
    Ug = fp.U.reshape(fp.n_vert, L1, 2)
    Us = [torch.tensor(Ug[m.columns()[0]].reshape(-1), device="cuda") for m in meshes]
    seq = []
    for m, h, U in zip(meshes, halos, Us):
        seq.append(m.jacobian(U))
    for h, (R, V) in zip(halos, seq):
        h.sum(R, V)
    seq_r = [m.residual(U) for m, U in zip(meshes, Us)]
    for h, R in zip(halos, seq_r):
        h.sum(R, None)
    fused = [(torch.full_like(R, float("nan")), torch.full_like(V, float("nan"))) for R, V in seq]
    for h, U, (R, V) in zip(halos, Us, fused):
        h.assemble(U, R, V)
    fused_r = [torch.full_like(R, float("nan")) for R in seq_r]
    for h, U, R in zip(halos, Us, fused_r):
        h.assemble(U, R)
    torch.cuda.synchronize()
    for p, m in enumerate(meshes):
        no = m.n_owned_dofs
        rp, _ = m.graph().to_host()
        nv = int(rp[no])
        assert fused[p][0][:no].cpu().numpy().tobytes() == seq[p][0][:no].cpu().numpy().tobytes()
        assert fused[p][1][:nv].cpu().numpy().tobytes() == seq[p][1][:nv].cpu().numpy().tobytes()
        assert fused_r[p][:no].cpu().numpy().tobytes() == seq_r[p][:no].cpu().numpy().tobytes()
        assert not torch.isnan(fused[p][1]).any()
    assert sum(m.last_launch_count() for m in meshes) > 0


def test_loopback_rejects_wrong_parts(torch_cuda):
    from paper_2204_04321_b200 import fo
    fp = mg.greenland_like(60.0, n_layers=3)
    part = fo.partition(fp.n_tri, 2)
    m0 = fo.Mesh.from_footprint(fp, part=part, my_part=0, n_parts=2)
    m1 = fo.Mesh.from_footprint(fp, part=part, my_part=1, n_parts=2)
    with pytest.raises(fo.FoError) as e:
        fo.Halo.loopback([m1, m0])
    assert e.value.status == fo.FO_ESTATE
    with pytest.raises(fo.FoError):
        fo.Halo.loopback([m0])


def test_nccl_halo_two_ranks(torch_cuda):
    """The NCCL transport: torchrun, 2 ranks on 2 GPUs, tools/halo_nccl_check.py
    (owned rows vs the single-domain assembly).  Skipped below 2 devices."""
    if torch_cuda.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (the round-end driver box has one)")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533",
                        os.path.join(ROOT, "tools", "halo_nccl_check.py")],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "halo_nccl_check OK" in r.stdout
