"""Footprint partition, local numbering (owned / ghost / column-only) and the
halo plan of the multi-GPU path (PAPER.md Import P:175,
Export P:185, owned-rows-first matrix P:250-255), tested on the host:
  * owned rows of every part carry exactly the global row pattern (bit-exact),
  * every global column is owned by exactly one part,
  * assembling each part with the ORACLE (on that part's triangles), placing
    the values in the part's local CSR and applying the library's halo plan
    reproduces the single-domain oracle Jacobian on every owned row;
  * the same exchange over torch.distributed gloo with world_size 2.
"""
import os

import numpy as np
import pytest

from paper_2204_04321_b200 import fo
from paper_2204_04321_b200 import meshgen as mg


@pytest.fixture(scope="module")
def lib():
    from paper_2204_04321_b200 import _build
    _build.build()
    return fo.lib()


def _workload(name):
    if name == "gris":
        return mg.greenland_like(70.0, n_layers=4)
    return mg.ismip_hom_a(nx=10, n_layers=3)


def _global_of_local_dofs(glob, L):
    L1 = L + 1
    node = (glob[:, None] * L1 + np.arange(L1)[None, :]).reshape(-1)
    return np.stack([2 * node, 2 * node + 1], axis=1).reshape(-1)


@pytest.mark.parametrize("name,P", [("C1", 2), ("C1", 3), ("gris", 4), ("gris", 7)])
def test_owned_rows_match_global_pattern(lib, ora_mod, name, P):
    fp = _workload(name)
    L = fp.n_layers
    part = fo.partition(fp.n_tri, P)
    grp, gcol = fo.graph_host(fp.n_vert, fp.tri, L)
    owners = np.zeros(fp.n_vert, dtype=np.int64)
    for p in range(P):
        glob, nA, nB, rp, col = fo.part_graph_host(fp.n_vert, fp.tri, L, part, P, p)
        owners[glob[:nA]] += 1
        g = _global_of_local_dofs(glob, L)
        n_owned = 2 * nA * (L + 1)
        for r in range(n_owned):
            loc = np.sort(g[col[rp[r]:rp[r + 1]]])
            gr = g[r]
            assert np.array_equal(loc, gcol[grp[gr]:grp[gr + 1]])
        # ghost rows exist, column-only rows are empty
        nk = 2 * (nA + nB) * (L + 1)
        assert np.all(np.diff(rp)[nk:] == 0)
        # local columns sorted ascending in local numbering
        for r in range(0, nk, 7):
            assert np.all(np.diff(col[rp[r]:rp[r + 1]]) > 0)
    assert np.all(owners == 1)


def _part_assembly(ora_mod, fp, part, P, p):
    """oracle values of part p's triangles placed into p's local CSR."""
    L = fp.n_layers
    glob, nA, nB, rp, col = fo.part_graph_host(fp.n_vert, fp.tri, L, part, P, p)
    sub = mg.sub_footprint_tris(fp, np.nonzero(part == p)[0])
    o = ora_mod.Oracle(sub)
    orp, ocol = o.graph()
    Rs, vs = o.jacobian(sub.U)
    sg = _global_of_local_dofs(sub.vertex_ids, L)          # sub dof -> global dof
    nG = 2 * fp.n_vert * (L + 1)
    rows = np.repeat(np.arange(orp.size - 1), np.diff(orp))
    key = sg[rows] * nG + sg[ocol]
    order = np.argsort(key)
    key, vs = key[order], vs[order]
    g = _global_of_local_dofs(glob, L)
    lrows = np.repeat(np.arange(rp.size - 1), np.diff(rp))
    lkey = g[lrows] * nG + g[col]
    pos = np.searchsorted(key, lkey)
    pos = np.minimum(pos, key.size - 1)
    hit = key[pos] == lkey
    vals = np.where(hit, vs[pos], 0.0)
    R = np.zeros(rp.size - 1)
    rloc = {int(x): i for i, x in enumerate(g)}
    for i, gd in enumerate(sg):
        R[rloc[int(gd)]] += Rs[i]
    return dict(glob=glob, nA=nA, rp=rp, col=col, vals=vals, R=R, g=g)


def _check_owned(ora_mod, fp, parts, P):
    L = fp.n_layers
    o = ora_mod.Oracle(fp)
    grp, gcol = o.graph()
    Rg, vg = o.jacobian(fp.U)
    for p in range(P):
        d = parts[p]
        n_owned = 2 * d["nA"] * (L + 1)
        for r in range(n_owned):
            gr = d["g"][r]
            seg = vg[grp[gr]:grp[gr + 1]]
            loc = d["vals"][d["rp"][r]:d["rp"][r + 1]]
            order = np.argsort(d["g"][d["col"][d["rp"][r]:d["rp"][r + 1]]])
            assert np.abs(loc[order] - seg).max() <= 1e-12 * np.abs(seg).max()
        assert np.abs(d["R"][:n_owned] - Rg[d["g"][:n_owned]]).max() <= 1e-12 * np.abs(Rg).max()


@pytest.mark.parametrize("name,P", [("C1", 2), ("gris", 3)])
def test_halo_plan_reproduces_single_domain(lib, ora_mod, name, P):
    fp = _workload(name)
    L = fp.n_layers
    part = fo.partition(fp.n_tri, P)
    parts = [_part_assembly(ora_mod, fp, part, P, p) for p in range(P)]
    plans = [fo.halo_plan_host(fp.n_vert, fp.tri, L, part, P, p) for p in range(P)]
    # "fake comm": p's contiguous send slices added into q's owned rows
    for p in range(P):
        for q, (sr, dr, sv, dv) in plans[p].items():
            assert np.all(np.diff(sr) == 1) and np.all(np.diff(sv) == 1)    # zero-copy slices
            np.add.at(parts[q]["R"], dr, parts[p]["R"][sr])
            np.add.at(parts[q]["vals"], dv, parts[p]["vals"][sv])
    _check_owned(ora_mod, fp, parts, P)


def _gloo_worker(rank, world, port, result_q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as ora_mod
        fp = _workload("gris")
        L = fp.n_layers
        part = fo.partition(fp.n_tri, world)
        me = _part_assembly(ora_mod, fp, part, world, rank)
        plans = {p: fo.halo_plan_host(fp.n_vert, fp.tri, L, part, world, p) for p in range(world)}
        # what I send: my ghost slices; what I receive: slices of others owning my columns
        reqs = []
        for q, (sr, dr, sv, dv) in plans[rank].items():
            buf = torch.tensor(np.concatenate([me["R"][sr], me["vals"][sv]]))
            reqs.append(dist.isend(buf, dst=q))
        for p in range(world):
            if p == rank or rank not in plans[p]:
                continue
            sr, dr, sv, dv = plans[p][rank]
            buf = torch.empty(len(sr) + len(sv), dtype=torch.float64)
            dist.recv(buf, src=p)
            b = buf.numpy()
            np.add.at(me["R"], dr, b[:len(sr)])
            np.add.at(me["vals"], dv, b[len(sr):])
        for r in reqs:
            r.wait()
        parts = {rank: me}
        # check my owned rows against the single-domain oracle
        o = ora_mod.Oracle(fp)
        grp, gcol = o.graph()
        Rg, vg = o.jacobian(fp.U)
        n_owned = 2 * me["nA"] * (L + 1)
        worst = 0.0
        for r in range(n_owned):
            gr = me["g"][r]
            seg = vg[grp[gr]:grp[gr + 1]]
            loc = me["vals"][me["rp"][r]:me["rp"][r + 1]]
            order = np.argsort(me["g"][me["col"][me["rp"][r]:me["rp"][r + 1]]])
            worst = max(worst, np.abs(loc[order] - seg).max() / np.abs(seg).max())
        rerr = np.abs(me["R"][:n_owned] - Rg[me["g"][:n_owned]]).max() / np.abs(Rg).max()
        result_q.put((rank, worst, rerr))
        del parts
    finally:
        dist.destroy_process_group()


def test_halo_exchange_gloo_world2(lib):
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = [q.get(timeout=5) for _ in range(2)]
    for rank, jerr, rerr in res:
        assert jerr <= 1e-12 and rerr <= 1e-12, (rank, jerr, rerr)
    assert all(p.exitcode == 0 for p in procs)
