"""NCCL halo check, one rank per GPU (torchrun --nproc-per-node N):
fo_halo_create (NCCL) -> fo_halo_import -> fo_assemble_jacobian -> fo_halo_sum
(and fo_assemble_jacobian_halo, bit for bit the same owned rows), then the owned rows of every rank against the single-domain assembly on the
same GPU (R <= 1e-12 max|R|, J <= 1e-11 row-scaled) and the imported ghost U
bit for bit.  Used by tests/test_gpu_halo.py::test_nccl_halo_two_ranks (only on
boxes with >= 2 GPUs).  Prints "halo_nccl_check OK" on rank 0.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_04321_b200 import fo, meshgen as mg  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    fp = mg.greenland_like(16.0)
    L1 = fp.n_layers + 1
    part = fo.partition(fp.n_tri, world)
    uid = [fo.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    m = fo.Mesh.from_footprint(fp, device=dev, part=part, my_part=rank, n_parts=world)
    halo = fo.Halo(m, uid[0], rank, world)
    glob, nA, nB, nC = m.columns()
    Ul = fp.U.reshape(fp.n_vert, L1, 2)[glob].reshape(-1).copy()
    Ul[2 * nA * L1:] = np.nan
    U = torch.tensor(Ul, device=f"cuda:{dev}")
    halo.import_(U)
    R, V = m.jacobian(U)
    halo.sum(R, V)
    # fo_assemble_jacobian_halo (export overlapped with the interior patches):
    # the owned rows bit for bit as the sequential call pair
    Rf2, Vf2 = torch.full_like(R, float("nan")), torch.full_like(V, float("nan"))
    halo.assemble(U, Rf2, Vf2)
    torch.cuda.synchronize()
    no_ = m.n_owned_dofs
    nv_ = int(m.graph().to_host()[0][no_])
    assert Rf2[:no_].cpu().numpy().tobytes() == R[:no_].cpu().numpy().tobytes(), "fused R"
    assert Vf2[:nv_].cpu().numpy().tobytes() == V[:nv_].cpu().numpy().tobytes(), "fused J"
    U, R, V = U.cpu().numpy(), R.cpu().numpy(), V.cpu().numpy()
    want = fp.U.reshape(fp.n_vert, L1, 2)[glob[nA:nA + nB]].reshape(-1)
    assert U[2 * nA * L1:2 * (nA + nB) * L1].tobytes() == want.tobytes(), "ghost U import"
    full = fo.Mesh.from_footprint(fp, device=dev)
    Rf, Vf = full.jacobian(torch.tensor(fp.U, device=f"cuda:{dev}"))
    grp, _ = full.graph().to_host()
    Rf, Vf = Rf.cpu().numpy(), Vf.cpu().numpy()
    n = glob[:, None] * L1 + np.arange(L1)
    g = np.stack([2 * n, 2 * n + 1], axis=2).reshape(-1)
    no = m.n_owned_dofs
    assert np.abs(R[:no] - Rf[g[:no]]).max() <= 1e-12 * np.abs(Rf).max(), "owned R"
    rp, col = m.graph().to_host()
    for r in range(no):
        seg = Vf[grp[g[r]]:grp[g[r] + 1]]
        loc = V[rp[r]:rp[r + 1]][np.argsort(g[col[rp[r]:rp[r + 1]]], kind="stable")]
        assert np.abs(loc - seg).max() <= 1e-11 * np.abs(seg).max(), f"owned J row {r}"
    dist.barrier()
    halo.close()
    if rank == 0:
        print("halo_nccl_check OK", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
