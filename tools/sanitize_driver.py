"""One pass over every libfo kernel on small inputs, for compute-sanitizer
(SURVEY.md 4.3 / VERDICT r1 item 4):  tools/gpu_sanitize.sh runs this under
memcheck, racecheck, synccheck and initcheck.

  python tools/sanitize_driver.py C1|C2

Kernels exercised: ka_ws_kernel (wedge and tetrahedral R + J, with the
in-kernel zero fill and, through the fused halo call, without), ka_patch_kernel
(residual-only instances, generic n, the round-1 R + J kernel),
zero_boundary_kernel, multi_fixup_kernel, lateral_kernel, the atomic
ablation, the quad-patch and coloured hexahedral kernels, the halo gather /
unpack-add kernels (loopback transport, sequential and fused) and the
Newton-consumer kernels (SpMV, line factor / solve, Krylov dots / update).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_04321_b200 import fo, meshgen as mg  # noqa: E402


def main(cfg):
    fp = mg.ismip_hom_a() if cfg == "C1" else mg.greenland_like(16.0)
    dev = "cuda"
    U = torch.tensor(fp.U, device=dev)
    m = fo.Mesh.from_footprint(fp)
    g = m.graph()
    R, V = m.jacobian(U)                        # zero kernel, patch kernel <1,1,0>, multi fix-up
    m.residual(U)                               # patch kernel <0,1,0>
    m.set_lateral(True)
    m.jacobian(U)                               # + lateral kernel
    m.set_lateral(False)
    m.set_element(1)
    m.jacobian(U)                               # tetrahedral instance <1,1,1>
    m.residual(U)
    m.set_element(0)
    m.set_scatter(fo.SCATTER_ATOMIC)
    m.jacobian(U)                               # atomic ablation kernel
    m.set_scatter(fo.SCATTER_OWNER)
    m2 = fo.Mesh.from_footprint(fp, params=dict(glen_n=1.0))
    m2.jacobian(U)                              # generic-n instance <1,0,0>
    fpt = mg.with_temperature(mg.ismip_hom_a(nx=8, n_layers=4))
    mt = fo.Mesh.from_footprint(fpt)
    mt.set_temperature(fpt.T_star, fpt.arrhenius["A0"], fpt.arrhenius["Q"])
    mt.jacobian(torch.tensor(fpt.U, device=dev))
    # Newton consumer kernels
    # inputs made by host-to-device copies: compute-sanitizer instruments only
    # libfo's kernels (--kernel-name kns=N2fo), so memory written by torch's own
    # kernels would read as uninitialised to initcheck
    x = torch.tensor(np.ones(m.n_dofs), device=dev)
    y = torch.tensor(np.zeros(m.n_dofs), device=dev)
    L = fo.lib()
    stream = torch.cuda.current_stream().cuda_stream
    fo.check(L.fo_spmv(m.handle, g.handle, fo._ptr(V), fo._ptr(x), fo._ptr(y), stream), "fo_spmv")
    fo.check(L.fo_line_factor(m.handle, g.handle, fo._ptr(V), stream), "fo_line_factor")
    fo.check(L.fo_line_solve(m.handle, fo._ptr(x), fo._ptr(y), stream), "fo_line_solve")
    Vk = torch.tensor(np.random.default_rng(1).random((4, m.n_dofs)), device=dev)
    h = torch.tensor(np.zeros(4), device=dev)
    fo.check(L.fo_krylov_dots(m.handle, m.n_dofs, 4, fo._ptr(Vk), m.n_dofs, fo._ptr(x), fo._ptr(h), stream),
             "fo_krylov_dots")
    fo.check(L.fo_krylov_update(m.handle, m.n_dofs, 4, fo._ptr(Vk), m.n_dofs, fo._ptr(h), fo._ptr(x), stream),
             "fo_krylov_update")
    # hexahedra
    fq = mg.to_quads(mg.slab(nx=10, n_layers=3, distort=0.1), 10)
    mq = fo.Mesh.from_footprint(fq)
    mq.jacobian(torch.tensor(fq.U, device=dev))     # quad-patch kernel (KH-patch) + zero fill + fix-up
    mq.residual(torch.tensor(fq.U, device=dev))     # coloured kernel, residual
    mq.set_scatter(fo.SCATTER_ATOMIC)
    mq.jacobian(torch.tensor(fq.U, device=dev))     # coloured R + J ablation
    # the round-1 single-warpgroup wedge kernel (R + J)
    m.set_scatter(fo.SCATTER_OWNER_1WG)
    m.jacobian(U)
    m.set_scatter(fo.SCATTER_OWNER)
    # halo kernels over the loopback transport (3 parts)
    part = fo.partition(fp.n_tri, 3)
    parts = [fo.Mesh.from_footprint(fp, part=part, my_part=p, n_parts=3) for p in range(3)]
    halos = fo.Halo.loopback(parts)
    L1 = fp.n_layers + 1
    Ug = fp.U.reshape(fp.n_vert, L1, 2)
    Us = [torch.tensor(Ug[pm.columns()[0]].reshape(-1), device=dev) for pm in parts]
    for hh, Ul in zip(halos, Us):
        hh.import_(Ul)
    outs = [pm.jacobian(Ul) for pm, Ul in zip(parts, Us)]
    for hh, (Rp, Vp) in zip(halos, outs):
        hh.sum(Rp, Vp)
    # fused assembly + export (side stream, split launches, zero kernel)
    for hh, Ul, (Rp, Vp) in zip(halos, Us, outs):
        hh.assemble(Ul, Rp, Vp)
    for hh, Ul, (Rp, Vp) in zip(halos, Us, outs):
        hh.assemble(Ul, Rp)
    torch.cuda.synchronize()
    assert np.isfinite(R.cpu().numpy()).all() and np.isfinite(V.cpu().numpy()).all()
    print(f"sanitize_driver {cfg} done", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C1")
