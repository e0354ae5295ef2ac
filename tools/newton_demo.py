"""NEXT-f2 demo + measurement: damped Newton / GMRES on C1 and C2 (convergence
history), and the SpMV / line-solve kernels' bandwidth at C3 (CUDA events).
usage: python tools/newton_demo.py  (one GPU)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time

import numpy as np
import torch

from paper_2204_04321_b200 import fo, meshgen as mg, newton


def solve(name, fp, **kw):
    mesh = fo.Mesh.from_footprint(fp)
    U = torch.tensor(fp.U, device="cuda")
    s = newton.NewtonSolver(mesh, restart=30, max_krylov=kw.pop("max_krylov", 600))
    torch.cuda.synchronize()
    t = time.perf_counter()
    rep = s.solve(U, **kw)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    f = rep.residual_norms
    print(json.dumps({"workload": name, "wedges": fp.n_elem, "converged": rep.converged,
                      "newton_steps": rep.newton_steps, "seconds": round(dt, 3),
                      "rel_residual": [float(f"{x / f[0]:.3e}") for x in f],
                      "krylov_iterations": rep.krylov_iterations, "alpha": rep.step_lengths}))


def kernel_bw():
    fp = mg.greenland_like_1_10()
    mesh = fo.Mesh.from_footprint(fp)
    U = torch.tensor(fp.U, device="cuda")
    s = newton.NewtonSolver(mesh, restart=2)
    mesh.jacobian(U, R=s.R, vals=s.vals)
    fo.check(fo.lib().fo_line_factor(mesh.handle, s.graph.handle, newton._p(s.vals), None), "factor")
    x = torch.randn(mesh.n_dofs, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    flush = torch.empty(512 * 2**20 // 8, dtype=torch.float64, device="cuda")
    out = {}
    for name, fn, nbytes in [
            ("spmv", lambda: s.spmv(x, y), 8 * s.graph.nnz + 16 * mesh.n_dofs),
            ("line_solve", lambda: s.precond(x, y), 8 * (mesh.n_dofs // 2) * 8 + 16 * mesh.n_dofs)]:
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        out[name] = {"ms": round(ms, 4), "algorithmic_bytes": nbytes, "GB_s": round(nbytes / ms / 1e6, 1)}
    print(json.dumps({"workload": "C3", "kernels": out}))


if __name__ == "__main__":
    solve("C1", mg.ismip_hom_a(), rtol=1e-10, krylov_rtol=1e-6)
    solve("C2", mg.greenland_like(16.0), rtol=1e-8, krylov_rtol=1e-4, max_newton=60, max_krylov=3000)
    kernel_bw()
