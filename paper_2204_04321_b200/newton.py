"""NEXT-f2: damped Newton with right-preconditioned GMRES(m) on libfo's kernels
(PAPER.md eq:linearsystem P:160-165 -- the paper solves
J(U) dU = -F(U) with preconditioned GMRES).

Every matrix operation runs in libfo: the R + J assembly (fo_assemble_jacobian),
y = J x (fo_spmv, column-structured CSR), the vertical-line preconditioner
(fo_line_factor / fo_line_solve) and the Krylov dot products / basis updates
(fo_krylov_dots / fo_krylov_update, fixed-order reductions).  PyTorch only
holds the device vectors (copies, scaling); the (m+1) x m Hessenberg least
squares is solved on the host with Givens rotations (m doubles per step).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import fo


def _p(t):
    return C.c_void_p(t.data_ptr())


@dataclass
class NewtonReport:
    converged: bool
    newton_steps: int
    residual_norms: list = field(default_factory=list)     # ||F(U_k)||_2
    krylov_iterations: list = field(default_factory=list)  # per Newton step
    step_lengths: list = field(default_factory=list)       # damping alpha per step


class NewtonSolver:
    """Newton for F(U) = 0 on one (single-domain) mesh."""

    def __init__(self, mesh: "fo.Mesh", restart: int = 30, max_krylov: int = 300):
        import torch
        if restart < 1 or restart > 63:
            raise ValueError("restart must be in [1, 63]")
        self.mesh = mesh
        self.graph = mesh.graph()
        self.n = mesh.n_dofs
        self.m = restart
        self.max_krylov = max_krylov
        dev = f"cuda:{mesh.device}"
        self.torch = torch
        self.V = torch.zeros((restart + 1, self.n), dtype=torch.float64, device=dev)
        self.vals = torch.zeros(self.graph.nnz, dtype=torch.float64, device=dev)
        self.R = torch.zeros(self.n, dtype=torch.float64, device=dev)
        self.w = torch.zeros(self.n, dtype=torch.float64, device=dev)
        self.z = torch.zeros(self.n, dtype=torch.float64, device=dev)
        self.h = torch.zeros(64, dtype=torch.float64, device=dev)
        self.stream = torch.cuda.current_stream(mesh.device).cuda_stream

    # -- libfo wrappers -------------------------------------------------
    def _check(self, st, where):
        fo.check(st, where)

    def spmv(self, x, y):
        self._check(fo.lib().fo_spmv(self.mesh.handle, self.graph.handle, _p(self.vals), _p(x), _p(y),
                                     C.c_void_p(self.stream)), "fo_spmv")

    def precond(self, r, z):
        self._check(fo.lib().fo_line_solve(self.mesh.handle, _p(r), _p(z), C.c_void_p(self.stream)),
                    "fo_line_solve")

    def dots(self, k, w):
        """V[:k] . w on the device -> host numpy (k values)."""
        self._check(fo.lib().fo_krylov_dots(self.mesh.handle, self.n, k, _p(self.V), self.n, _p(w),
                                            _p(self.h), C.c_void_p(self.stream)), "fo_krylov_dots")
        return self.h[:k].cpu().numpy()

    def update(self, k, coef, w):
        """w -= sum_j coef_j V_j."""
        self.h[:k].copy_(self.torch.from_numpy(np.ascontiguousarray(coef, dtype=np.float64)))
        self._check(fo.lib().fo_krylov_update(self.mesh.handle, self.n, k, _p(self.V), self.n, _p(self.h),
                                              _p(w), C.c_void_p(self.stream)), "fo_krylov_update")

    def norm(self, w):
        V0 = self.V[0].clone()
        self.V[0].copy_(w)
        d = self.dots(1, w)[0]
        self.V[0].copy_(V0)
        return math.sqrt(max(d, 0.0))

    # -- GMRES(m), right preconditioning: J M^-1 y = b, x = M^-1 y -------
    def gmres(self, b, x, rtol):
        """solve J x = b (x overwritten, initial guess 0); returns iterations."""
        torch = self.torch
        x.zero_()
        beta0 = self.norm(b)
        if beta0 == 0.0:
            return 0
        r = b.clone()
        its = 0
        while its < self.max_krylov:
            beta = self.norm(r)
            if beta <= rtol * beta0:
                break
            self.V[0].copy_(r).div_(beta)
            H = np.zeros((self.m + 1, self.m))
            cs, sn = np.zeros(self.m), np.zeros(self.m)
            g = np.zeros(self.m + 1)
            g[0] = beta
            j_done = 0
            for j in range(self.m):
                self.precond(self.V[j], self.z)
                self.spmv(self.z, self.w)
                # classical Gram-Schmidt, twice (CGS2)
                hcol = self.dots(j + 1, self.w)
                self.update(j + 1, hcol, self.w)
                h2 = self.dots(j + 1, self.w)
                self.update(j + 1, h2, self.w)
                hcol = hcol + h2
                hn = self.norm(self.w)
                H[:j + 1, j] = hcol
                H[j + 1, j] = hn
                if hn > 0.0:
                    self.V[j + 1].copy_(self.w).div_(hn)
                for i in range(j):   # apply previous rotations
                    t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                    H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                    H[i, j] = t
                d = math.hypot(H[j, j], H[j + 1, j])
                cs[j], sn[j] = (1.0, 0.0) if d == 0.0 else (H[j, j] / d, H[j + 1, j] / d)
                H[j, j] = d
                H[j + 1, j] = 0.0
                g[j + 1] = -sn[j] * g[j]
                g[j] = cs[j] * g[j]
                its += 1
                j_done = j + 1
                if abs(g[j + 1]) <= rtol * beta0 or its >= self.max_krylov or hn == 0.0:
                    break
            y = np.zeros(j_done)
            for i in range(j_done - 1, -1, -1):
                y[i] = (g[i] - H[i, i + 1:j_done] @ y[i + 1:]) / H[i, i]
            # x += M^-1 (V y): accumulate V y into w (w = 0 - sum(-y_j) V_j)
            self.w.zero_()
            self.update(j_done, -y, self.w)
            self.precond(self.w, self.z)
            x.add_(self.z)
            # r = b - J x
            self.spmv(x, self.w)
            r = b - self.w
        return its

    # -- damped Newton -------------------------------------------------
    def residual(self, U, R):
        self.mesh.residual(U, R=R)

    def solve(self, U, rtol: float = 1e-9, max_newton: int = 40, krylov_rtol: float = 1e-4) -> NewtonReport:
        """U (device, overwritten) <- the solution of F(U) = 0; stops when
        ||F(U)|| <= rtol ||F(U_0)||.  Backtracking on ||F||: alpha = 1, 1/2,
        ... until ||F(U - alpha dU)|| <= (1 - 1e-4 alpha) ||F(U)||."""
        torch = self.torch
        rep = NewtonReport(False, 0)
        dU = torch.zeros_like(U)
        Rt = torch.zeros_like(U)
        Ut = torch.zeros_like(U)
        self.mesh.jacobian(U, R=self.R, vals=self.vals)
        f0 = self.norm(self.R)
        rep.residual_norms.append(f0)
        f = f0
        for it in range(max_newton):
            if f <= rtol * f0:
                rep.converged = True
                break
            self._check(fo.lib().fo_line_factor(self.mesh.handle, self.graph.handle, _p(self.vals),
                                                C.c_void_p(self.stream)), "fo_line_factor")
            its = self.gmres(self.R, dU, krylov_rtol)
            rep.krylov_iterations.append(its)
            alpha = 1.0
            while True:
                torch.sub(U, dU, alpha=alpha, out=Ut)
                self.residual(Ut, Rt)
                ft = self.norm(Rt)
                if ft <= (1.0 - 1e-4 * alpha) * f or alpha < 1e-6:
                    break
                alpha *= 0.5
            U.copy_(Ut)
            rep.step_lengths.append(alpha)
            rep.newton_steps = it + 1
            self.mesh.jacobian(U, R=self.R, vals=self.vals)
            f = self.norm(self.R)
            rep.residual_norms.append(f)
        else:
            rep.converged = f <= rtol * f0
        if f <= rtol * f0:
            rep.converged = True
        return rep
