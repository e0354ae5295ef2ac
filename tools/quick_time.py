"""quick device timing of the assembly kernels on one config (dev tool)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2204_04321_b200 import fo, meshgen as mg  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
t0 = time.time()
fp = mg.by_name(name)
print(f"{name}: n_tri {fp.n_tri} n_elem {fp.n_elem} gen {time.time()-t0:.1f}s", flush=True)
t0 = time.time()
mesh = fo.Mesh.from_footprint(fp)
g = mesh.graph()
print(f"mesh+graph {time.time()-t0:.1f}s nnz {g.nnz}", flush=True)
U = torch.tensor(fp.U, device="cuda")
R = torch.empty(mesh.n_dofs, dtype=torch.float64, device="cuda")
V = torch.empty(g.nnz, dtype=torch.float64, device="cuda")
import os
modes = [int(x) for x in os.environ.get('FO_SCATTERS', '1,0').split(',')]
whats = os.environ.get('FO_WHAT', 'residual,jacobian').split(',')
for sc in modes:
    try:
        mesh.set_scatter(sc)
    except Exception as e:
        print("scatter", sc, e); continue
    for what in whats:
        for _ in range(3):
            mesh.residual(U, R) if what == "residual" else mesh.jacobian(U, g, R, V)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10
        e0.record()
        for _ in range(n):
            mesh.residual(U, R) if what == "residual" else mesh.jacobian(U, g, R, V)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(f"scatter {sc} {what}: {ms:.3f} ms  {fp.n_elem/ms/1e3:.1f} Melem/s  "
              f"HBM-alg {(8*g.nnz + 16*mesh.n_nodes*2)/ms/1e6:.0f} GB/s", flush=True)
