"""quick device timing of the tetrahedral path on C3 (three tets per prism):
the warp-specialised kernel (scatter 0) and the round-1 patch kernel (3) (dev tool)."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2204_04321_b200 import fo, meshgen as mg  # noqa: E402

fp = mg.greenland_like_1_10()
m = fo.Mesh.from_footprint(fp)
m.set_element(1)
g = m.graph()
U = torch.tensor(fp.U, device="cuda")
R = torch.empty(m.n_dofs, dtype=torch.float64, device="cuda")
V = torch.empty(g.nnz, dtype=torch.float64, device="cuda")
for sc in (0, 3):
    m.set_scatter(sc)
    for _ in range(3):
        m.jacobian(U, g, R, V)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        m.jacobian(U, g, R, V)
    b.record()
    torch.cuda.synchronize()
    print(f"C3-tet scatter {sc} R+J {a.elapsed_time(b) / 10:.3f} ms", flush=True)
