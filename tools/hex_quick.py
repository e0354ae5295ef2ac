"""quick device timing of the hexahedral path (700 x 700 quads x 10 layers,
4.9 M hexahedra): owner-computes patches (default) and the coloured
read-modify-write ablation (FO_SCATTER_ATOMIC on a quad mesh) (dev tool)."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2204_04321_b200 import fo, meshgen as mg  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 700
fq = mg.to_quads(mg.ismip_hom_a(nx=nx, n_layers=10), nx)
mq = fo.Mesh.from_footprint(fq)
gq = mq.graph()
Uq = torch.tensor(fq.U, device="cuda")
Rq = torch.empty(mq.n_dofs, dtype=torch.float64, device="cuda")
Vq = torch.empty(gq.nnz, dtype=torch.float64, device="cuda")
for sc, tag in ((fo.SCATTER_OWNER, "owner"), (fo.SCATTER_ATOMIC, "coloured")):
    mq.set_scatter(sc)
    for f, name in ((lambda: mq.jacobian(Uq, gq, Rq, Vq), "hex RJ"), (lambda: mq.residual(Uq, Rq), "hex R")):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            f()
        b.record()
        torch.cuda.synchronize()
        print(tag, name, round(a.elapsed_time(b) / 5, 3), "ms", flush=True)
