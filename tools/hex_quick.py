import sys, os, json, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2204_04321_b200 import fo, meshgen as mg
fq = mg.to_quads(mg.ismip_hom_a(nx=700, n_layers=10), 700)
mq = fo.Mesh.from_footprint(fq); gq = mq.graph()
Uq = torch.tensor(fq.U, device="cuda"); Rq = torch.empty(mq.n_dofs, dtype=torch.float64, device="cuda"); Vq = torch.empty(gq.nnz, dtype=torch.float64, device="cuda")
for f, name in ((lambda: mq.jacobian(Uq, gq, Rq, Vq), "hex RJ"), (lambda: mq.residual(Uq, Rq), "hex R")):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(5)]; b.record(); torch.cuda.synchronize()
    print(name, a.elapsed_time(b) / 5, "ms")
