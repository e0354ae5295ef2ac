"""Measurement of the NEXT rows on one B200 (C3, 4.80 M wedges): device time
per assembly (CUDA events, median of 10, 512 MB written between calls) for
  base     R + J, wedges (the bench.py step without the halo)
  r_only   R only
  f3       R + J with the in-kernel Arrhenius flow factor
  f1       R + J + the lateral margin term kernel
  f4       R + J with three P1 tetrahedra per prism
usage: python tools/next_rows_bench.py > profiles/<tag>_next_rows.jsonl"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_04321_b200 import fo, meshgen as mg  # noqa: E402

fp = mg.with_temperature(mg.greenland_like_1_10())
mesh = fo.Mesh.from_footprint(fp)
g = mesh.graph()
U = torch.tensor(fp.U, device="cuda")
R = torch.empty(mesh.n_dofs, dtype=torch.float64, device="cuda")
V = torch.empty(g.nnz, dtype=torch.float64, device="cuda")
flush = torch.empty(512 * 2**20 // 8, dtype=torch.float64, device="cuda")


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        flush.fill_(0.5)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def line(name, ms, note):
    print(json.dumps({"variant": name, "workload": "C3", "wedges": fp.n_elem, "ms": round(ms, 4),
                      "Melem_s": round(fp.n_elem / ms / 1e3, 1), "launches": mesh.last_launch_count(),
                      "note": note}), flush=True)


jac = lambda: mesh.jacobian(U, g, R, V)
line("base", timeit(jac), "R + J, wedges, warp-specialised owner-computes kernel")
line("r_only", timeit(lambda: mesh.residual(U, R)), "R only")
mesh.set_temperature(fp.T_star, fp.arrhenius["A0"], fp.arrhenius["Q"])
line("f3_temperature", timeit(jac), "R + J, A = A0 exp(-Q/RT*) per wedge in-kernel")
mesh.set_temperature(None)
mesh.set_lateral(True)
line("f1_lateral", timeit(jac), "R + J + lateral margin term kernel")
mesh.set_lateral(False)
mesh.set_element(1)
line("f4_tet3", timeit(jac), "R + J, three P1 tetrahedra per prism (14.4 M tets), warp-specialised kernel")
line("f4_tet3_r_only", timeit(lambda: mesh.residual(U, R)), "R only, tetrahedra")

# hexahedra on a quadrilateral footprint of C3 size (700 x 700 quads x 10 layers)
fq = mg.to_quads(mg.ismip_hom_a(nx=700, n_layers=10), 700)
mq = fo.Mesh.from_footprint(fq)
gq = mq.graph()
Uq = torch.tensor(fq.U, device="cuda")
Rq = torch.empty(mq.n_dofs, dtype=torch.float64, device="cuda")
Vq = torch.empty(gq.nnz, dtype=torch.float64, device="cuda")
ms = timeit(lambda: mq.jacobian(Uq, gq, Rq, Vq))
print(json.dumps({"variant": "f4_hex8", "workload": "700x700 quads x 10 layers", "wedges": fq.n_elem,
                  "ms": round(ms, 4), "Melem_s": round(fq.n_elem / ms / 1e3, 1), "launches": mq.last_launch_count(),
                  "note": "R + J, 8-node trilinear hexahedra, quad-patch owner-computes kernel"}), flush=True)
mq.set_scatter(fo.SCATTER_ATOMIC)
ms = timeit(lambda: mq.jacobian(Uq, gq, Rq, Vq))
print(json.dumps({"variant": "f4_hex8_coloured", "workload": "700x700 quads x 10 layers", "wedges": fq.n_elem,
                  "ms": round(ms, 4), "Melem_s": round(fq.n_elem / ms / 1e3, 1), "launches": mq.last_launch_count(),
                  "note": "R + J, hexahedra, coloured read-modify-write ablation"}), flush=True)
mq.set_scatter(fo.SCATTER_OWNER)
ms = timeit(lambda: mq.residual(Uq, Rq))
print(json.dumps({"variant": "f4_hex8_r_only", "workload": "700x700 quads x 10 layers", "wedges": fq.n_elem,
                  "ms": round(ms, 4), "Melem_s": round(fq.n_elem / ms / 1e3, 1), "launches": mq.last_launch_count(),
                  "note": "R only, hexahedra"}), flush=True)
