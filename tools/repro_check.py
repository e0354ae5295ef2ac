"""run-to-run bitwise check of the C3 assembly (dev tool): repeats R + J and
R-only assemblies into NaN-filled buffers and reports differing entries."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2204_04321_b200 import fo, meshgen as mg  # noqa: E402

fp = mg.greenland_like_1_10()
mesh = fo.Mesh.from_footprint(fp)
U = torch.tensor(fp.U, device="cuda")
g = mesh.graph()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
ref = None
for rep in range(reps):
    R = torch.full((mesh.n_dofs,), float("nan"), dtype=torch.float64, device="cuda")
    vals = torch.full((g.nnz,), float("nan"), dtype=torch.float64, device="cuda")
    mesh.jacobian(U, R=R, vals=vals)
    Rr = torch.full((mesh.n_dofs,), float("nan"), dtype=torch.float64, device="cuda")
    mesh.residual(U, R=Rr)
    torch.cuda.synchronize()
    cur = [x.cpu().numpy() for x in (R, vals, Rr)]
    nan = [int(np.isnan(x).sum()) for x in cur]
    if ref is None:
        ref = cur
        print("rep 0 nan counts", nan, flush=True)
        continue
    diffs = []
    for name, a, b in zip(("R", "vals", "Rr"), ref, cur):
        d = np.nonzero(a.view(np.int64) != b.view(np.int64))[0]
        diffs.append((name, d.size, d[:5].tolist(), [float(a[i] - b[i]) for i in d[:3]]))
    print(f"rep {rep} nan {nan} diffs {diffs}", flush=True)
