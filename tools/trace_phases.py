"""phase timeline of ka_patch_kernel (dev tool; library built with -DFO_TRACE).
Per SM: how long both resident CTAs were in the element phase (A), both in
the gather/store phase (B), or one in each."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2204_04321_b200 import fo, meshgen as mg  # noqa: E402

fp = mg.by_name("C3")
mesh = fo.Mesh.from_footprint(fp)
g = mesh.graph()
U = torch.tensor(fp.U, device="cuda")
R = torch.empty(mesh.n_dofs, dtype=torch.float64, device="cuda")
V = torch.empty(g.nnz, dtype=torch.float64, device="cuda")
for _ in range(3):
    mesh.jacobian(U, g, R, V)
torch.cuda.synchronize()
S, NMAX = 24, 8192
buf = (ctypes.c_ulonglong * (NMAX * S))()
assert fo.lib().fo_debug_trace(buf, NMAX * S) == 0
tr = np.frombuffer(buf, dtype=np.uint64).reshape(NMAX, S).astype(np.int64)
L = fp.n_layers
npatch = int((tr[:, 1] > 0).sum())
tr = tr[:npatch]
t0 = tr[:, 1].min()
sm = tr[:, 0]
# intervals: A_k = [prev end, end of A_k], B_k = [end A_k, end B_k]
ev = []
for p in range(npatch):
    prev = tr[p, 1]
    for k in range(L + 1):
        a_end = tr[p, 2 + 2 * k] if k < L else tr[p, 2 + 2 * k - 1]
        if k < L:
            ev.append((sm[p], prev - t0, a_end - t0, "A"))
            b_end = tr[p, 3 + 2 * k]
            ev.append((sm[p], a_end - t0, b_end - t0, "B"))
            prev = b_end
        else:
            ev.append((sm[p], prev - t0, tr[p, 2 + 2 * L] - t0, "B"))
tot = {"AA": 0, "BB": 0, "AB": 0, "A": 0, "B": 0, "idle": 0}
span = max(e[2] for e in ev)
for s in np.unique(sm):
    es = [e for e in ev if e[0] == s]
    pts = sorted(set([e[1] for e in es] + [e[2] for e in es] + [0, span]))
    for a, b in zip(pts[:-1], pts[1:]):
        m = (a + b) / 2
        st = sorted(e[3] for e in es if e[1] <= m < e[2])
        key = "".join(st) if st else "idle"
        tot[key if key in tot else "AB"] = tot.get(key if key in tot else "AB", 0) + (b - a)
T = sum(tot.values())
print(f"patches {npatch}, span {span/1e3:.1f} us, per-SM time shares:",
      {k: f"{100*v/T:.1f}%" for k, v in tot.items()})
da = [tr[p, 2] - tr[p, 1] for p in range(npatch)]
dA = np.array([[tr[p, 2 + 2 * k] - (tr[p, 1 + 2 * k] if k else tr[p, 1]) for k in range(L)] for p in range(npatch)])
dB = np.array([[tr[p, 3 + 2 * k] - tr[p, 2 + 2 * k] for k in range(L)] for p in range(npatch)])
print(f"mean phase A {dA.mean()/1e3:.2f} us (first {dA[:,0].mean()/1e3:.2f}), mean phase B {dB.mean()/1e3:.2f} us, "
      f"patch lifetime {(tr[:, 2 + 2 * L] - tr[:, 1]).mean()/1e3:.1f} us")
