"""Per-rank device time of the partitioned assembly on ONE GPU (dev tool):
for N in the arguments, build the C4xN footprint (the weak-scaling workload of
bench.py), create the part mesh of rank r (default 0 and N-1) and time
fo_assemble_jacobian on it (CUDA events, median of 10).  Without the NCCL
exchange, this is what each rank computes per step at N GPUs.
usage: python tools/part_time.py 2 4 8 > profiles/<tag>_part_times.jsonl"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_04321_b200 import fo, meshgen as mg  # noqa: E402


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


for arg in sys.argv[1:]:
    N = int(arg)
    t0 = time.time()
    fp = mg.greenland_like_1_10(scale=float(N))
    gen_s = time.time() - t0
    part = fo.partition(fp.n_tri, N)
    for r in sorted({0, N - 1}):
        t0 = time.time()
        mesh = fo.Mesh.from_footprint(fp, part=part, my_part=r, n_parts=N)
        g = mesh.graph()
        setup_s = time.time() - t0
        glob, nA, nB, nC = mesh.columns()
        L = fp.n_layers
        U = torch.tensor(fp.U.reshape(fp.n_vert, L + 1, 2)[glob].reshape(-1), device="cuda")
        R = torch.empty(mesh.n_dofs, dtype=torch.float64, device="cuda")
        V = torch.empty(g.nnz, dtype=torch.float64, device="cuda")
        ms = timeit(lambda: mesh.jacobian(U, g, R, V))
        print(json.dumps({"workload": f"C4x{N}", "rank": r, "n_parts": N, "wedges": mesh.n_elems,
                          "owned_cols": nA, "ghost_cols": nB, "coupling_only_cols": nC, "nnz": g.nnz,
                          "ms": round(ms, 4), "Melem_s": round(mesh.n_elems / ms / 1e3, 1),
                          "gen_s": round(gen_s, 1), "setup_s": round(setup_s, 1)}), flush=True)
        del mesh, g, U, R, V
        torch.cuda.empty_cache()
