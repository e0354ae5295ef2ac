#!/usr/bin/env python
"""bench.py -- FO-Stokes residual + Newton-Jacobian assembly throughput on B200.

Metric (BASELINE.json): "FO-Stokes Jacobian+residual assembly Melem/s per GPU,
% HBM roofline, 1-8 GPU".  One step = one Total Fill of PAPER.md P:388:
fo_assemble_jacobian (R and J in one pass) at N = 1; at N > 1
fo_halo_import -> fo_assemble_jacobian_halo (assembly with the ghost-row sum
overlapped; --halo sequential: fo_assemble_jacobian then fo_halo_sum), on a
synthetic extruded Greenland-like mesh with 10 layers:
  N = 1: config C3 (1-10 km graded footprint sized to the paper's 479,930
         triangles), 4.8 M wedges;
  N > 1: config C4, the C3 recipe refined to N x 479,930 triangles, footprint
         partitioned into N Hilbert-contiguous parts (weak scaling), NCCL halo;
  --config C3 / C5 at N > 1: that mesh split into N parts (strong scaling,
         BASELINE.json's "C3 ... 1 and 8 B200" and "C5 ... 8 B200" configs).
value = all wedges of all ranks per second / 1e6 (Melem/s, whole job), timed
with CUDA events around every step (L2 flushed between steps, outside the
events), max over ranks; the line also carries the per-GPU figure (the
metric's "per GPU") and, at N > 1, the scaling efficiency of P:531-535 against
the one-GPU time of the base mesh measured in the same run.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config auto|C3|C4|C5] [--loopback P] [--halo fused|sequential]

--loopback P (N = 1): also time the P-part split of the workload on the one
GPU through the library's halo path (loopback transport), both the sequential
(fo_halo_import -> fo_assemble_jacobian -> fo_halo_sum on every part) and the
fused (fo_halo_import -> fo_assemble_jacobian_halo) step: the multi-GPU code
path end to end.

--impl reference runs the CPU oracle (oracle/, the serial C++ FE assembly the
CUDA path is validated against) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FO-Stokes Jacobian+residual assembly Melem/s per GPU, % HBM roofline, 1-8 GPU"
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 148 SMs x 64 FP64 FMA/clk x 2 x max clock


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scatter", type=int, default=0, choices=[0, 1, 2, 3],
                    help="0 owner-computes (default: the warp-specialised kernel), 1 atomic, 2 warp-specialised, 3 round-1 patch kernel")
    ap.add_argument("--cpu-sample-tris", type=int, default=40000, help="oracle sample per host core")
    ap.add_argument("--ref-sample-tris", type=int, default=3000, help="reference-arm sample per host core")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--config", default="auto", choices=["auto", "C3", "C4", "C5"],
                    help="auto: C3 at N = 1, C4 x N (weak) at N > 1; C3 / C5: strong scaling at N > 1")
    ap.add_argument("--loopback", type=int, default=0, help="N = 1: also time P parts through the halo path")
    ap.add_argument("--halo", choices=["fused", "sequential"], default="fused",
                    help="N > 1: fo_assemble_jacobian_halo (export overlapped with the interior patches, "
                         "default) or fo_assemble_jacobian then fo_halo_sum")
    ap.add_argument("--no-eta", action="store_true", help="N > 1: skip the one-GPU base run of the efficiency")
    ap.add_argument("--no-next-rows", action="store_true",
                    help="N = 1: skip the SURVEY.md 8(f) f4 lines (tetrahedra on C3, hexahedra 700 x 700 x 10)")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def workload(n_gpus: int, config: str = "auto"):
    """(footprint, config name, scaling, base config of the efficiency)"""
    from paper_2204_04321_b200 import meshgen as mg
    if config == "C5":
        return mg.antarctica_like(), "C5", ("strong" if n_gpus > 1 else "weak"), "C5"
    if config == "C3" or (config == "auto" and n_gpus == 1):
        return mg.greenland_like_1_10(), "C3", ("strong" if n_gpus > 1 else "weak"), "C3"
    return mg.greenland_like_1_10(scale=float(n_gpus)), f"C4x{n_gpus}", "weak", "C3"


def scaling_efficiency(t1_ms: float, n1: int, tn_ms: float, nn: int, n: int) -> float:
    """eta = ((t_1 / N_1) / (t_n / N_n)) / n, N = wedges
    (weak scaling: N_n = n N_1, perfect eta = 1 at t_n = t_1; strong scaling:
    N_n = N_1, perfect at t_n = t_1 / n)."""
    return (t1_ms / n1) / (tn_ms / nn) / n


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def kernel_src_hash() -> str:
    """sha256 (16 hex) of the CUDA/C++ sources and the build flags: an ncu
    capture summary carries the hash of the build it measured, and bench flags
    a capture taken on other kernel code."""
    import glob
    import hashlib
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2204_04321_b200", "csrc")
    for f in sorted(glob.glob(os.path.join(csrc, "*"))):
        if f.endswith((".cu", ".cuh", ".h", ".cpp")):
            h.update(os.path.basename(f).encode())
            h.update(open(f, "rb").read())
    h.update(os.environ.get("FO_EXTRA_NVCC_FLAGS", "").encode())
    return h.hexdigest()[:16]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except (FileNotFoundError, OSError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.2)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def algorithmic_bytes(n_elem, nnz, n_nodes, n_cols, n_tri, has_A):
    """J values written once, R written, U read, column
    records (x, y, s, H, beta), triangle connectivity, per-wedge A if a field."""
    return 8 * nnz + 16 * n_nodes + 16 * n_nodes + 40 * n_cols + 12 * n_tri + (8 * n_elem if has_A else 0)


# the R + J assembly kernel each --scatter mode launches (name in the ncu
# launch list, mangled-name fragment in the ptxas log)
DOMINANT_KERNEL = {0: ("ka_ws_kernel", "ka_ws_kernelILb1E"), 1: ("assemble_atomic_kernel", "assemble_atomic_kernelILb1ELb1E"),
                   2: ("ka_ws_kernel", "ka_ws_kernelILb1E"), 3: ("ka_patch_kernel", "ka_patch_kernelILb1ELb1ELb0E")}


def ncu_summary(config_name, kernel_name=None):
    """dram traffic / fp64 counts of the dominant kernel from the committed ncu
    capture; `matches_build` says whether it was taken on these kernel sources."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    if d.get("config") != config_name:
        return None
    if kernel_name is not None and kernel_name not in d.get("kernel", ""):
        return None   # a capture of another kernel says nothing about this one
    d["matches_build"] = d.get("src_hash") == kernel_src_hash()
    return d


def roofline_entry(alg_bytes, kernel_ms, kernel_ms_total, step_ms_total, n_elems, peak_gbs, peak_src, prof,
                   kernel_name):
    """the bench line's `roofline` object for the dominant kernel: HBM fraction
    of the algorithmic bytes per launch, FP64 fraction of the ncu-counted flops
    (committed capture `prof`, may be None), and the binding roof.  When the
    binding roof is FP64 (plain fp64 ALU arithmetic, no tensor cores: DESIGN.md
    section 7) the object reports "bound": "alu" against the derived FP64 peak
    and keeps the metric's HBM fraction under "hbm"."""
    achieved = alg_bytes / (kernel_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak_gbs, "unit": "GB/s", "frac": achieved / peak_gbs,
            "traffic": prof.get("dram_bytes_per_launch") if prof else None, "kernel": kernel_name,
            "kernel_ms": kernel_ms, "kernel_share_of_step": kernel_ms_total / max(step_ms_total, 1e-12),
            "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peak_src,
            "bytes_formula": "8 nnz + 32 N_nodes + 40 N_cols + 12 N_tri (SURVEY.md 8(d) d3)"}
    fpw = prof.get("fp64_flop_per_wedge") if prof else None
    if fpw:
        tfl = fpw * n_elems / (kernel_ms / 1e3) / 1e12
        fp64 = {"achieved": tfl, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": tfl / FP64_PEAK_TFLOPS,
                "flop_per_wedge": fpw, "peak_source": "derived: 148 SM x 64 DFMA/clk x 2 x 1.965 GHz",
                "flop_source": prof.get("source")}
        binding = "fp64" if fp64["frac"] > roof["frac"] else "hbm"
        roof["min_roof"] = {"binding": binding, "frac": max(fp64["frac"], roof["frac"])}
        if binding == "fp64":
            hbm = {k: roof.pop(k) for k in ("achieved", "peak", "unit", "frac", "peak_source", "bytes_formula",
                                            "algorithmic_bytes_per_launch")}
            roof.pop("bound")
            roof = {"bound": "alu", "achieved": fp64["achieved"], "peak": fp64["peak"], "unit": "TFLOP/s",
                    "frac": fp64["frac"], "traffic": roof.pop("traffic"), **roof,
                    "flop_per_wedge": fpw, "peak_source": fp64["peak_source"],
                    "flop_source": fp64["flop_source"], "hbm": hbm}
        else:
            roof["fp64"] = fp64
    if prof:
        roof["ncu"] = {k: prof.get(k) for k in ("fp64_pipe_pct", "registers_per_thread", "warps_active_pct",
                                                 "l1_data_pipe_pct", "shared_wavefronts", "shared_bank_conflicts",
                                                 "l2_red_sectors_per_s", "src_hash", "matches_build")
                       if prof.get(k) is not None}
        if not prof.get("matches_build", False):
            roof["ncu"]["stale"] = ("capture taken on other kernel sources: flop_per_wedge and traffic "
                                    "are the captured build's")
    return roof


def _host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


_FORK_FP = None   # the workload, inherited by the forked oracle processes


def _oracle_worker(args):
    """one process: the oracle's R + Dual<12> Jacobian on one Hilbert-contiguous
    part of the sample (graph built untimed), `reps` timed calls after a common
    start barrier; returns the seconds of each call."""
    t0, t1, reps, barrier = args
    fp = _FORK_FP
    from oracle import oracle as ora
    from paper_2204_04321_b200 import meshgen as mg
    sub = mg.sub_footprint(fp, t0, t1)
    o = ora.Oracle(sub)
    o.graph()
    barrier.wait()
    out = []
    for _ in range(reps):
        a = time.perf_counter()
        o.jacobian(sub.U)
        out.append(time.perf_counter() - a)
    return out


def oracle_parallel(fp, n_tri_sample, procs, reps=1):
    """SURVEY.md 8(d) d5 (all cores): P processes, one per host core, each
    assembling one Hilbert-contiguous part of the sample (the paper's MPI
    rank per core); per call the slowest process's time counts.
    Returns (seconds per call for each rep, sample triangles, wedges)."""
    import multiprocessing as mp
    from oracle import oracle as ora
    global _FORK_FP
    ora.build()
    _FORK_FP = fp
    nt = min(n_tri_sample, fp.n_tri)
    procs = max(1, min(procs, nt))
    ctx = mp.get_context("fork")
    barrier = ctx.Manager().Barrier(procs)
    bounds = [(i * nt) // procs for i in range(procs + 1)]
    with ctx.Pool(procs) as pool:
        res = pool.map(_oracle_worker, [(bounds[i], bounds[i + 1], reps, barrier) for i in range(procs)], chunksize=1)
    per_rep = [max(r[k] for r in res) for k in range(reps)]
    return per_rep, nt, nt * fp.n_layers


ORACLE_COMPILER = "g++ -O2 -std=c++17 (no fast-math, no threads), oracle/fo_oracle.cpp"


def cpu_baseline_oracle(fp, n_tri_sample_per_core, one_core_tris=6000):
    """The oracle as it stands (serial C++ per process, Dual<12> AD Jacobian) on
    every host core: a sample of n_tri_sample_per_core triangles per core (the
    whole workload if smaller), split into Hilbert-contiguous parts; plus the
    1-core figure of SURVEY.md 8(d) d5 (one process, median of 3 calls after a
    warm-up, on the first one_core_tris triangles)."""
    cores = _host_cores()
    secs, nt, nw = oracle_parallel(fp, n_tri_sample_per_core * cores, cores)
    dt = secs[0]
    s1, nt1, nw1 = oracle_parallel(fp, one_core_tris, 1, reps=4)
    t1 = statistics.median(s1[1:])
    return {"value": nw / dt / 1e6, "unit": "Melem/s", "cores": cores, "kind": "oracle",
            "sample": f"first {nt} triangles x {fp.n_layers} layers = {nw} wedges of {fp.name}, split into "
                      f"{cores} Hilbert-contiguous parts, one oracle process per core (R + Dual<12> AD "
                      f"Jacobian, -O2); wall time of the slowest process {dt:.2f} s",
            "seconds": dt,
            "one_core": {"value": nw1 / t1 / 1e6, "unit": "Melem/s", "cores": 1,
                         "sample": f"first {nt1} triangles x {fp.n_layers} layers = {nw1} wedges, one process, "
                                   f"median of 3 calls after a warm-up", "seconds": t1},
            "cpu_model": cpu_model(), "compiler": ORACLE_COMPILER}


def small_config_lines(dev, flush, stream):
    """SURVEY.md 8(d) d5 per config: the small configurations C1 (ISMIP-HOM A,
    4 000 wedges) and C2 (Greenland-like 16 km, ~300 k wedges) -- one R + J
    assembly on the GPU (median of 10 after warm-up, CUDA events) and one
    whole-config oracle evaluation on ONE host core (median of 2 after a warm-up
    for C1, one evaluation for C2)."""
    import torch
    from paper_2204_04321_b200 import fo, meshgen as mg
    out = {}
    for name, make, reps in (("C1", mg.ismip_hom_a, 3), ("C2", lambda: mg.greenland_like(16.0), 1)):
        fpc = make()
        m = fo.Mesh.from_footprint(fpc, device=dev.index)
        g = m.graph()
        U = torch.tensor(fpc.U, device=dev)
        R = torch.empty(m.n_dofs, dtype=torch.float64, device=dev)
        V = torch.empty(g.nnz, dtype=torch.float64, device=dev)
        for _ in range(3):
            m.jacobian(U, g, R, V)
        ms = statistics.median(time_steps(lambda: m.jacobian(U, g, R, V), 10, flush, stream))
        secs, nt, nw = oracle_parallel(fpc, fpc.n_tri, 1, reps=reps)
        t1 = statistics.median(secs[1:] if reps > 1 else secs)
        out[name] = {"wedges": fpc.n_elem, "gpu_ms": ms, "gpu_Melem_s": fpc.n_elem / ms / 1e3,
                     "oracle_1core_s": t1, "oracle_1core_Melem_s": nw / t1 / 1e6}
        m.close()
    return out


def run_reference(args):
    """--impl reference: the CPU oracle timed on the host cores (rank 0 only),
    one process per core on a Hilbert-contiguous split of a bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    fp, name, scaling, _ = workload(args.gpus, args.config)
    cores = _host_cores()
    secs, nt, nw = oracle_parallel(fp, args.ref_sample_tris * cores, cores, reps=args.warmup + args.steps)
    times = secs[args.warmup:]
    tot = sum(times)
    value = nw * args.steps / tot / 1e6
    sample = (f"{nw} wedges per step (first {nt} triangles of {fp.name}) split over {cores} host cores, "
              f"one oracle process per core, R + Dual<12> AD Jacobian")
    line = {"metric": METRIC, "value": value, "unit": "Melem/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{name}: {fp.name}, sample of {nt} triangles x {fp.n_layers} layers",
                       "n_elem": nw},
            "cpu_baseline": {"value": value, "unit": "Melem/s", "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model(), "compiler": ORACLE_COMPILER},
            "e2e": {"value": value, "unit": "Melem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def time_steps(step, steps, flush, stream):
    """CUDA-event time of each of `steps` calls of step() on `stream`, the L2
    flushed (512 MB written) before each, outside the events; ms per step."""
    import torch
    evs = []
    for _ in range(steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def single_gpu_base(fp, steps, warmup, dev, flush, stream):
    """the one-GPU time of the efficiency's base mesh (single domain, same protocol)"""
    import torch
    from paper_2204_04321_b200 import fo
    m = fo.Mesh.from_footprint(fp, device=dev.index)
    g = m.graph()
    U = torch.tensor(fp.U, dtype=torch.float64, device=dev)
    R = torch.empty(m.n_dofs, dtype=torch.float64, device=dev)
    V = torch.empty(g.nnz, dtype=torch.float64, device=dev)
    for _ in range(max(warmup, 3)):
        m.jacobian(U, g, R, V)
    ms = time_steps(lambda: m.jacobian(U, g, R, V), steps, flush, stream)
    n = m.n_elems
    del R, V, U, g
    m.close()
    return sum(ms) / len(ms), n


def loopback_run(fp, P, steps, warmup, dev, flush, stream):
    """--loopback P: the workload split into P parts on this one GPU, every
    step = fo_halo_import on every part -> fo_assemble_jacobian on every part
    -> fo_halo_sum on every part (loopback transport: the library's halo plans,
    staging, gather / unpack-add kernels; device copies for the transfers)."""
    import torch
    from paper_2204_04321_b200 import fo
    L1 = fp.n_layers + 1
    part = fo.partition(fp.n_tri, P)
    meshes = [fo.Mesh.from_footprint(fp, device=dev.index, part=part, my_part=p, n_parts=P) for p in range(P)]
    halos = fo.Halo.loopback(meshes)
    Ug = fp.U.reshape(fp.n_vert, L1, 2)
    st = []
    for m in meshes:
        g = m.graph()
        st.append((m, g, torch.tensor(Ug[m.columns()[0]].reshape(-1), device=dev),
                   torch.empty(m.n_dofs, dtype=torch.float64, device=dev),
                   torch.empty(g.nnz, dtype=torch.float64, device=dev)))

    def step_seq():
        for h, (m, g, U, R, V) in zip(halos, st):
            h.import_(U)
        for m, g, U, R, V in st:
            m.jacobian(U, g, R, V)
        for h, (m, g, U, R, V) in zip(halos, st):
            h.sum(R, V)

    def step_fused():
        for h, (m, g, U, R, V) in zip(halos, st):
            h.import_(U)
        for h, (m, g, U, R, V) in zip(halos, st):
            h.assemble(U, R, V)

    res = {}
    for name, step in (("sequential", step_seq), ("fused", step_fused)):
        for _ in range(max(warmup, 3)):
            step()
        ms = time_steps(step, steps, flush, stream)
        t = sum(ms) / len(ms)
        res[name] = {"ms_per_step": t, "value": fp.n_elem / (t / 1e3) / 1e6}
    recv = [h.info() for h in halos]
    out = {"parts": P, "ms_per_step": res["fused"]["ms_per_step"], "value": res["fused"]["value"],
           "unit": "Melem/s", "sequential": res["sequential"], "fused": res["fused"],
           "halo_values_received_per_step": int(sum(r[1] + r[2] for r in recv)),
           "max_neighbours": int(max(r[0] for r in recv)),
           "note": "P parts of the workload on one GPU with the loopback transport (the multi-GPU code path, "
                   "one device): sequential = fo_halo_import -> fo_assemble_jacobian -> fo_halo_sum on every "
                   "part; fused = fo_halo_import -> fo_assemble_jacobian_halo (ghost rows sent while the "
                   "interior patches run)"}
    for h in halos:
        h.close()
    for m, g, U, R, V in st:
        m.close()
    return out


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    from paper_2204_04321_b200 import _build, fo

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        _build.build()
    if world > 1:
        dist.barrier()

    fp, cfg_name, scaling, base_cfg = workload(world, args.config)
    L = fp.n_layers
    if world == 1:
        mesh = fo.Mesh.from_footprint(fp, device=local)
        U_local = fp.U
        halo = None
    else:
        part = fo.partition(fp.n_tri, world)
        mesh = fo.Mesh.from_footprint(fp, device=local, part=part, my_part=rank, n_parts=world)
        glob = mesh.columns()[0]
        U_local = fp.U.reshape(fp.n_vert, L + 1, 2)[glob].reshape(-1)
        obj = [fo.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        halo = fo.Halo(mesh, obj[0], rank, world)
    mesh.set_scatter(args.scatter)
    graph = mesh.graph()
    glob, nA, nB, nC = mesh.columns()
    n_cols = nA + nB
    n_tri_local = mesh.n_elems // L
    U = torch.tensor(U_local, dtype=torch.float64, device=dev)
    R = torch.empty(mesh.n_dofs, dtype=torch.float64, device=dev)
    V = torch.empty(graph.nnz, dtype=torch.float64, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=dev)   # 512 MB > 126 MB L2
    stream = torch.cuda.current_stream()

    def step():
        if halo is None:
            mesh.jacobian(U, graph, R, V)
            return
        halo.import_(U)
        if args.halo == "fused":   # fo_assemble_jacobian_halo: ghost rows sent while the interior runs
            halo.assemble(U, R, V)
        else:
            mesh.jacobian(U, graph, R, V)
            halo.sum(R, V)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    launches_per_step = mesh.last_launch_count()
    if halo is not None:
        nn, _, _ = halo.info()
        launches_per_step += 4 * nn   # gather + scatter-add kernels of the halo (upper bound)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    mesh.kernel_timing(True)
    evs = []
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for _ in range(args.steps):
        flush.zero_()                        # evict inputs from L2 (outside the timed span)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    mesh.kernel_timing(False)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    kern_ms, kern_n = mesh.kernel_time_ms()
    tot_ms = sum(step_ms)
    elems = mesh.n_elems
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        e = torch.tensor([elems], dtype=torch.float64, device=dev)
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
        elems = int(e.item())
    value = elems * args.steps / (tot_ms / 1e3) / 1e6

    # roofline of the dominant kernel (ka_patch_kernel), this rank
    peak, peak_src = measured_peaks()
    has_A = fp.A_elem is not None
    alg = algorithmic_bytes(mesh.n_elems, graph.nnz, mesh.n_nodes, n_cols, n_tri_local, has_A)
    # per STEP: a fused halo step (N > 1) launches the kernel twice (boundary
    # and interior patches), each over part of the patches
    kavg = kern_ms / max(args.steps, 1)
    kname, ksym = DOMINANT_KERNEL[args.scatter]
    prof = ncu_summary(cfg_name, kname)
    roof = roofline_entry(alg, kavg, kern_ms, sum(step_ms), mesh.n_elems, peak, peak_src, prof, kname)
    res = _build.ptxas_resources(ksym)
    if res is not None:
        roof["ptxas"] = {"registers_per_thread": res[0], "spill_bytes": res[1], "source": "ptxas -v of this build"}

    # residual only (KR), the same timing protocol
    r_ms = []
    for _ in range(max(args.warmup, 3)):
        mesh.residual(U, R)
    for _ in range(args.steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        if halo is None:
            mesh.residual(U, R)
        elif args.halo == "fused":
            halo.import_(U)
            halo.assemble(U, R)
        else:
            halo.import_(U)
            mesh.residual(U, R)
            halo.sum(R, None)
        b.record(stream)
        r_ms.append((a, b))
    torch.cuda.synchronize()
    r_tot = sum(a.elapsed_time(b) for a, b in r_ms)
    if world > 1:
        t = torch.tensor([r_tot], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        r_tot = float(t.item())
    r_bytes = 32 * mesh.n_nodes + 40 * n_cols + 12 * n_tri_local
    residual_only = {"value": elems * args.steps / (r_tot / 1e3) / 1e6, "unit": "Melem/s",
                     "ms_per_step": r_tot / args.steps,
                     "hbm_frac": r_bytes / (r_tot / args.steps / 1e3) / 1e9 / peak,
                     "bytes_formula": "32 N_nodes + 40 N_cols + 12 N_tri (U read, R written, geometry)"}

    # the paper's timed unit, 100 R + J evaluations captured in
    # one CUDA graph (N = 1; no L2 flush inside: the 1.7 GB of values exceed L2)
    graph100 = None
    if world == 1:
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        with torch.cuda.stream(gs):
            mesh.jacobian(U, graph, R, V)
        stream.wait_stream(gs)
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg):
            for _ in range(100):
                mesh.jacobian(U, graph, R, V)
        cg.replay()
        torch.cuda.synchronize()
        reps = []
        for _ in range(3):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            cg.replay()
            b.record(stream)
            b.synchronize()
            reps.append(a.elapsed_time(b))
        g_ms = statistics.median(reps)
        graph100 = {"evaluations": 100, "ms": g_ms, "ms_per_eval": g_ms / 100,
                    "value": mesh.n_elems * 100 / (g_ms / 1e3) / 1e6, "unit": "Melem/s",
                    "note": "median of 3 replays of one CUDA graph of 100 fo_assemble_jacobian calls"}
        del cg

    # end to end through the C ABI with host buffers (pinned)
    e2e = None
    if world == 1 and args.e2e_steps > 0:
        Uh = torch.tensor(U_local, dtype=torch.float64).pin_memory()
        Rh = torch.empty(mesh.n_dofs, dtype=torch.float64).pin_memory()
        Vh = torch.empty(graph.nnz, dtype=torch.float64).pin_memory()
        mesh.jacobian_host(Uh, Rh, Vh, graph)          # warm-up (staging allocation)
        tms = []
        for _ in range(args.e2e_steps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            mesh.jacobian_host(Uh, Rh, Vh, graph)
            b.record(stream)
            b.synchronize()
            tms.append(a.elapsed_time(b))
        e2e = {"value": mesh.n_elems * len(tms) / (sum(tms) / 1e3) / 1e6, "unit": "Melem/s",
               "h2d_bytes_per_step": 8 * mesh.n_dofs, "d2h_bytes_per_step": 8 * (mesh.n_dofs + graph.nnz),
               "api": "fo_assemble_jacobian_host (pinned host U in, R and CSR values out)"}
    elif world > 1 and args.e2e_steps > 0:
        n_owned = mesh.n_owned_dofs
        owned_vals = int(graph.row_ptr_host()[n_owned])
        Uh = torch.tensor(U_local[:n_owned], dtype=torch.float64).pin_memory()
        Rh = torch.empty(n_owned, dtype=torch.float64).pin_memory()
        Vh = torch.empty(owned_vals, dtype=torch.float64).pin_memory()
        tms = []
        for _ in range(args.e2e_steps):
            dist.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            U[:n_owned].copy_(Uh, non_blocking=True)
            step()
            Rh.copy_(R[:n_owned], non_blocking=True)
            Vh.copy_(V[:owned_vals], non_blocking=True)
            b.record(stream)
            b.synchronize()
            tms.append(a.elapsed_time(b))
        t = torch.tensor([sum(tms)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": elems * len(tms) / (float(t.item()) / 1e3) / 1e6, "unit": "Melem/s",
               "h2d_bytes_per_step": 8 * n_owned, "d2h_bytes_per_step": 8 * (n_owned + owned_vals),
               "api": "torch H2D of owned U -> fo_halo_import -> fo_assemble_jacobian_halo (or fo_assemble_jacobian + "
                      "fo_halo_sum with --halo sequential) -> D2H owned rows"}

    # N > 1: the efficiency of P:531-535 against the base mesh on one GPU, timed
    # by rank 0 in this run with the same protocol (C3 for the weak series)
    eta = None
    if world > 1 and not args.no_eta:
        dist.barrier()
        if rank == 0:
            from paper_2204_04321_b200 import meshgen as mg
            fb = fp if base_cfg == cfg_name else (mg.greenland_like_1_10() if base_cfg == "C3" else mg.antarctica_like())
            t1, n1 = single_gpu_base(fb, args.steps, args.warmup, dev, flush, stream)
            tn = tot_ms / args.steps
            eta = {"eta": scaling_efficiency(t1, n1, tn, elems, world), "scaling": scaling,
                   "t1_ms": t1, "n1_wedges": n1, "tn_ms": tn, "nn_wedges": elems, "n": world,
                   "base": f"{base_cfg} single domain on GPU 0 of this run",
                   "formula": "((t1/N1)/(tn/Nn))/n, N = wedges (PAPER.md P:531-535)"}
        dist.barrier()

    # SURVEY.md 8(f) f4 at N = 1 (not part of the step): R + J with three P1
    # tetrahedra per prism on the same C3 mesh, and 8-node hexahedra on a
    # 700 x 700 quad footprint x 10 layers (4.9 M elements, 548 M nonzeros);
    # device time per assembly with the step's protocol (median, L2 flushed)
    next_rows = None
    if world == 1 and not args.no_next_rows:
        def med_ms(fn, n=7):
            for _ in range(3):
                fn()
            out = []
            for _ in range(n):
                flush.fill_(0.5)
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                b.synchronize()
                out.append(a.elapsed_time(b))
            return statistics.median(out)
        from paper_2204_04321_b200 import meshgen as mg
        mesh.set_element(1)
        t_ms = med_ms(lambda: mesh.jacobian(U, graph, R, V))
        mesh.set_element(0)
        fq = mg.to_quads(mg.ismip_hom_a(nx=700, n_layers=10), 700)
        mq = fo.Mesh.from_footprint(fq, device=dev.index)
        gq = mq.graph()
        Uq = torch.tensor(fq.U, device=dev)
        Rq = torch.empty(mq.n_dofs, dtype=torch.float64, device=dev)
        Vq = torch.empty(gq.nnz, dtype=torch.float64, device=dev)
        h_ms = med_ms(lambda: mq.jacobian(Uq, gq, Rq, Vq))
        next_rows = {
            "f4_tet3": {"elements": 3 * mesh.n_elems, "ms": t_ms, "value": 3 * mesh.n_elems / t_ms / 1e3,
                        "unit": "Melem/s", "workload": "C3, three P1 tetrahedra per prism (reading L22)"},
            "f4_hex8": {"elements": mq.n_elems, "nnz": gq.nnz, "ms": h_ms, "value": mq.n_elems / h_ms / 1e3,
                        "unit": "Melem/s", "workload": "700 x 700 quads x 10 layers, 8-node trilinear hexahedra "
                                                       "(reading L23)"},
            "note": "R + J device time per assembly, median of 7 after 3 warm-ups, 512 MB written before each"}
        del mq, gq, Uq, Rq, Vq

    loop = None
    if world == 1 and args.loopback > 1:
        loop = loopback_run(fp, args.loopback, args.steps, args.warmup, dev, flush, stream)
        loop["vs_single_domain"] = (tot_ms / args.steps) / loop["ms_per_step"]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_oracle(fp, args.cpu_sample_tris)
        cpu["per_config"] = small_config_lines(dev, flush, stream)

    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Melem/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded " + ("Antarctica" if cfg_name == "C5" else "Greenland") +
                    "-like footprint, SIA velocity; SURVEY.md 8(d) d1)",
            "per_gpu": {"value": value / world, "unit": "Melem/s per GPU",
                        "note": "the metric's per-GPU figure (value = whole job over all GPUs)"},
            "scaling_efficiency": eta, "loopback": loop,
            "build": {"src_hash": kernel_src_hash(), "extra_nvcc_flags": os.environ.get("FO_EXTRA_NVCC_FLAGS", ""),
                      "seed": "meshgen SplitMix64 defaults (C3 seed 1, C5 seed 2)"},
            "config": {"workload": f"{cfg_name}: {fp.name}, {fp.n_tri} triangles x {L} layers = "
                                   f"{fp.n_elem} wedges, {world} part(s)",
                       "wedges_per_gpu": mesh.n_elems, "nnz_per_gpu": graph.nnz, "n_dofs_per_gpu": mesh.n_dofs,
                       "parallelism": f"footprint partition x{world}" + (f", NCCL halo ({args.halo})" if world > 1 else ""),
                       "config": cfg_name,
                       "scatter": {0: "owner-computes", 1: "atomic", 2: "owner-computes (ws)", 3: "owner-computes (round-1 kernel)"}[args.scatter],
                       "l2": "1.7 GB of CSR values written per step (> 126 MB L2) and a 512 MB buffer "
                             "written between timed steps"},
            "roofline": roof, "residual_only": residual_only, "graph_100": graph100, "next_rows": next_rows,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk, "cpu_baseline": cpu,
            "per_step_ms": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
