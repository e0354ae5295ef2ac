"""Build libfo.so in-tree: nvcc for sm_100a, C++17, -lineinfo.

    python -m paper_2204_04321_b200._build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import json
import os
import re
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libfo.so")
STAMP = os.path.join(LIB_DIR, "libfo.stamp.json")     # flags + compiler of the built library
PTXAS_LOG = os.path.join(LIB_DIR, "ptxas.txt")         # -Xptxas -v output (registers, spills)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    """NCCL headers and library shipped with the torch wheel (nvidia-nccl)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        inc = os.path.join(base, "nccl", "include")
        lib = os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel)")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _extra_flags():
    return os.environ.get("FO_EXTRA_NVCC_FLAGS", "").split()


def _nvcc_version():
    try:
        return subprocess.run([NVCC, "--version"], capture_output=True, text=True).stdout.strip().splitlines()[-1]
    except OSError:
        return "?"


def _stamp():
    return {"extra_flags": _extra_flags(), "nvcc": _nvcc_version(), "arch": ARCH}


def _stale():
    if not os.path.exists(LIB):
        return True
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "fo.h"), __file__]
    t = os.path.getmtime(LIB)
    if any(os.path.getmtime(d) > t for d in deps):
        return True
    # a library built with other flags (e.g. FO_EXTRA_NVCC_FLAGS experiment
    # switches) or another compiler is rebuilt, never silently reused
    try:
        return json.load(open(STAMP)) != _stamp()
    except (OSError, ValueError):
        return True


def ptxas_resources(kernel_substr: str):
    """(registers, spill stores + loads in bytes) of the first kernel whose
    mangled name contains kernel_substr, from the last build's ptxas -v log;
    None when unknown."""
    try:
        txt = open(PTXAS_LOG).read().splitlines()
    except OSError:
        return None
    for i, ln in enumerate(txt):
        if "Compiling entry function" in ln and kernel_substr in ln:
            regs = spill = None
            for ln2 in txt[i + 1:i + 6]:
                m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln2)
                if m:
                    spill = int(m.group(1)) + int(m.group(2))
                m = re.search(r"Used (\d+) registers", ln2)
                if m:
                    regs = int(m.group(1))
            return regs, spill
    return None


def _compile(src, inc):
    obj = os.path.join(LIB_DIR, os.path.basename(src) + ".o")
    extra = _extra_flags()
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", *extra, "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v",
           "-I", os.path.join(ROOT, "include"), "-I", inc, "-c", src, "-o", obj]
    if src.endswith(".cpp"):   # host code: the -D switches of FO_EXTRA_NVCC_FLAGS apply too
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-fvisibility=hidden", "-Wall",
               *[f for f in extra if f.startswith("-D")],
               "-I", os.path.join(ROOT, "include"), "-I", inc,
               "-I", os.path.join(os.path.dirname(os.path.dirname(NVCC)), "include"),
               "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, obj, r


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    inc, nlib = nccl_paths()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda src: _compile(src, inc), sources()))
    objs, log = [], []
    for src, obj, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        log.append(r.stderr)
        objs.append(obj)
    link = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-L", nlib, "-l:libnccl.so.2",
            "-Xlinker", "-rpath", "-Xlinker", nlib]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link of libfo.so failed")
    for o in objs:
        os.remove(o)
    with open(PTXAS_LOG, "w") as f:
        f.write("".join(log))
    with open(STAMP, "w") as f:
        json.dump(_stamp(), f)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
