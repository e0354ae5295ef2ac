"""write profiles/ncu_summary.json from one ncu --set full capture of the
assembly kernel (dram traffic per launch, FP64 flops per wedge from the SASS
thread-instruction counts; DFMA = 2 flops).
usage: python tools/ncu_summary.py X.ncu-rep CONFIG N_WEDGES [out.json]"""
import csv
import io
import json
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (kernel_src_hash: the capture records the build it measured)

rep, cfg, nw = sys.argv[1], sys.argv[2], float(sys.argv[3])
out = sys.argv[4] if len(sys.argv) > 4 else "profiles/ncu_summary.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]


def metric(name):
    i = h.index(name)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[i], 1)
    return float(v[i]) * scale


src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(x for x in rows if "Source" in x and "Thread Instructions Executed" in x)
si, ti = hdr.index("Source"), hdr.index("Thread Instructions Executed")
cnt = {"DFMA": 0, "DADD": 0, "DMUL": 0}
for x in rows:
    if len(x) > ti and x is not hdr:
        m = re.search(r"\b(DFMA|DADD|DMUL)\b", x[si])
        if m:
            try:
                cnt[m.group(1)] += int(x[ti])
            except ValueError:
                pass
flops = 2 * cnt["DFMA"] + cnt["DADD"] + cnt["DMUL"]
d = {"config": cfg, "kernel": h and v[h.index("Kernel Name")] if "Kernel Name" in h else "",
     "source": f"ncu --set full capture {rep.split('/')[-1]}",
     "gpu_time_ms": metric("gpu__time_duration.sum") / 1e6 if u[h.index("gpu__time_duration.sum")] == "nsecond"
     else float(v[h.index("gpu__time_duration.sum")]),
     "dram_bytes_read": metric("dram__bytes_read.sum"), "dram_bytes_write": metric("dram__bytes_write.sum"),
     "fp64_instr_per_wedge": {k: c / nw for k, c in cnt.items()},
     "fp64_flop_per_wedge": flops / nw}
d["dram_bytes_per_launch"] = d["dram_bytes_read"] + d["dram_bytes_write"]
d["src_hash"] = bench.kernel_src_hash()
try:
    d["git_head"] = subprocess.run(["git", "rev-parse", "--short=12", "HEAD"], capture_output=True,
                                   text=True).stdout.strip() or None
except OSError:
    d["git_head"] = None


def raw(name):
    return float(v[h.index(name)].replace(",", "")) if name in h else None


# SURVEY.md 8(d) d4 report items
d["fp64_pipe_pct"] = raw("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed")
d["registers_per_thread"] = raw("launch__registers_per_thread")
d["warps_active_pct"] = raw("sm__warps_active.avg.pct_of_peak_sustained_active")
d["l1_data_pipe_pct"] = raw("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed")
d["shared_wavefronts"] = raw("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
d["shared_bank_conflicts"] = raw("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
red = raw("lts__t_sectors_srcunit_tex_op_red.sum")
d["l2_red_sectors"] = red
if red is not None:
    d["l2_red_sectors_per_s"] = red / (d["gpu_time_ms"] / 1e3)
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d, indent=1))
