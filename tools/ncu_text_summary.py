"""human-readable summary of one ncu --set full capture (dev tool).
usage: python tools/ncu_text_summary.py X.ncu-rep > profiles/<tag>_ncu_summary.txt"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
d = dict(zip(r[0], r[2]))
u = dict(zip(r[0], r[1]))
keys = [
    "Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
]
for k in keys:
    if k in d:
        print(f"{k:75s} {d[k]:>22s} {u.get(k, '')}")
st = {k: float(v.replace(",", "")) for k, v in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v}
tot = sum(st.values())
print("\nwarp stall samples (share of all samples):")
for k, v in sorted(st.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * v / tot:5.1f}%")
