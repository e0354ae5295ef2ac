"""dynamic FP64 (DFMA/DMUL/DADD) and total warp-instructions per code section,
per wedge (dev tool).  usage: ... --print-source cuda,sass > s.csv; python tools/ncu_fp64_sections.py s.csv n_wedges"""
import csv
import re
import sys

sys.path.insert(0, "tools")
from ncu_sections import section  # noqa: E402

rows = list(csv.reader(open(sys.argv[1])))
nw = float(sys.argv[2])
cur, curline = "", 0
fp, tot = {}, {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            curline = int(r[0])
        except ValueError:
            pass
        continue
    if len(r) > 8 and r[0] == "" and r[2].startswith("0x"):
        try:
            ex = int(r[7])       # Instructions Executed (warp level)
        except ValueError:
            continue
        op = r[3].strip().split()
        opn = op[0] if op else ""
        if opn.startswith("@"):
            opn = op[1] if len(op) > 1 else ""
        k = section(cur, curline)
        tot[k] = tot.get(k, 0) + ex
        if re.match(r"D(FMA|MUL|ADD)", opn):
            fp[k] = fp.get(k, 0) + ex
T = sum(tot.values())
F = sum(fp.values())
print(f"per wedge: {32 * T / nw:.0f} thread-instr, {32 * F / nw:.0f} FP64 (DFMA/DMUL/DADD)")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:20]:
    print(f"{32 * v / nw:7.0f} instr  {32 * fp.get(k, 0) / nw:7.0f} fp64   {k}")
