"""aggregate ncu source-page stall samples per CUDA source line (dev tool).
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv; python tools/ncu_lines.py s.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur_file = ""
agg = {}
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) > 6 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            s = int(r[4])
        except ValueError:
            continue
        agg[(cur_file, int(r[0]))] = (s, r[1][:100])
tot = sum(v[0] for v in agg.values())
print("total samples", tot)
for (f, ln), (s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100*s/tot:5.1f}% {f}:{ln}  {src}")
