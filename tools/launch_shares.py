"""summarise an ncu --metrics gpu__time_duration.sum launch list (dev tool)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    name = r[4].split("(")[0]
    tot[name] += float(r[14]) / 1e3
    cnt[name] += 1
allt = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{100*v/allt:6.2f}%  {v/cnt[k]:10.1f} us/launch  x{cnt[k]:3d}  {k}")
