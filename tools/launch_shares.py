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

# the R + J step alone (bench.py's timed unit at N = 1): the warp-specialised
# wedge kernel and the multi fix-up, per launch (the launch list also holds the
# warm-up, residual-only, graph, e2e and next-row kernels)
ws = [k for k in tot if k.endswith("ka_ws_kernel<1, 0>")]
fx = [k for k in tot if k.endswith("multi_fixup_kernel")]
if ws and fx:
    a = tot[ws[0]] / cnt[ws[0]]
    b = tot[fx[0]] / cnt[fx[0]]
    print(f"step (R + J, C3): {ws[0]} {a:.1f} us + {fx[0]} {b:.1f} us per step; "
          f"share of the dominant kernel {100 * a / (a + b):.2f}%")
