"""where do STL/LDL (register spills) sit? innermost source line per spill (dev tool).
usage: nvdisasm -gi x.cubin > x.sass; python tools/spill_lines.py x.sass <kernel-substring>"""
import re
import sys

lines = open(sys.argv[1]).read().split("\n")
pat = sys.argv[2]
start = next(i for i, l in enumerate(lines) if ".section" in l and ".text." in l and pat in l)
cur, cnt, fresh = None, {}, True
for l in lines[start + 1:]:
    if ".section" in l and ".text." in l:
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if fresh:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
        fresh = False
        continue
    if "/*" in l and ";" in l:
        fresh = True
        if "STL" in l or "LDL" in l:
            key = (cur, "STL" if "STL" in l else "LDL")
            cnt[key] = cnt.get(key, 0) + 1
for k, v in sorted(cnt.items(), key=lambda kv: -kv[1])[:40]:
    print(v, k)
