"""stall samples of the KA-patch kernel grouped by code section (dev tool).
usage: ncu -i X --page source --csv --print-source cuda,sass > s.csv; python tools/ncu_sections.py s.csv"""
import csv
import re
import sys

src = {}
for f in ("paper_2204_04321_b200/csrc/fo_element_v4.cuh", "paper_2204_04321_b200/csrc/fo_owner.cu"):
    try:
        src[f.split("/")[-1]] = open(f).read().split("\n")
    except OSError:
        pass


def section(fname, ln):
    lines = src.get(fname)
    if not lines:
        return fname
    # nearest preceding marker comment "// ----" (element) or function name (owner)
    for i in range(min(ln, len(lines)) - 1, -1, -1):
        l = lines[i]
        if fname.endswith(".cuh") and ("// ----" in l or "if (w.go)" in l):
            return fname + ": " + l.strip()[:60]
        if fname.endswith(".cu") and re.match(r"^(template|__global__|__device__|struct|// phase|static)", l):
            return fname + ": " + l.strip()[:60]
    return fname



if __name__ == "__main__":
    rows = list(csv.reader(open(sys.argv[1])))
    cur = ""
    agg = {}
    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 6 and r[0] not in ("", "Line No") and r[2] == "-":
            try:
                s, ln = int(r[4]), int(r[0])
            except ValueError:
                continue
            k = section(cur, ln)
            agg[k] = agg.get(k, 0) + s
    tot = sum(agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:25]:
        print(f"{100 * v / tot:5.1f}%  {k}")


def stall_breakdown(path, want_file="fo_owner.cu"):
    """per section: samples split by stall reason (columns 31..47 of the SASS rows)."""
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    names = hdr[31:48]
    cur, curline, agg = "", 0, {}
    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 48 and r[0] not in ("", "Line No") and r[2] == "-":
            curline = int(r[0])
            continue
        if len(r) > 48 and r[0] == "" and r[2].startswith("0x"):
            k = section(cur, curline)
            d = agg.setdefault(k, [0] * len(names))
            for i in range(len(names)):
                try:
                    d[i] += int(r[31 + i])
                except ValueError:
                    pass
    for k, d in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:8]:
        tot = sum(d)
        top = sorted(zip(names, d), key=lambda x: -x[1])[:5]
        print(f"{tot:8d} {k[:70]}\n         " + ", ".join(f"{n[6:]} {100 * v / max(tot, 1):.0f}%" for n, v in top))
