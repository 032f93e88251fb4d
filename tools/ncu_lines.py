"""Per-source-line totals of an ncu capture (needs -lineinfo builds):
instructions executed and warp-stall samples, hottest first.

usage: ncu -i rep.ncu-rep -k regex:KERNEL --page source --csv --print-source cuda,sass > x.csv
       python tools/ncu_lines.py x.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
items, fname = [], "?"
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit():
        try:
            items.append((int(r[7] or 0), int(r[4] or 0), fname, int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
te = sum(i[0] for i in items) or 1
ts = sum(i[1] for i in items) or 1
print(f"total warp instructions {te}, stall samples {ts}")
for e, s, f, ln, src in sorted(items, key=lambda x: -x[1])[:n]:
    print(f"{100 * e / te:5.1f}% inst {100 * s / ts:5.1f}% stall  {f}:{ln:<5} {src}")
