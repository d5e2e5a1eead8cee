"""Hottest SASS instructions (warp-stall samples) of one kernel in an
`ncu -i X.ncu-rep --page source --csv --print-source sass` export.

  python tools/sass_hot.py export.csv KERNEL_SUBSTR [top=25] [context=0]
"""
import csv
import sys

path, sub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
ctx = int(sys.argv[4]) if len(sys.argv) > 4 else 0
rows = list(csv.reader(open(path)))
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        sections.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
sec = next(s for s in sections if sub in s["name"])
hdr, data = sec["rows"][0], sec["rows"][1:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
num = lambda v: int(v) if v.isdigit() else 0
total = sum(num(r[iS]) for r in data)
print(sec["name"][:120], "samples", total)
agg = {}
for r in data:
    for i in stalls:
        agg[hdr[i]] = agg.get(hdr[i], 0) + num(r[i])
print("stall mix:", sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:8])
order = sorted(range(len(data)), key=lambda i: -num(data[i][iS]))[:top]
for i in sorted(order) if ctx else order:
    lo, hi = (i - ctx, i + 1) if ctx else (i, i + 1)
    for j in range(max(lo, 0), hi):
        r = data[j]
        st = sorted(((num(r[k]), hdr[k][6:]) for k in stalls), reverse=True)[:2]
        mark = "*" if j == i else " "
        print(f"{mark}{r[0][-5:]} {r[iS]:>5} {r[iE]:>8}  {r[1].strip()[:70]:70} {st}")
    if ctx:
        print()
