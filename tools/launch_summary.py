"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel count, total and mean time, and share of the listed time.

  python tools/launch_summary.py launches.csv [--skip N] [--last N]
"""
import csv
import re
import sys
from collections import OrderedDict


def short(name):
    if name.startswith("void "):
        name = name[5:]
    return re.sub(r"\(.*$", "", name)[:110]


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else 0
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        t = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "usecond":
            t *= 1e3
        elif r["Metric Unit"] == "msecond":
            t *= 1e6
        rows.append((short(r["Kernel Name"]), r["Grid Size"], t))
    rows = rows[skip:]
    if last:
        rows = rows[-last:]
    agg = OrderedDict()
    for n, g, t in rows:
        c, s = agg.get((n, g), (0, 0.0))
        agg[(n, g)] = (c + 1, s + t)
    total = sum(s for _, s in agg.values())
    print(f"{'kernel':<112} {'grid':>14} {'n':>4} {'mean us':>9} {'share':>6}")
    for (n, g), (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n:<112} {g:>14} {c:>4} {s / c / 1e3:>9.2f} {100 * s / total:>5.1f}%")
    print(f"total {total / 1e3:.1f} us over {len(rows)} launches")


if __name__ == "__main__":
    main()
