"""Key metrics of an `ncu --set full` capture exported with
`ncu -i X.ncu-rep --page raw --csv` (one row per profiled launch).

  python tools/ncu_summary.py raw.csv [--json traffic.json --key NAME --match SUBSTR]
"""
import csv
import json
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % elapsed"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % active"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    traffic = {}
    for v in vals:
        name = v[idx["Kernel Name"]]
        print(f"== {name[:150]}  grid {v[idx['Grid Size']]} block {v[idx['Block Size']]}")
        for m, label in METRICS:
            if m in idx:
                print(f"   {label:<24} {v[idx[m]]:>14} {units[idx[m]]}")
        if "dram__bytes_read.sum" in idx:
            t = (to_bytes(v[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]]) +
                 to_bytes(v[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]]))
            traffic.setdefault(name, t)
    if "--json" in sys.argv:
        out = sys.argv[sys.argv.index("--json") + 1]
        key = sys.argv[sys.argv.index("--key") + 1]
        match = sys.argv[sys.argv.index("--match") + 1]
        try:
            d = json.load(open(out))
        except (OSError, ValueError):
            d = {}
        for n, t in traffic.items():
            if match in n:
                d[key] = t
                break
        json.dump(d, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
