#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and
an `ncu --set full` report into a markdown table for profiles/.

    python tools/ncu_summary.py <launches.csv> [<prof.ncu-rep>] > profiles/<name>.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_registers", "CTA/SM (reg limit)"),
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    k, v = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        try:
            d[r[k]].append(float(r[v]))
        except ValueError:
            pass
    tot = sum(sum(x) for n, x in d.items() if not n.startswith("k_partition"))
    print("## Launch list (ncu, serialised, cold cache: compare shares, not absolutes)\n")
    print("| kernel | launches | mean µs | share of block work |")
    print("|---|---|---|---|")
    for n, x in sorted(d.items(), key=lambda t: -sum(t[1])):
        share = "setup" if n.startswith("k_partition") else f"{100 * sum(x) / tot:.1f}%"
        print(f"| `{n.split('(')[0]}` | {len(x)} | {sum(x) / len(x) / 1e3:.2f} | {share} |")
    print()


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    cols = [(hdr.index(m), name, units[hdr.index(m)]) for m, name in METRICS if m in hdr]
    print("## ncu --set full (one launch per kernel)\n")
    print("| kernel | " + " | ".join(f"{n} ({u})" if u else n for _, n, u in cols) + " |")
    print("|---|" + "---|" * len(cols))
    seen = set()
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        if name in seen:
            continue
        seen.add(name)
        print(f"| `{name}` | " + " | ".join(r[i] for i, _, _ in cols) + " |")
    print()


if __name__ == "__main__":
    launches(sys.argv[1])
    if len(sys.argv) > 2:
        full(sys.argv[2])
