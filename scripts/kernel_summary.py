"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name.

    python scripts/kernel_summary.py gpurun_out/launches.csv [--steps N]
"""

import csv
import sys
from collections import defaultdict


def load(path):
    rows = []
    with open(path, newline="") as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(unit, 1e-3)
        rows.append((r["Kernel Name"], v * scale))
    return rows


def main():
    path = sys.argv[1]
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 1
    rows = load(path)
    agg = defaultdict(lambda: [0, 0.0])
    for name, us in rows:
        short = name.split("(")[0].replace("void ", "")
        agg[short][0] += 1
        agg[short][1] += us
    total = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {total / steps:.1f} us of kernel time per step ({steps} steps)")
    print(f"{'kernel':60s} {'n/step':>7s} {'us/step':>9s} {'share':>6s}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n / steps:7.1f} {us / steps:9.1f} {100 * us / total:5.1f}%")


if __name__ == "__main__":
    main()
