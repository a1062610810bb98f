"""Per-launch list (first step) of an ncu gpu__time_duration csv: python scripts/launch_list.py file.csv [steps]"""
import csv, sys
rows = []
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    us = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}[r["Metric Unit"]]
    rows.append((r["Kernel Name"].split("(")[0].replace("void ", ""), r["Grid Size"], r["Block Size"], us))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n = len(rows) // steps
for i, (k, g, b, us) in enumerate(rows[:n]):
    print(f"{i:3d} {k[:40]:40s} {g:>14s} {us:8.1f}")
print("total", sum(r[3] for r in rows[:n]))
