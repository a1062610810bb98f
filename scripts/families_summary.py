"""Markdown summary of the kernel-family ncu evidence (scripts/gpu_families.sh):

    python scripts/families_summary.py gpurun_out > profiles/r02_ncu_families.md

Part 1 -- every launch of scripts/profile_families.py (one C1 step + one dense refresh at 32 streams,
compaction, encoders, count increment, one ingest step, one ConvLSTM step): duration, DRAM bytes and
achieved DRAM GB/s against the measured HBM peak.  Part 2 -- the `--set full` capture of one
instance per family: DRAM / L2 / tensor-pipe utilisation, issue activity, occupancy, top stalls.
ncu times are cold-cache and serialised (replay): use them for shares and traffic, not as bench values.
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def launches(path):
    per = OrderedDict()
    for r in csv.DictReader(l for l in open(path) if l.startswith('"')):
        key = (int(r["ID"]), r["Kernel Name"])
        per.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNITS.get(
            r["Metric Unit"], 1.0)
    return per


FULL = [
    ("gpu__time_duration.sum", "us", 1e6),
    ("dram__bytes_read.sum", "DRAM rd MB", 1e-6),
    ("dram__bytes_write.sum", "DRAM wr MB", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1),
    ("lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed", "L2 %", 1),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor %", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %", 1),
]


def full_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    head, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        val = dict(zip(head, row))
        unit = dict(zip(head, units))
        cells = [val.get("Kernel Name", "?")[:46]]
        for key, _, scale in FULL:
            k = key if key in val else next((h for h in head if h.endswith(key)), None)
            try:
                v = float(val[k].replace(",", "")) * UNITS.get(unit.get(k, ""), 1.0) if k else float("nan")
            except (ValueError, KeyError):
                v = float("nan")
            if key == "gpu__time_duration.sum":
                cells.append(f"{v * 1e6:.1f}")
            elif key.startswith("dram__bytes"):
                cells.append(f"{v * 1e-6:.2f}")
            else:
                cells.append(f"{v:.1f}")
        stalls = [(h, val[h]) for h in head if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
        top = sorted(((float(v or 0), h) for h, v in stalls), reverse=True)[:3]
        cells.append(", ".join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
                               f" {v:.1f}" for v, h in top))
        res.append(cells)
    return res


def main(d):
    peak, src = peak_gbs()
    print("# Kernel-family ncu evidence (round 2)\n")
    print(f"HBM peak for the fractions: {peak:.0f} GB/s ({src}, MEASURED_PEAKS.json).  ncu times are cold-cache and")
    print("serialised (replay): shares and traffic, not bench values.\n")
    print("## 1. Every launch of `scripts/profile_families.py` (32 streams)\n")
    print("| # | kernel | us | DRAM read MB | DRAM write MB | DRAM GB/s | % of HBM peak |")
    print("|---|---|---|---|---|---|---|")
    for (lid, name), m in launches(os.path.join(d, "fam_launch.csv")).items():
        t = m.get("gpu__time_duration.sum", 0.0)
        rb, wb = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
        gbs = (rb + wb) / t / 1e9 if t else 0.0
        print(f"| {lid} | `{name.split('(')[0][:60]}` | {t * 1e6:.1f} | {rb / 1e6:.2f} | {wb / 1e6:.2f} | {gbs:.0f} | "
              f"{100 * gbs / peak:.1f} |")
    print("\n## 2. `ncu --set full` of one instance per family\n")
    print("| kernel | " + " | ".join(lbl for _, lbl, _ in FULL) + " | top stalls (cycles / issue) |")
    print("|---" * (len(FULL) + 2) + "|")
    for rep in sorted(glob.glob(os.path.join(d, "fam_*.ncu-rep"))):
        for cells in full_rows(rep):
            print("| " + " | ".join(f"`{c}`" if i == 0 else c for i, c in enumerate(cells)) + " |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")
