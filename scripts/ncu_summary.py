"""Key metrics of a one-kernel `ncu --set full` report (for profiles/):
    python scripts/ncu_summary.py gpurun_out/prof_conv.ncu-rep > profiles/r01_ncu_dec3.txt"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("Kernel Name", "kernel"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed", "L2 <- SM sectors % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1/TEX throughput %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    for row in rows[2:]:
        val = dict(zip(head, row))
        unit = dict(zip(head, units))
        for key, label in KEYS:
            if key not in val:
                key = next((h for h in head if h.endswith("." + key) and val.get(h)), key)
            if key in val:
                print(f"{label:32s} {val[key]} {unit.get(key, '')}".rstrip())
        stalls = [(h, val[h]) for h in head if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
        top = sorted(((float(v or 0), h) for h, v in stalls), reverse=True)[:6]
        print("top stall reasons (cycles per issued instruction):")
        for v, h in top:
            print(f"   {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {v:.2f}")
        print()


if __name__ == "__main__":
    main(sys.argv[1])
