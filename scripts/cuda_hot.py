"""Warp-stall samples and executed instructions per CUDA source line of an ncu report:

    python scripts/cuda_hot.py rep.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, rows, tot = "?", [], 0
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        smp, ins = int(r[4] or 0), int(r[7] or 0)
    except (ValueError, IndexError):
        continue
    rows.append((smp, ins, fname, r[0], r[1].strip()[:100]))
    tot += smp
print("samples", tot)
for smp, ins, f, ln, src in sorted(rows, reverse=True)[:n]:
    print(f"{100 * smp / max(tot, 1):5.1f}% {ins:>9} {f}:{ln:5s} {src}")
