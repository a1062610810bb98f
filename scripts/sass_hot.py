"""Top SASS instructions by warp-stall samples from an ncu report: python scripts/sass_hot.py rep.ncu-rep [N]"""
import csv, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr = r[1]; rows = [dict(zip(hdr, x)) for x in r[2:] if len(x) == len(hdr)]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in rows)
print("instructions", len(rows), "samples", tot)
idx = sorted(range(len(rows)), key=lambda i: -int(rows[i]["Warp Stall Sampling (All Samples)"] or 0))[:n]
for i in sorted(idx):
    d = rows[i]
    print(f"{i:5d} {d['Warp Stall Sampling (All Samples)']:>6} {d['Instructions Executed']:>8}  {d['Source'][:90]}")
