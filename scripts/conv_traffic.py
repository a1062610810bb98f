"""DRAM bytes of the conv launches of one step, from an ncu --csv metrics log:
    python scripts/conv_traffic.py gpurun_out/conv_traffic_s32.csv --sessions 32 > profiles/r01_conv_traffic_s32.json
(bench.py reports the sum as roofline.traffic when its workload matches)."""
import argparse
import csv
import json
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--sessions", type=int, default=32)
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    rows = [r for r in csv.DictReader(l for l in open(args.csv) if l.startswith('"'))]
    per = defaultdict(dict)
    for r in rows:
        per[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = float(r["Metric Value"]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r["Metric Unit"], 1.0)
    launches = []
    for (lid, name), m in sorted(per.items(), key=lambda kv: int(kv[0][0])):
        if "dram__bytes_read.sum" in m:
            launches.append({"kernel": name.split("(")[0], "dram_read": m["dram__bytes_read.sum"],
                             "dram_write": m.get("dram__bytes_write.sum", 0.0)})
    tot = sum(l["dram_read"] + l["dram_write"] for l in launches) / args.steps
    print(json.dumps({"model": "evflownet-256", "sessions": args.sessions, "launches_per_step": len(launches) // args.steps,
                      "dram_bytes_per_step": tot, "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                      "-k regex:k_conv, one C1 step (python scripts/profile_step.py --steps 1 --sessions 32)",
                      "launches": launches}, indent=1))


if __name__ == "__main__":
    main()
