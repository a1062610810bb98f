"""C4 sweep only (bench.c4_config): python scripts/c4_bench.py"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2303_04670_b200 as evc  # noqa: E402

r = bench.c4_config(evc, iters=10)
print(f"dense {r['dense_us']:.1f} us")
for row in r["sweep"]:
    print(f"{row['live_tiles']:6.3f}  scatter {row['scatter_us']:8.1f}  fused {row['fused_us']:8.1f}  "
          f"scatter/dense {row['sparse_over_dense']:.3f}  performed/dense {row['performed_over_dense']:.4f}")
print(json.dumps(r))
