"""Per-launch side-by-side of two ncu launch lists (gpu__time_duration.sum) of the same program.

    python scripts/launch_diff.py a.csv b.csv
"""
import sys
sys.path.insert(0, "scripts")
from kernel_summary import load  # noqa: E402

a, b = load(sys.argv[1]), load(sys.argv[2])
ta = tb = 0.0
for i, ((na, ua), (nb, ub)) in enumerate(zip(a, b)):
    ta += ua
    tb += ub
    print(f"{i:3d} {na[:44]:44s} {ua:9.1f} {ub:9.1f} {ub / ua if ua else 0:6.2f}  {nb[:30] if nb != na else ''}")
print(f"total {ta:.1f} {tb:.1f} us")
