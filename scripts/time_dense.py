"""Time Graph.dense_pass (refresh) of C1 at S streams."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2303_04670_b200 as evc  # noqa: E402
from paper_2303_04670_b200 import configs  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 32
spec = configs.evflownet_spec(tp=0.0)
g = evc.build(spec, evc.WeightManifest.random_tensors(spec, 0), refresh_interval=0, sessions=S)
x = torch.rand((S, 4, 256, 256), device="cuda")
for _ in range(2):
    g.dense_pass(x if S > 1 else x[0])
torch.cuda.synchronize()
if "--prof" in sys.argv:
    torch.cuda.profiler.start()
    g.dense_pass(x if S > 1 else x[0])
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    sys.exit(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(5):
    g.dense_pass(x if S > 1 else x[0])
e1.record()
torch.cuda.synchronize()
print(f"dense_pass S={S}: {e0.elapsed_time(e1) / 5:.2f} ms device, {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms wall")
