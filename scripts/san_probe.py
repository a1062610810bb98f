"""Small C1 session (2 increments) for compute-sanitizer runs."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))

import paper_2303_04670_b200 as evc  # noqa: E402
from paper_2303_04670_b200 import configs  # noqa: E402
from test_gpu_graph import evflownet_inputs  # noqa: E402

spec = configs.evflownet_spec(tp=0.0)
weights = evc.WeightManifest.random_tensors(spec, 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
xs = evflownet_inputs(n)
g = evc.build(spec, weights, refresh_interval=0, cuda_graph=len(sys.argv) > 2 and sys.argv[2] == "1")
g.dense_pass(xs[0])
for i in range(1, n + 1):
    g.incr_step(evc.step_increment(xs[i - 1], xs[i], spec.tile))
print("ok")
