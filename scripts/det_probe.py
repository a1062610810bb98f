"""Hash every step's output / flags / meters of the 64-increment C1 session (determinism probe)."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))

import numpy as np  # noqa: E402

import paper_2303_04670_b200 as evc  # noqa: E402
from paper_2303_04670_b200 import configs  # noqa: E402
from test_gpu_graph import evflownet_inputs  # noqa: E402

spec = configs.evflownet_spec(tp=0.0)
weights = evc.WeightManifest.random_tensors(spec, 0)
xs = evflownet_inputs(64)
hx = hashlib.sha1(b"".join(x.cpu().numpy().tobytes() for x in xs)).hexdigest()[:12]
for rep_i in range(2):
    g = evc.build(spec, weights, refresh_interval=0)
    g.dense_pass(xs[0])
    lines = []
    for i in range(1, 65):
        yup, y, rep = g.incr_step(evc.step_increment(xs[i - 1], xs[i], spec.tile))
        h = hashlib.sha1(y.detach().cpu().numpy().tobytes() + yup.mask.numpy().tobytes()).hexdigest()[:10]
        lines.append(f"{i} {h} " + " ".join(f"{k}={p}" for k, (p, _) in sorted(rep.per_node.items())))
    Path(f"gpurun_out/det_{sys.argv[1]}_{rep_i}.txt").write_text(f"inputs {hx}\n" + "\n".join(lines) + "\n")
print("done", hx)
