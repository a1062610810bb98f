"""ncu target: C2 E2Depth-style UNet incremental steps (8 streams, ~1 % voxel density); optional --scatter ids."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_04670_b200 as evc  # noqa: E402
from paper_2303_04670_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sessions", type=int, default=8)
ap.add_argument("--rate", type=float, default=2.0e5)
ap.add_argument("--scatter", default="")
args = ap.parse_args()
S = args.sessions
spec = configs.unet_e2depth_spec(tp=0.0)
g = evc.build(spec, evc.WeightManifest.random_tensors(spec, 0), refresh_interval=0, sessions=S,
              scatter_convs=tuple(x for x in args.scatter.split(",") if x))
xs = bench.make_inputs(lambda sd: bench.c2_frames(evc, sd, 8, args.rate), list(range(S)))
g.dense_pass(xs[0])
for i in range(1, 5):
    g.step_from_encodings(xs[i - 1], xs[i])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(5, 7):
    g.step_from_encodings(xs[i - 1], xs[i])
e1.record()
torch.cuda.synchronize()
print(f"C2 S={S} rate={args.rate:g} scatter={args.scatter!r}: {e0.elapsed_time(e1) / 2:.3f} ms/step")
torch.cuda.profiler.start()
g.step_from_encodings(xs[6], xs[7])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print([(n.spec.id, n.out_shape, tuple(int(v) for v in n.weight.shape)) for n in g.nodes if n.kind == "conv"][:6])
