"""ncu target: the C4 scatter conv's launches at 0.5 % and 20 % clustered live tiles (Graph path)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2303_04670_b200 as evc  # noqa: E402
from paper_2303_04670_b200.graph import ModelSpec, NodeSpec  # noqa: E402

C, H, W, CO = 64, 480, 640, 128
spec = ModelSpec("c4", (C, H, W), [NodeSpec("conv", "conv", ["input"], {"out_channels": CO, "kernel": [3, 3],
                                                                       "stride": 1, "padding": 1})], "conv")
rng = np.random.default_rng(0)
wt = (rng.standard_normal((CO, C, 3, 3)) * np.sqrt(2.0 / (C * 9))).astype(np.float32)
g = evc.build(spec, {"conv.weight": wt}, refresh_interval=0, cuda_graph=False, scatter_convs=("conv",))
g.dense_pass(torch.zeros(C, H, W, device="cuda"))
gh, gw = -(-H // 6), -(-W // 6)
v, f = g.input_slot()
for d in (0.005, 0.2):
    f2 = rng.random((gh, gw)) < d
    px = np.repeat(np.repeat(f2, 6, 0), 6, 1)[:H, :W]
    v.copy_(torch.from_numpy((rng.standard_normal((C, H, W)) * px[None]).astype(np.float32)).cuda().unsqueeze(0))
    f.copy_(torch.from_numpy(np.broadcast_to(f2, (C, gh, gw)).copy()).cuda().unsqueeze(0))
    g._run_program()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    g._run_program()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
