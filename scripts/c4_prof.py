"""One C4 inc_conv2d call at 0.5 % clustered density under the profiler (launch list)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2303_04670_b200 as evc  # noqa: E402

C, H, W, CO = 64, 480, 640, 128
rng = np.random.default_rng(0)
wt = torch.from_numpy((rng.standard_normal((CO, C, 3, 3)) * 0.05).astype(np.float32)).cuda()
params = evc.ConvParams.from_weight(wt.cpu().numpy(), 1, 1)
f2 = rng.random((80, 107)) < 0.005
flags = np.broadcast_to(f2, (C, 80, 107)).copy()
px = np.repeat(np.repeat(f2, 6, 0), 6, 1)[:H, :W]
x = evc.IncrementTensor(torch.from_numpy((rng.standard_normal((C, H, W)) * px[None]).astype(np.float32)).cuda(),
                        evc.TileMask(torch.from_numpy(flags).cuda(), evc.TileShape(6, 6)))
for _ in range(3):
    evc.inc_conv2d(x, wt, params, evc.FlopCounter())
torch.cuda.synchronize()
torch.cuda.profiler.start()
evc.inc_conv2d(x, wt, params, evc.FlopCounter())
torch.cuda.synchronize()
torch.cuda.profiler.stop()
