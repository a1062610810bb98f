"""Eager C1 sessions (as tests/test_gpu_determinism.py) + light per-step sums of the
dec3 upsample input and the dec3 sparsify flags, to locate a run-to-run difference."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))

import torch  # noqa: E402

import paper_2303_04670_b200 as evc  # noqa: E402
from paper_2303_04670_b200 import configs  # noqa: E402
from test_gpu_graph import evflownet_inputs  # noqa: E402

spec = configs.evflownet_spec(tp=0.0)
weights = evc.WeightManifest.random_tensors(spec, 0)
xs = evflownet_inputs(12)
byid = {n.id: n for n in spec.topo_order()}
xin = byid["dec3_up"].inputs[0]


def run():
    g = evc.build(spec, weights, refresh_interval=0, cuda_graph=False)
    g.dense_pass(xs[0])
    rec = []
    for i in range(1, len(xs)):
        yup, y, rep = g.incr_step(evc.step_increment(xs[i - 1], xs[i], spec.tile))
        xv, xf = g._slot_view(xin)
        _, sf = g._slot_view("dec3_sp")
        rec.append((float(xv.sum(dtype=torch.float64)), int(xf.sum(dtype=torch.int64)), int(sf.sum(dtype=torch.int64)),
                    rep.per_node["dec3"][0], y.detach().cpu().numpy().tobytes()))
    return rec


a = run()
for k in range(3):
    b = run()
    for i, (ra, rb) in enumerate(zip(a, b)):
        if ra != rb:
            print(f"run {k} step {i}: x sum {ra[0]!r} vs {rb[0]!r}; x flags {ra[1]} vs {rb[1]}; "
                  f"dec3_sp flags {ra[2]} vs {rb[2]}; dec3 perf {ra[3]} vs {rb[3]}; y same {ra[4] == rb[4]}")
            break
    else:
        print(f"run {k}: identical")
