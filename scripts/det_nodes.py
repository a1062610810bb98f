"""Find the first node whose flags / values differ between sessions fed the same increments."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))

import paper_2303_04670_b200 as evc  # noqa: E402
from paper_2303_04670_b200 import configs  # noqa: E402
from test_gpu_graph import evflownet_inputs  # noqa: E402

cg = sys.argv[1] == "1" if len(sys.argv) > 1 else True
spec = configs.evflownet_spec(tp=0.0)
weights = evc.WeightManifest.random_tensors(spec, 0)
xs = evflownet_inputs(12)


def run():
    g = evc.build(spec, weights, refresh_interval=0, cuda_graph=cg)
    g.dense_pass(xs[0])
    rec = []
    for i in range(1, len(xs)):
        _, _, rep = g.incr_step(evc.step_increment(xs[i - 1], xs[i], spec.tile))
        d = {}
        for nid in g._slots:
            v, f = g._slot_view(nid)
            d[nid] = (hashlib.sha1(f.cpu().numpy().tobytes()).hexdigest()[:8],
                      hashlib.sha1(v.detach().cpu().numpy().tobytes()).hexdigest()[:8])
        rec.append((d, dict(rep.per_node)))
    return rec


a = run()
order = [n.id for n in spec.topo_order()]
for k in range(4):
    b = run()
    for i, ((da, pa), (db, pb)) in enumerate(zip(a, b)):
        bad = [n for n in order if n in da and da[n] != db[n]]
        badp = {n: (pa[n], pb[n]) for n in pa if pa[n] != pb[n]}
        if bad or badp:
            print(f"run {k} step {i}: first differing slots {bad[:4]} -> {[(da[n], db[n]) for n in bad[:2]]}; meters {badp}")
            break
    else:
        print(f"run {k}: identical")
