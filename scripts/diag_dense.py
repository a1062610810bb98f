"""Per-node dense-pass error of C1 vs the oracle at several session counts (diagnostic)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2303_04670_b200 as evc
from paper_2303_04670_b200 import configs
from oracle import evincr_np as O

spec = configs.evflownet_spec(tp=0.0)
w = evc.WeightManifest.random_tensors(spec, 0)
st = evc.generate_events(seed=0, duration_us=52_000, rate_hz=1.0e6, n_objects=8, sensor_size=(256, 256))
win = evc.slice_window(st, 50_000, 50_000)
x = torch.cat([evc.encode(win, evc.EncoderKind("count")), evc.encode(win, evc.EncoderKind("timestamp"))])
og = O.OracleGraph(spec.to_dict(), w, refresh_interval=0)
ref = og._dense(x.cpu().numpy(), False)
for S in [int(a) for a in sys.argv[1:]] or [1, 8, 32]:
    g = evc.build(spec, w, refresh_interval=0, sessions=S)
    g._eval_dense(x.unsqueeze(0).expand(S, *x.shape).contiguous() if S > 1 else x, mutate=False)
    torch.cuda.synchronize()
    rows = []
    for n in g.nodes:
        nid = n.spec.id
        if n.kind == "conv" and n.fused_act is not None:
            continue
        v, _ = g._slot_view(nid)
        v = v[0].cpu().numpy()
        r = ref[nid]
        if not np.abs(v).max() and np.abs(r).max():
            continue
        sc = max(1.0, float(np.abs(r).max()))
        rows.append((nid, float(np.abs(v - r).max()), sc, float(np.abs(v - r).max()) / sc))
    print(f"S={S}")
    for r in rows:
        print(f"  {r[0]:12s} abs {r[1]:.3e} scale {r[2]:.3e} rel {r[3]:.3e}")
    cfg = {n.spec.id: (int(n.plan.cfg.thin), int(n.plan.cfg.row), int(n.plan.cfg.bn), int(n.plan.cfg.splits))
           for n in g.nodes if n.kind == "conv"}
    print("  cfg", cfg)
    g._clear_increments()
    del g
