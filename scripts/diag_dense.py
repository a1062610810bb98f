"""Per-node dense-pass error of C1 at several session counts, against an f64 restatement of the
oracle (oracle/evincr_np.py with F32 -> float64) and against the f32 oracle itself (diagnostic)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2303_04670_b200 as evc
from paper_2303_04670_b200 import configs
from oracle import evincr_np as O

N = 16
spec = configs.evflownet_spec(tp=0.0)
w = evc.WeightManifest.random_tensors(spec, 0)
st = evc.generate_events(seed=0, duration_us=50_000 + 1_000 * (N + 1), rate_hz=1.0e6, n_objects=8, sensor_size=(256, 256))
win = evc.slice_window(st, 50_000, 50_000)
x = torch.cat([evc.encode(win, evc.EncoderKind("count")), evc.encode(win, evc.EncoderKind("timestamp"))])
og = O.OracleGraph(spec.to_dict(), w, refresh_interval=0)
ref = og._dense(x.cpu().numpy(), False)
f32 = O.F32
O.F32 = np.float64
og64 = O.OracleGraph(spec.to_dict(), {k: np.asarray(v, np.float64) for k, v in w.items()}, refresh_interval=0)
r64 = og64._dense(x.cpu().numpy().astype(np.float64), False)
O.F32 = f32
for S in [int(a) for a in sys.argv[1:]] or [1, 8, 32]:
    g = evc.build(spec, w, refresh_interval=0, sessions=S)
    g._eval_dense(x.unsqueeze(0).expand(S, *x.shape).contiguous() if S > 1 else x, mutate=False)
    torch.cuda.synchronize()
    print(f"S={S}   node  kind  scale  gpu-vs-f32oracle  gpu-vs-f64  f32oracle-vs-f64")
    for n in g.nodes:
        nid = n.spec.id
        if n.kind == "conv" and n.fused_act is not None:
            continue
        v, _ = g._slot_view(nid)
        v = v[0].cpu().numpy().astype(np.float64)
        r, d = ref[nid].astype(np.float64), r64[nid]
        if not np.abs(v).max() and np.abs(r).max():
            continue
        sc = max(1.0, float(np.abs(d).max()))
        print(f"  {nid:12s} {n.kind:9s} {sc:9.3e} {np.abs(v - r).max() / sc:.3e} {np.abs(v - d).max() / sc:.3e} "
              f"{np.abs(r - d).max() / sc:.3e}")
    cfg = {n.spec.id: (int(n.plan.cfg.thin), int(n.plan.cfg.row), int(n.plan.cfg.bn), int(n.plan.cfg.splits))
           for n in g.nodes if n.kind == "conv"}
    print("  cfg", cfg)
    g._clear_increments()
    del g
