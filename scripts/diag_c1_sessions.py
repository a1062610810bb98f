"""C1 at S sessions: dense-pass and per-increment integrated-output error vs the oracle for sessions
{0, S-1} (diagnostic for the accumulation-chain accuracy of the S >= 8 conv configurations)."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2303_04670_b200 as evc
from paper_2303_04670_b200 import configs, shard
from oracle import evincr_np as O

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8


def stream_inputs(seed, n):
    st = evc.generate_events(seed=seed, duration_us=50_000 + 1_000 * (n + 1), rate_hz=1.0e6, n_objects=8,
                             sensor_size=(256, 256))
    return torch.stack([torch.cat([evc.encode(w, evc.EncoderKind("count")), evc.encode(w, evc.EncoderKind("timestamp"))])
                        for w in (evc.slice_window(st, 50_000 + 1_000 * i, 50_000) for i in range(n + 1))])


def err(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max()) / max(1.0, float(np.abs(b).max()))


spec = configs.evflownet_spec(tp=0.0)
w = evc.WeightManifest.random_tensors(spec, 0)
seeds = shard.stream_seeds(0, S)
check = sorted({0, S - 1})
xs = torch.stack([stream_inputs(sd, N) for sd in seeds], dim=1).contiguous()
g = evc.build(spec, w, refresh_interval=0, sessions=S)
ogs = {s: O.OracleGraph(spec.to_dict(), w, refresh_interval=0) for s in check}
y0 = g.dense_pass(xs[0] if S > 1 else xs[0][0]).cpu().numpy().reshape(S, *spec_out) if False else None
y0 = g.dense_pass(xs[0] if S > 1 else xs[0][0]).cpu().numpy()
if S == 1:
    y0 = y0[None]
tag = os.environ.get("TAG", "")
print(f"[{tag}] S={S} dense err", [round(err(y0[s], ogs[s].dense_pass(xs[0, s].cpu().numpy())), 7) for s in check])
worst = 0.0
for i in range(1, N + 1):
    g.step_from_encodings(xs[i - 1] if S > 1 else xs[i - 1][0], xs[i] if S > 1 else xs[i][0])
    es = []
    for s in check:
        rv, rf = O.step_increment(xs[i - 1, s].cpu().numpy(), xs[i, s].cpu().numpy(), 6, 6)
        _, oy, _ = ogs[s].incr_step(rv, rf)
        es.append(err(g.integrated_output(session=s).cpu().numpy(), oy))
    worst = max(worst, *es)
print(f"[{tag}] S={S} worst integrated err over {N} increments {worst:.3e}")
d = g.dense_oracle(xs[N] if S > 1 else xs[N][0])
print(f"[{tag}] S={S} drift vs GPU dense recompute", [g.drift(d, session=s) if S > 1 else g.drift(d) for s in check])
