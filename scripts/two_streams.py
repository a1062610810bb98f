"""Feasibility: two half-batch graphs (S/2 streams each) replayed on two CUDA streams concurrently vs one S graph."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_04670_b200 as evc  # noqa: E402
from paper_2303_04670_b200 import configs  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 32
K = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = configs.evflownet_spec(tp=0.0)
w = evc.WeightManifest.random_tensors(spec, 0)
n = 24
xs = bench.make_inputs(lambda sd: bench.c1_frames(evc, sd, n), list(range(S)))


def time_it(graphs, streams, parts):
    for g, p in zip(graphs, parts):
        g.dense_pass(xs[0][p])
    torch.cuda.synchronize()
    ts = []
    for i in range(1, n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        e0.record(cur)
        for g, st, p in zip(graphs, streams, parts):
            st.wait_event(e0)
            with torch.cuda.stream(st):
                g.step_from_encodings(xs[i - 1][p], xs[i][p])
        for st in streams:
            cur.wait_stream(st)
        e1.record(cur)
        torch.cuda.synchronize()
        if i > 3:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


one = evc.build(spec, w, refresh_interval=0, sessions=S)
t1 = time_it([one], [torch.cuda.Stream()], [slice(0, S)])
del one
h = S // K
gs = [evc.build(spec, w, refresh_interval=0, sessions=h) for _ in range(K)]
t2 = time_it(gs, [torch.cuda.Stream() for _ in range(K)], [slice(k * h, (k + 1) * h) for k in range(K)])
print(f"S={S}: one graph {t1:.3f} ms/step ({S / t1 * 1e3:.0f} inc/s); {K} x {h} on {K} streams {t2:.3f} ms/step "
      f"({S / t2 * 1e3:.0f} inc/s)")
