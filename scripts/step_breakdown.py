"""Per-launch device time of one eager C1 incr_step (CUDA events around every launch, L2 warm).

    python scripts/step_breakdown.py [--sessions S] [--steps N]
"""
import argparse
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_04670_b200 as evc  # noqa: E402
from paper_2303_04670_b200 import _lib, configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sessions", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    args = ap.parse_args()
    S = args.sessions
    spec = configs.evflownet_spec(tp=0.0)
    g = evc.build(spec, evc.WeightManifest.random_tensors(spec, 0), refresh_interval=0, sessions=S, cuda_graph=False)
    xs = bench.make_inputs(lambda sd: bench.c1_frames(evc, sd, 4 + args.steps), list(range(S)))
    g.dense_pass(xs[0] if S > 1 else xs[0][0])
    for i in range(1, 3):
        g.step_from_encodings(xs[i - 1], xs[i])
    names = {n for _, _, n in g._program}
    acc = defaultdict(float)
    order = []
    for i in range(3, 3 + args.steps):
        _lib.check(g.lib.evc_diff_mask(xs[i - 1].data_ptr(), xs[i].data_ptr(), xs[0][0].numel(), g._desc(g.input_id),
                                       S, _lib.stream_ptr()), "diff")
        timed = (names, [])
        g._run_program(timed=timed)
        torch.cuda.synchronize()
        for j, (n, e0, e1) in enumerate(timed[1]):
            key = (j, n)
            acc[key] += e0.elapsed_time(e1) * 1e3 / args.steps
            if i == 3:
                order.append(key)
    prog = [p for p in g._program]
    tot = 0.0
    by = defaultdict(float)
    for j, n in order:
        us = acc[(j, n)]
        tot += us
        by[n] += us
        print(f"{j:3d} {n:20s} {us:8.1f}")
    print(f"sum {tot:.1f} us per step (S={S})")
    for n, us in sorted(by.items(), key=lambda kv: -kv[1]):
        print(f"   {n:20s} {us:8.1f}")


if __name__ == "__main__":
    main()
