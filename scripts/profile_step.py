"""Profile target: C1 EV-FlowNet incremental steps between cudaProfilerStart/Stop.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py [--steps 2] [--eager]

Only the profiled steps (diff_mask + the incr_step launch sequence) are
captured; setup (stream generation, encoding, dense pass) is excluded.
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_04670_b200 as evc  # noqa: E402
from paper_2303_04670_b200 import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--sessions", type=int, default=1)
    ap.add_argument("--eager", action="store_true")
    args = ap.parse_args()
    S = args.sessions
    spec = configs.evflownet_spec(tp=0.0)
    g = evc.build(spec, evc.WeightManifest.random_tensors(spec, 0), refresh_interval=0, sessions=S,
                  cuda_graph=not args.eager)
    xs = bench.make_inputs(lambda sd: bench.c1_frames(evc, sd, 5 + args.steps), list(range(S)))
    g.dense_pass(xs[0] if S > 1 else xs[0][0])
    for i in range(1, 4):
        g.step_from_encodings(xs[i - 1], xs[i])
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for i in range(4, 4 + args.steps):
        g.step_from_encodings(xs[i - 1], xs[i])
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled", args.steps, "steps;", g.kernel_launches_per_step() + 1, "libevconv launches per step")


if __name__ == "__main__":
    main()
