"""Host-side cost of the e2e serving loop (bench.measure_e2e_events): wall per step, and a cProfile of
one 63-step run, to see whether the Python loop or the device bounds the end-to-end rate."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_04670_b200 as evc  # noqa: E402
from paper_2303_04670_b200 import configs  # noqa: E402
from paper_2303_04670_b200 import shard as _shard  # noqa: E402


def main():
    S = 32
    spec = configs.evflownet_spec(tp=0.0)
    g = evc.build(spec, evc.WeightManifest.random_tensors(spec, 0), refresh_interval=64, sessions=S)
    seeds = _shard.stream_seeds(0, S)
    streams = {sd: bench.c1_stream(evc, sd, 70) for sd in seeds}
    n = 63
    taus = [[bench.WINDOW_US + bench.SHIFT_US * i for i in range(n + 1)] for _ in range(S)]
    recs = [evc.pack_records(streams[sd]) for sd in seeds]
    ts = [streams[sd].t for sd in seeds]
    pipe = evc.EventPipeline(g, (256, 256), "count+timestamp", window_us=bench.WINDOW_US)
    y = g._y_run[g.output_ids[0]]
    out_host = torch.empty((n, *y.shape), dtype=torch.float32).pin_memory()
    pipe.run(recs, ts, [t[:3] for t in taus], out_host[:2])
    torch.cuda.synchronize()
    for _ in range(2):
        t0 = time.perf_counter()
        pipe.run(recs, ts, taus, out_host)
        print(f"e2e run: {n * S / (time.perf_counter() - t0):.0f} increments/s")
    pr = cProfile.Profile()
    pr.enable()
    pipe.run(recs, ts, taus, out_host)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
