"""ncu target: every kernel family of the library once, between cudaProfilerStart / Stop.

    ncu --profile-from-start off --metrics <...> --csv --log-file gpurun_out/families.csv \
        python scripts/profile_families.py [--sessions 32]

Families (north_star: compaction, gather, scatter, nonlinearity, GEMM tiles, binning):
  one C1 incremental step at S sessions (diff_mask, sparsify, tiles act / add / add_act,
  up_sparsify, fused / persistent / thin convs, integrate, meter_step); one C1 dense refresh
  (to_hwc, act_dense, copy_dense, upsample, sumsq); evc_compact over 1 Mi flags; encode of one C1
  window as count / timestamp / voxel (bin_events: keys, radix sort, runs); count_increment;
  one EventPipeline step of S sessions (ingest_ring, encode_windows); one ConvLSTM step (mul).
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_04670_b200 as evc  # noqa: E402
from paper_2303_04670_b200 import _lib, configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sessions", type=int, default=32)
    args = ap.parse_args()
    S = args.sessions
    spec = configs.evflownet_spec(tp=0.0)
    w = evc.WeightManifest.random_tensors(spec, 0)
    g = evc.build(spec, w, refresh_interval=0, sessions=S)
    xs = bench.make_inputs(lambda sd: bench.c1_frames(evc, sd, 6), list(range(S)))
    g.dense_pass(xs[0])
    for i in range(1, 4):
        g.step_from_encodings(xs[i - 1], xs[i])
    # other families' inputs
    flags = (torch.rand(1 << 20, device="cuda") < 0.02).to(torch.uint8)
    idx = torch.empty(1 << 20, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    scr = torch.zeros(int(_lib.lib().evc_compact_scratch(flags.numel())), dtype=torch.int32, device="cuda")
    stream = evc.generate_events(seed=0, duration_us=60_000, rate_hz=1.0e6, n_objects=8, sensor_size=(256, 256))
    wp, wc = evc.slice_window(stream, 50_000, 50_000), evc.slice_window(stream, 51_000, 50_000)
    evc.encode(wp, evc.EncoderKind("count"))
    rspec = configs.recurrent_unet_spec(levels=2, base=8, in_shape=(2, 48, 64))
    rg = evc.build(rspec, evc.WeightManifest.random_tensors(rspec, 0), refresh_interval=0)
    rx = torch.randn(2, 48, 64, device="cuda")
    rg.dense_pass(rx)
    streams = [evc.generate_events(seed=s, duration_us=56_000, rate_hz=1.0e6, n_objects=8, sensor_size=(256, 256))
               for s in range(S)]
    gi = evc.build(spec, w, refresh_interval=0, sessions=S)
    pipe = evc.EventPipeline(gi, (256, 256), "count+timestamp", window_us=50_000)
    out = torch.empty((2, S, 2, 256, 256), dtype=torch.float32).pin_memory()
    pipe.run([evc.pack_records(s) for s in streams], [s.t for s in streams], [[50_000, 51_000, 52_000]] * S, out)
    torch.cuda.synchronize()

    torch.cuda.profiler.start()
    g.step_from_encodings(xs[3], xs[4])                       # incremental step, all S sessions
    g.dense_pass(xs[4])                                       # dense refresh
    _lib.check(_lib.lib().evc_compact(_lib.ptr(flags), flags.numel(), _lib.ptr(idx), _lib.ptr(cnt), _lib.ptr(scr),
                                      _lib.stream_ptr()), "compact")
    for kind in ("count", "timestamp", "voxel:5"):
        evc.encode(wc, evc.parse_encoder(kind))
    evc.count_increment(wp, wc, spec.tile)
    pipe.run([evc.pack_records(s) for s in streams], [s.t for s in streams], [[54_000, 55_000]] * S, out[:1])
    rg.incr_step(evc.step_increment(rx, rx + (torch.rand_like(rx) < 0.02) * torch.randn_like(rx), rspec.tile))
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled the kernel families at", S, "sessions")


if __name__ == "__main__":
    main()
