"""EV-FlowNet 256x256 incremental inference benchmark (BASELINE.json metric), plus the C2 / C3 / C4
configurations of BASELINE.json as sub-results of the same JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--sessions S] [--impl ours|reference]
                    [--configs c2,c3,c4 | --configs none]

A "step" is one incremental pass (step_increment + Graph.incr_step, plus the
refresh when due -- the reference's timed region, bench.py:196-209) for each of
the S independent event streams this rank owns (default 32 per GPU: the C5
layout of 256 streams over 8 GPUs; every launch serves all S streams).  A
second, single-stream pass reports the batch-1 per-increment latency
(p50_increment_latency_ms).  Inputs are count(2) + timestamp(2) encodings of
seeded synthetic 1 MHz streams (generate_events, 8 objects, 256x256), 50 ms
windows shifted by 1 ms (~2 % of elements change per increment), encoded on the
GPU before timing and resident in HBM.  Weights: seeded He-normal
(WeightManifest.random_tensors), t_p = 0, refresh every 64 increments: one dense
refresh is timed on its own and 1/64 of it is added to every step
(``refresh_amortized_ms``), so ``value`` is the steady-state rate with refreshes.

``value`` is the whole-job rate (increments/s over all ranks, the driver's
scaling input); ``value_per_gpu`` = value / N is the metric's per-GPU figure.
``--gpus N`` without torchrun re-launches this script under
``torch.distributed.run`` with N ranks (one GPU each, NCCL, 127.0.0.1).
Streams shard across ranks with no collective on the data path (scaling
"weak": rank r owns streams r*S .. r*S+S-1); rank 0 prints one JSON line with
the max-over-ranks device time.  ``--impl reference`` times the CPU reference
algorithm (the oracle port of evincr's per-channel loop) on the host cores.
At N = 1 the line also carries ``configs``: C2 (E2Depth UNet, 5-bin voxels,
264x352, 1 / 3 / 5 % density), C3 (ResNet-18, 2x180x240 counts) and C4 (one
64->128 3x3 conv at 480x640, sparse vs the library's own dense conv over
0.5-20 % live tiles), each with its rate, p50 latency, conv roofline and a
bounded CPU baseline.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2303_04670_b200 import shard as _shard  # noqa: E402  (no CUDA needed)

METRIC = "EV-FlowNet increments/sec/GPU and p50 per-increment latency at 2% density"
UNIT = "increments/s"
WINDOW_US, SHIFT_US, RATE_HZ = 50_000, 1_000, 1.0e6
C1_ALG_BYTES = 42.5e6  # minimal bytes per C1 increment (live input, acc r/w, weights, outputs)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


def dist_env():
    return _shard.dist_env()


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md)
# ---------------------------------------------------------------------------


class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def c1_stream(evc, seed, n_windows):
    return evc.generate_events(seed=seed, duration_us=WINDOW_US + SHIFT_US * n_windows, rate_hz=RATE_HZ,
                               n_objects=8, sensor_size=(256, 256))


def c1_frames(evc, seed, n_windows, stream=None):
    """C1 input frames: count(2) + timestamp(2) of a seeded 1 MHz 256x256 stream, 50 ms windows / 1 ms."""
    import torch

    stream = stream or c1_stream(evc, seed, n_windows)
    xs = []
    for i in range(n_windows):
        w = evc.slice_window(stream, WINDOW_US + SHIFT_US * i, WINDOW_US)
        xs.append(torch.cat([evc.encode(w, evc.EncoderKind("count")), evc.encode(w, evc.EncoderKind("timestamp"))]))
    return torch.stack(xs)


C2_RATES = {"1%": 2.0e5, "3%": 2.0e6, "5%": 3.8e6}  # voxel increment density on 264x352 (calibrated)


def c2_frames(evc, seed, n_windows, rate):
    """C2 input frames: 5-bin voxel grids of a 260x346 stream, zero-padded bottom / right to 264x352."""
    import torch

    stream = evc.generate_events(seed=seed, duration_us=WINDOW_US + SHIFT_US * n_windows, rate_hz=rate,
                                 n_objects=8, sensor_size=(260, 346))
    xs = [torch.nn.functional.pad(evc.encode(evc.slice_window(stream, WINDOW_US + SHIFT_US * i, WINDOW_US),
                                             evc.parse_encoder("voxel:5")), (0, 6, 0, 4))
          for i in range(n_windows)]
    return torch.stack(xs)


def c3_frames(evc, seed, n_windows, rate=2.0e5):
    """C3 input frames: count(2) of a 180x240 stream (N-Caltech101 shape)."""
    import torch

    stream = evc.generate_events(seed=seed, duration_us=WINDOW_US + SHIFT_US * n_windows, rate_hz=rate,
                                 n_objects=8, sensor_size=(180, 240))
    return torch.stack([evc.encode(evc.slice_window(stream, WINDOW_US + SHIFT_US * i, WINDOW_US),
                                   evc.EncoderKind("count")) for i in range(n_windows)])


def make_inputs(frames, seeds):
    import torch

    return torch.stack([frames(sd) for sd in seeds], dim=1).contiguous()  # (n_windows, S, C, H, W)


def timed_steps(g, xs, steps, warmup, world=1, clocks_index=None):
    """Dense pass on window 0, `warmup` untimed steps, then `steps` timed steps (CUDA events on
    the step stream, L2 flushed by a 256 MiB write before each).  Refreshes run in-line when due."""
    import torch

    S = g.S
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=xs.device)

    def frame(i):
        return xs[i] if S > 1 else xs[i][0]

    def step(i):
        g.step_from_encodings(frame(i - 1), frame(i))
        if g.refresh_due:
            g.dense_pass(frame(i))

    g.dense_pass(frame(0))
    for i in range(1, 1 + warmup):
        step(i)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    refreshes = 0
    clk = Clocks(clocks_index) if clocks_index is not None else None
    if clk:
        clk.__enter__()
    try:
        for j in range(steps):
            flush.fill_(float(j))  # evict L2 between timed steps (256 MiB > 126 MB L2)
            i = 1 + warmup + j
            evs[j][0].record()
            will_refresh = g.refresh_interval and g.step_count + 1 >= g.refresh_interval
            step(i)
            refreshes += bool(will_refresh)
            evs[j][1].record()
        torch.cuda.synchronize()
    finally:
        if clk:
            clk.__exit__()
    if world > 1:
        dist.barrier()
    del flush
    return [a.elapsed_time(b) for a, b in evs], refreshes, clk


def time_refresh(g, x, reps=3):
    """Device time of one dense refresh (dense_pass) of all S sessions, ms (median of `reps`)."""
    import torch

    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        g.dense_pass(x)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def pct(sorted_ts, q):
    return sorted_ts[min(len(sorted_ts) - 1, int(round(q * (len(sorted_ts) - 1))))]


def run_ours(args):
    import torch

    import paper_2303_04670_b200 as evc
    from paper_2303_04670_b200 import configs

    rank, world, local = dist_env()
    # test knob: EVC_BENCH_SHARE_GPU=1 runs every rank on GPU 0 over gloo (the N > 1 logic on a
    # one-GPU box); the product path is one rank per GPU over NCCL
    share = os.environ.get("EVC_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cdev = None if share else dev  # device of the max-over-ranks reduction tensors
    spec = configs.evflownet_spec(tp=0.0)
    weights = evc.WeightManifest.random_tensors(spec, 0)
    S = args.sessions
    n_win = 1 + args.warmup + args.steps + 1
    seeds = _shard.stream_seeds(rank, S)
    streams = {sd: c1_stream(evc, sd, max(n_win, 66)) for sd in seeds}  # (the e2e leg runs 64 increments)
    xs = make_inputs(lambda sd: c1_frames(evc, sd, n_win, streams[sd]), seeds)  # resident in HBM before timing
    density = float((xs[1:] != xs[:-1]).float().mean())
    g = evc.build(spec, weights, refresh_interval=64, sessions=S)
    times, refreshes, clk = timed_steps(g, xs, args.steps, args.warmup, world, dev.index or 0)
    # one refresh per 64 increments: timed on its own, 1/64 of it added to every step
    refresh_ms = time_refresh(g, xs[0] if S > 1 else xs[0][0])
    steps_cost = sum(times) + refresh_ms * max(0.0, args.steps / 64.0 - refreshes)
    total_ms = _shard.job_time_ms(steps_cost, world, cdev)  # max over ranks
    total_ms_nr = _shard.job_time_ms(sum(times), world, cdev)  # (every rank joins each collective)
    value = _shard.aggregate_rate(args.steps, S, world, total_ms)
    steady = sorted(times)
    p50, p99 = statistics.median(steady), pct(steady, 0.99)
    launches = g.kernel_launches_per_step() + 1  # + diff_mask
    gpu_launches = args.steps * launches + refreshes * g.dense_launches()
    lat = None
    if S > 1 and not args.no_latency_pass:  # single-stream latency (batch 1), same workload
        g1 = evc.build(spec, weights, refresh_interval=64, sessions=1)
        t1, _, _ = timed_steps(g1, xs[:, :1].contiguous(), min(args.steps, 32), args.warmup, world)
        s1 = sorted(t1)
        lat = {"sessions": 1, "p50_ms": statistics.median(s1), "p99_ms": pct(s1, 0.99), "steps": len(s1)}
        del g1
    roof = conv_roofline(g, xs, evc)
    e2e = measure_e2e_events(evc, g, [streams[sd] for sd in seeds], args, S, world, cdev)
    e2e["frames_pipeline"] = measure_e2e(g, xs, args, S, world, cdev)
    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "value_per_gpu": value / world,
            "config": {"workload": (f"C1 EV-FlowNet 256x256 (4-ch count+timestamp), ~2% increment density, batch 1 "
                                    f"per stream; {S} independent streams per GPU batched into every launch "
                                    f"(C5 layout: 256 streams over 8 GPUs = 32 per GPU)"),
                       "sessions_per_gpu": S, "streams_total": S * world, "t_p": 0.0, "refresh_interval": 64,
                       "window_us": WINDOW_US, "shift_us": SHIFT_US, "increment_density": density,
                       "l2": "flushed between timed steps (256 MiB write, excluded from step events)",
                       "refresh": ("one dense refresh per 64 increments: timed separately and 1/64 of it added to "
                                   "every step without an in-line refresh"),
                       "parallelism": f"streams sharded over {world} GPU(s) (rank r owns streams r*S..r*S+S-1), "
                                      f"no collective"},
            "p50_ms": p50, "p99_ms": p99, "refreshes_in_timed_region": refreshes,
            "refresh_ms": refresh_ms, "refresh_amortized_ms": refresh_ms / 64.0,
            "value_no_refresh": _shard.aggregate_rate(args.steps, S, world, total_ms_nr),
            "p50_increment_latency_ms": (lat or {}).get("p50_ms", p50 if S == 1 else None),
            "latency_single_stream": lat,
            "clocks": clk.summary(), "gpu_launches": gpu_launches, "roofline": roof, "e2e": e2e,
        }
    if rank == 0:  # roofline.achieved = t_roof / t_p50 per increment
        hbm, bf16, _src = peaks()
        f_inc = roof["algorithmic_flops_per_step"] / S
        t_roof = max(f_inc / (0.5 * bf16 * 1e12), C1_ALG_BYTES / (hbm * 1e9)) * 1e6
        p50_inc = out["p50_increment_latency_ms"]
        out["latency_roofline"] = {
            "t_roof_us": t_roof, "alg_flops_per_increment": f_inc, "alg_bytes_per_increment": C1_ALG_BYTES,
            "frac_batch1": t_roof / (p50_inc * 1e3) if p50_inc else None,
            "frac_amortized": t_roof / (out["ms_per_step"] * 1e3 / S),
            "definition": "t_roof = max(F_alg / TF32 peak, B_alg / HBM peak) per increment (SURVEY 8(d)); "
                          "frac = t_roof / p50 single-stream latency, or / amortised per-increment time at S streams"}
    if world > 1 and args.gpus != world and rank == 0:
        out["config"]["gpus_flag_mismatch"] = f"--gpus {args.gpus} but WORLD_SIZE {world}"
    del g, xs
    torch.cuda.empty_cache()
    if rank == 0 and world == 1:
        want = [c for c in args.configs.split(",") if c and c != "none"]
        if want:
            out["configs"] = sub_configs(evc, configs, want, args)
    if world > 1:
        dist.barrier()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(budget_s=args.cpu_budget)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def conv_roofline(g, xs, evc, nsteps=8):
    """Time every conv launch of a few eager steps with CUDA events on the launching stream;
    achieved = reference-meter FLOPs (algorithmic) / conv time, peak = the TF32 tensor peak."""
    import torch

    from paper_2303_04670_b200 import _lib

    hbm, bf16, src = peaks()
    S = g.S
    g2 = evc.build(g.spec, _weights_of(g), refresh_interval=0, sessions=S, cuda_graph=False)
    g2.dense_pass(xs[0] if S > 1 else xs[0][0])
    prog = g2._program
    gemm_ms, gemm_flops, step_ms = [], [], []
    nsteps = min(nsteps, xs.shape[0] - 1)
    conv_idx = [n.meter_idx for n in g2.nodes if n.kind == "conv"]
    for i in range(1, 1 + nsteps):
        _lib.check(g2.lib.evc_diff_mask(xs[i - 1].data_ptr(), xs[i].data_ptr(), xs[0][0].numel(),
                                        g2._desc(g2.input_id), S, _lib.stream_ptr()), "diff")
        timed = ({"conv_fused", "conv_gemm"}, [])
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        g2._run_program(timed=timed)
        s1.record()
        torch.cuda.synchronize()
        gemm_ms.append(sum(a.elapsed_time(b) for _, a, b in timed[1]))
        step_ms.append(s0.elapsed_time(s1))
        gemm_flops.append(int(g2._perf_step[conv_idx].sum()))
    t = sum(gemm_ms) / len(gemm_ms) / 1e3
    f = sum(gemm_flops) / len(gemm_flops)
    achieved = f / t / 1e12
    peak = 0.5 * bf16  # dense TF32 tensor peak = 1/2 measured bf16
    n_launch = sum(1 for _, _, n in prog if n in ("conv_fused", "conv_gemm"))
    traffic, tsrc = None, None
    tp = ROOT / "profiles" / "r02_conv_traffic_s32.json"
    if tp.exists():  # ncu DRAM bytes of the same launches (one step), committed under profiles/
        tj = json.loads(tp.read_text())
        if tj.get("sessions") == S and tj.get("launches_per_step") == n_launch and g.spec.name == tj.get("model"):
            traffic, tsrc = tj["dram_bytes_per_step"], f"profiles/{tp.name} ({tj['source']})"
    del g2
    return {"bound": "tensor", "kernel": f"conv_fused (all {n_launch} conv layers incl. fused mask/meter/activation, per step)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
            "frac_of_3xtf32_ceiling": achieved / (peak / 3.0),  # fp32 accuracy: three TF32 MMAs per product
            "traffic_unit": "bytes per step", "traffic_source": tsrc,
            "peak_source": f"0.5 x {src} bf16 ({bf16} TF) as the TF32 tensor peak",
            "algorithmic_flops_per_step": f, "gemm_ms_per_step": t * 1e3, "gemm_launches_per_step": n_launch,
            "gemm_share_of_eager_step": (sum(gemm_ms) / sum(step_ms)) if step_ms else None}


def _weights_of(g):
    out = {}
    for n in g.nodes:
        if n.weight is not None:
            out[f"{n.spec.id}.weight"] = n.weight.cpu().numpy()
            if n.bias is not None:
                out[f"{n.spec.id}.bias"] = n.bias.cpu().numpy()
    return out


def measure_e2e(g, xs, args, S, world=1, dev=None):
    """Same metric through the public serving API with host buffers: every step uploads
    its new encodings from pinned memory, runs step_from_encodings (+refresh) and
    downloads its integrated output (serving.StreamPipeline overlaps those copies with
    the neighbouring steps' compute).  Wall clock incl. Python, from the first upload to
    the last download."""
    import torch

    from paper_2303_04670_b200.serving import StreamPipeline

    n = min(args.steps, xs.shape[0] - 2)
    host = xs[: n + 1].cpu().pin_memory()
    y = g._y_run[g.output_ids[0]]
    out_host = torch.empty((n, *y.shape), dtype=torch.float32).pin_memory()
    pipe = StreamPipeline(g)
    g.dense_pass(xs[0] if S > 1 else xs[0][0])
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    t0 = time.perf_counter()
    pipe.run(host, out_host, dense_first=False)
    wall = time.perf_counter() - t0
    wall = _shard.job_time_ms(wall * 1e3, world, dev) / 1e3  # slowest rank (every rank ran n steps)
    return {"value": n * S * world / wall, "unit": UNIT, "h2d_bytes_per_step": int(host[0].numel() * 4),
            "d2h_bytes_per_step": int(out_host[0].numel() * 4), "ms_per_step": wall / n * 1e3,
            "copies": "H2D / D2H on a copy stream, overlapped with the neighbouring steps' compute"}


E2E_RUNS = 3  # end-to-end runs of 63 increments each; `value` is their median


def measure_e2e_events(evc, g, streams, args, S, world=1, dev=None):
    """The metric end to end from raw events (serving.EventPipeline): every step uploads only the
    packed EVB records that arrived since the previous window end (13 B per event, pinned), bins
    the windows on the device, runs step_increment + incr_step (+ refresh) and downloads the
    integrated output.  Wall clock incl. Python, first upload to last download; the median of
    E2E_RUNS runs (all reported in `run_values`)."""
    import torch

    n = 63  # one dense pass (the first window) per 64 windows: the steady state of refresh_interval 64
    taus = [[WINDOW_US + SHIFT_US * i for i in range(n + 1)] for _ in range(S)]
    recs = [evc.pack_records(st) for st in streams]
    ts = [st.t for st in streams]
    pipe = evc.EventPipeline(g, (256, 256), "count+timestamp", window_us=WINDOW_US)
    y = g._y_run[g.output_ids[0]]
    out_host = torch.empty((n, *y.shape), dtype=torch.float32).pin_memory()
    pipe.run(recs, ts, [t[:3] for t in taus], out_host[:2])  # warm-up (allocations, graph capture)
    torch.cuda.synchronize()
    walls = []
    for _ in range(E2E_RUNS):  # the host loop's wall clock is noisy on a shared box: median of runs
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        t0 = time.perf_counter()
        pipe.run(recs, ts, taus, out_host)
        wall = time.perf_counter() - t0
        walls.append(_shard.job_time_ms(wall * 1e3, world, dev) / 1e3)
    wall = statistics.median(walls)
    steady = pipe.h2d_bytes[1:]
    return {"value": n * S * world / wall, "unit": UNIT, "h2d_bytes_per_step": int(sum(steady) / len(steady)),
            "d2h_bytes_per_step": int(out_host[0].numel() * 4), "ms_per_step": wall / n * 1e3,
            "runs": len(walls), "run_values": [round(n * S * world / w, 1) for w in walls],
            "h2d_bytes_first_window": int(pipe.h2d_bytes[0]),
            "copies": ("raw events in: each step's new packed EVB records (13 B/event) of every stream H2D from "
                       "pinned memory, device ring + binning (evc_ingest_ring, evc_encode_windows), the step, "
                       "the integrated output D2H; copies overlapped with the neighbouring steps' compute")}


# ---------------------------------------------------------------------------
# C2 / C3 / C4 sub-results (N = 1)
# ---------------------------------------------------------------------------


def graph_config(evc, spec, frames, S, steps, warmup, cpu_fn, cpu_budget, label):
    """Rate (S sessions), single-stream p50 latency, conv roofline and CPU baseline of one model config."""
    import torch

    weights = evc.WeightManifest.random_tensors(spec, 0)
    n_win = 1 + warmup + steps + 1
    xs = make_inputs(frames, _shard.stream_seeds(0, S))
    density = float((xs[1:] != xs[:-1]).float().mean())
    g = evc.build(spec, weights, refresh_interval=64, sessions=S)
    times, refreshes, _ = timed_steps(g, xs, steps, warmup)
    refresh_ms = time_refresh(g, xs[0] if S > 1 else xs[0][0], reps=1)
    cost = sum(times) + refresh_ms * max(0.0, steps / 64.0 - refreshes)
    roof = conv_roofline(g, xs, evc, nsteps=4)
    del g
    g1 = evc.build(spec, weights, refresh_interval=64, sessions=1)
    t1, _, _ = timed_steps(g1, xs[:, :1].contiguous(), steps, warmup)
    del g1, xs
    torch.cuda.empty_cache()
    s1 = sorted(t1)
    res = {"workload": label, "sessions": S, "increment_density": density, "steps": steps,
           "value": steps * S / (cost / 1e3), "unit": UNIT, "ms_per_step": cost / steps,
           "p50_ms_per_step": statistics.median(times), "refresh_ms": refresh_ms,
           "p50_increment_latency_ms": statistics.median(s1), "p99_increment_latency_ms": pct(s1, 0.99),
           "roofline": {k: roof[k] for k in ("bound", "achieved", "peak", "unit", "frac", "algorithmic_flops_per_step",
                                             "gemm_ms_per_step", "gemm_share_of_eager_step")}}
    if cpu_fn is not None and cpu_budget > 0:
        res["cpu_baseline"] = run_cpu(cpu_fn, cpu_budget)
    return res


def c4_config(evc, iters=10, cpu_budget=0.0):
    """C4: one 64 -> 128 3x3 conv (stride 1, pad 1) at 480x640 inside a device Graph (input ->
    conv), incremental on a tile-clustered increment (fraction d of the 6x6 tiles live in all 64
    channels) vs the same library's dense conv of the full input.  Sparse paths: the
    input-stationary scatter conv (mask/meter kernel + evc_conv_scatter: compaction, gather -> GEMM
    -> scatter-add, per-tile sum) and the output-stationary fused conv (input shadow + any-channel
    map + evc_conv_fused).  Times = CUDA events around the conv's launches, median of `iters`."""
    import numpy as np
    import torch

    from paper_2303_04670_b200.graph import ModelSpec, NodeSpec

    C, H, W, CO = 64, 480, 640, 128
    spec = ModelSpec("c4-conv", (C, H, W), [NodeSpec("conv", "conv", ["input"],
                                                      {"out_channels": CO, "kernel": [3, 3], "stride": 1,
                                                       "padding": 1})], "conv")
    rng = np.random.default_rng(0)
    wt = (rng.standard_normal((CO, C, 3, 3)) * np.sqrt(2.0 / (C * 9))).astype(np.float32)
    graphs = {"scatter": evc.build(spec, {"conv.weight": wt}, refresh_interval=0, sessions=1, cuda_graph=False,
                                   scatter_convs=("conv",)),
              "fused": evc.build(spec, {"conv.weight": wt}, refresh_interval=0, sessions=1, cuda_graph=False)}
    x_dense = torch.from_numpy(rng.standard_normal((C, H, W)).astype(np.float32)).cuda()
    g = graphs["fused"]
    g.dense_pass(x_dense)
    dts = []
    for _ in range(iters):  # dense: the conv's launches of the dense program (input shadow + dense conv)
        g._load_input(x_dense)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g._dense_program(False)
        e1.record()
        torch.cuda.synchronize()
        dts.append(e0.elapsed_time(e1) * 1e3)
    g._clear_increments()
    t_dense = statistics.median(dts)
    graphs["scatter"].dense_pass(x_dense)
    gh, gw = -(-H // 6), -(-W // 6)
    names = {"to_hwc", "tile_any", "conv_fused", "conv_mask", "conv_gemm", "conv_scatter"}
    rows = []
    for d in (0.005, 0.01, 0.02, 0.05, 0.10, 0.20):
        f2 = rng.random((gh, gw)) < d
        px = np.repeat(np.repeat(f2, 6, 0), 6, 1)[:H, :W]
        vals = torch.from_numpy((rng.standard_normal((C, H, W)) * px[None]).astype(np.float32)).cuda()
        flags = torch.from_numpy(np.broadcast_to(f2, (C, gh, gw)).copy()).cuda().to(torch.uint8)
        row = {"live_tiles": d, "mask": "clustered", "dense_us": t_dense}
        for name, gg in graphs.items():
            ts, perf = [], 0
            v, f = gg.input_slot()
            for it in range(iters + 2):
                v.copy_(vals.unsqueeze(0))
                f.copy_(flags.unsqueeze(0))
                torch.cuda.synchronize()
                timed = (names, [])
                gg._run_program(timed=timed)
                torch.cuda.synchronize()
                if it >= 2:  # (the first two calls settle the region / tile state of the new mask)
                    ts.append(sum(a.elapsed_time(b) for _, a, b in timed[1]) * 1e3)
                    perf = int(gg._perf_step[0, 0])
            row[f"{name}_us"] = statistics.median(ts)
            row["performed_over_dense"] = perf / gg._dense_static[0]
        row["sparse_us"] = row["scatter_us"]
        row["sparse_over_dense"] = row["scatter_us"] / t_dense
        rows.append(row)
    cross = max([r["live_tiles"] for r in rows if r["sparse_us"] < t_dense], default=None)
    del graphs, g
    torch.cuda.empty_cache()
    res = {"workload": "C4 single 3x3 conv 64->128 @480x640, tile-clustered increments (Graph, conv launches timed)",
           "dense_us": t_dense, "sweep": rows, "sparse_faster_than_dense_up_to": cross,
           "sparse_path": "input-stationary scatter conv (evc_conv_mask + evc_conv_scatter)"}
    if cpu_budget > 0:
        res["cpu_baseline"] = run_cpu(("c4", 0.02), cpu_budget)
    return res


def sub_configs(evc, configs, want, args):
    steps = max(4, min(args.steps, 16))
    warmup = args.warmup
    n_win = 1 + warmup + steps + 1
    budget = args.sub_cpu_budget if not args.no_cpu_baseline else 0.0
    out = {}
    if "c2" in want:
        spec = configs.unet_e2depth_spec(tp=0.0)
        for name, rate in C2_RATES.items():
            out[f"C2_{name}"] = graph_config(
                evc, spec, lambda sd, r=rate: c2_frames(evc, sd, n_win, r), 8, steps, warmup,
                ("c2", rate) if name == "1%" else None, budget,
                f"C2 E2Depth-style UNet (levels 4, base 32) on 5-bin voxels 264x352, ~{name} increment density, "
                f"8 streams batched")
    if "c3" in want:
        out["C3"] = graph_config(evc, configs.resnet18_spec(tp=0.0), lambda sd: c3_frames(evc, sd, n_win), 32, steps,
                                 warmup, ("c3", 2.0e5), budget,
                                 "C3 ResNet-18 (fc 101) on 2x180x240 count histograms, 32 streams batched")
    if "c4" in want:
        out["C4"] = c4_config(evc, cpu_budget=budget)
    return out


# ---------------------------------------------------------------------------
# CPU reference arm (oracle port of evincr's algorithm)
# ---------------------------------------------------------------------------


def _cpu_worker(seed, n_incr, budget_s, q):
    import paper_2303_04670_b200.configs as configs  # spec only (no CUDA)
    from paper_2303_04670_b200.graph import WeightManifest
    from paper_2303_04670_b200.synth import generate_events
    from oracle import evincr_np as O

    spec = configs.evflownet_spec(tp=0.0)
    weights = WeightManifest.random_tensors(spec, 0)
    stream = generate_events(seed=seed, duration_us=WINDOW_US + SHIFT_US * (n_incr + 1), rate_hz=RATE_HZ,
                             n_objects=8, sensor_size=(256, 256))

    def enc(i):
        lo, hi = O.slice_window(stream.t, WINDOW_US + SHIFT_US * i, WINDOW_US)
        a = O.encode(stream.t, stream.x, stream.y, stream.p, lo, hi, WINDOW_US + SHIFT_US * i, WINDOW_US, 256, 256,
                     "count")
        b = O.encode(stream.t, stream.x, stream.y, stream.p, lo, hi, WINDOW_US + SHIFT_US * i, WINDOW_US, 256, 256,
                     "timestamp")
        return np.concatenate([a, b])

    g = O.OracleGraph(spec.to_dict(), weights, refresh_interval=64, conv_impl="refalg")
    prev = enc(0)
    g.dense_pass(prev)
    times = []
    t_start = time.perf_counter()
    for i in range(1, n_incr + 1):
        cur = enc(i)  # encoding is outside the reference's timed region (bench.py:184)
        t0 = time.perf_counter()
        dv, df = O.step_increment(prev, cur, 6, 6)
        g.incr_step(dv, df)
        if g.refresh_due:
            g.refresh(cur)
        times.append(time.perf_counter() - t0)
        prev = cur
        if time.perf_counter() - t_start > budget_s:
            break
    q.put(times)


def cpu_baseline(budget_s=20.0, procs=1, n_incr=64):
    """Time the reference algorithm on the host cores; returns the cpu_baseline dict."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    cores = len(os.sched_getaffinity(0))
    env_threads = os.environ.get("OPENBLAS_NUM_THREADS")
    if procs > 1:
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ps = [ctx.Process(target=_cpu_worker, args=(1000 + r, n_incr, budget_s, q)) for r in range(procs)]
    t0 = time.perf_counter()
    for p in ps:
        p.start()
    res = [q.get() for _ in ps]
    for p in ps:
        p.join()
    wall = time.perf_counter() - t0
    if env_threads is None:
        os.environ.pop("OPENBLAS_NUM_THREADS", None)
    else:
        os.environ["OPENBLAS_NUM_THREADS"] = env_threads
    n = sum(len(r) for r in res)
    busy = max(sum(r) for r in res)
    allt = sorted(t for r in res for t in r)
    threads = procs if procs > 1 else int(env_threads or cores)
    return {"value": n / busy if procs == 1 else n / max(sum(r) for r in res), "unit": UNIT, "cores": threads,
            "kind": "port", "p50_ms": 1e3 * statistics.median(allt),
            "sample": f"{n} C1 increments (step_increment+incr_step, reference per-channel conv loop), "
                      f"{procs} process(es), OpenBLAS threads {'1' if procs > 1 else (env_threads or 'default')}, "
                      f"{cores} host cores visible, wall {wall:.1f}s"}


def _cpu_sub_worker(kind, param, budget_s, q):
    """Reference algorithm (oracle port, per-channel conv loop) on one C2 / C3 / C4 sample."""
    import paper_2303_04670_b200.configs as configs  # specs only (no CUDA)
    from paper_2303_04670_b200.graph import WeightManifest
    from paper_2303_04670_b200.synth import generate_events
    from oracle import evincr_np as O

    times = []
    if kind == "c4":
        rng = np.random.default_rng(0)
        C, H, W, CO = 64, 480, 640, 128
        wt = (rng.standard_normal((CO, C, 3, 3)) * np.sqrt(2.0 / (C * 9))).astype(np.float32)
        f2 = rng.random((-(-H // 6), -(-W // 6))) < param
        px = np.repeat(np.repeat(f2, 6, 0), 6, 1)[:H, :W]
        vals = (rng.standard_normal((C, H, W)) * px[None]).astype(np.float32)
        flags = np.broadcast_to(f2, (C, *f2.shape)).copy()
        t_start = time.perf_counter()
        while not times or time.perf_counter() - t_start < budget_s:
            t0 = time.perf_counter()
            O.inc_conv2d_refalg(vals, flags, 6, 6, wt, 1, 1)
            times.append(time.perf_counter() - t0)
        q.put(times)
        return
    if kind == "c2":
        spec = configs.unet_e2depth_spec(tp=0.0)
        hw, enc, pad = (260, 346), ("voxel", 5), (4, 6)
    else:
        spec = configs.resnet18_spec(tp=0.0)
        hw, enc, pad = (180, 240), ("count", 1), (0, 0)
    weights = WeightManifest.random_tensors(spec, 0)
    stream = generate_events(seed=0, duration_us=WINDOW_US + SHIFT_US * 40, rate_hz=param, n_objects=8,
                             sensor_size=hw)

    def frame(i):
        lo, hi = O.slice_window(stream.t, WINDOW_US + SHIFT_US * i, WINDOW_US)
        x = O.encode(stream.t, stream.x, stream.y, stream.p, lo, hi, WINDOW_US + SHIFT_US * i, WINDOW_US, *hw,
                     enc[0], bins=enc[1])
        return np.pad(x, ((0, 0), (0, pad[0]), (0, pad[1])))

    g = O.OracleGraph(spec.to_dict(), weights, refresh_interval=64, conv_impl="refalg")
    prev = frame(0)
    g.dense_pass(prev)
    t_start = time.perf_counter()
    for i in range(1, 39):
        cur = frame(i)
        t0 = time.perf_counter()
        g.incr_step(*O.step_increment(prev, cur, 6, 6))
        times.append(time.perf_counter() - t0)
        prev = cur
        if time.perf_counter() - t_start > budget_s:
            break
    q.put(times)


def run_cpu(job, budget_s):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_cpu_sub_worker, args=(job[0], job[1], budget_s, q))
    t0 = time.perf_counter()
    p.start()
    times = q.get()
    p.join()
    cores = len(os.sched_getaffinity(0))
    what = {"c2": "C2 increments (step_increment + incr_step)", "c3": "C3 increments (step_increment + incr_step)",
            "c4": f"C4 inc_conv2d calls at {job[1]:.0%} clustered live tiles"}[job[0]]
    return {"value": len(times) / sum(times), "unit": UNIT if job[0] != "c4" else "calls/s",
            "cores": int(os.environ.get("OPENBLAS_NUM_THREADS", cores)), "kind": "port",
            "p50_ms": 1e3 * statistics.median(times),
            "sample": f"{len(times)} {what}, reference per-channel conv loop (oracle port), OpenBLAS threads "
                      f"{os.environ.get('OPENBLAS_NUM_THREADS', 'default')}, {cores} host cores visible, "
                      f"wall {time.perf_counter() - t0:.1f}s"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    procs = max(1, min(cores, args.ref_procs or cores))
    budget = args.cpu_budget
    cb = cpu_baseline(budget_s=budget, procs=procs, n_incr=args.steps)
    out = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": "C1 EV-FlowNet 256x256 (4-ch count+timestamp), ~2% increment density",
                      "streams_total": procs, "t_p": 0.0, "refresh_interval": 64},
           "p50_ms": cb["p50_ms"], "cpu_baseline": cb,
           "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def relaunch(n):
    """--gpus N without a launcher: re-exec this script under torch.distributed.run with N ranks."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sessions", type=int, default=int(os.environ.get("EVC_SESSIONS", "32")))
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-procs", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-latency-pass", action="store_true")
    ap.add_argument("--configs", default="c2,c3,c4",
                    help="sub-results at N = 1: comma list of c2, c3, c4 (or 'none')")
    ap.add_argument("--sub-cpu-budget", type=float, default=8.0, help="CPU seconds per sub-config baseline")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args.gpus)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
