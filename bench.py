"""EV-FlowNet 256x256 incremental inference benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--sessions S] [--impl ours|reference]

A "step" is one incremental pass (step_increment + Graph.incr_step, plus the
refresh when due -- the reference's timed region, bench.py:196-209) for each of
the S independent event streams this rank owns (default 32 per GPU: the C5
layout of 256 streams over 8 GPUs; every launch serves all S streams).  A
second, single-stream pass reports the batch-1 per-increment latency
(p50_increment_latency_ms).  Inputs are count(2) +
timestamp(2) encodings of seeded synthetic 1 MHz streams (generate_events,
8 objects, 256x256), 50 ms windows shifted by 1 ms (~2 % of elements change
per increment), encoded on the GPU before timing and resident in HBM.
Weights: seeded He-normal (WeightManifest.generate), t_p = 0, refresh every 64.

Multi-GPU (torchrun): streams shard across ranks with no collective on the
data path (scaling "weak"); rank 0 prints one JSON line with the max-over-ranks
device time.  ``--impl reference`` times the CPU reference algorithm (the
oracle port of evincr's per-channel loop) on the host cores instead.
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


def make_inputs(evc, n_windows, seeds, device):
    import torch

    per = []
    for seed in seeds:
        stream = evc.generate_events(seed=seed, duration_us=WINDOW_US + SHIFT_US * n_windows, rate_hz=RATE_HZ,
                                     n_objects=8, sensor_size=(256, 256))
        xs = []
        for i in range(n_windows):
            w = evc.slice_window(stream, WINDOW_US + SHIFT_US * i, WINDOW_US)
            xs.append(torch.cat([evc.encode(w, evc.EncoderKind("count")), evc.encode(w, evc.EncoderKind("timestamp"))]))
        per.append(torch.stack(xs))
    return torch.stack(per, dim=1).contiguous()  # (n_windows, S, 4, 256, 256)


def timed_run(evc, spec, weights, S, steps, warmup, rank, world, dev):
    """Build an S-session graph, warm up, and time `steps` steps with CUDA events (L2 flushed between)."""
    import torch

    n_win = 1 + warmup + steps + 1
    seeds = _shard.stream_seeds(rank, S)
    xs = make_inputs(evc, n_win, seeds, dev)  # resident in HBM before timing
    density = float((xs[1:] != xs[:-1]).float().mean())
    g = evc.build(spec, weights, refresh_interval=64, sessions=S)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def dense(i):
        return g.dense_pass(xs[i] if S > 1 else xs[i][0])

    def step(i):
        g.step_from_encodings(xs[i - 1], xs[i])
        if g.refresh_due:
            dense(i)

    dense(0)
    for i in range(1, 1 + warmup):
        step(i)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    refreshes = 0
    with Clocks(dev.index or 0) as clk:
        for j in range(steps):
            flush.fill_(float(j))  # evict L2 between timed steps (256 MiB > 126 MB L2)
            i = 1 + warmup + j
            evs[j][0].record()
            will_refresh = g.refresh_interval and g.step_count + 1 >= g.refresh_interval
            step(i)
            refreshes += bool(will_refresh)
            evs[j][1].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times = [a.elapsed_time(b) for a, b in evs]
    del flush
    return g, xs, times, refreshes, clk, density


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
    res = timed_run(evc, spec, weights, S, args.steps, args.warmup, rank, world, dev)
    g, xs, times, refreshes, clk, density = res
    total_ms = _shard.job_time_ms(sum(times), world, cdev)  # max over ranks
    value = _shard.aggregate_rate(args.steps, S, world, total_ms)
    steady = sorted(times)
    p50 = statistics.median(steady)
    p99 = steady[min(len(steady) - 1, int(round(0.99 * (len(steady) - 1))))]
    launches = g.kernel_launches_per_step() + 1  # + diff_mask
    gpu_launches = args.steps * launches + refreshes * g.dense_launches()
    lat = None
    if S > 1 and not args.no_latency_pass:  # single-stream latency (batch 1), same workload
        g1, _, t1, _, _, _ = timed_run(evc, spec, weights, 1, min(args.steps, 32), args.warmup, rank, world, dev)
        s1 = sorted(t1)
        lat = {"sessions": 1, "p50_ms": statistics.median(s1),
               "p99_ms": s1[min(len(s1) - 1, int(round(0.99 * (len(s1) - 1))))], "steps": len(s1)}
        del g1
    # -- per-kernel timing of the conv GEMMs (dominant kernel) on the launching stream
    roof = conv_roofline(g, xs, args, evc)
    e2e = measure_e2e(g, xs, args, S, world, cdev)
    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": (f"C1 EV-FlowNet 256x256 (4-ch count+timestamp), ~2% increment density, batch 1 "
                                    f"per stream; {S} independent streams per GPU batched into every launch "
                                    f"(C5 layout: 256 streams over 8 GPUs = 32 per GPU)"),
                       "sessions_per_gpu": S, "streams_total": S * world, "t_p": 0.0, "refresh_interval": 64,
                       "window_us": WINDOW_US, "shift_us": SHIFT_US, "increment_density": density,
                       "l2": "flushed between timed steps (256 MiB write, excluded from step events)",
                       "parallelism": f"streams sharded over {world} GPU(s), no collective"},
            "p50_ms": p50, "p99_ms": p99, "refreshes_in_timed_region": refreshes,
            "p50_increment_latency_ms": (lat or {}).get("p50_ms", p50 if S == 1 else None),
            "latency_single_stream": lat,
            "clocks": clk.summary(), "gpu_launches": gpu_launches, "roofline": roof, "e2e": e2e,
        }
    if world > 1:
        dist.barrier()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(budget_s=args.cpu_budget)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def conv_roofline(g, xs, args, evc):
    """Time every conv GEMM launch of a few steps with CUDA events on the launching
    stream; achieved = reference-meter FLOPs (algorithmic) / GEMM time."""
    import torch

    from paper_2303_04670_b200 import _lib

    hbm, bf16, src = peaks()
    # replay the same windows eagerly with events around the GEMM launches
    g2 = evc.build(g.spec, {k: v for k, v in _weights_of(g).items()}, refresh_interval=0, sessions=g.S,
                   cuda_graph=False)
    S = g.S
    g2.dense_pass(xs[0] if S > 1 else xs[0][0])
    prog = g2._program
    gemm_ms, gemm_flops, step_ms = [], [], []
    nsteps = min(8, xs.shape[0] - 1)
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
    tp = Path(__file__).resolve().parent / "profiles" / "r01_conv_traffic_s32.json"
    if tp.exists():  # ncu DRAM bytes of the same 16 launches (one step), committed under profiles/
        tj = json.loads(tp.read_text())
        if tj.get("sessions") == S and tj.get("launches_per_step") == n_launch_expected(g2):
            traffic, tsrc = tj["dram_bytes_per_step"], f"profiles/{tp.name} ({tj['source']})"
    return {"bound": "tensor", "kernel": "conv_fused (all 16 conv layers incl. fused mask/meter/activation, per step)", "achieved": achieved,
            "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes per step",
            "traffic_source": tsrc,
            "peak_source": f"0.5 x {src} bf16 ({bf16} TF) as the TF32 tensor peak",
            "algorithmic_flops_per_step": f, "gemm_ms_per_step": t * 1e3, "gemm_launches_per_step": n_launch,
            "gemm_share_of_eager_step": (sum(gemm_ms) / sum(step_ms)) if step_ms else None}


def n_launch_expected(g):
    return sum(1 for _, _, n in g._program if n in ("conv_fused", "conv_gemm"))


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
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
