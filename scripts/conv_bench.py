"""Isolated timing of the fused conv kernel on the C1 layer geometries.

    python scripts/conv_bench.py [--iters 50] [--mode incr|dense] [--splits N] [--layers dec3,res0a]

Each layer runs with all input tiles live (worst case of an increment) or in
dense mode; CUDA events around `iters` back-to-back launches (L2 warm).
Prints us/launch, the reference-meter FLOPs rate and the executed 3xTF32 rate.
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_04670_b200 import _lib, configs  # noqa: E402
from paper_2303_04670_b200.tensors import ConvPlan, grid_shape  # noqa: E402


def layers():
    spec = configs.evflownet_spec()
    shapes = spec.infer_shapes()
    for n in spec.topo_order():
        if n.kind == "conv":
            ish = shapes[n.inputs[0]]
            yield n.id, ish, n.attrs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--mode", default="incr")
    ap.add_argument("--splits", type=int, default=0)
    ap.add_argument("--layers", default="")
    ap.add_argument("--act", type=int, default=1)
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--sessions", type=int, default=1)
    ap.add_argument("--cin", type=int, default=0)
    ap.add_argument("--subpixel", action="store_true",
                    help="what-if: decoder convs on the low-res input with 4x output channels")
    args = ap.parse_args()
    want = set(args.layers.split(",")) if args.layers else None
    lib = _lib.lib()
    dev = torch.device("cuda")
    s = _lib.stream_ptr()
    tot = 0.0
    for nid, (c, h, w), at in layers():
        if want and nid not in want:
            continue
        if args.cin:  # what-if: the same layer with another input channel count
            c = args.cin
        k = int(at["kernel"][0])
        st, pad, co = int(at.get("stride", 1)), int(at.get("padding", 0)), int(at["out_channels"])
        if args.subpixel and nid.startswith("dec"):
            h, w, co = h // 2, w // 2, 4 * co
        wt = torch.randn(co, c, k, k, device=dev) * (2.0 / (c * k * k)) ** 0.5
        S = args.sessions
        plan = ConvPlan(wt, st, pad, h, w, 6, 6, S, max_splits=args.splits)
        ho, wo = int(plan.g.Ho), int(plan.g.Wo)
        x = torch.randn(S, c, h, w, device=dev)
        gh, gw = grid_shape((c, h, w), type("T", (), {"h": 6, "w": 6})())[1:]
        fl = torch.ones(S, c, gh, gw, dtype=torch.uint8, device=dev)
        y = torch.zeros(S, co, ho, wo, device=dev)
        ya = torch.zeros_like(y)
        acc = torch.zeros_like(y)
        gho, gwo = -(-ho // 6), -(-wo // 6)
        yf = torch.zeros(S, co, gho, gwo, dtype=torch.uint8, device=dev)
        din = _lib.tdesc(x.data_ptr(), fl.data_ptr(), c * h * w, c * gh * gw, c, h, w, 6, 6)
        dout = _lib.tdesc(y.data_ptr(), yf.data_ptr(), co * ho * wo, co * gho * gwo, co, ho, wo, 6, 6)
        dact = _lib.tdesc(ya.data_ptr(), yf.data_ptr(), co * ho * wo, co * gho * gwo, co, ho, wo, 6, 6)
        fany = torch.ones(S * gh * gw, dtype=torch.uint8, device=dev)
        mpart = torch.zeros(S * plan.ctas * 2, dtype=torch.int64, device=dev)
        pre = plan.prep(din)
        _lib.check(pre[0](*pre[1], s), "to_hwc")
        dense = args.mode == "dense"
        act = (0, 0.0, acc.data_ptr(), acc[0].numel(), dact) if args.act else None
        fn, fa = plan.fused(din, None if act else dout, fany=fany.data_ptr(), mpart=mpart.data_ptr(),
                            act=act, dense=dense)
        for _ in range(3):
            _lib.check(fn(*fa, s), "conv_fused")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            fn(*fa, s)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / args.iters
        tot += us
        if args.trace:
            cfg = plan.cfg
            n_cta = int(lib.evc_conv_fused_ctas(plan.g, cfg)) * S
            tb = torch.zeros(n_cta * 16, dtype=torch.int64, device=dev)
            lib.evc_conv_trace(tb.data_ptr())
            fn, fa = plan.fused(din, None if act else dout, fany=fany.data_ptr(), mpart=mpart.data_ptr(),
                                act=act, dense=dense)
            _lib.check(fn(*fa, s), "conv_fused")
            torch.cuda.synchronize()
            lib.evc_conv_trace(None)
            t = tb.view(n_cta, 16).cpu().numpy().astype(np.float64)
            g0 = t[:, 15] - t[:, 15].min()
            names = {1: "live", 2: "tmem", 3: "tma0", 4: "land0", 12: "mma0", 11: "tmaN", 5: "mmaN", 10: "side",
                     6: "accbar", 7: "tmemld", 8: "csync", 9: "emit", 13: "end"}
            line = "   ".join(f"{nm}={np.median(t[:, i]) / 1965:.2f}" for i, nm in names.items())
            print(f"    trace (us from CTA start, median): {line}")
            print(f"    CTA start spread: median {np.median(g0) / 1e3:.2f} us, max {g0.max() / 1e3:.2f} us; "
                  f"CTA duration median {np.median(t[:, 13]) / 1965:.2f} us max {t[:, 13].max() / 1965:.2f}")
        flops = 2.0 * k * k * c * co * ho * wo * S
        cfg = plan.cfg
        print(f"{nid:6s} {c:4d}x{h:3d}x{w:3d} -> {co:3d}x{ho:3d}x{wo:3d} k{k} s{st}  bn={cfg.bn:3d} r={cfg.rh}x{cfg.rw} "
              f"splits={cfg.splits:2d}  {us:8.1f} us  {flops / us * 1e-6:7.1f} TFLOP/s alg  "
              f"{3 * flops * (-(-c // 32) * 32 / c) / us * 1e-6:7.1f} TFLOP/s executed", flush=True)
    print(f"total {tot:.1f} us")


if __name__ == "__main__":
    main()
