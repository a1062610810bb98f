"""C4: one 64 -> 128 3x3 conv increment on 480 x 640; sparse (inc_conv2d,
tile-clustered and pixel-uniform masks) vs the same library's dense conv, over densities.

    python scripts/c4_sweep.py [--iters 20]

Prints per density: sparse us, dense us, speed-up, reference-meter FLOPs and the crossover."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2303_04670_b200 as evc  # noqa: E402

C, H, W, CO = 64, 480, 640, 128


def timeit(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    rng = np.random.default_rng(0)
    wt = torch.from_numpy((rng.standard_normal((CO, C, 3, 3)) * np.sqrt(2.0 / (C * 9))).astype(np.float32)).cuda()
    params = evc.ConvParams.from_weight(wt.cpu().numpy(), 1, 1)
    gh, gw = -(-H // 6), -(-W // 6)
    x_dense = torch.from_numpy(rng.standard_normal((C, H, W)).astype(np.float32)).cuda()
    t_dense = timeit(lambda: evc.dense_conv2d(x_dense, wt, None, 1, 1), args.iters)
    print(f"C4 dense conv 64->128 3x3 @480x640: {t_dense:.1f} us ({2 * 9 * C * CO * H * W / t_dense * 1e-6:.1f} TFLOP/s)")
    print(f"{'density':>8} {'mask':>10} {'sparse_us':>10} {'speedup':>8} {'performed/dense':>16}")
    cross = {}
    for kind in ("clustered", "uniform"):
        for d in (0.005, 0.01, 0.02, 0.05, 0.10, 0.20):
            if kind == "clustered":
                f2 = rng.random((gh, gw)) < d
                flags = np.broadcast_to(f2, (C, gh, gw)).copy()
                px = np.repeat(np.repeat(f2, 6, 0), 6, 1)[:H, :W]
                vals = (rng.standard_normal((C, H, W)) * px[None]).astype(np.float32)
            else:
                vals = (rng.standard_normal((C, H, W)) * (rng.random((C, H, W)) < d)).astype(np.float32)
                flags = None
            xv = torch.from_numpy(vals).cuda()
            if flags is None:
                x = evc.IncrementTensor(xv, evc.make_tile_mask(xv, evc.TileShape(6, 6)))
            else:
                x = evc.IncrementTensor(xv, evc.TileMask(torch.from_numpy(flags).cuda(), evc.TileShape(6, 6)))
            meter = evc.FlopCounter()
            evc.inc_conv2d(x, wt, params, meter)
            t = timeit(lambda: evc.inc_conv2d(x, wt, params, evc.FlopCounter()), args.iters)
            frac = meter.performed / meter.dense_equiv
            print(f"{d:8.3f} {kind:>10} {t:10.1f} {t_dense / t:8.2f} {frac:16.3f}")
            if t < t_dense:
                cross[kind] = d
    print("sparse faster than dense up to density:", cross)


if __name__ == "__main__":
    main()
