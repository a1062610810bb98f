"""CPU check of the sub-pixel rewrite of "2x bilinear upsample -> 3x3 conv" (csrc/subpixel.cu):
the composed weights (tensors.compose_subpixel) applied to the edge-replicated low-res input, plus
the border-line correction evc_subpixel_border computes (minus the off-image taps of W . U(clamp)),
equal the oracle's conv of the upsample (tensors.py:259-282, 205-228) to float32 rounding."""

import numpy as np
import pytest

from oracle import evincr_np as O
from paper_2303_04670_b200.tensors import compose_subpixel


def subpixel_conv(x, w):
    ci, h, wd = x.shape
    co = w.shape[0]
    wc = compose_subpixel(w).astype(np.float64)
    xp = np.pad(x.astype(np.float64), ((0, 0), (1, 1), (1, 1)), mode="edge")
    lo = np.zeros((4 * co, h, wd))
    for dy in range(3):
        for dx in range(3):
            lo += np.einsum("oi,ihw->ohw", wc[:, :, dy, dx], xp[:, dy:dy + h, dx:dx + wd])
    H, W = 2 * h, 2 * wd
    out = np.zeros((co, H, W))
    for a in range(2):
        for b in range(2):
            out[:, a::2, b::2] = lo[2 * a + b::4]
    u = O.dense_upsample(x, 2, "bilinear").astype(np.float64)
    w64 = w.astype(np.float64)
    for Y in range(H):
        for X in range(W):
            if 0 < Y < H - 1 and 0 < X < W - 1:
                continue
            for kh in range(3):
                for kw in range(3):
                    yy, xx = Y + kh - 1, X + kw - 1
                    if 0 <= yy < H and 0 <= xx < W:
                        continue
                    out[:, Y, X] -= w64[:, :, kh, kw] @ u[:, min(max(yy, 0), H - 1), min(max(xx, 0), W - 1)]
    return out


@pytest.mark.parametrize("ci,co,h,w", [(5, 3, 7, 9), (3, 16, 4, 4), (2, 2, 1, 6)])
def test_subpixel_composition_matches_upsample_conv(ci, co, h, w):
    rng = np.random.default_rng(ci * 100 + co)
    x = rng.standard_normal((ci, h, w)).astype(np.float32)
    wt = rng.standard_normal((co, ci, 3, 3)).astype(np.float32)
    ref = O.dense_conv2d(O.dense_upsample(x, 2, "bilinear"), wt, None, 1, 1)
    got = subpixel_conv(x, wt)
    assert np.abs(got - ref).max() <= 1e-5 * max(1.0, np.abs(ref).max())


def test_subpixel_taps_sum_to_one():
    """Every phase's composed weights carry each kernel tap with total weight 1 (bilinear taps)."""
    w = np.zeros((1, 1, 3, 3), np.float32)
    for kh in range(3):
        for kw in range(3):
            w[:] = 0
            w[0, 0, kh, kw] = 1
            c = compose_subpixel(w)
            assert np.allclose(c.reshape(4, 9).sum(1), 1.0)
