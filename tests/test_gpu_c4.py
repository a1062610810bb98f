"""C4 at full size: one 64 -> 128 3x3 conv increment on 480 x 640.

The numpy oracle's value path is too slow at this size, so parity uses what does not
depend on size: the FLOP meter and the output mask bit-exact against the oracle's
meter-only path (conv_meter, increment_ops.py:144-194), the values against an
independent torch fp32 convolution (TF32 off) restricted to the active sites, and
linearity inc(a) + inc(b) = inc(a + b) on the union mask.
"""

import numpy as np
import pytest
import torch

import paper_2303_04670_b200 as evc
from oracle import evincr_np as O
from evc_testutil import close

pytestmark = pytest.mark.gpu

C, H, W, CO = 64, 480, 640, 128


def _incr(vals, flags):
    return evc.IncrementTensor(torch.from_numpy(vals).cuda(), evc.TileMask(torch.from_numpy(flags).cuda(),
                                                                              evc.TileShape(6, 6)))


def _case(d, clustered, seed):
    rng = np.random.default_rng(seed)
    gh, gw = -(-H // 6), -(-W // 6)
    if clustered:  # the same live tiles in all channels
        flags = np.broadcast_to(rng.random((gh, gw)) < d, (C, gh, gw)).copy()
        vals = (rng.standard_normal((C, H, W)) * O.flags_to_pixels(flags, 6, 6, H, W)).astype(np.float32)
    else:  # pixel-uniform: i.i.d. live pixels, the mask is their tiles
        vals = (rng.standard_normal((C, H, W)) * (rng.random((C, H, W)) < d)).astype(np.float32)
        flags = O.tile_flags(vals, 6, 6)
    return vals, flags


def _weights():
    rng = np.random.default_rng(11)
    return (rng.standard_normal((CO, C, 3, 3)) * np.sqrt(2.0 / (C * 9))).astype(np.float32)


def _torch_conv(vals, wt):
    prev = torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32
    torch.backends.cudnn.allow_tf32 = torch.backends.cuda.matmul.allow_tf32 = False
    try:
        y = torch.nn.functional.conv2d(torch.from_numpy(vals).cuda()[None], torch.from_numpy(wt).cuda(), padding=1)[0]
    finally:
        torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32 = prev
    return y.cpu().numpy()


@pytest.mark.parametrize("d,clustered", [(0.005, True), (0.02, True), (0.2, True), (0.01, False)])
def test_c4_full_size_vs_meter_oracle_and_fp32(d, clustered):
    vals, flags = _case(d, clustered, 3)
    wt = _weights()
    meter = evc.FlopCounter()
    y = evc.inc_conv2d(_incr(vals, flags), torch.from_numpy(wt).cuda(), evc.ConvParams.from_weight(wt, 1, 1), meter)
    perf, dense, act = O.conv_meter(flags, 6, 6, H, W, CO, 3, 3, 1, 1)
    assert (meter.performed, meter.dense_equiv) == (perf, dense)
    oflags = np.broadcast_to(O.tiles_any(act[None], 6, 6), (CO, -(-H // 6), -(-W // 6)))
    assert np.array_equal(y.mask.numpy(), oflags)
    ref = _torch_conv(vals, wt)
    ref[:, ~act] = 0.0
    assert close(y.values.cpu().numpy(), ref, 1e-5)


def test_c4_linearity():
    va, fa = _case(0.03, True, 5)
    vb, fb = _case(0.03, False, 6)
    wt = torch.from_numpy(_weights()).cuda()
    p = evc.ConvParams.from_weight(_weights(), 1, 1)
    fu = fa | fb
    ya = evc.inc_conv2d(_incr(va, fu), wt, p, evc.FlopCounter())
    yb = evc.inc_conv2d(_incr(vb, fu), wt, p, evc.FlopCounter())
    yab = evc.inc_conv2d(_incr(va + vb, fu), wt, p, evc.FlopCounter())
    assert np.array_equal(ya.mask.numpy(), yab.mask.numpy())
    assert close((ya.values + yb.values).cpu().numpy(), yab.values.cpu().numpy(), 1e-5)
