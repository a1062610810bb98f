"""Recurrent ConvLSTM graphs on the GPU engine vs the oracle.

The `delay` node (graph.py NODE_KINDS) feeds h_{t-1} / c_{t-1} of every ConvLSTM cell; the
oracle's incremental delay rules are pinned to the frame-by-frame recurrence on CPU
(tests/test_recurrent.py).  Here the device Graph runs the same specs: integrated outputs
within 1e-4 every step, output masks and per-node FLOP meters against the oracle (flips
counted and printed), the delayed state (held / pending) against the oracle's, and drift
after the run against a GPU dense recompute.
"""

import numpy as np
import pytest
import torch

import paper_2303_04670_b200 as evc
from paper_2303_04670_b200 import configs
from oracle import evincr_np as O
from evc_testutil import max_err

pytestmark = pytest.mark.gpu


def np_(t):
    return t.detach().cpu().numpy()


def _voxel_frames(n, seed, rate):
    stream = evc.generate_events(seed=seed, duration_us=50_000 + 1_000 * (n + 1), rate_hz=rate, n_objects=8,
                                 sensor_size=(260, 346))
    return [torch.nn.functional.pad(evc.encode(evc.slice_window(stream, 50_000 + 1_000 * i, 50_000),
                                               evc.parse_encoder("voxel:5")), (0, 6, 0, 4)).contiguous()
            for i in range(n + 1)]


def _run(spec, weights, xs, S_check=None):
    g = evc.build(spec, weights, refresh_interval=0)
    og = O.OracleGraph(spec.to_dict(), weights, refresh_interval=0)
    e0 = max_err(np_(g.dense_pass(xs[0])), og.dense_pass(np_(xs[0])))
    assert e0 <= 1e-4, e0
    worst, flips, perf_rel, exact, nodes = 0.0, 0, 0.0, 0, 0
    for i in range(1, len(xs)):
        rv, rf = O.step_increment(np_(xs[i - 1]), np_(xs[i]), 6, 6)
        yup, y, rep = g.incr_step(evc.step_increment(xs[i - 1], xs[i], spec.tile))
        (ov, of), oy, orep = og.incr_step(rv, rf)
        flips += int((yup.mask.numpy() != of).sum())
        for k, (p, d) in rep.per_node.items():
            rp = orep["per_node"][k][0]
            nodes += 1
            exact += int(p == rp)
            perf_rel = max(perf_rel, abs(p - rp) / max(1, d))
        worst = max(worst, max_err(np_(y), oy))
    fg, fo = g.state_fingerprint(), og.state_fingerprint()
    held = max(max_err(fg[k], fo[k]) for k in fo if k.endswith(".held") or k.endswith(".pend"))
    d = g.drift(g.dense_oracle(xs[-1]))
    return worst, flips, perf_rel, exact, nodes, held, d, float(np.abs(np_(g.integrated_output())).max())


def test_small_convlstm_unet_64_increments_vs_oracle():
    spec = configs.recurrent_unet_spec(levels=2, base=8, in_shape=(2, 48, 64))
    weights = evc.WeightManifest.random_tensors(spec, 1)
    rng = np.random.default_rng(4)
    x = rng.standard_normal(spec.input_shape).astype(np.float32)
    xs = [torch.from_numpy(x).cuda()]
    for _ in range(64):
        x = x.copy()
        m = rng.random(x.shape) < 0.02
        x[m] += rng.standard_normal(int(m.sum())).astype(np.float32)
        xs.append(torch.from_numpy(x).cuda())
    worst, flips, perf_rel, exact, nodes, held, d, scale = _run(spec, weights, xs)
    print(f"ConvLSTM UNet 2x48x64, 64 increments: max err {worst:.2e}, output-mask flips {flips}, "
          f"exact meters {exact}/{nodes}, max meter rel {perf_rel:.2e}, delay state err {held:.2e}, drift {d:.2e}")
    assert worst <= 1e-4 and held <= 1e-4
    # value-derived intermediate masks (sparsify of [x, h_prev]) may flip at rounding zeros; one flipped
    # 6x6 tile moves a layer's meter of this small map by ~1e-3 of dense
    assert exact >= 0.99 * nodes and perf_rel <= 2e-3 and flips <= 8
    assert d <= 1e-4 * max(1.0, scale)


def test_e2depth_convlstm_voxel_c2_shape_vs_oracle():
    """E2Depth-style recurrent UNet (3 ConvLSTM encoder stages) on 5-bin voxels at the C2 shape."""
    spec = configs.recurrent_unet_spec(levels=3, base=16, in_shape=(5, 264, 352))
    weights = evc.WeightManifest.random_tensors(spec, 0)
    xs = _voxel_frames(8, seed=5, rate=2.0e5)
    worst, flips, perf_rel, exact, nodes, held, d, scale = _run(spec, weights, xs)
    print(f"recurrent UNet 5x264x352, 8 increments: max err {worst:.2e}, flips {flips}, exact meters "
          f"{exact}/{nodes}, delay state err {held:.2e}, drift {d:.2e}")
    assert worst <= 1e-4 and held <= 1e-4 and perf_rel <= 1e-4 and exact >= 0.95 * nodes
    assert d <= 1e-4 * max(1.0, scale)


def test_convlstm_sessions_match_oracle_per_session():
    spec = configs.recurrent_unet_spec(levels=1, base=8, in_shape=(2, 36, 48))
    weights = evc.WeightManifest.random_tensors(spec, 2)
    S = 3
    rng = np.random.default_rng(9)
    x = rng.standard_normal((S, *spec.input_shape)).astype(np.float32)
    g = evc.build(spec, weights, refresh_interval=0, sessions=S)
    ogs = [O.OracleGraph(spec.to_dict(), weights, refresh_interval=0) for _ in range(S)]
    g.dense_pass(torch.from_numpy(x).cuda())
    for s in range(S):
        ogs[s].dense_pass(x[s])
    for _ in range(10):
        prev, x = x, x.copy()
        m = rng.random(x.shape) < 0.03
        x[m] += rng.standard_normal(int(m.sum())).astype(np.float32)
        g.step_from_encodings(torch.from_numpy(prev).cuda(), torch.from_numpy(x).cuda())
        for s in range(S):
            _, oy, _ = ogs[s].incr_step(*O.step_increment(prev[s], x[s], 6, 6))
            assert max_err(np_(g.integrated_output(session=s)), oy) <= 1e-4, s


def test_convlstm_refresh_keeps_recurrence():
    spec = configs.recurrent_unet_spec(levels=1, base=8, in_shape=(2, 36, 48))
    weights = evc.WeightManifest.random_tensors(spec, 6)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(spec.input_shape).astype(np.float32)
    g = evc.build(spec, weights, refresh_interval=4)
    og = O.OracleGraph(spec.to_dict(), weights, refresh_interval=4)
    g.dense_pass(torch.from_numpy(x).cuda())
    og.dense_pass(x)
    for _ in range(12):
        prev, x = x, x.copy()
        m = rng.random(x.shape) < 0.03
        x[m] += rng.standard_normal(int(m.sum())).astype(np.float32)
        _, y, _ = g.incr_step(evc.step_increment(torch.from_numpy(prev).cuda(), torch.from_numpy(x).cuda(), spec.tile))
        _, oy, _ = og.incr_step(*O.step_increment(prev, x, 6, 6))
        if g.refresh_due:
            y = g.refresh(torch.from_numpy(x).cuda())
            oy = og.refresh(x)
        assert max_err(np_(y), oy) <= 1e-4
