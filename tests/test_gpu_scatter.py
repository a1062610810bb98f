"""Input-stationary scatter conv (evc_conv_scatter, csrc/conv_scatter.cu) against the oracle.

inc_conv2d (increment_ops.py:126-194) through the scatter path: values within 1e-5 normwise
(3xTF32, fp32 accumulate), output tile flags and the FLOP meter bit-exact; in a Graph over several
steps whose live tiles move (tiles that die are zeroed exactly: TileMask soundness); and C4 at full
size (64 -> 128, 480 x 640) at 2 % and 20 % tile-clustered density.
"""

import numpy as np
import pytest
import torch

import paper_2303_04670_b200 as evc
from paper_2303_04670_b200 import increment_ops
from oracle import evincr_np as O
from evc_testutil import max_err

pytestmark = pytest.mark.gpu


def _clustered(rng, c, h, w, d, th=6, tw=6):
    f2 = rng.random((-(-h // th), -(-w // tw))) < d
    px = O.flags_to_pixels(np.broadcast_to(f2, (c, *f2.shape)), th, tw, h, w)
    v = (rng.standard_normal((c, h, w)) * px).astype(np.float32)
    return v, O.tile_flags(v, th, tw)


def _uniform(rng, c, h, w, d, th=6, tw=6):
    v = (rng.standard_normal((c, h, w)) * (rng.random((c, h, w)) < d)).astype(np.float32)
    return v, O.tile_flags(v, th, tw)


def _check(vals, flags, wt, pad, monkeypatch, tol=1e-5):
    monkeypatch.setattr(increment_ops, "SCATTER_PATH_BELOW", 1.01)  # force the scatter path
    x = evc.IncrementTensor(torch.from_numpy(vals).cuda(), evc.TileMask(torch.from_numpy(flags).cuda(), evc.TileShape(6, 6)))
    meter = evc.FlopCounter()
    params = evc.ConvParams.from_weight(wt, 1, pad)
    y = evc.inc_conv2d(x, torch.from_numpy(wt).cuda(), params, meter)
    ry, rf, rperf, rde = O.inc_conv2d(vals, flags, 6, 6, wt, 1, pad)
    assert np.array_equal(y.mask.numpy(), rf)
    assert (meter.performed, meter.dense_equiv) == (rperf, rde)
    e = max_err(y.values.cpu().numpy(), ry)
    assert e <= tol, e
    return e


@pytest.mark.parametrize("shape,k,pad,d,kind", [
    ((64, 128, 96, 128), 3, 1, 0.02, "clustered"),
    ((64, 128, 96, 128), 3, 1, 0.2, "clustered"),
    ((64, 128, 96, 128), 3, 1, 0.6, "clustered"),
    ((32, 16, 61, 85), 3, 1, 0.1, "clustered"),      # ragged edge tiles, one channel block
    ((40, 24, 50, 70), 3, 1, 0.002, "uniform"),      # C_in not a multiple of 32, C_out of 16
    ((16, 32, 48, 64), 1, 0, 0.3, "clustered"),      # 1x1
    ((8, 8, 36, 36), 3, 1, 0.0, "clustered"),        # no live tile at all
])
def test_scatter_conv_vs_oracle(shape, k, pad, d, kind, monkeypatch):
    c_in, c_out, h, w = shape
    rng = np.random.default_rng(hash(shape) % 2**32)
    wt = (rng.standard_normal((c_out, c_in, k, k)) * np.sqrt(2.0 / (c_in * k * k))).astype(np.float32)
    vals, flags = (_clustered if kind == "clustered" else _uniform)(rng, c_in, h, w, d)
    _check(vals, flags, wt, pad, monkeypatch)


@pytest.mark.parametrize("d", [0.02, 0.2])
def test_scatter_conv_c4_full_size(d, monkeypatch):
    rng = np.random.default_rng(0)
    wt = (rng.standard_normal((128, 64, 3, 3)) * np.sqrt(2.0 / (64 * 9))).astype(np.float32)
    vals, flags = _clustered(rng, 64, 480, 640, d)
    e = _check(vals, flags, wt, 1, monkeypatch)
    print(f"C4 scatter at {d:.0%} clustered: max err {e:.2e}")


def test_scatter_conv_in_graph_moving_tiles():
    """A Graph conv on the scatter path over steps whose live tiles move: every step's output
    increment (values, flags, meter) against the oracle, incl. tiles that die (zeroed once)."""
    spec = evc.ModelSpec.from_dict({"name": "sc", "input": {"id": "input", "shape": [48, 72, 90]}, "tile": [6, 6],
                                    "output": "conv", "nodes": [{"id": "conv", "kind": "conv", "inputs": ["input"],
                                                                 "out_channels": 40, "kernel": [3, 3], "stride": 1,
                                                                 "padding": 1}]})
    weights = evc.WeightManifest.random_tensors(spec, 4)
    S = 3
    g = evc.build(spec, weights, refresh_interval=0, sessions=S, scatter_convs=("conv",))
    assert g._by_id["conv"].scatter
    ogs = [O.OracleGraph(spec.to_dict(), weights, refresh_interval=0) for _ in range(S)]
    rng = np.random.default_rng(7)
    x0 = rng.standard_normal((S, 48, 72, 90)).astype(np.float32)
    g.dense_pass(torch.from_numpy(x0).cuda())
    for s in range(S):
        ogs[s].dense_pass(x0[s])
    for step in range(5):
        incs = [_clustered(rng, 48, 72, 90, [0.05, 0.3, 0.02, 0.0, 0.15][step]) for _ in range(S)]
        g.incr_step_batch(torch.from_numpy(np.stack([v for v, _ in incs])).cuda(),
                          torch.from_numpy(np.stack([f for _, f in incs]).astype(np.uint8)).cuda())
        ov, of = g._slot_view("conv")
        ov, of = ov.cpu().numpy(), of.cpu().numpy().astype(bool)
        for s in range(S):
            (rv, rf), ry, rep = ogs[s].incr_step(*incs[s])
            assert np.array_equal(of[s], rf), (step, s)
            assert max_err(ov[s], rv) <= 1e-5, (step, s)
            assert {k: v[0] for k, v in g.step_report(session=s).per_node.items()} == \
                {k: v[0] for k, v in rep["per_node"].items()}
            assert max_err(g.integrated_output(session=s).cpu().numpy(), ry) <= 1e-5
