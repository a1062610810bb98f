"""The overlapped serving loop (serving.StreamPipeline) against the serial loop of the
reference's bench (bench.py:196-209): identical outputs, step for step, bit-for-bit."""

import numpy as np
import pytest
import torch

import paper_2303_04670_b200 as evc
from paper_2303_04670_b200.graph import WeightManifest
from paper_2303_04670_b200.models import build_plain_cnn
from paper_2303_04670_b200.serving import StreamPipeline

pytestmark = pytest.mark.gpu


def _frames(n, S, shape, seed=0):
    g = np.random.default_rng(seed)
    x = np.zeros((n + 1, S, *shape), np.float32)
    x[0] = g.standard_normal((S, *shape)).astype(np.float32)
    for i in range(1, n + 1):  # ~3 % of the pixels change per window
        x[i] = x[i - 1]
        m = g.random((S, *shape)) < 0.03
        x[i][m] = g.standard_normal(int(m.sum())).astype(np.float32)
    return torch.from_numpy(x)


@pytest.mark.parametrize("S", [1, 3])
@pytest.mark.parametrize("cuda_graph", [True, False])
def test_pipeline_matches_serial_loop(S, cuda_graph):
    spec = build_plain_cnn(depth=3, channels=8, tp=0.0, in_shape=(2, 36, 36))
    w = WeightManifest.random_tensors(spec, 1)
    n = 9
    frames = _frames(n, S, (2, 36, 36))
    # serial loop
    g1 = evc.build(spec, w, refresh_interval=4, sessions=S, cuda_graph=cuda_graph)
    dev = frames.cuda()
    g1.dense_pass(dev[0] if S > 1 else dev[0][0])
    ref = []
    for i in range(1, n + 1):
        g1.step_from_encodings(dev[i - 1], dev[i])
        if g1.refresh_due:
            g1.dense_pass(dev[i] if S > 1 else dev[i][0])
        ref.append(g1._y_run[g1.output_ids[0]].cpu().numpy().copy())
    # overlapped loop
    g2 = evc.build(spec, w, refresh_interval=4, sessions=S, cuda_graph=cuda_graph)
    host = frames.pin_memory()
    out = torch.empty((n, *g2._y_run[g2.output_ids[0]].shape), dtype=torch.float32).pin_memory()
    assert StreamPipeline(g2).run(host, out) == n
    for i in range(n):
        assert np.array_equal(out[i].numpy().view(np.uint32), ref[i].view(np.uint32)), i


def test_pipeline_needs_pinned_buffers():
    spec = build_plain_cnn(depth=1, channels=4, tp=0.0, in_shape=(2, 12, 12))
    g = evc.build(spec, WeightManifest.random_tensors(spec, 0), refresh_interval=0)
    with pytest.raises(ValueError):
        StreamPipeline(g).run(torch.zeros(3, 2, 12, 12), torch.zeros(2, 2, 12, 12))
