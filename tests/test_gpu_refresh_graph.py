"""The dense refresh as a captured CUDA graph (graph.py dense_pass: first run eager, then one capture and
replays) is bit-identical to the eager dense pass, and the batched resets (evc_fill_segments) leave the
increment state exactly as the eager path does: the same inputs through both graphs give bit-identical
outputs for dense passes, refreshes and the increments after them (graph.py:503-565, 573-630)."""

import numpy as np
import pytest
import torch

import paper_2303_04670_b200 as evc
from paper_2303_04670_b200 import configs

pytestmark = pytest.mark.gpu


def _frames(n, shape, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, *shape)).astype(np.float32)
    for i in range(1, n):  # sparse changes between frames
        m = rng.random(shape) < 0.03
        x[i] = np.where(m, x[i], x[i - 1])
    return torch.from_numpy(x).cuda()


@pytest.mark.parametrize("which", ["plain_tp", "evflownet_s2"])
def test_captured_refresh_matches_eager(which):
    if which == "plain_tp":
        spec = evc.build_plain_cnn(depth=3, channels=16, tp=1e-3, in_shape=(2, 48, 64))
        S, shape = 1, (2, 48, 64)
    else:
        spec = configs.evflownet_spec(tp=0.0)
        S, shape = 2, (4, 256, 256)
    w = evc.WeightManifest.random_tensors(spec, 3)
    gs = {cg: evc.build(spec, w, refresh_interval=0, sessions=S, cuda_graph=cg) for cg in (True, False)}
    xs = _frames(10, (S, *shape) if S > 1 else shape, 11)
    outs = {True: [], False: []}
    for cg, g in gs.items():
        for i in range(10):
            if i in (0, 3, 6):  # eager run, capture + replay, replay
                outs[cg].append(g.dense_pass(xs[i]).cpu().numpy())
            else:
                if S > 1:
                    g.step_from_encodings(xs[i - 1], xs[i])
                else:
                    g.incr_step(evc.step_increment(xs[i - 1], xs[i], g.tile))
                outs[cg].append(g.integrated_output(session=0).cpu().numpy())
    assert gs[True]._dense_graph is not None  # the later dense passes were graph replays
    for a, b in zip(outs[True], outs[False]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
