"""Run-to-run determinism of the device path: two fresh sessions fed the same increments
must produce bit-identical outputs, increment flags and per-node performed-FLOP meters.
(No float atomics on the data path: split-K reduces in a fixed order over DSMEM, norm
partials fold in a fixed order -- see DESIGN.md.)"""

import hashlib
import os

import numpy as np
import pytest
import torch

import paper_2303_04670_b200 as evc
from paper_2303_04670_b200 import configs
from test_gpu_graph import evflownet_inputs

pytestmark = pytest.mark.gpu


def _run(spec, weights, xs, cuda_graph):
    g = evc.build(spec, weights, refresh_interval=0, cuda_graph=cuda_graph)
    g.dense_pass(xs[0])
    out = []
    for i in range(1, len(xs)):
        yup, y, rep = g.incr_step(evc.step_increment(xs[i - 1], xs[i], spec.tile))
        slots = {nid: hashlib.sha1(f.cpu().numpy().tobytes()).hexdigest()[:10]
                 for nid in g._slots for f in [g._slot_view(nid)[1]]} if os.environ.get("EVC_DET_SLOTS") else {}
        out.append((y.detach().cpu().numpy().copy(), yup.mask.numpy().copy(), dict(rep.per_node), slots))
    return out


@pytest.mark.parametrize("cuda_graph", [True, False])
def test_evflownet_bitwise_reproducible(cuda_graph):
    spec = configs.evflownet_spec(tp=0.0)
    weights = evc.WeightManifest.random_tensors(spec, 0)
    xs = evflownet_inputs(12)
    a = _run(spec, weights, xs, cuda_graph)
    for _ in range(2):
        b = _run(spec, weights, xs, cuda_graph)
        for i, ((ya, fa, pa, sa), (yb, fb, pb, sb)) in enumerate(zip(a, b)):
            assert sa == sb, (i, [k for k in sa if sa[k] != sb[k]])  # every node's tile flags
            assert np.array_equal(fa, fb), i
            assert np.array_equal(ya.view(np.uint32), yb.view(np.uint32)), (i, float(np.abs(ya - yb).max()))
            bad = {k: (pa[k], pb[k]) for k in pa if pa[k] != pb[k]}
            assert not bad, (i, bad)
