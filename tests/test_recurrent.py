"""Recurrent-state extension: ConvLSTM graphs through `delay` nodes.

CPU checks of the oracle's incremental delay rules against the frame semantics they restate:
the integrated output of dense_pass(x_0) + incr_step(dx_1) + ... + incr_step(dx_t) must equal
the plain frame-by-frame recurrent network y_t = net(x_t, h_{t-1}, c_{t-1}) (h_{-1} = c_{-1} = 0),
computed here by running the oracle's dense evaluator once per frame with each delay node fed
its source's value of the previous frame.  Also: spec validation of the new kind.
"""

import numpy as np
import pytest

from oracle import evincr_np as O
from paper_2303_04670_b200 import configs
from paper_2303_04670_b200.graph import GraphError, ModelSpec, NodeSpec, ShapeError, WeightManifest
from evc_testutil import max_err


def frames(shape, n, seed, density=0.04):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(shape).astype(np.float32)
    out = [x]
    for _ in range(n):
        x = x.copy()
        m = rng.random(shape) < density
        x[m] += rng.standard_normal(int(m.sum())).astype(np.float32)
        out.append(x)
    return out


def frame_recurrence(spec, weights, xs):
    """y_t of the frame-by-frame recurrent network (no increments anywhere)."""
    og = O.OracleGraph(spec.to_dict(), weights, refresh_interval=0)
    delays = [n for n in og.order if n["kind"] == "delay"]
    prev = {n["id"]: np.zeros(og.shapes[n["id"]], np.float32) for n in delays}
    ys = []
    for x in xs:
        for n in delays:
            og.state[n["id"]]["held"] = prev[n["id"]]
        vals = og._dense(x, False)
        prev = {n["id"]: vals[n["source"]].copy() for n in delays}
        ys.append(vals[og.out_ids[0]])
    return ys


@pytest.mark.parametrize("tp", [0.0])
def test_incremental_convlstm_equals_frame_recurrence(tp):
    spec = configs.recurrent_unet_spec(levels=2, base=4, in_shape=(2, 36, 48), tp=tp)
    weights = WeightManifest.random_tensors(spec, 3)
    xs = frames(spec.input_shape, 12, seed=1)
    ref = frame_recurrence(spec, weights, xs)
    og = O.OracleGraph(spec.to_dict(), weights, refresh_interval=0)
    y0 = og.dense_pass(xs[0])
    assert max_err(y0, ref[0]) <= 1e-5
    worst = 0.0
    for t in range(1, len(xs)):
        _, y, _ = og.incr_step(*O.step_increment(xs[t - 1], xs[t], 6, 6))
        worst = max(worst, max_err(y, ref[t]))
        # the delayed state is the previous frame's hidden state
        fp = og.state_fingerprint()
        assert np.abs(fp["enc0_lstm_hprev.held"]).max() > 0
    assert worst <= 1e-4, worst
    # recurrence matters: the output differs from the stateless (zero-state) network
    og0 = O.OracleGraph(spec.to_dict(), weights, refresh_interval=0)
    assert max_err(og0.dense_oracle(xs[-1]), ref[-1]) > 1e-3


def test_refresh_reanchors_recurrent_state():
    spec = configs.recurrent_unet_spec(levels=1, base=4, in_shape=(2, 24, 30))
    weights = WeightManifest.random_tensors(spec, 5)
    xs = frames(spec.input_shape, 8, seed=2)
    ref = frame_recurrence(spec, weights, xs)
    og = O.OracleGraph(spec.to_dict(), weights, refresh_interval=3)
    og.dense_pass(xs[0])
    for t in range(1, len(xs)):
        _, y, _ = og.incr_step(*O.step_increment(xs[t - 1], xs[t], 6, 6))
        if og.refresh_due:
            y = og.refresh(xs[t])  # dense re-run of frame t with h_{t-1}: same frame value
        assert max_err(y, ref[t]) <= 1e-4, t
        assert max_err(og.dense_oracle(xs[t]), ref[t]) <= 1e-5


def test_recurrent_spec_shapes_and_validation():
    spec = configs.recurrent_unet_spec()  # C2 shape
    shapes = spec.infer_shapes()
    assert shapes[spec.output] == (1, 264, 352)
    assert shapes["enc2_lstm_h"] == (128, 33, 44)
    assert sum(1 for n in spec.nodes if n.kind == "delay") == 6
    bad = [NodeSpec("d", "delay", [], {"source": "nope", "shape": [1, 4, 4]}),
           NodeSpec("y", "add", ["input", "d"], {})]
    with pytest.raises(GraphError, match="delay source"):
        ModelSpec("bad", (1, 4, 4), bad, "y").topo_order()
    wrong = [NodeSpec("d", "delay", [], {"source": "y", "shape": [2, 4, 4]}),
             NodeSpec("y", "relu", ["input"], {})]
    with pytest.raises(ShapeError, match="differs from its source"):
        ModelSpec("bad", (1, 4, 4), wrong, "y").infer_shapes()
    with pytest.raises(GraphError, match="takes no inputs"):
        ModelSpec("bad", (1, 4, 4), [NodeSpec("d", "delay", ["input"], {"source": "d", "shape": [1, 4, 4]})],
                  "d").topo_order()
