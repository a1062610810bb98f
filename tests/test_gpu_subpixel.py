"""Sub-pixel decoder convs (csrc/subpixel.cu, ConvPlan._init_subpixel) against the oracle.

A Graph node chain upsample(2x bilinear) -> sparsify(t_p = 0) -> conv(3x3) runs as ONE composed
3x3 conv on the low-res input (4 x C_out channels) plus a border-line correction.  Checked per step
against the oracle's unfused chain: output flags and per-node FLOP meters bit-exact, values within
1e-5 normwise, over moving sparsity, ragged tiles, image borders, several sessions and a refresh;
and against the same Graph built without the sub-pixel form (it is opt-in: EVC_SUBPIXEL=1).
"""

import numpy as np
import pytest
import torch

import paper_2303_04670_b200 as evc
from oracle import evincr_np as O
from evc_testutil import max_err

pytestmark = pytest.mark.gpu


def _spec(c, h, w, co, act=True, tail=True):
    nodes = [{"id": "up", "kind": "upsample", "inputs": ["input"], "factor": 2, "mode": "bilinear"},
             {"id": "sp", "kind": "sparsify", "inputs": ["up"], "tp": 0.0},
             {"id": "conv", "kind": "conv", "inputs": ["sp"], "out_channels": co, "kernel": [3, 3], "stride": 1,
              "padding": 1}]
    out = "conv"
    if act:
        nodes.append({"id": "act", "kind": "relu", "inputs": ["conv"]})
        out = "act"
    if tail:
        nodes += [{"id": "sp2", "kind": "sparsify", "inputs": [out], "tp": 0.0},
                  {"id": "head", "kind": "conv", "inputs": ["sp2"], "out_channels": 2, "kernel": [1, 1], "stride": 1,
                   "padding": 0},
                  {"id": "tanh", "kind": "tanh", "inputs": ["head"]}]
        out = "tanh"
    return evc.ModelSpec.from_dict({"name": "subpix", "input": {"id": "input", "shape": [c, h, w]}, "tile": [6, 6],
                                    "output": out, "nodes": nodes})


def _increment(rng, c, h, w, d):
    gh, gw = -(-h // 6), -(-w // 6)
    f2 = rng.random((gh, gw)) < d
    px = O.flags_to_pixels(np.broadcast_to(f2, (c, gh, gw)), 6, 6, h, w)
    v = (rng.standard_normal((c, h, w)) * px).astype(np.float32)
    return v, O.tile_flags(v, 6, 6)


@pytest.fixture(autouse=True)
def _subpixel_on(monkeypatch):
    monkeypatch.setenv("EVC_SUBPIXEL", "1")  # opt-in path (tensors.SUBPIXEL_MAX_COUT)


@pytest.mark.parametrize("c,h,w,co,S,fused", [(66, 32, 40, 16, 2, 0), (20, 23, 31, 32, 3, 0), (8, 12, 12, 16, 1, 0),
                                              (41, 14, 18, 16, 2, 0), (72, 12, 14, 16, 1, 0),  # chunks 32+9, 40
                                              (66, 32, 40, 16, 2, 1), (20, 23, 31, 32, 3, 1)])  # one-launch form
def test_subpixel_chain_vs_oracle(c, h, w, co, S, fused, monkeypatch):
    if fused:  # evc_subpixel_input_border (input pass + border GEMM in one launch)
        monkeypatch.setenv("EVC_SUBPIX_FUSED", "1")
    spec = _spec(c, h, w, co)
    weights = evc.WeightManifest.random_tensors(spec, 5)
    g = evc.build(spec, weights, refresh_interval=0, sessions=S)
    assert g._by_id["conv"].plan.subpixel
    ogs = [O.OracleGraph(spec.to_dict(), weights, refresh_interval=0) for _ in range(S)]
    rng = np.random.default_rng(c + h)
    x0 = rng.standard_normal((S, c, h, w)).astype(np.float32)
    y0 = g.dense_pass(torch.from_numpy(x0).cuda())
    for s in range(S):
        r0 = ogs[s].dense_pass(x0[s])
        assert max_err((y0[s] if S > 1 else y0).cpu().numpy(), r0) <= 1e-5
    worst = 0.0
    for step, d in enumerate([0.05, 0.3, 0.0, 1.0, 0.1, 0.02]):
        incs = [_increment(rng, c, h, w, d) for _ in range(S)]
        g.incr_step_batch(torch.from_numpy(np.stack([v for v, _ in incs])).cuda(),
                          torch.from_numpy(np.stack([f for _, f in incs]).astype(np.uint8)).cuda())
        cv, cf = g._slot_view("act")
        cv, cf = cv.cpu().numpy(), cf.cpu().numpy().astype(bool)
        for s in range(S):
            (rv, rf), ry, rep = ogs[s].incr_step(*incs[s])
            assert {k: v[0] for k, v in g.step_report(session=s).per_node.items()} == \
                {k: v[0] for k, v in rep["per_node"].items()}, (step, s)
            assert np.array_equal(g._slot_view("tanh")[1][s].cpu().numpy().astype(bool), rf), (step, s)
            e = max_err(g.integrated_output(session=s).cpu().numpy(), ry)
            worst = max(worst, e)
            assert e <= 1e-5, (step, s, e)
    print(f"sub-pixel chain C={c} {h}x{w} -> {co} S={S}{' (one launch)' if fused else ''}: max err {worst:.2e}")


def test_subpixel_matches_unfused_graph(monkeypatch):
    """The same Graph with and without the sub-pixel form: act values within 1e-5, flags and
    meters identical, for every step (including the dead-region zero restore)."""
    c, h, w, co, S = 34, 20, 26, 16, 2
    spec = _spec(c, h, w, co, tail=False)
    weights = evc.WeightManifest.random_tensors(spec, 9)
    g1 = evc.build(spec, weights, refresh_interval=0, sessions=S)
    monkeypatch.setenv("EVC_SUBPIXEL", "0")
    g2 = evc.build(spec, weights, refresh_interval=0, sessions=S)
    assert g1._by_id["conv"].plan.subpixel and not g2._by_id["conv"].plan.subpixel
    rng = np.random.default_rng(3)
    x0 = torch.from_numpy(rng.standard_normal((S, c, h, w)).astype(np.float32)).cuda()
    g1.dense_pass(x0)
    g2.dense_pass(x0)
    for d in [0.1, 0.0, 0.5, 0.0, 0.03]:
        incs = [_increment(rng, c, h, w, d) for _ in range(S)]
        v = torch.from_numpy(np.stack([a for a, _ in incs])).cuda()
        f = torch.from_numpy(np.stack([b for _, b in incs]).astype(np.uint8)).cuda()
        g1.incr_step_batch(v, f)
        g2.incr_step_batch(v, f)
        a1, f1 = g1._slot_view("act")
        a2, f2 = g2._slot_view("act")
        assert torch.equal(f1, f2)
        assert max_err(a1.cpu().numpy(), a2.cpu().numpy()) <= 1e-5
        # values outside the live output tiles are exact zeros in both
        dead = ~O.flags_to_pixels(f1.cpu().numpy().astype(bool).reshape(-1, *f1.shape[-2:]), 6, 6,
                                  2 * h, 2 * w).reshape(a1.shape)
        assert not np.any(a1.cpu().numpy()[dead])
        for s in range(S):
            assert g1.step_report(session=s).per_node == g2.step_report(session=s).per_node
