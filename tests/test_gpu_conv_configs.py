"""Oracle parity of every fused-conv launch configuration (evc_conv_fused_config branches).

The conv launch configuration depends on the layer geometry, the session count S and the
EVC_FORCE_* / EVC_NO_* knobs (csrc/conv_fused.cu evc_conv_fused_config): thin CUDA-core path,
tap mode, row mode, packed row mode, BN 16..256, cluster split-K, persistent vs one-shot CTAs,
one vs two CTAs per SM.  Each case below pins one branch at a C1 layer shape,
runs two chained increments through a device Graph of S sessions, and compares selected sessions
with the oracle (oracle/evincr_np.py, pinned to the reference by tests/golden):

* ``plain``  input -> conv -> output: conv values (<= 1e-5 normwise), output tile flags and the
  per-step FLOP meter bit-exact (increment_ops.py:126-194);
* ``chain``  input -> sparsify -> conv -> relu -> sparsify -> conv: the conv epilogue runs the
  activation delta and the t_p = 0 sparsify and writes the next conv's input shadow
  (graph.py:573-630 semantics), checked through the second conv's output and every meter.
"""

import zlib

import numpy as np
import pytest
import torch

import paper_2303_04670_b200 as evc
from paper_2303_04670_b200 import _lib
from oracle import evincr_np as O
from evc_testutil import max_err

pytestmark = pytest.mark.gpu

# name: (c_in, c_out, k, stride, pad, H, W, S, live tile fraction, env, expected cfg fields)
CASES = {
    "enc0_thin": (4, 32, 3, 2, 1, 256, 256, 8, 0.3, {}, {"thin": 1}),
    "enc1_tap_persist": (32, 64, 3, 2, 1, 128, 128, 8, 0.9, {}, {"row": 0, "bn": 64, "splits": 1}),
    "enc1_tap_oneshot": (32, 64, 3, 2, 1, 128, 128, 8, 0.9, {"EVC_NO_PERSIST": "1"}, {"row": 0, "bn": 64}),
    "enc2_tap_s32": (64, 128, 3, 2, 1, 64, 64, 32, 0.95, {}, {"row": 0, "bn": 128}),
    "enc3_tap_bn128_s32": (128, 256, 3, 2, 1, 32, 32, 32, 0.95, {}, {"row": 0, "bn": 128}),
    "tap_bn256_s2": (64, 256, 3, 2, 1, 128, 128, 2, 0.9, {}, {"row": 0, "bn": 256}),
    "enc3_tap_s4": (128, 256, 3, 2, 1, 32, 32, 4, 0.95, {}, {"row": 0}),
    "enc3_split_s1": (128, 256, 3, 2, 1, 32, 32, 1, 0.95, {}, {"row": 0}),
    "res_tap_s32": (256, 256, 3, 1, 1, 16, 16, 32, 0.97, {}, {"row": 0, "bn": 128}),
    "res_tap_s8": (256, 256, 3, 1, 1, 16, 16, 8, 0.97, {}, {"row": 0, "bn": 128}),
    "res_row_split_s1": (256, 256, 3, 1, 1, 16, 16, 1, 0.97, {}, {"row": 1, "bn": 64}),
    "res_forced_split3_s2": (256, 256, 3, 1, 1, 16, 16, 2, 0.97, {"EVC_FORCE_SPLITS": "3"}, {"splits": 3}),
    "dec0_tap_s32": (512, 128, 3, 1, 1, 32, 32, 32, 0.95, {}, {"row": 0, "bn": 128}),
    "dec0_tap_s8": (512, 128, 3, 1, 1, 32, 32, 8, 0.95, {}, {"row": 0, "bn": 128}),
    # opt-in persistent BN = 128 (split-small TMEM layout): more items than SMs
    "enc2_persist128_s32": (64, 128, 3, 2, 1, 64, 64, 32, 0.95, {"EVC_PERSIST128": "1"}, {"row": 0, "bn": 128}),
    "dec0_persist128_s32": (512, 128, 3, 1, 1, 32, 32, 32, 0.95, {"EVC_PERSIST128": "1"}, {"row": 0, "bn": 128}),
    "dec0_row_s2": (512, 128, 3, 1, 1, 32, 32, 2, 0.95, {}, {"row": 1, "bn": 64}),
    "dec1_row_bn64_s8": (258, 64, 3, 1, 1, 64, 64, 8, 0.88, {}, {"row": 1, "bn": 64}),
    "dec1_row_oneshot_s8": (258, 64, 3, 1, 1, 64, 64, 8, 0.88, {"EVC_NO_PERSIST": "1"}, {"row": 1}),
    "dec1_tap_forced_s8": (258, 64, 3, 1, 1, 64, 64, 8, 0.88, {"EVC_NO_ROW": "1"}, {"row": 0}),
    "dec2_packed_s8": (130, 32, 3, 1, 1, 128, 128, 8, 0.82, {}, {"row": 2, "bn": 32}),
    "dec2_unpacked_s8": (130, 32, 3, 1, 1, 128, 128, 8, 0.82, {"EVC_NO_PACK": "1"}, {"row": 1, "bn": 32}),
    "dec3_packed_bn16_s4": (66, 16, 3, 1, 1, 256, 256, 4, 0.83, {}, {"row": 2, "bn": 16}),
    "dec3_packed_occ1_s4": (66, 16, 3, 1, 1, 256, 256, 4, 0.83, {"EVC_NO_OCC2": "1"}, {"row": 2}),
    "dec3_tap_rw8_s4": (66, 16, 3, 1, 1, 256, 256, 4, 0.83, {"EVC_NO_ROW": "1", "EVC_FORCE_RW": "8"},
                        {"row": 0, "rw": 8}),
    "mid_tap_bn32_forced": (128, 128, 3, 2, 1, 64, 64, 8, 0.6, {"EVC_FORCE_BN": "32"}, {"row": 0, "bn": 32}),
    "mid_tap_bn16_forced": (64, 64, 3, 1, 1, 64, 64, 8, 0.6, {"EVC_FORCE_BN": "16", "EVC_NO_ROW": "1"},
                            {"row": 0, "bn": 16}),
    "k5_row_s8": (32, 32, 5, 1, 2, 64, 64, 8, 0.5, {}, {"row": 1}),
    "pred_thin_1x1_s8": (16, 2, 1, 1, 0, 256, 256, 8, 0.7, {}, {"thin": 1}),
    "pred_thin_1x1_64ch": (64, 2, 1, 1, 0, 64, 64, 32, 0.7, {}, {"thin": 1}),
}


def _spec(name, c_in, c_out, k, stride, pad, h, w, chain):
    conv = {"kind": "conv", "out_channels": c_out, "kernel": [k, k], "stride": stride, "padding": pad}
    if not chain:
        nodes = [dict(id="c", inputs=["input"], **conv)]
        out = "c"
    else:
        nodes = [{"id": "sp0", "kind": "sparsify", "inputs": ["input"], "tp": 0.0},
                 dict(id="c", inputs=["sp0"], **conv),
                 {"id": "a", "kind": "relu", "inputs": ["c"]},
                 {"id": "sp1", "kind": "sparsify", "inputs": ["a"], "tp": 0.0},
                 {"id": "c2", "kind": "conv", "inputs": ["sp1"], "out_channels": 16, "kernel": [3, 3], "stride": 1,
                  "padding": 1}]
        out = "c2"
    return evc.ModelSpec.from_dict({"name": name, "input": {"id": "input", "shape": [c_in, h, w]}, "tile": [6, 6],
                                    "output": out, "nodes": nodes})


def _increment(rng, shape, density):
    c, h, w = shape
    gh, gw = -(-h // 6), -(-w // 6)
    flags = rng.random((c, gh, gw)) < density
    px = O.flags_to_pixels(flags, 6, 6, h, w)
    v = (rng.standard_normal(shape).astype(np.float32) * px).astype(np.float32)
    return v, O.tile_flags(v, 6, 6)


@pytest.mark.parametrize("chain", [False, True], ids=["plain", "chain"])
@pytest.mark.parametrize("case", sorted(CASES))
def test_conv_config_vs_oracle(case, chain, monkeypatch):
    c_in, c_out, k, stride, pad, h, w, S, dens, env, expect = CASES[case]
    for key in ("EVC_NO_PERSIST", "EVC_NO_ROW", "EVC_NO_PACK", "EVC_NO_OCC2", "EVC_FORCE_BN", "EVC_FORCE_SPLITS",
                "EVC_FORCE_RW"):
        monkeypatch.delenv(key, raising=False)
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    spec = _spec(case, c_in, c_out, k, stride, pad, h, w, chain)
    weights = evc.WeightManifest.random_tensors(spec, 3)
    weights["c.bias"] = np.random.default_rng(9).standard_normal(c_out).astype(np.float32)
    g = evc.build(spec, weights, refresh_interval=0, sessions=S)
    node = g._by_id["c"]
    assert node.plan.path == "fused"
    cfg = {f: int(getattr(node.plan.cfg, f)) for f in ("thin", "row", "bn", "rw", "splits")}
    for f, v in expect.items():
        assert cfg[f] == v, (case, cfg)
    if chain and not cfg["thin"]:
        assert node.fused_sp is not None and node.fused_act is not None  # the epilogue runs act + sparsify
    rng = np.random.default_rng(zlib.crc32(case.encode()))
    x0 = rng.standard_normal((S, c_in, h, w)).astype(np.float32)
    # fp32-grade tolerance: 3xTF32 drops the lo*lo term (~2^-22 per product) and sums in another order
    # than numpy's sgemm; the normwise error grows like sqrt(K), so the 1e-5 bar is
    # scaled for reductions deeper than C1's 3x3x128 = 1152
    tol = 1e-5 * max(1.0, (c_in * k * k / 1152) ** 0.5)
    check = sorted({0, S // 2, S - 1})
    ogs = {s: O.OracleGraph(spec.to_dict(), weights, refresh_interval=0) for s in check}
    y0 = g.dense_pass(torch.from_numpy(x0 if S > 1 else x0[0]).cuda())
    y0 = y0.cpu().numpy().reshape(S, *y0.shape[-3:])
    for s in check:
        e = max_err(y0[s], ogs[s].dense_pass(x0[s]))
        assert e <= tol, (case, "dense", s, e)
    for step in range(2):
        incs = [_increment(rng, (c_in, h, w), dens if step == 0 else dens / 3) for _ in range(S)]
        vals = torch.from_numpy(np.stack([v for v, _ in incs])).cuda()
        flags = torch.from_numpy(np.stack([f for _, f in incs]).astype(np.uint8)).cuda()
        g.incr_step_batch(vals, flags)
        torch.cuda.synchronize()
        ov, of = g._slot_view(spec.output)
        ov, of = ov.cpu().numpy(), of.cpu().numpy().astype(bool)
        for s in check:
            (rv, rf), ry, rep = ogs[s].incr_step(*incs[s])
            assert np.array_equal(of[s], rf), (case, step, s, int((of[s] != rf).sum()))
            e = max_err(ov[s], rv)
            assert e <= tol, (case, step, s, e)
            mine = {kk: v[0] for kk, v in g.step_report(session=s).per_node.items()}
            assert mine == {kk: v[0] for kk, v in rep["per_node"].items()}, (case, step, s)
            e = max_err(g.integrated_output(session=s).cpu().numpy(), ry)
            assert e <= tol, (case, step, s, e)
    _lib.check(0, "ok")
