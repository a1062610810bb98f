"""Pin the CPU oracle (oracle/evincr_np.py) against the reference's own outputs.

The fixtures were produced by tests/golden/make_golden.py importing the
real ``evincr`` 0.1.0.  Masks, index lists, FLOP counts and encodings must
match bit-exactly; float values within the SPEC tolerances.
"""

import json

import numpy as np
import pytest

from oracle import evincr_np as O
from evc_testutil import GOLDEN, close, unpack


def test_conv_cases(golden):
    n = len({k.split("/")[1] for k in golden.conv.files})
    assert n >= 60
    for i in range(n):
        c = unpack(golden.conv, f"conv/{i}")
        th, tw = (int(v) for v in c["tile"])
        for impl in (O.inc_conv2d, O.inc_conv2d_refalg):
            y, f, perf, de = impl(c["x"], c["flags"], th, tw, c["w"], int(c["stride"]), int(c["pad"]))
            assert np.array_equal(f, c["yflags"]), (i, impl.__name__)
            assert perf == int(c["performed"]) and de == int(c["dense"]), (i, impl.__name__)
            assert close(y, c["y"]), (i, impl.__name__)
            assert np.array_equal(O.active_index_list(f), np.flatnonzero(c["yflags"]))


def test_upsample(golden):
    for mode in ("nearest", "bilinear"):
        for fct in (2, 4):
            c = unpack(golden.ops, f"up_{mode}_{fct}")
            y, f = O.inc_upsample(c["x"], c["flags"], 6, 6, fct, mode)
            assert np.array_equal(f, c["yflags"])
            assert np.array_equal(y, c["y"])  # same float32 op sequence -> bit-exact


def test_maxpool(golden):
    for key in ("pool_2x2_s2", "pool_3x3_s2", "pool_3x2_s1"):
        c = unpack(golden.ops, key)
        acc = c["acc0"].copy()
        for s in range(c["x"].shape[0]):
            y, f, acc = O.inc_maxpool(c["x"][s], c["flags"][s], 6, 6, acc, tuple(int(v) for v in c["win"]),
                                      int(c["stride"]))
            assert np.array_equal(f, c["yflags"][s])
            assert np.array_equal(y, c["y"][s])
        assert np.array_equal(acc, c["acc"])


@pytest.mark.parametrize("kind", ["relu", "sigmoid", "tanh", "leaky_relu"])
def test_activation(golden, kind):
    c = unpack(golden.ops, f"act_{kind}")
    acc = c["acc0"].copy()
    for s in range(c["x"].shape[0]):
        y, f, acc = O.inc_activation(c["x"][s], c["flags"][s], acc, kind)
        assert np.array_equal(f, c["flags"][s])
        assert np.array_equal(y, c["y"][s])
    assert np.array_equal(acc, c["acc"])


def test_mul(golden):
    c = unpack(golden.ops, "mul")
    sa, sb = c["sa0"].copy(), c["sb0"].copy()
    for s in range(c["a"].shape[0]):
        y, f, sa, sb = O.inc_mul(c["a"][s], c["fa"][s], c["b"][s], c["fb"][s], sa, sb)
        assert np.array_equal(f, c["yflags"][s])
        assert np.array_equal(y, c["y"][s])
    assert np.array_equal(sa, c["sa"]) and np.array_equal(sb, c["sb"])


def test_linear(golden):
    c = unpack(golden.ops, "linear")
    assert np.array_equal(O.flatten_runs(c["x"], 6, 6), c["runflags"].reshape(-1))
    y, perf, de = O.inc_linear(c["x"], 6, 6, c["w"])
    assert perf == int(c["performed"]) and de == int(c["dense"])
    assert close(y, c["y"].reshape(-1))


@pytest.mark.parametrize("name", ["sp_pinned", "sp_tp", "sp_zero"])
def test_sparsify(golden, name):
    c = unpack(golden.ops, name)
    st = O.sparsify_state(c["x0"].shape, tp=float(c["tp"]), k=0.0 if name != "sp_pinned" else 0.37)
    if float(c["tp"]) > 0:
        O.sparsify_reset(st, c["x0"])
    assert st["k"] == float(c["k_init"]) and st["norm_ema"] == float(c["norm_init"])
    for s in range(c["x"].shape[0]):
        y, f = O.sparsify_step(c["x"][s], 6, 6, st)
        assert np.array_equal(y, c["y"][s])
        assert np.array_equal(f, c["yflags"][s])
        assert np.array_equal(st["delta"], c["delta"][s])
        assert st["k"] == float(c["k"][s]) and st["norm_ema"] == float(c["norm"][s])


def test_tile_mask(golden):
    c = unpack(golden.ops, "tilemask")
    assert np.array_equal(O.tile_flags(c["x"], 4, 7), c["flags"])


@pytest.mark.parametrize("key", ["enc_count", "enc_timestamp", "enc_voxel5", "enc_voxel3"])
def test_encode(golden, key):
    c = unpack(golden.enc, key)
    h, w = (int(v) for v in c["hw"])
    kind = key.split("_")[1].rstrip("0123456789")
    for i, tau in enumerate(c["taus"]):
        lo, hi = O.slice_window(c["t"], int(tau), 50_000)
        assert (lo, hi) == tuple(int(v) for v in c["win"][i])
        out = O.encode(c["t"], c["x"], c["y"], c["p"], lo, hi, int(tau), 50_000, h, w, kind, int(c["bins"]))
        assert np.array_equal(out, c["out"][i])  # bit-exact, voxel included


@pytest.mark.parametrize("name", ["plain", "plain_tp", "unet", "delayed", "custom"])
def test_graph(golden, name):
    specs = json.loads((GOLDEN / "graph_specs.json").read_text())
    c = unpack(golden.graph, name)
    g = O.OracleGraph(specs[name], c["weights"], refresh_interval=3)
    y0 = g.dense_pass(c["xin"])
    assert close(y0, c["y0"], 1e-5)
    perf = json.loads(str(c["perf_json"]))
    for s in range(4):
        st = c["steps"][str(s)]
        yup, y, rep = g.incr_step(st["x"], st["flags"])
        assert np.array_equal(yup[1], st["yupflags"])
        assert close(yup[0], st["yup"], 1e-4)
        assert close(y, st["y"], 1e-4)
        assert {k: list(v) for k, v in rep["per_node"].items()} == perf[str(s)]
        assert rep["false_tile_frac"] == json.loads(str(st["ff"]))
        assert g.refresh_due == bool(st["due"])
    fp = g.state_fingerprint()
    assert set(fp) == set(c["fingerprint"])
    for k, v in fp.items():
        assert close(v, c["fingerprint"][k], 1e-4), k
    assert {k: list(v) for k, v in g.flop_report().items()} == json.loads(str(c["flops"]))


