"""GPU parity of every operator against the reference's golden vectors and the oracle.

Masks, active index lists, FLOP meters and encodings: bit-exact.
Values: within the SPEC tolerances (1e-5 for single ops, normwise).
"""

import numpy as np
import pytest
import torch

import paper_2303_04670_b200 as evc
from oracle import evincr_np as O
from evc_testutil import close, unpack

pytestmark = pytest.mark.gpu


def np_(t):
    return t.detach().cpu().numpy()


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def incr(vals, flags, tile=(6, 6)):
    return evc.IncrementTensor(T(vals.astype(np.float32)), evc.TileMask(T(flags), evc.TileShape(*tile)))


def test_library_loaded_from_tree():
    from paper_2303_04670_b200 import _lib
    lib = _lib.lib()
    assert lib._name.endswith("paper_2303_04670_b200/libevconv.so")


def test_conv_golden(golden):
    n = len({k.split("/")[1] for k in golden.conv.files})
    for i in range(n):
        c = unpack(golden.conv, f"conv/{i}")
        tile = tuple(int(v) for v in c["tile"])
        x = incr(c["x"], c["flags"], tile)
        w = c["w"]
        meter = evc.FlopCounter()
        y = evc.inc_conv2d(x, T(w), evc.ConvParams.from_weight(w, int(c["stride"]), int(c["pad"])), meter)
        assert np.array_equal(y.mask.numpy(), c["yflags"]), i
        assert meter.performed == int(c["performed"]) and meter.dense_equiv == int(c["dense"]), i
        assert close(np_(y.values), c["y"], 1e-5), i
        assert np.array_equal(np_(y.mask.active_indices()), np.flatnonzero(c["yflags"])), i


@pytest.mark.parametrize("kernel", ["tc", "simt"])
@pytest.mark.parametrize("shape,k,st,pad,d", [((64, 120, 160), 3, 1, 1, 0.02), ((32, 64, 64), 3, 2, 1, 0.3),
                                              ((256, 16, 16), 3, 1, 1, 0.9), ((66, 64, 64), 3, 1, 1, 0.5),
                                              ((16, 64, 64), 1, 1, 0, 0.7), ((2, 45, 61), 7, 2, 3, 0.4),
                                              ((512, 32, 32), 3, 1, 1, 1.0), ((130, 40, 44), 3, 1, 1, 0.6)])
def test_conv_vs_oracle(shape, k, st, pad, d, kernel, monkeypatch):
    from paper_2303_04670_b200 import tensors
    monkeypatch.setattr(tensors, "CONV_KERNEL", kernel)
    rng = np.random.default_rng(7)
    c, h, w = shape
    gh, gw = -(-h // 6), -(-w // 6)
    flags = rng.random((c, gh, gw)) < d
    vals = rng.standard_normal(shape).astype(np.float32) * O.flags_to_pixels(flags, 6, 6, h, w)
    cout = 16 if c < 64 else 128
    wt = (rng.standard_normal((cout, c, k, k)) * np.sqrt(2.0 / (c * k * k))).astype(np.float32)
    meter = evc.FlopCounter()
    y = evc.inc_conv2d(incr(vals, flags), T(wt), evc.ConvParams.from_weight(wt, st, pad), meter)
    ry, rf, perf, de = O.inc_conv2d(vals, flags, 6, 6, wt, st, pad)
    assert np.array_equal(y.mask.numpy(), rf)
    assert (meter.performed, meter.dense_equiv) == (perf, de)
    assert close(np_(y.values), ry, 1e-5)


def test_dense_conv_bias():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((5, 33, 47)).astype(np.float32)
    w = rng.standard_normal((7, 5, 3, 3)).astype(np.float32)
    b = rng.standard_normal(7).astype(np.float32)
    for st, pad in ((1, 1), (2, 0), (2, 1)):
        y = evc.dense_conv2d(T(x), T(w), T(b), st, pad)
        assert close(np_(y), O.dense_conv2d(x, w, b, st, pad), 1e-5)


def test_upsample_golden(golden):
    for mode in ("nearest", "bilinear"):
        for f in (2, 4):
            c = unpack(golden.ops, f"up_{mode}_{f}")
            y = evc.inc_upsample(incr(c["x"], c["flags"]), f, mode)
            assert np.array_equal(y.mask.numpy(), c["yflags"])
            assert np.array_equal(np_(y.values), c["y"])  # same float32 rounding sequence
            assert np.array_equal(np_(evc.dense_upsample(T(c["x"]), f, mode)), O.dense_upsample(c["x"], f, mode))


def test_maxpool_golden(golden):
    for key in ("pool_2x2_s2", "pool_3x3_s2", "pool_3x2_s1"):
        c = unpack(golden.ops, key)
        st = evc.AccState(T(c["acc0"]))
        win = tuple(int(v) for v in c["win"])
        for s in range(c["x"].shape[0]):
            y = evc.inc_maxpool(incr(c["x"][s], c["flags"][s]), st, win, int(c["stride"]))
            assert np.array_equal(y.mask.numpy(), c["yflags"][s])
            assert np.array_equal(np_(y.values), c["y"][s])
        assert np.array_equal(np_(st.x_acc), c["acc"])


def test_maxpool_stride_gaps():
    rng = np.random.default_rng(3)
    vals = rng.standard_normal((2, 30, 30)).astype(np.float32)
    flags = rng.random((2, 5, 5)) < 0.3
    vals *= O.flags_to_pixels(flags, 6, 6, 30, 30)
    acc = rng.standard_normal((2, 30, 30)).astype(np.float32)
    st = evc.AccState(T(acc))
    y = evc.inc_maxpool(incr(vals, flags), st, (2, 2), 9)
    ry, rf, racc = O.inc_maxpool(vals, flags, 6, 6, acc, (2, 2), 9)
    assert np.array_equal(y.mask.numpy(), rf) and np.array_equal(np_(y.values), ry)


@pytest.mark.parametrize("kind", ["relu", "sigmoid", "tanh", "leaky_relu"])
def test_activation_golden(golden, kind):
    c = unpack(golden.ops, f"act_{kind}")
    st = evc.AccState(T(c["acc0"]))
    fn = evc.resolve_activation(kind)
    for s in range(c["x"].shape[0]):
        y = evc.inc_activation(incr(c["x"][s], c["flags"][s]), st, fn)
        assert np.array_equal(y.mask.numpy(), c["flags"][s])
        if kind in ("relu", "leaky_relu"):
            assert np.array_equal(np_(y.values), c["y"][s])
        else:
            assert close(np_(y.values), c["y"][s], 2e-6)
    assert np.array_equal(np_(st.x_acc), c["acc"])


def test_mul_add_golden(golden):
    c = unpack(golden.ops, "mul")
    sa, sb = evc.AccState(T(c["sa0"])), evc.AccState(T(c["sb0"]))
    for s in range(c["a"].shape[0]):
        a, b = incr(c["a"][s], c["fa"][s]), incr(c["b"][s], c["fb"][s])
        y = evc.inc_mul(a, b, sa, sb)
        assert np.array_equal(y.mask.numpy(), c["yflags"][s])
        assert np.array_equal(np_(y.values), c["y"][s])
        z = evc.inc_add(a, b)
        ry, rf = O.inc_add(c["a"][s], c["fa"][s], c["b"][s], c["fb"][s])
        assert np.array_equal(z.mask.numpy(), rf) and np.array_equal(np_(z.values), ry)
    assert np.array_equal(np_(sa.x_acc), c["sa"]) and np.array_equal(np_(sb.x_acc), c["sb"])


def test_linear_golden(golden):
    c = unpack(golden.ops, "linear")
    x = incr(c["x"], c["flags"])
    flat = evc.flatten_increment(x)
    assert np.array_equal(flat.mask.numpy(), c["runflags"])
    meter = evc.FlopCounter()
    y = evc.inc_linear(flat, T(c["w"]), meter)
    assert (meter.performed, meter.dense_equiv) == (int(c["performed"]), int(c["dense"]))
    assert close(np_(y.values), c["y"], 1e-5)
    assert bool(y.mask.flags.all())


@pytest.mark.parametrize("name", ["sp_pinned", "sp_tp", "sp_zero"])
def test_sparsify_golden(golden, name):
    c = unpack(golden.ops, name)
    st = evc.SparsifyState(c["x0"].shape, tp=float(c["tp"]), k=0.37 if name == "sp_pinned" else 0.0)
    if float(c["tp"]) > 0:
        st.reset(T(c["x0"]))
        assert st.k == pytest.approx(float(c["k_init"]), rel=1e-6)
        st.k = float(c["k_init"])  # pin k so every rounding decision is comparable bit-for-bit
        st.norm_ema = float(c["norm_init"])
    for s in range(c["x"].shape[0]):
        y = evc.sparsify_step(incr(c["x"][s], c["flags"][s]), st)
        assert np.array_equal(np_(y.values), c["y"][s]), s
        assert np.array_equal(y.mask.numpy(), c["yflags"][s]), s
        assert np.array_equal(np_(st.delta), c["delta"][s]), s
        assert st.norm_ema == pytest.approx(float(c["norm"][s]), rel=1e-6)
        assert st.k == pytest.approx(float(c["k"][s]), rel=1e-6)
        if float(c["tp"]) > 0:
            st.k, st.norm_ema = float(c["k"][s]), float(c["norm"][s])


def test_tile_mask_and_compact(golden):
    c = unpack(golden.ops, "tilemask")
    m = evc.make_tile_mask(T(c["x"]), evc.TileShape(4, 7))
    assert np.array_equal(m.numpy(), c["flags"])
    rng = np.random.default_rng(0)
    for n, p in ((1, 1.0), (4095, 0.5), (4097, 0.01), (300_001, 0.3), (1 << 20, 0.999)):
        f = rng.random((1, 1, n)) < p
        idx = evc.TileMask(T(f), evc.TileShape(1, 1)).active_indices()
        assert np.array_equal(np_(idx), np.flatnonzero(f))


@pytest.mark.parametrize("key", ["enc_count", "enc_timestamp", "enc_voxel5", "enc_voxel3"])
def test_encode_golden(golden, key):
    c = unpack(golden.enc, key)
    h, w = (int(v) for v in c["hw"])
    s = evc.EventStream((h, w), c["t"], c["x"], c["y"], c["p"])
    kind = key.split("_")[1]
    enc = evc.parse_encoder("voxel:" + kind[5:] if kind.startswith("voxel") else kind)
    for i, tau in enumerate(c["taus"]):
        win = evc.slice_window(s, int(tau), 50_000)
        out = evc.encode(win, enc)
        assert np.array_equal(np_(out), c["out"][i]), (key, i)


def test_step_increment_and_integrate():
    rng = np.random.default_rng(5)
    prev = rng.integers(0, 3, (4, 50, 70)).astype(np.float32)
    cur = prev.copy()
    cur[:, 10:20, 30:44] += 1
    cur[1, 0, 0] = -0.0
    x = evc.step_increment(T(prev), T(cur), evc.TileShape())
    rv, rf = O.step_increment(prev, cur, 6, 6)
    assert np.array_equal(np_(x.values), rv) and np.array_equal(x.mask.numpy(), rf)
    y = evc.integrate(T(prev), x)
    assert np.array_equal(np_(y), O.integrate(prev, rv, rf, 6, 6))


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    from paper_2303_04670_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "_initialized", False)
    monkeypatch.setattr(_lib, "LIB_PATH", tmp_path / "missing.so")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        evc.make_tile_mask(torch.zeros(1, 6, 6), evc.TileShape())


@pytest.mark.parametrize("kind", ["relu", "leaky_relu", "tanh"])
def test_add_act_equals_add_then_activation(kind):
    """evc_add_act (graph fusion of an add read only by an activation) is bit-identical to
    evc_add followed by evc_act_delta (increment_ops.py:226-238)."""
    from paper_2303_04670_b200 import _lib
    lib = _lib.lib()
    rng = np.random.default_rng(5)
    C, H, W = 24, 30, 36
    gh, gw = 5, 6
    fa, fb = rng.random((C, gh, gw)) < 0.3, rng.random((C, gh, gw)) < 0.3
    a = (rng.standard_normal((C, H, W)) * O.flags_to_pixels(fa, 6, 6, H, W)).astype(np.float32)
    b = (rng.standard_normal((C, H, W)) * O.flags_to_pixels(fb, 6, 6, H, W)).astype(np.float32)
    acc0 = rng.standard_normal((C, H, W)).astype(np.float32)
    code = _lib.ACT[kind]
    ta, tb = T(a), T(b)
    tfa, tfb = T(fa.astype(np.uint8)), T(fb.astype(np.uint8))

    def desc(v, f):
        return _lib.tdesc(v.data_ptr(), f.data_ptr(), 0, 0, C, H, W, 6, 6)

    # unfused
    s_v, s_f = torch.zeros_like(ta), torch.zeros_like(tfa)
    y1, f1, acc1 = torch.zeros_like(ta), torch.zeros_like(tfa), T(acc0)
    assert lib.evc_add(desc(ta, tfa), desc(tb, tfb), desc(s_v, s_f), 1, _lib.stream_ptr()) == 0
    assert lib.evc_act_delta(desc(s_v, s_f), acc1.data_ptr(), acc1.numel(), desc(y1, f1), code, 0.01, 1,
                             _lib.stream_ptr()) == 0
    # fused
    y2, f2, acc2 = torch.zeros_like(ta), torch.zeros_like(tfa), T(acc0)
    assert lib.evc_add_act(desc(ta, tfa), desc(tb, tfb), acc2.data_ptr(), acc2.numel(), desc(y2, f2), code, 0.01, 1,
                           _lib.stream_ptr()) == 0
    torch.cuda.synchronize()
    assert np.array_equal(np_(y1).view(np.uint32), np_(y2).view(np.uint32))
    assert np.array_equal(np_(acc1).view(np.uint32), np_(acc2).view(np.uint32))
    assert np.array_equal(np_(f1), np_(f2)) and np.array_equal(np_(f2).astype(bool), fa | fb)


@pytest.mark.parametrize("C", [4, 12, 32])
def test_shadow_layouts_hilo_and_fp32(C):
    """evc_to_hwc (include/evconv.h shadow layout): with cp > 0 each channel is a TF32 head
    plus an exact tail (head + tail == value bit for bit, head has 13 zero low bits); with
    cp < 0 the pixel holds the fp32 values themselves -- the same numbers in half the bytes."""
    from paper_2303_04670_b200 import _lib
    lib = _lib.lib()
    rng = np.random.default_rng(C)
    H, W, S = 14, 17, 2
    cp = -(-C // 4) * 4 if C % 32 else C
    x = rng.standard_normal((S, C, H, W)).astype(np.float32)
    tx = T(x)
    flags = torch.ones((S, C, -(-H // 6), -(-W // 6)), dtype=torch.uint8, device="cuda")
    d = _lib.tdesc(tx.data_ptr(), flags.data_ptr(), C * H * W, flags[0].numel(), C, H, W, 6, 6)
    hl = torch.zeros((S, H, W, 2 * cp), dtype=torch.float32, device="cuda")
    f32 = torch.zeros((S, H, W, cp), dtype=torch.float32, device="cuda")
    assert lib.evc_to_hwc(d, hl.data_ptr(), hl[0].numel(), cp, W, S, _lib.stream_ptr()) == 0
    assert lib.evc_to_hwc(d, f32.data_ptr(), f32[0].numel(), -cp, W, S, _lib.stream_ptr()) == 0
    torch.cuda.synchronize()
    want = x.transpose(0, 2, 3, 1)
    got = np_(f32)
    assert np.array_equal(got[..., :C].view(np.uint32), want.view(np.uint32))
    h = np_(hl)
    if cp % 32 == 0:  # 32-channel chunks [heads | tails]
        h = h.reshape(S, H, W, cp // 32, 2, 32)
        heads, tails = h[..., 0, :].reshape(S, H, W, cp), h[..., 1, :].reshape(S, H, W, cp)
    else:
        heads, tails = h[..., :cp], h[..., cp:]
    assert np.array_equal((heads[..., :C] + tails[..., :C]).view(np.uint32), want.view(np.uint32))
    assert not np.any(heads.view(np.uint32) & 0x1FFF)
