"""CPU-only checks of the host side: the C-ABI library, specs, weights, streams."""

import hashlib
import json
import re
import tempfile

import numpy as np
import pytest

import paper_2303_04670_b200 as evc
from paper_2303_04670_b200 import _lib, configs
from oracle import evincr_np as O
from evc_testutil import GOLDEN, ROOT


def header_symbols():
    text = (ROOT / "include" / "evconv.h").read_text()
    return sorted(set(re.findall(r"\b(evc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load(require_cuda=False)
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.evc_version() == _lib.ABI_VERSION


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_conv_table_host_helper():
    lib = _lib.load(require_cuda=False)
    g = _lib.EvcConvGeom(3, 4, 3, 3, 2, 1, 13, 17, 7, 9, 6, 6)
    n = lib.evc_conv_table_len(g)
    tab = np.zeros(n, np.int32)
    assert lib.evc_conv_table_fill(g, tab.ctypes.data) == 0
    ho, wo, kh, kw, K, ghi, gwi, gho, gwo, rows, cols, kdec, rt, ct, boxr, boxc = tab[:16]
    assert (ho, wo, kh, kw, K, ghi, gwi, gho, gwo) == (7, 9, 3, 3, 27, 3, 3, 2, 2)
    # in-bounds tap counts per output row equal the oracle's
    L, inb = O.conv_live_taps(np.ones((1, 3, 3), bool), 6, 6, 13, 17, 3, 3, 2, 1)
    inr = tab[rows:rows + 7 * 6].reshape(7, 6)[:, 2]
    inc = tab[cols:cols + 9 * 6].reshape(9, 6)[:, 2]
    assert np.array_equal(np.outer(inr, inc), inb)


def _table(c_in, c_out, k, st, pad, h, w, th, tw):
    lib = _lib.load(require_cuda=False)
    ho, wo = O.conv_out_hw(h, w, k, k, st, pad)
    g = _lib.EvcConvGeom(c_in, c_out, k, k, st, pad, h, w, ho, wo, th, tw)
    tab = np.zeros(lib.evc_conv_table_len(g), np.int32)
    assert lib.evc_conv_table_fill(g, tab.ctypes.data) == 0
    return tab


def _meter_from_table(tab, flags, c_out):
    """The split used by the conv_mask kernels: weighted live count + border padding term."""
    ho, wo, kh, kw, K, ghi, gwi, gho, gwo, rows, cols, kdec, rt, ct, boxr, boxc = (int(v) for v in tab[:16])
    R = tab[rows:rows + ho * (3 + kh)].reshape(ho, 3 + kh)
    Cc = tab[cols:cols + wo * (3 + kw)].reshape(wo, 3 + kw)
    RT, CT = tab[rt:rt + ghi].astype(np.int64), tab[ct:ct + gwi].astype(np.int64)
    c_in = flags.shape[0]
    if not flags.any():
        return 0
    if flags.all():
        return 2 * kh * kw * c_in * c_out * ho * wo
    term1 = int((flags.astype(np.int64) * RT[None, :, None] * CT[None, None, :]).sum())
    border = 0
    for u in range(ho):
        for v in range(wo):
            d = kh * kw - R[u, 2] * Cc[v, 2]
            if d == 0 or R[u, 1] == 0 or Cc[v, 1] == 0:
                continue
            box = flags[:, R[u, 0]:R[u, 0] + R[u, 1], Cc[v, 0]:Cc[v, 0] + Cc[v, 1]]
            border += d * int(box.reshape(c_in, -1).any(axis=1).sum())
    # the device sums the same border term over host-grouped boxes
    grp, ngrp = int(tab[16]), int(tab[17])
    G = tab[grp:grp + 5 * ngrp].reshape(ngrp, 5)
    border_g = sum(int(d) * int(flags[:, a0:a0 + na, b0:b0 + nb].reshape(c_in, -1).any(axis=1).sum())
                   for a0, na, b0, nb, d in G)
    assert border_g == border
    return 2 * c_out * (term1 + border)


def test_meter_decomposition_matches_reference(golden):
    """The weighted-count + border-term meter equals the reference's per-channel
    loop on every golden conv case (pinned on CPU, no GPU needed)."""
    from evc_testutil import unpack
    n = len({k.split("/")[1] for k in golden.conv.files})
    for i in range(n):
        c = unpack(golden.conv, f"conv/{i}")
        th, tw = (int(v) for v in c["tile"])
        cin, h, w = c["x"].shape
        cout, _, k, _ = c["w"].shape
        tab = _table(cin, cout, k, int(c["stride"]), int(c["pad"]), h, w, th, tw)
        assert _meter_from_table(tab, c["flags"], cout) == int(c["performed"]), i


def _specs():
    return json.loads((GOLDEN / "graph_specs.json").read_text())


@pytest.mark.parametrize("name", ["plain", "plain_tp", "unet", "delayed", "custom"])
def test_spec_roundtrip_and_topo(name):
    d = _specs()[name]
    spec = evc.ModelSpec.from_dict(d)
    assert spec.to_dict() == d
    assert [n.id for n in spec.topo_order()] == [n["id"] for n in O.topo_order(d)]
    with tempfile.TemporaryDirectory() as td:
        spec.save(f"{td}/m.yaml")
        assert evc.ModelSpec.load(f"{td}/m.yaml").to_dict() == d


def test_builders_match_reference_specs():
    s = _specs()
    assert evc.build_plain_cnn(depth=3, channels=6, tp=0.0, in_shape=(2, 24, 30), pool_every=2).to_dict() == s["plain"]
    assert evc.build_unet(evc.UNetConfig(levels=3, base_channels=4, in_shape=(2, 24, 32), tp=0.0,
                                         upsample_mode="bilinear")).to_dict() == s["unet"]
    assert evc.build_delayed_unet(evc.UNetConfig(levels=3, base_channels=4, in_shape=(5, 16, 24),
                                                 tp=0.0)).to_dict() == s["delayed"]


def test_spec_errors():
    N = evc.NodeSpec
    cyc = evc.ModelSpec("c", (1, 8, 8), [N("a", "relu", ["b"]), N("b", "relu", ["a"])], "a")
    with pytest.raises(evc.CycleError):
        cyc.topo_order()
    bad = evc.ModelSpec("c", (1, 8, 8), [N("a", "conv", ["input"], {"out_channels": 2, "kernel": [9, 9]})], "a")
    with pytest.raises(evc.ShapeError):
        bad.infer_shapes()
    with pytest.raises(evc.GraphError):
        evc.ModelSpec("c", (1, 8, 8), [N("a", "add", ["input"])], "a").topo_order()
    with pytest.raises(evc.GraphError):
        evc.ModelSpec("c", (1, 8, 8), [N("a", "nope", ["input"])], "a").topo_order()


def test_weight_generation_matches_reference():
    dig = json.loads((GOLDEN / "host_digests.json").read_text())["weights"]
    specs = {"plain": evc.build_plain_cnn(3, 6, 0.0, (2, 24, 30)),
             "unet": evc.build_unet(evc.UNetConfig(levels=3, base_channels=4, in_shape=(2, 24, 32)))}
    for name, spec in specs.items():
        with tempfile.TemporaryDirectory() as td:
            man = evc.WeightManifest.generate(spec, seed=3, out_dir=td)
            assert hashlib.sha256(man.blob_path.read_bytes()).hexdigest() == dig[name]["sha256"]
            assert man.entries == dig[name]["entries"]
            t = evc.WeightManifest.load(f"{td}/weights.yaml").tensors()
            r = evc.WeightManifest.random_tensors(spec, 3)
            assert all(np.array_equal(t[k], r[k]) for k in r)


def test_weight_manifest_errors():
    spec = evc.build_plain_cnn(1, 2, 0.0, (1, 8, 8))
    with tempfile.TemporaryDirectory() as td:
        man = evc.WeightManifest.generate(spec, seed=0, out_dir=td)
        man.entries[0]["length"] += 4
        with pytest.raises(evc.WeightError):
            man.tensors()


def test_generate_events_matches_reference():
    dig = json.loads((GOLDEN / "host_digests.json").read_text())["synth"]
    for key, ref in dig.items():
        seed, dur, rate, nobj, hw = key.split("_")
        h, w = (int(v) for v in hw.split("x"))
        s = evc.generate_events(int(seed), int(dur), float(rate), int(nobj), (h, w))
        hsh = hashlib.sha256()
        for a in (s.t, s.x, s.y, s.p):
            hsh.update(np.ascontiguousarray(a).tobytes())
        assert len(s) == ref["n"] and hsh.hexdigest() == ref["sha256"], key


def test_event_io_roundtrip():
    s = evc.generate_events(1, 20_000, 2e5, 2, (30, 40))
    with tempfile.TemporaryDirectory() as td:
        evc.write_events(s, f"{td}/a.evb")
        evc.write_events(s, f"{td}/a.csv")
        assert evc.read_events(f"{td}/a.evb") == s
        assert evc.read_events(f"{td}/a.csv", sensor_size=(30, 40)) == s


def test_slice_window_matches_oracle():
    s = evc.generate_events(2, 60_000, 2e5, 3, (20, 20))
    for tau in (0, 10, 50_000, 55_500, 60_000, 90_000):
        w = evc.slice_window(s, tau, 50_000)
        assert (w.lo, w.hi) == O.slice_window(s.t, tau, 50_000)


def test_config_specs():
    c1 = configs.evflownet_spec()
    assert len(c1.nodes) == 58 and c1.parameter_count() == 3_535_128
    assert c1.infer_shapes()[c1.output] == (2, 256, 256)
    c3 = configs.resnet18_spec()
    assert len(c3.nodes) == 67
    sh = c3.infer_shapes()
    assert sh["stem_pool"] == (64, 44, 59) and sh["s3b1_act"] == (512, 6, 8) and sh["fc"] == (101, 1, 1)
    c2 = configs.unet_e2depth_spec()
    assert len(c2.nodes) == 47


def _c1_conv_cfgs(S):
    lib = _lib.load(require_cuda=False)
    spec = configs.evflownet_spec()
    shapes = spec.infer_shapes()
    out = {}
    for n in spec.topo_order():
        if n.kind != "conv":
            continue
        c, h, w = shapes[n.inputs[0]]
        k, st, pad = int(n.attrs["kernel"][0]), int(n.attrs.get("stride", 1)), int(n.attrs.get("padding", 0))
        co = int(n.attrs["out_channels"])
        ho, wo = O.conv_out_hw(h, w, k, k, st, pad)
        g = _lib.EvcConvGeom(c, co, k, k, st, pad, h, w, ho, wo, 6, 6)
        cfg = _lib.EvcConvCfg()
        assert lib.evc_conv_fused_config(g, S, 0, cfg) == 0
        out[n.id] = (cfg.thin, cfg.row, cfg.bn, cfg.splits)
        assert lib.evc_conv_fused_ctas(g, cfg) > 0
    return out


def test_conv_launch_configuration_rules():
    """evc_conv_fused_config: CUDA-core path for the 4-channel input and the
    2-channel heads; packed row mode for the thin decoders; row mode for C_out <= 64; tap mode with
    128-channel blocks for wide layers at many streams, row mode at one stream; split-K when the
    grid is shorter than the SM count."""
    s32, s1 = _c1_conv_cfgs(32), _c1_conv_cfgs(1)
    for cfgs in (s32, s1):
        assert cfgs["enc0"][0] == 1 and all(cfgs[f"pred{i}"][0] == 1 for i in range(4))
        assert cfgs["dec3"][1:3] == (2, 16) and cfgs["dec2"][1:3] == (2, 32)
        assert cfgs["dec1"][1:3] == (1, 64)
        assert cfgs["enc1"][1] == 0  # stride 2: tap mode
    for nid in ("res0a", "res0b", "res1a", "res1b", "dec0"):
        assert s32[nid][1] == 0 and s32[nid][2] == 128, (nid, s32[nid])
        assert s1[nid][1] == 1, (nid, s1[nid])
    assert s32["enc3"][1:] == (0, 128, 1) and s32["res0a"][3] == 1  # 128 CTAs: no split-K
    assert s1["res0a"][3] >= 2 and s1["enc3"][3] >= 2  # short grids: cluster split-K


def test_window_bounds_match_slice_window():
    """serving.window_bounds (all windows of the e2e loop at once) == slice_window per window."""
    from paper_2303_04670_b200.serving import window_bounds

    st = evc.generate_events(seed=3, duration_us=80_000, rate_hz=2.0e5, n_objects=4, sensor_size=(64, 64))
    taus = [0, 5, 1_000, 30_000, 50_000, 50_001, 79_999, 80_000, 95_000]
    for delta in (1, 1_000, 50_000):
        lo, hi = window_bounds(st.t, taus, delta)
        for i, tau in enumerate(taus):
            w = evc.slice_window(st, tau, delta)
            assert (int(lo[i]), int(hi[i])) == (w.lo, w.hi), (tau, delta)
