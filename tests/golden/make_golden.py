"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``evincr`` 0.1.0 from /root/reference/pkg/src and records
inputs + outputs of the hot-path functions on small seeded cases.  The
fixtures pin ``oracle/evincr_np.py`` (tests/test_oracle_golden.py) and are
read directly by the GPU parity tests.
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import evincr as ev  # noqa: E402
from evincr import increment_ops as iops  # noqa: E402

OUT = Path(__file__).resolve().parent
F32 = np.float32


def rand_increment(rng, shape, tile, p_live):
    c, h, w = shape
    gh, gw = -(-h // tile[0]), -(-w // tile[1])
    flags = rng.random((c, gh, gw)) < p_live
    px = np.repeat(np.repeat(flags, tile[0], 1), tile[1], 2)[:, :h, :w]
    vals = (rng.standard_normal(shape).astype(F32) * px).astype(F32)
    return vals, flags


def conv_cases(rng):
    recs = []
    geoms = []
    for k in (1, 3, 5, 7):
        for st in (1, 2):
            for pad in sorted({0, k // 2, min(k, 3)}):
                for tile in ((6, 6), (4, 5), (1, 1), (3, 7)):
                    geoms.append((k, st, pad, tile))
    rng.shuffle(geoms)
    for i, (k, st, pad, tile) in enumerate(geoms[:72]):
        cin = int(rng.integers(1, 6))
        cout = int(rng.integers(1, 6))
        h = int(rng.integers(k, 19))
        w = int(rng.integers(k, 21))
        p_live = [0.0, 0.1, 0.35, 0.7, 1.0][i % 5]
        vals, flags = rand_increment(rng, (cin, h, w), tile, p_live)
        wt = rng.standard_normal((cout, cin, k, k)).astype(F32)
        mask = ev.TileMask(flags, ev.TileShape(*tile))
        meter = ev.FlopCounter()
        y = iops.inc_conv2d(ev.IncrementTensor(vals, mask), wt, ev.ConvParams.from_weight(wt, st, pad), meter)
        recs.append(dict(x=vals, flags=flags, w=wt, stride=st, pad=pad, tile=np.array(tile),
                         y=y.values, yflags=y.mask.flags, performed=meter.performed, dense=meter.dense_equiv))
    return recs


def op_cases(rng):
    d = {}
    tile = ev.TileShape(6, 6)
    # upsample
    for mode in ("nearest", "bilinear"):
        for f in (2, 4):
            vals, flags = rand_increment(rng, (3, 13, 17), (6, 6), 0.3)
            y = ev.inc_upsample(ev.IncrementTensor(vals, ev.TileMask(flags, tile)), f, mode)
            d[f"up_{mode}_{f}"] = dict(x=vals, flags=flags, y=y.values, yflags=y.mask.flags)
    # maxpool sequences
    for win, st in (((2, 2), 2), ((3, 3), 2), ((3, 2), 1)):
        acc0 = rng.standard_normal((3, 15, 14)).astype(F32)
        state = iops.AccState(acc0.copy())
        xs, fs, ys, yfs = [], [], [], []
        for _ in range(4):
            vals, flags = rand_increment(rng, (3, 15, 14), (6, 6), 0.4)
            y = ev.inc_maxpool(ev.IncrementTensor(vals, ev.TileMask(flags, tile)), state, win, st)
            xs.append(vals); fs.append(flags); ys.append(y.values); yfs.append(y.mask.flags)
        d[f"pool_{win[0]}x{win[1]}_s{st}"] = dict(acc0=acc0, x=np.stack(xs), flags=np.stack(fs), y=np.stack(ys),
                                                  yflags=np.stack(yfs), acc=state.x_acc, win=np.array(win), stride=st)
    # activations
    for kind in ("relu", "sigmoid", "tanh", "leaky_relu"):
        acc0 = rng.standard_normal((4, 14, 13)).astype(F32)
        state = iops.AccState(acc0.copy())
        fn = ev.resolve_activation(kind, 0.01)
        xs, fs, ys = [], [], []
        for _ in range(5):
            vals, flags = rand_increment(rng, (4, 14, 13), (6, 6), 0.5)
            y = ev.inc_activation(ev.IncrementTensor(vals, ev.TileMask(flags, tile)), state, fn)
            xs.append(vals); fs.append(flags); ys.append(y.values)
        d[f"act_{kind}"] = dict(acc0=acc0, x=np.stack(xs), flags=np.stack(fs), y=np.stack(ys), acc=state.x_acc)
    # mul
    sa0 = rng.standard_normal((2, 9, 11)).astype(F32)
    sb0 = rng.standard_normal((2, 9, 11)).astype(F32)
    sa, sb = iops.AccState(sa0.copy()), iops.AccState(sb0.copy())
    xa, fa_, xb, fb_, ys, yfs = [], [], [], [], [], []
    for _ in range(4):
        a, fa = rand_increment(rng, (2, 9, 11), (6, 6), 0.5)
        b, fb = rand_increment(rng, (2, 9, 11), (6, 6), 0.5)
        y = ev.inc_mul(ev.IncrementTensor(a, ev.TileMask(fa, tile)), ev.IncrementTensor(b, ev.TileMask(fb, tile)), sa, sb)
        xa.append(a); fa_.append(fa); xb.append(b); fb_.append(fb); ys.append(y.values); yfs.append(y.mask.flags)
    d["mul"] = dict(sa0=sa0, sb0=sb0, a=np.stack(xa), fa=np.stack(fa_), b=np.stack(xb), fb=np.stack(fb_),
                    y=np.stack(ys), yflags=np.stack(yfs), sa=sa.x_acc, sb=sb.x_acc)
    # linear
    vals, flags = rand_increment(rng, (3, 10, 9), (6, 6), 0.4)
    vals[0, 0, :3] = 0.0  # zero a few live values so value-derived runs differ from tile flags
    mat = rng.standard_normal((7, 270)).astype(F32)
    x = ev.IncrementTensor(vals, ev.TileMask(flags, tile))
    flat = ev.flatten_increment(x)
    meter = ev.FlopCounter()
    y = ev.inc_linear(flat, mat, meter)
    d["linear"] = dict(x=vals, flags=flags, w=mat, y=y.values, runflags=flat.mask.flags,
                       performed=meter.performed, dense=meter.dense_equiv)
    # sparsify: pinned k, and tp > 0 tracking
    for name, tp, k in (("sp_pinned", 0.0, 0.37), ("sp_tp", 0.05, 0.0), ("sp_zero", 0.0, 0.0)):
        shape = (3, 11, 13)
        st = ev.SparsifyState(shape, tp=tp, k=k)
        x0 = rng.standard_normal(shape).astype(F32)
        if tp > 0:
            st.reset(x0)
        k0, n0 = st.k, st.norm_ema
        xs, fs, ys, yfs, ks, norms, deltas = [], [], [], [], [], [], []
        for _ in range(6):
            vals, flags = rand_increment(rng, shape, (6, 6), 0.5)
            y = ev.sparsify_step(ev.IncrementTensor(vals, ev.TileMask(flags, tile)), st)
            xs.append(vals); fs.append(flags); ys.append(y.values); yfs.append(y.mask.flags)
            ks.append(st.k); norms.append(st.norm_ema); deltas.append(st.delta.copy())
        d[name] = dict(x0=x0, tp=tp, k_init=k0, norm_init=n0, x=np.stack(xs), flags=np.stack(fs), y=np.stack(ys),
                       yflags=np.stack(yfs), k=np.array(ks), norm=np.array(norms), delta=np.stack(deltas))
    # make_tile_mask incl. -0.0 and partial tiles
    t = rng.standard_normal((3, 17, 20)).astype(F32)
    t[rng.random(t.shape) < 0.9] = 0.0
    t[0, 0, 0] = -0.0
    d["tilemask"] = dict(x=t, flags=ev.make_tile_mask(t, ev.TileShape(4, 7)).flags)
    return d


def encode_cases():
    d = {}
    for seed, kind, hw, rate in ((1, "count", (40, 52), 2e5), (2, "timestamp", (40, 52), 2e5),
                                 (3, "voxel:5", (26, 34), 3e5), (4, "voxel:3", (30, 30), 4e5)):
        s = ev.generate_events(seed=seed, duration_us=60_000, rate_hz=rate, n_objects=3, sensor_size=hw)
        enc = ev.parse_encoder(kind)
        outs, wins = [], []
        for tau in (10_000, 50_000, 51_000, 60_000):
            w = ev.slice_window(s, tau, 50_000)
            outs.append(ev.encode(w, enc))
            wins.append((w.lo, w.hi))
        d[f"enc_{kind.replace(':', '')}"] = dict(t=s.t, x=s.x, y=s.y, p=s.p, hw=np.array(hw), out=np.stack(outs),
                                               win=np.array(wins), taus=np.array([10_000, 50_000, 51_000, 60_000]),
                                               bins=enc.bins)
    return d


def custom_spec():
    N = ev.NodeSpec
    nodes = [
        N("sp0", "sparsify", ["input"], {"tp": 0.0}),
        N("c0", "conv", ["sp0"], {"out_channels": 6, "kernel": [3, 3], "stride": 1, "padding": 1}),
        N("a0", "leaky_relu", ["c0"], {"alpha": 0.05}),
        N("sp1", "sparsify", ["a0"], {"tp": 0.0}),
        N("c1", "conv", ["sp1"], {"out_channels": 6, "kernel": [3, 3], "stride": 2, "padding": 1}),
        N("g", "sigmoid", ["c1"]),
        N("t", "tanh", ["c1"]),
        N("m", "mul", ["g", "t"]),
        N("pool", "maxpool", ["a0"], {"window": [2, 2], "stride": 2}),
        N("sum", "add", ["m", "pool"]),
        N("up", "upsample", ["sum"], {"factor": 2, "mode": "nearest"}),
        N("cat", "concat", ["up", "a0"]),
        N("sp2", "sparsify", ["cat"], {"tp": 0.0}),
        N("c2", "conv", ["sp2"], {"out_channels": 4, "kernel": [5, 5], "stride": 1, "padding": 2}),
        N("r2", "relu", ["c2"]),
        N("fc", "linear", ["r2"], {"out_features": 5}),
    ]
    return ev.ModelSpec("custom-mix", (3, 24, 20), nodes, output="r2", aux_outputs=["fc"])


def graph_cases():
    specs = {
        "plain": ev.build_plain_cnn(depth=3, channels=6, tp=0.0, in_shape=(2, 24, 30), pool_every=2),
        "plain_tp": ev.build_plain_cnn(depth=3, channels=6, tp=0.02, in_shape=(2, 24, 30)),
        "unet": ev.build_unet(ev.UNetConfig(levels=3, base_channels=4, in_shape=(2, 24, 32), tp=0.0,
                                            upsample_mode="bilinear")),
        "delayed": ev.build_delayed_unet(ev.UNetConfig(levels=3, base_channels=4, in_shape=(5, 16, 24), tp=0.0)),
        "custom": custom_spec(),
    }
    recs = {}
    for gi, (name, spec) in enumerate(specs.items()):
        with tempfile.TemporaryDirectory() as td:
            man = ev.WeightManifest.generate(spec, seed=10 + gi, out_dir=td)
            weights = {k: v.copy() for k, v in man.tensors().items()}
        g = ev.build(spec, weights, refresh_interval=3)
        rng = np.random.default_rng(100 + gi)
        shape = spec.input_shape
        x = rng.standard_normal(shape).astype(F32)
        xin = x.copy()
        y0 = g.dense_pass(x)
        steps = []
        for s in range(4):
            vals, flags = rand_increment(rng, shape, (spec.tile.h, spec.tile.w), 0.25 if s != 2 else 0.0)
            yup, y, rep = g.incr_step(ev.IncrementTensor(vals, ev.TileMask(flags, spec.tile)))
            x = x + vals
            steps.append(dict(x=vals, flags=flags, yup=yup.values, yupflags=yup.mask.flags, y=y,
                              perf=rep.per_node, ff=rep.false_tile_frac, due=g.refresh_due,
                              oracle=g.dense_oracle(x), drift=g.drift(g.dense_oracle(x))))
        fp = g.state_fingerprint()
        recs[name] = dict(spec=spec.to_dict(), weights=weights, xin=xin, y0=y0,
                          steps=steps, fingerprint=fp, flops=g.flop_report().per_node)
    return recs


def synth_digests():
    out = {}
    for seed, dur, rate, nobj, hw in ((0, 30_000, 1e5, 2, (64, 64)), (7, 115_000, 1e6, 8, (256, 256)),
                                      (3, 0, 1e5, 2, (10, 10)), (5, 20_000, 3e5, 8, (260, 346))):
        s = ev.generate_events(seed=seed, duration_us=dur, rate_hz=rate, n_objects=nobj, sensor_size=hw)
        h = hashlib.sha256()
        for a in (s.t, s.x, s.y, s.p):
            h.update(np.ascontiguousarray(a).tobytes())
        out[f"{seed}_{dur}_{int(rate)}_{nobj}_{hw[0]}x{hw[1]}"] = dict(n=len(s), sha256=h.hexdigest())
    return out


def weight_digests():
    out = {}
    for name, spec in (("plain", ev.build_plain_cnn(3, 6, 0.0, (2, 24, 30))),
                       ("unet", ev.build_unet(ev.UNetConfig(levels=3, base_channels=4, in_shape=(2, 24, 32))))):
        with tempfile.TemporaryDirectory() as td:
            man = ev.WeightManifest.generate(spec, seed=3, out_dir=td)
            blob = man.blob_path.read_bytes()
            out[name] = dict(sha256=hashlib.sha256(blob).hexdigest(), entries=man.entries)
    return out


def pack(prefix, d, store):
    """Flatten nested dicts/lists into npz keys."""
    if isinstance(d, dict):
        for k, v in d.items():
            pack(f"{prefix}/{k}" if prefix else str(k), v, store)
    elif isinstance(d, (list, tuple)) and d and isinstance(d[0], dict):
        for i, v in enumerate(d):
            pack(f"{prefix}/{i}", v, store)
    else:
        store[prefix] = np.asarray(d)


def main():
    rng = np.random.default_rng(20240304)
    store = {}
    for i, r in enumerate(conv_cases(rng)):
        pack(f"conv/{i}", r, store)
    np.savez_compressed(OUT / "conv_cases.npz", **store)
    store = {}
    pack("", op_cases(rng), store)
    np.savez_compressed(OUT / "op_cases.npz", **store)
    store = {}
    pack("", encode_cases(), store)
    np.savez_compressed(OUT / "encode_cases.npz", **store)
    recs = graph_cases()
    store = {}
    specs = {}
    for name, r in recs.items():
        specs[name] = r.pop("spec")
        perf = {}
        for si, st in enumerate(r["steps"]):
            perf[str(si)] = {k: list(v) for k, v in st.pop("perf").items()}
            st["ff"] = json.dumps(st["ff"])
        r["flops"] = json.dumps({k: list(v) for k, v in r["flops"].items()})
        r["perf_json"] = json.dumps(perf)
        pack(name, r, store)
    np.savez_compressed(OUT / "graph_cases.npz", **store)
    (OUT / "graph_specs.json").write_text(json.dumps(specs, indent=1))
    (OUT / "host_digests.json").write_text(json.dumps({"synth": synth_digests(), "weights": weight_digests()}, indent=1))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
