"""Device event ingest, checked against the oracle (oracle/evincr_np.py,
pinned to the reference encoders by tests/golden): EVB records unpacked on the GPU (also from an
out-of-order file), the count increment from only the entering / leaving events, and the
serving pipeline that uploads only each step's new packed records into per-session device rings,
bins the windows on the device and runs the graph -- encodings bit-exact and integrated outputs
within 1e-4 of the oracle fed by O.encode + O.step_increment (events.py:251-302)."""

import numpy as np
import pytest
import torch

import paper_2303_04670_b200 as evc
from oracle import evincr_np as O
from evc_testutil import max_err

pytestmark = pytest.mark.gpu


def _stream(seed=3, size=(96, 128)):
    return evc.generate_events(seed=seed, duration_us=120_000, rate_hz=4e5, n_objects=5, sensor_size=size)


def _oracle_enc(s, tau, delta, kind, bins=1):
    lo, hi = O.slice_window(s.t, tau, delta)
    return O.encode(s.t, s.x, s.y, s.p, lo, hi, tau, delta, *s.sensor_size, kind, bins=bins)


def _bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("shuffle", [False, True])
def test_upload_evb_encodings_vs_oracle(tmp_path, shuffle):
    s = _stream()
    path = tmp_path / "s.evb"
    if shuffle:  # an out-of-order file: read_events stable-sorts it (events.py:64-66)
        rec = evc.pack_records(s)
        perm = np.random.default_rng(0).permutation(len(rec))
        with open(path, "wb") as f:
            f.write(evc.events._EVB_HEADER.pack(evc.events.EVB_MAGIC, *s.sensor_size, len(rec)))
            f.write(rec[perm].tobytes())
        s = evc.read_events(path)
    else:
        evc.write_events(s, path)
    d = evc.upload_evb(path)
    assert d == s
    for got, want in zip(d.device_columns(), (s.t.view(np.int64), s.x.view(np.int16), s.y.view(np.int16), s.p)):
        assert np.array_equal(got.cpu().numpy()[: len(s)], np.asarray(want))
    w = evc.slice_window(d, 80_000, 50_000)
    for kind, bins in (("count", 1), ("timestamp", 1), ("voxel", 5)):
        enc = evc.parse_encoder(kind if kind != "voxel" else "voxel:5")
        a = evc.encode(w, enc).cpu().numpy()
        assert np.array_equal(_bits(a), _bits(_oracle_enc(s, 80_000, 50_000, kind, bins))), kind


@pytest.mark.parametrize("delta,shift", [(50_000, 1_000), (50_000, 7_000), (10_000, 30_000), (50_000, 0),
                                         (20_000, 500)])
def test_count_increment_vs_oracle(delta, shift):
    s = _stream(seed=7)
    tile = evc.TileShape(6, 6)
    for tau in (5_000, 60_000, 90_000):  # the first window starts before the stream
        wp, wc = evc.slice_window(s, tau, delta), evc.slice_window(s, tau + shift, delta)
        inc = evc.count_increment(wp, wc, tile)
        rv, rf = O.step_increment(_oracle_enc(s, tau, delta, "count"), _oracle_enc(s, tau + shift, delta, "count"), 6, 6)
        assert np.array_equal(_bits(inc.values.cpu().numpy()), _bits(rv))
        assert np.array_equal(inc.mask.numpy(), rf)


def test_count_increment_rejects_backward_windows():
    s = _stream()
    with pytest.raises(ValueError):
        evc.count_increment(evc.slice_window(s, 80_000, 50_000), evc.slice_window(s, 70_000, 50_000),
                            evc.TileShape(6, 6))


@pytest.mark.parametrize("ring", [1 << 17, 1 << 15])
def test_event_pipeline_vs_oracle(ring):
    """S = 3 sessions at 1 ms shifts; the small ring wraps every few steps."""
    S, n, size, delta = 3, 8, (60, 84), 20_000
    spec = evc.build_plain_cnn(depth=3, channels=8, tp=0.0, in_shape=(4, *size))
    weights = evc.WeightManifest.random_tensors(spec, 1)
    streams = [evc.generate_events(seed=20 + s, duration_us=delta + 1_000 * (n + 2), rate_hz=1.0e6, n_objects=4,
                                   sensor_size=size) for s in range(S)]
    taus = [[delta + 1_000 * i for i in range(n + 1)] for _ in range(S)]
    g = evc.build(spec, weights, refresh_interval=0, sessions=S)
    pipe = evc.EventPipeline(g, size, "count+timestamp", window_us=delta, ring=ring)
    out = torch.empty((n, S, *g.shapes[spec.output]), dtype=torch.float32).pin_memory()
    pipe.run([evc.pack_records(st) for st in streams], [st.t for st in streams], taus, out)
    torch.cuda.synchronize()

    def enc(st, tau):
        return np.concatenate([_oracle_enc(st, tau, delta, "count"), _oracle_enc(st, tau, delta, "timestamp")])

    for s in range(S):
        og = O.OracleGraph(spec.to_dict(), weights, refresh_interval=0)
        prev = enc(streams[s], taus[s][0])
        og.dense_pass(prev)
        for i in range(1, n + 1):
            cur = enc(streams[s], taus[s][i])
            _, oy, _ = og.incr_step(*O.step_increment(prev, cur, 6, 6))
            assert max_err(out[i - 1, s].numpy(), oy) <= 1e-4, (s, i)
            prev = cur
        # the device encoding of the last window is bit-identical to the reference encoders
        assert np.array_equal(_bits(pipe.enc[n % len(pipe.enc)][s].cpu().numpy()), _bits(prev))
    steady = pipe.h2d_bytes[1:]
    assert max(steady) < 13 * S * 2_000 + 8 * 7 * S  # only the ~1k new events per session and step
