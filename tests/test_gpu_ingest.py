"""Device event ingest: EVB records unpacked on the GPU, and the
count-encoding increment from only the entering / leaving events -- both bit-exact
against the reference path (read_events + encode + step_increment)."""

import numpy as np
import pytest
import torch

import paper_2303_04670_b200 as evc

pytestmark = pytest.mark.gpu


def _stream(seed=3, size=(96, 128)):
    return evc.generate_events(seed=seed, duration_us=120_000, rate_hz=4e5, n_objects=5, sensor_size=size)


def test_upload_evb_builds_the_same_columns(tmp_path):
    s = _stream()
    path = tmp_path / "s.evb"
    evc.write_events(s, path)
    d = evc.upload_evb(path)
    assert d == s
    for got, want in zip(d.device_columns(), (s.t.view(np.int64), s.x.view(np.int16), s.y.view(np.int16), s.p)):
        assert np.array_equal(got.cpu().numpy()[: len(s)], np.asarray(want))
    w = evc.slice_window(d, 80_000, 50_000)
    for kind in ("count", "timestamp", "voxel:5"):
        enc = evc.parse_encoder(kind)
        a = evc.encode(w, enc).cpu().numpy()
        b = evc.encode(evc.slice_window(s, 80_000, 50_000), enc).cpu().numpy()
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), kind


@pytest.mark.parametrize("delta,shift", [(50_000, 1_000), (50_000, 7_000), (10_000, 30_000), (50_000, 0),
                                         (20_000, 500)])
def test_count_increment_is_the_encoding_diff(delta, shift):
    s = _stream(seed=7)
    tile = evc.TileShape(6, 6)
    count = evc.EncoderKind("count")
    for tau in (5_000, 60_000, 90_000):  # the first window starts before the stream
        wp, wc = evc.slice_window(s, tau, delta), evc.slice_window(s, tau + shift, delta)
        inc = evc.count_increment(wp, wc, tile)
        ref = evc.step_increment(evc.encode(wp, count), evc.encode(wc, count), tile)
        assert np.array_equal(inc.values.cpu().numpy().view(np.uint32), ref.values.cpu().numpy().view(np.uint32))
        assert np.array_equal(inc.mask.numpy(), ref.mask.numpy())


def test_count_increment_rejects_backward_windows():
    s = _stream()
    with pytest.raises(ValueError):
        evc.count_increment(evc.slice_window(s, 80_000, 50_000), evc.slice_window(s, 70_000, 50_000),
                            evc.TileShape(6, 6))
