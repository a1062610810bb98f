"""Golden replay / sweep reports (reference bench.py:140-265) from the REAL reference.

Run in the build container only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_replay_golden.py

Writes tests/golden/replay_cases.npz: the stream, the weights and the report columns of a
small `replay(mode="both")` and a `sweep("tp", ...)`, for tests/test_gpu_replay.py.
"""

from __future__ import annotations

import csv
import io
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import evincr as ev  # noqa: E402
from evincr import bench as rb  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    spec = ev.build_plain_cnn(depth=3, channels=6, tp=0.0, in_shape=(2, 32, 40))
    with tempfile.TemporaryDirectory() as td:
        man = ev.WeightManifest.generate(spec, seed=4, out_dir=td)
        weights = {k: v.copy() for k, v in man.tensors().items()}
    stream = ev.generate_events(seed=9, duration_us=62_000, rate_hz=1.5e5, n_objects=3, sensor_size=(32, 40))
    enc = ev.EncoderKind("count")
    rep = rb.replay(spec, weights, stream, enc, window_us=50_000, shift_us=1_000, mode="both",
                    refresh_interval=5, max_steps=10)
    buf = io.StringIO()
    with tempfile.TemporaryDirectory() as td:
        rep.write_csv(Path(td) / "r.csv")
        text = (Path(td) / "r.csv").read_text()
    rows = list(csv.reader(io.StringIO(text)))
    sw = rb.sweep("tp", [0.0, 0.05], spec, weights, stream, enc, window_us=50_000, shift_us=2_000, mode="both",
                  refresh_interval=4, max_steps=6)
    store = {f"w/{k}": v for k, v in weights.items()}
    store.update(t=stream.t, x=stream.x, y=stream.y, p=stream.p, sensor=np.array(stream.sensor_size),
                 spec=json.dumps(spec.to_dict()), csv=json.dumps(rows),
                 summary=json.dumps(rep.summary(), default=float), sweep=json.dumps(sw, default=float),
                 dense_flops=np.int64(rb.static_dense_flops(spec)))
    np.savez_compressed(OUT / "replay_cases.npz", **store)
    print("wrote replay_cases.npz:", len(rows) - 1, "steps,", len(sw), "sweep rows")


if __name__ == "__main__":
    main()
