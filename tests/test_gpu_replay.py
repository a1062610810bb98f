"""The device replay harness (bench_report.py) against the reference's bench.replay / sweep reports
(golden: tests/golden/make_replay_golden.py, reference bench.py:140-265): same CSV schema, and
every non-wall-clock column equal -- FLOP meters and false-tile fractions exactly, drift within
the float tolerance of the graph parity tests."""

import csv
import json

import numpy as np
import pytest

import paper_2303_04670_b200 as evc
from paper_2303_04670_b200 import bench_report as R
from evc_testutil import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def case():
    d = np.load(GOLDEN / "replay_cases.npz")
    spec = evc.ModelSpec.from_dict(json.loads(str(d["spec"])))
    weights = {k[2:]: d[k] for k in d.files if k.startswith("w/")}
    h, w = (int(v) for v in d["sensor"])
    stream = evc.EventStream((h, w), d["t"], d["x"], d["y"], d["p"])
    return dict(spec=spec, weights=weights, stream=stream, rows=json.loads(str(d["csv"])),
                sweep=json.loads(str(d["sweep"])), dense=int(d["dense_flops"]))


def test_replay_report_matches_reference(case, tmp_path):
    assert R.static_dense_flops(case["spec"]) == case["dense"]
    rep = R.replay(case["spec"], case["weights"], case["stream"], evc.EncoderKind("count"), window_us=50_000,
                   shift_us=1_000, mode="both", refresh_interval=5, max_steps=10)
    rep.write_csv(tmp_path / "r.csv")
    ours = list(csv.reader(open(tmp_path / "r.csv")))
    ref = case["rows"]
    assert ours[0] == ref[0] and len(ours) == len(ref)
    for a, b in zip(ours[1:], ref[1:]):
        for col, x, y in zip(ref[0], a, b):
            if col.startswith("wall_"):
                assert float(x) > 0.0
            elif col == "drift":
                assert abs(float(x) - float(y)) <= 1e-4, (col, x, y)
            else:
                assert x == y, (a[0], col, x, y)
    s = rep.summary()
    assert s["steps"] == 10 and s["performed_flops"] == sum(int(r[3]) for r in ref[1:])


def test_sweep_rows_match_reference(case):
    rows = R.sweep("tp", [0.0, 0.05], case["spec"], case["weights"], case["stream"], evc.EncoderKind("count"),
                   window_us=50_000, shift_us=2_000, mode="both", refresh_interval=4, max_steps=6)
    for a, b in zip(rows, case["sweep"]):
        assert (a["param"], a["value"]) == (b["param"], b["value"])
        assert a["mean_input_false_frac"] == pytest.approx(b["mean_input_false_frac"], abs=1e-12)
        assert a["mean_flop_reduction_pct"] == pytest.approx(b["mean_flop_reduction_pct"], abs=1e-9)
        assert a["mean_drift"] == pytest.approx(b["mean_drift"], rel=1e-3, abs=1e-4)


def test_replay_argument_errors(case):
    with pytest.raises(ValueError):
        R.replay(case["spec"], case["weights"], case["stream"], evc.EncoderKind("count"), mode="bogus")
    with pytest.raises(ValueError):
        R.sweep("depth", [1], case["spec"], case["weights"], case["stream"], evc.EncoderKind("count"))
