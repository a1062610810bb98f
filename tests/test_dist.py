"""World-size-2 CPU (gloo) tests of the multi-GPU layout.

Streams are independent sessions: rank r owns streams r*S .. r*S + S - 1, there is no
collective on the data path, and the job time is the max over ranks.  Each rank here
also advances its own streams through the CPU oracle and checks them against a
single-process run of the same seeds (sharding must not change any stream's result).
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import evincr_np as O
from paper_2303_04670_b200 import shard
from paper_2303_04670_b200.graph import WeightManifest
from paper_2303_04670_b200.models import build_plain_cnn
from paper_2303_04670_b200.synth import generate_events

S = 2  # streams per rank


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _stream_outputs(seed, steps=3):
    """Integrated output of one stream after `steps` increments (oracle, tiny CNN)."""
    spec = build_plain_cnn(depth=2, channels=4, tp=0.0, in_shape=(2, 24, 24))
    weights = WeightManifest.random_tensors(spec, 0)
    g = O.OracleGraph(spec.to_dict(), weights, refresh_interval=0)
    ev = generate_events(seed=seed, duration_us=60_000, rate_hz=2e4, n_objects=2, sensor_size=(24, 24))

    def enc(i):
        lo, hi = O.slice_window(ev.t, 50_000 + 1_000 * i, 50_000)
        return O.encode(ev.t, ev.x, ev.y, ev.p, lo, hi, 50_000 + 1_000 * i, 50_000, 24, 24, "count")

    prev = enc(0)
    g.dense_pass(prev)
    y = None
    for i in range(1, steps + 1):
        cur = enc(i)
        _, y, _ = g.incr_step(*O.step_increment(prev, cur, 6, 6))
        prev = cur
    return y


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, _ = shard.dist_env()
        seeds = shard.stream_seeds(r, S)
        outs = {sd: _stream_outputs(sd) for sd in seeds}
        gathered = [None] * w
        dist.all_gather_object(gathered, seeds)
        job = shard.job_time_ms(10.0 + 5.0 * r, w)
        q.put((r, w, gathered, job, {sd: o.tolist() for sd, o in outs.items()}))
    finally:
        dist.destroy_process_group()


def test_two_ranks_shard_streams_and_time_max():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    all_seeds = res[0][2]
    assert all_seeds == res[1][2]
    flat = [sd for part in all_seeds for sd in part]
    assert sorted(flat) == list(range(world * S)), "every stream owned by exactly one rank"
    assert all(r[3] == 15.0 for r in res), "job time is the max over ranks"
    # sharding does not change any stream: each rank's outputs equal a single-process run
    for r in res:
        for sd, y in r[4].items():
            assert np.array_equal(np.asarray(y, np.float32), _stream_outputs(sd)), sd


def test_single_process_defaults():
    assert shard.stream_seeds(0, 3) == [0, 1, 2]
    assert shard.job_time_ms(7.5, 1) == 7.5
    assert shard.aggregate_rate(64, 32, 8, 1000.0) == pytest.approx(64 * 32 * 8)
