"""Multi-GPU layout of independent event streams.

Streams are independent sessions (graph.py:423-429): rank r of N owns
the S streams r*S .. r*S + S - 1, weights are replicated, and there is no collective on
the data path.  The only cross-rank step is reporting: the job's wall time is the
maximum of the per-rank device times (the slowest rank finishes the job).
"""

from __future__ import annotations

import os


def dist_env():
    """(rank, world_size, local_rank) from the torchrun environment (defaults: one process)."""
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def stream_seeds(rank: int, sessions: int) -> list:
    """Seeds (= global stream ids) of the streams rank `rank` owns."""
    return [rank * sessions + s for s in range(sessions)]


def job_time_ms(local_ms: float, world: int, device=None) -> float:
    """Max over ranks of the per-rank timed-region duration (a no-op for one process).

    Uses the default process group (NCCL on the GPU box, gloo in the CPU tests)."""
    if world <= 1:
        return float(local_ms)
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(local_ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_rate(steps: int, sessions: int, world: int, job_ms: float) -> float:
    """Whole-job increments per second: every rank advances `sessions` streams per step."""
    return steps * sessions * world / (job_ms / 1e3)
