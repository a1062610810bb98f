"""Host-I/O-overlapped serving loop over a :class:`~paper_2303_04670_b200.graph.Graph`.

The reference's timed loop (reference bench.py:196-209) is strictly serial: encode the
next window, ``step_increment``, ``incr_step``, read the output.  On a GPU the host
copies of one step can run under the compute of its neighbours: while step i runs on
the compute stream, a copy stream uploads frame i + 1 and downloads step i - 1's
integrated output.  Every step still moves its own input host -> device and its own
result device -> host; only the ordering changes, so each step's output is bit-identical
to the serial loop (tests/test_gpu_serving.py).

Buffers: a ring of three device frames (frame i is ``cur`` of step i and ``prev`` of
step i + 1, so the upload of frame i + 2 may only overwrite frame i - 1 after step i
finished), and two device snapshots of the integrated output (the graph updates it in
place every step).
"""

from __future__ import annotations

import torch


class StreamPipeline:
    """Run consecutive increments of a graph with uploads / downloads overlapped.

    ``host_frames``: pinned host tensor ``(n + 1, S, C, H, W)`` (``(n + 1, C, H, W)`` for
    one session) of encoded windows; frame 0 is the dense-pass input.
    ``out_host``: pinned host tensor ``(n, *integrated_output_shape)``; row i - 1 receives
    the integrated output after increment i.
    A refresh (dense pass) runs in-line whenever the graph reports it due, as in the
    reference's bench loop.
    """

    def __init__(self, graph):
        self.g = graph
        dev = graph.device
        self.copy = torch.cuda.Stream(device=dev)
        self.compute = torch.cuda.current_stream(dev)

    def run(self, host_frames: torch.Tensor, out_host: torch.Tensor, *, dense_first: bool = True) -> int:
        g = self.g
        n = host_frames.shape[0] - 1
        if n < 1:
            return 0
        if not (host_frames.is_pinned() and out_host.is_pinned()):
            raise ValueError("StreamPipeline: host_frames and out_host must be pinned")
        y = g._y_run[g.output_ids[0]]
        one = g.S == 1 and host_frames.dim() == 4
        frames = [torch.empty(host_frames.shape[1:], dtype=host_frames.dtype, device=g.device) for _ in range(3)]
        snaps = [torch.empty_like(y) for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(3)]     # frame k uploaded
        ev_done = [torch.cuda.Event() for _ in range(3)]   # step using frame k as `cur` finished
        ev_snap = [torch.cuda.Event() for _ in range(2)]   # snapshot k written
        ev_out = [torch.cuda.Event() for _ in range(2)]    # snapshot k downloaded
        cs, cp = self.compute, self.copy

        def upload(i):
            k = i % 3
            with torch.cuda.stream(cp):
                if i >= 3:
                    cp.wait_event(ev_done[(i - 2) % 3])  # frame i - 3 was `prev` of step i - 2
                frames[k].copy_(host_frames[i], non_blocking=True)
                ev_in[k].record(cp)

        upload(0)
        if n >= 1:
            upload(1)
        cs.wait_event(ev_in[0])
        if dense_first:
            g.dense_pass(frames[0])
        ev_done[0].record(cs)
        for i in range(1, n + 1):
            if i + 1 <= n:
                upload(i + 1)
            k, kp = i % 3, (i - 1) % 3
            cs.wait_event(ev_in[k])
            g.step_from_encodings(frames[kp], frames[k])
            if g.refresh_due:
                g.dense_pass(frames[k])
            j = i % 2
            if i >= 3:
                cs.wait_event(ev_out[j])  # snapshot j's previous download finished
            snaps[j].copy_(y)
            ev_snap[j].record(cs)
            ev_done[k].record(cs)
            with torch.cuda.stream(cp):
                cp.wait_event(ev_snap[j])
                out_host[i - 1].copy_(snaps[j][0] if one else snaps[j], non_blocking=True)
                ev_out[j].record(cp)
            if i >= 2:
                ev_out[(i - 1) % 2].synchronize()  # the host holds step i - 1's result
        ev_out[n % 2].synchronize()
        return n
